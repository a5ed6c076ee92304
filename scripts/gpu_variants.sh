cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for mb in 0 4 6 8; do
  UUV_B200_LIB=build/variants/lib_mb$mb.so timeout 600 python scripts/sweep.py --cases cfg2,bluerov,cfg3,cfg2_k8,cfg5_physics --sizes 4096,262144,1048576 > gpurun_out/sweep_mb$mb.jsonl 2> gpurun_out/sweep_mb$mb.err
  echo "mb$mb exit $?"
done
