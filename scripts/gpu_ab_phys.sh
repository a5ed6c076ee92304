# Interleaved A/B of the physics + task kernels between the in-tree build and
# build/variants/lib_$AB_OLD.so (GPU tests first, on the in-tree build).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/abp_*.jsonl
if [ -z "$AB_NO_TESTS" ]; then
  timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_ab.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_ab.log
fi
for rep in 1 2; do for v in new ${AB_OLD:-old}; do
  if [ $v = new ]; then unset UUV_B200_LIB; else export UUV_B200_LIB=build/variants/lib_$v.so; fi
  timeout 600 python scripts/sweep.py --cases ${AB_CASES:-bluerov,cfg2,cfg5_physics,cfg2_k8,task_cfg4,task_cfg5} --sizes ${AB_SIZES:-4096,65536,1048576} >> gpurun_out/abp_$v.jsonl 2>&1; echo "$v exit $?"
done; done
