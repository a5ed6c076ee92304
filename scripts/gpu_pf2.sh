cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/pytest_pf.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_pf.log
timeout 600 python scripts/sweep.py --cases cfg2,bluerov,cfg3,cfg5_physics,cfg2_k8 --sizes 4096,65536,1048576,4194304 > gpurun_out/sweep_simple.jsonl 2>&1; echo "sweep simple exit $?"
UUV_B200_LIB=build/variants/lib_persist.so timeout 600 python scripts/sweep.py --cases cfg2,bluerov,cfg3,cfg5_physics,cfg2_k8 --sizes 4096,65536,1048576,4194304 > gpurun_out/sweep_persist.jsonl 2>&1; echo "sweep persist exit $?"
timeout 600 python bench.py --steps 1000 --warmup 20 > gpurun_out/bench.log 2>&1; echo "bench exit $?"
