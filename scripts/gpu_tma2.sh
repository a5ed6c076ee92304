cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
UUV_STEP_KERNEL=tma timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -q -p no:cacheprovider -x > gpurun_out/pytest_tma.log 2>&1; echo "pytest tma exit $?"; tail -3 gpurun_out/pytest_tma.log
UUV_STEP_KERNEL=tma timeout 600 python scripts/sweep.py --cases cfg2,bluerov,cfg3,cfg5_physics,cfg2_k8 --sizes 4096,65536,1048576,4194304 > gpurun_out/sweep_tma.jsonl 2>&1; echo "sweep tma exit $?"
timeout 600 python scripts/sweep.py --cases cfg2,bluerov,cfg3,cfg5_physics,cfg2_k8 --sizes 4096,65536,1048576,4194304 > gpurun_out/sweep_direct.jsonl 2>&1; echo "sweep direct exit $?"
