cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python scripts/sweep.py --cases cfg2,bluerov,cfg3,cfg5_physics,cfg2_k8 --sizes 4096,65536,1048576,4194304 > gpurun_out/sweep_tma.jsonl 2>&1; echo "sweep tma exit $?"
UUV_STEP_KERNEL=direct timeout 600 python scripts/sweep.py --cases cfg2,bluerov,cfg3,cfg5_physics,cfg2_k8 --sizes 4096,65536,1048576,4194304 > gpurun_out/sweep_direct.jsonl 2>&1; echo "sweep direct exit $?"
timeout 600 python bench.py --steps 1000 --warmup 20 > gpurun_out/bench.log 2>&1; echo "bench exit $?"
