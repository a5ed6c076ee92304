cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python scripts/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1; echo "e2e exit $?"; cat gpurun_out/e2e_probe.log
timeout 600 python scripts/sweep.py --cases cfg3 --sizes 4096,65536,1048576,4194304 > gpurun_out/sweep_mixed.jsonl 2>&1; echo "sweep exit $?"; cat gpurun_out/sweep_mixed.jsonl
timeout 600 python bench.py --steps 1000 --warmup 20 > gpurun_out/bench.log 2>&1; echo "bench exit $?"
