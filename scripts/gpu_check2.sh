cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py --steps 1000 --warmup 20 > gpurun_out/bench.log 2>&1; echo "bench exit $?"
timeout 600 python scripts/sweep.py > gpurun_out/sweep_dm.jsonl 2>&1; echo "sweep exit $?"
