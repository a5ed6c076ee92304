cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 1000 --warmup 20 > gpurun_out/bench.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench.log | cut -c1-150
timeout 900 python bench.py --impl reference --steps 200 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"; tail -1 gpurun_out/bench_ref.log | cut -c1-200
timeout 600 python scripts/sweep.py > gpurun_out/sweep_final.jsonl 2>&1; echo "sweep exit $?"
timeout 600 python scripts/sweep.py --cases task_cfg4,task_cfg5 --sizes 4096,65536,1048576 > gpurun_out/sweep_task.jsonl 2>&1; echo "task sweep exit $?"
