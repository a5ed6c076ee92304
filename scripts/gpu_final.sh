# End-of-round evidence on the final tree: GPU tests, smoke, bench (+ reference arm),
# sweeps, launch list and ncu --set full captures (scripts/gpu_profiles.sh).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 1000 --warmup 20 > gpurun_out/bench.log 2>&1; echo "bench exit $?"
timeout 900 python bench.py --impl reference --steps 200 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"
timeout 900 python scripts/sweep.py > gpurun_out/sweep_final.jsonl 2>&1; echo "sweep exit $?"
timeout 600 python scripts/sweep.py --cases task_cfg4,task_cfg5 --sizes 4096,65536,1048576 > gpurun_out/sweep_task.jsonl 2>&1; echo "task sweep exit $?"
timeout 600 python scripts/bench_tasks.py > gpurun_out/bench_tasks.jsonl 2>&1; echo "tasks exit $?"
timeout 600 python scripts/bench_cem.py > gpurun_out/bench_cem.jsonl 2>&1; echo "cem exit $?"
bash scripts/gpu_profiles.sh
