cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/sweep.py --cases task_cfg4,task_cfg5 --sizes 4096,65536,1048576 > gpurun_out/sweep_task2.jsonl 2>&1; echo "task sweep exit $?"; cat gpurun_out/sweep_task2.jsonl
