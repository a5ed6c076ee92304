cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/pytest_pf.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_pf.log
timeout 600 python scripts/sweep.py --cases cfg2,bluerov,cfg3,cfg5_physics,cfg2_k8 --sizes 4096,65536,1048576,4194304 > gpurun_out/sweep_pf1.jsonl 2>&1; echo "sweep pf1 exit $?"
UUV_STEP_WAVES=2 timeout 600 python scripts/sweep.py --cases cfg2,bluerov,cfg3,cfg5_physics,cfg2_k8 --sizes 1048576,4194304 > gpurun_out/sweep_pf2.jsonl 2>&1; echo "sweep pf2 exit $?"
UUV_STEP_WAVES=1000000 timeout 600 python scripts/sweep.py --cases cfg2,bluerov,cfg3,cfg5_physics,cfg2_k8 --sizes 4096,65536,1048576,4194304 > gpurun_out/sweep_pfoff.jsonl 2>&1; echo "sweep pfoff exit $?"
timeout 600 python scripts/sweep.py --cases task_cfg4,task_cfg5 --sizes 4096,65536,1048576 > gpurun_out/sweep_task.jsonl 2>&1; echo "sweep task exit $?"
