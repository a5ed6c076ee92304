cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
timeout 600 python scripts/bench_tasks.py > gpurun_out/bench_tasks.jsonl 2>&1; echo "tasks exit $?"; cat gpurun_out/bench_tasks.jsonl | cut -c1-300
UUV_BENCH_GPU_OVERRIDE=0 UUV_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29541 scripts/bench_tasks.py --envs-per-gpu 65536 --steps 100 > gpurun_out/bench_tasks_2rank.jsonl 2>&1
echo "tasks 2rank exit $?"; tail -2 gpurun_out/bench_tasks_2rank.jsonl | cut -c1-300
timeout 120 python scripts/profile_step.py --n 1048576 --case cfg2_k8 > gpurun_out/prof/plain_k8.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step -s 5 -c 1 \
    -o gpurun_out/prof/k_step_cfg2_k8_1m python scripts/profile_step.py --n 1048576 --case cfg2_k8 > gpurun_out/prof/ncu_k8.log 2>&1
echo "ncu k8 exit $?"
python scripts/ncu_summary.py gpurun_out/prof/k_step_cfg2_k8_1m.ncu-rep > gpurun_out/prof/k_step_cfg2_k8_1m.md 2>&1
ncu -i gpurun_out/prof/k_step_cfg2_k8_1m.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/k_step_cfg2_k8_1m_sass.csv 2>/dev/null
gzip -9 gpurun_out/prof/k_step_cfg2_k8_1m_sass.csv
rm -f gpurun_out/prof/*.ncu-rep
