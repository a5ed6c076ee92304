# ncu captures of the task-step and policy-step kernels at small N (one GPU, one tool per call).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
python scripts/profile_step.py --case task_cfg5 --n 4096 --steps 20 && \
python scripts/profile_step.py --case policy --n 512 --steps 30 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_task_step -s 10 -c 1 \
  -o gpurun_out/prof/task_cfg5_4096 python scripts/profile_step.py --case task_cfg5 --n 4096 --steps 20 > gpurun_out/prof/ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_task_step -s 10 -c 1 \
  -o gpurun_out/prof/policy_512 python scripts/profile_step.py --case policy --n 512 --steps 30 > gpurun_out/prof/ncu2.log 2>&1
for r in task_cfg5_4096 policy_512; do
  python scripts/ncu_summary.py gpurun_out/prof/$r.ncu-rep > gpurun_out/prof/$r.md 2>&1
  ncu -i gpurun_out/prof/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/${r}_sass.csv 2>/dev/null
  gzip -f gpurun_out/prof/${r}_sass.csv
  gzip -f gpurun_out/prof/$r.ncu-rep
done
ls -la gpurun_out/prof
