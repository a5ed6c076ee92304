cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
python scripts/profile_step.py --case task_cfg5 --n 1048576 --steps 6 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_task_step -s 3 -c 1 \
  -o gpurun_out/prof/task_cfg5_1m python scripts/profile_step.py --case task_cfg5 --n 1048576 --steps 6 > gpurun_out/prof/ncu4.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof/task_cfg5_1m.ncu-rep > gpurun_out/prof/task_cfg5_1m.md 2>&1
ncu -i gpurun_out/prof/task_cfg5_1m.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/task_cfg5_1m_sass.csv 2>/dev/null
ncu -i gpurun_out/prof/task_cfg5_1m.ncu-rep --page source --csv --print-source cuda > gpurun_out/prof/task_cfg5_1m_src.csv 2>/dev/null
gzip -f gpurun_out/prof/task_cfg5_1m_sass.csv gpurun_out/prof/task_cfg5_1m_src.csv
rm -f gpurun_out/prof/task_cfg5_1m.ncu-rep
cat gpurun_out/prof/task_cfg5_1m.md
