# Round-1 evidence for profiles/: launch list of the bench command + ncu --set full
# captures of the step kernel (bench workload, and 1M envs for the HBM-bound regime).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/prof/bench_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv \
    python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-serve > gpurun_out/prof/ncu_launches.log 2>&1; echo "launches exit $?"
python scripts/ncu_summary.py --launches gpurun_out/prof/launches.csv > gpurun_out/prof/launches.md 2>&1
for case in "4096 cfg2" "1048576 cfg2" "1048576 bluerov"; do
  set -- $case
  timeout 120 python scripts/profile_step.py --n $1 --case $2 > gpurun_out/prof/plain_$2_$1.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step -s 5 -c 1 \
      -o gpurun_out/prof/k_step_$2_$1 python scripts/profile_step.py --n $1 --case $2 > gpurun_out/prof/ncu_$2_$1.log 2>&1
  echo "ncu $2 $1 exit $?"
  python scripts/ncu_summary.py gpurun_out/prof/k_step_$2_$1.ncu-rep > gpurun_out/prof/k_step_$2_$1.md 2>&1
  ncu -i gpurun_out/prof/k_step_$2_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/k_step_$2_$1_sass.csv 2>/dev/null
  gzip -9 gpurun_out/prof/k_step_$2_$1_sass.csv
done
# keep one full report (the bench workload) for local inspection, drop the others
gzip -9 gpurun_out/prof/k_step_cfg2_4096.ncu-rep
rm -f gpurun_out/prof/*.ncu-rep
du -sh gpurun_out/prof
