cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
python scripts/profile_step.py --case policy --n 512 --steps 40 || exit 1
ncu --section WarpStateStats --section SourceCounters --warp-sampling-interval 0 --import-source on \
  --clock-control none -k regex:k_task_step -s 20 -c 10 -o gpurun_out/prof/pol512 \
  python scripts/profile_step.py --case policy --n 512 --steps 40 > gpurun_out/prof/ncu_pol.log 2>&1
ncu -i gpurun_out/prof/pol512.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/pol512_sass.csv 2>/dev/null
gzip -f gpurun_out/prof/pol512_sass.csv; rm -f gpurun_out/prof/pol512.ncu-rep
tail -2 gpurun_out/prof/ncu_pol.log
