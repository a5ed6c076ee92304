# Dense warp-state sampling of the latency-bound headline kernel (cfg2, 4096 envs).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
python scripts/profile_step.py --case cfg2 --n 4096 --steps 30 || exit 1
ncu --section WarpStateStats --section SourceCounters --warp-sampling-interval 0 --import-source on \
  --clock-control none -k regex:k_step -s 20 -c 5 -o gpurun_out/prof/lat4096 \
  python scripts/profile_step.py --case cfg2 --n 4096 --steps 30 > gpurun_out/prof/ncu_lat.log 2>&1
ncu -i gpurun_out/prof/lat4096.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/lat4096_sass.csv 2>/dev/null
gzip -f gpurun_out/prof/lat4096_sass.csv; rm -f gpurun_out/prof/lat4096.ncu-rep
tail -3 gpurun_out/prof/ncu_lat.log
