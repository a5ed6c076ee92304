cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv \
    python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-serve > gpurun_out/prof/ncu_launches.log 2>&1; echo "launches exit $?"
python scripts/ncu_summary.py --launches gpurun_out/prof/launches.csv > gpurun_out/prof/launches.md 2>&1
head -30 gpurun_out/prof/launches.md
