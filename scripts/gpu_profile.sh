set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep exit $?"
# launch list of the bench command (cold-cache, serialised: compare shares)
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches exit $?"
timeout 120 python scripts/profile_step.py --n 4096 --case cfg2 > gpurun_out/plain_prof.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step -s 5 -c 2 \
    -o gpurun_out/prof_step_cfg2 python scripts/profile_step.py --n 4096 --case cfg2 > gpurun_out/ncu_full_cfg2.log 2>&1; echo "ncu full cfg2 exit $?"
timeout 120 python scripts/profile_step.py --n 1048576 --case cfg2 > gpurun_out/plain_prof1m.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step -s 5 -c 1 \
    -o gpurun_out/prof_step_cfg2_1m python scripts/profile_step.py --n 1048576 --case cfg2 > gpurun_out/ncu_full_1m.log 2>&1; echo "ncu full 1m exit $?"
cat gpurun_out/sweep.jsonl
