cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./build/latency_probe > gpurun_out/latency_probe.log 2>&1; echo "probe exit $?"; cat gpurun_out/latency_probe.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv \
    python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches exit $?"
timeout 120 python scripts/profile_step.py --n 4096 --case cfg2 > gpurun_out/plain_c4k.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step -s 5 -c 1 \
    -o gpurun_out/r01_k_step_cfg2_4096 python scripts/profile_step.py --n 4096 --case cfg2 > gpurun_out/ncu_c4k.log 2>&1; echo "ncu c4k exit $?"
timeout 120 python scripts/profile_step.py --n 1048576 --case cfg2 > gpurun_out/plain_c1m.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step -s 5 -c 1 \
    -o gpurun_out/r01_k_step_cfg2_1m python scripts/profile_step.py --n 1048576 --case cfg2 > gpurun_out/ncu_c1m.log 2>&1; echo "ncu c1m exit $?"
timeout 120 python scripts/profile_step.py --n 1048576 --case bluerov > gpurun_out/plain_b1m.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step -s 5 -c 1 \
    -o gpurun_out/r01_k_step_bluerov_1m python scripts/profile_step.py --n 1048576 --case bluerov > gpurun_out/ncu_b1m.log 2>&1; echo "ncu b1m exit $?"
