cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 1000 --warmup 20 > gpurun_out/bench.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench.log | cut -c1-200
timeout 600 python scripts/sweep.py > gpurun_out/sweep_ac.jsonl 2>&1; echo "sweep exit $?"
timeout 120 python scripts/profile_step.py --n 1048576 --case bluerov > gpurun_out/plain_b1m.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step -s 5 -c 1 \
    -o gpurun_out/prof_ac_bluerov_1m python scripts/profile_step.py --n 1048576 --case bluerov > gpurun_out/ncu_b1m.log 2>&1; echo "ncu b1m exit $?"
timeout 120 python scripts/profile_step.py --n 4096 --case cfg2 > gpurun_out/plain_c4k.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step -s 5 -c 1 \
    -o gpurun_out/prof_ac_cfg2_4k python scripts/profile_step.py --n 4096 --case cfg2 > gpurun_out/ncu_c4k.log 2>&1; echo "ncu c4k exit $?"
timeout 120 python scripts/profile_step.py --n 1048576 --case cfg2 > gpurun_out/plain_c1m.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step -s 5 -c 1 \
    -o gpurun_out/prof_ac_cfg2_1m python scripts/profile_step.py --n 1048576 --case cfg2 > gpurun_out/ncu_c1m.log 2>&1; echo "ncu c1m exit $?"
