#!/bin/bash
# Round-2 profiling on one GPU: the bench's launch list and `ncu --set full` captures of the
# dominant kernels.  Outputs under gpurun_out/prof/ (summarised into profiles/r02 by
# scripts/ncu_summary.py).  Each capture runs only after its command exited 0 without ncu.
cd "$(dirname "$0")/.."
P=gpurun_out/prof; mkdir -p $P
NCU="ncu --clock-control none"
python scripts/profile_step.py --case cfg2 --n 4096 --steps 5 --rollout 20 > $P/plain.log 2>&1 || exit 1
$NCU --metrics gpu__time_duration.sum -c 600 --csv --log-file $P/launches.csv \
    python bench.py --steps 20 --warmup 5 --no-serve --no-cpu-baseline > $P/launches.log 2>&1
$NCU --set full --import-source on -k regex:k_rollout -c 1 -f -o $P/k_rollout_cfg2_4096 \
    python scripts/profile_step.py --case cfg2 --n 4096 --steps 5 --rollout 20 > $P/ncu1.log 2>&1
$NCU --set full --import-source on -k regex:k_step -s 3 -c 1 -f -o $P/k_step_cfg2_4096 \
    python scripts/profile_step.py --case cfg2 --n 4096 --steps 5 > $P/ncu2.log 2>&1
for c in ${EXTRA_CASES:-}; do
  $NCU --set full --import-source on -k regex:${c%%:*} -s 3 -c 1 -f -o $P/${c##*:} \
      python scripts/profile_step.py --case ${c#*:} --n 1048576 --steps 5 > $P/ncu_${c##*:}.log 2>&1
done
ls -la $P
