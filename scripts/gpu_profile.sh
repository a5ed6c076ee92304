#!/bin/bash
# Profiling on one GPU: the bench's launch list and `ncu --set full` captures of the dominant
# kernels, summarised ON THE BOX (raw-page markdown, SASS/source CSV) so only small files
# come back in gpurun_out/prof/.  Each capture runs after its command exited 0 without ncu.
#   CASES: lines "name:kernel_regex:skip:profile_step.py args" (default: the bench's step kernels)
cd "$(dirname "$0")/.."
P=gpurun_out/prof; mkdir -p $P
NCU="ncu --clock-control none"
python scripts/profile_step.py --case cfg2 --n 4096 --steps 5 --rollout 20 > $P/plain.log 2>&1 || exit 1
if [ -z "${SKIP_LAUNCHES:-}" ]; then
  $NCU --metrics gpu__time_duration.sum -c 800 --csv --log-file $P/launches.csv \
      python bench.py --steps 20 --warmup 5 --no-serve --no-cpu-baseline > $P/launches.log 2>&1
  python scripts/ncu_summary.py --launches $P/launches.csv > $P/launches.md
  gzip -f $P/launches.csv
fi
# one case per line: name:kernel_regex:launches_to_skip:profile_step.py arguments
DEFAULT_CASES="k_rollout_cfg2_4096:k_rollout:0:--case cfg2 --n 4096 --steps 5 --rollout 20
k_step_cfg2_4096:k_step:2:--case cfg2 --n 4096 --steps 5"
CASES=${CASES:-$DEFAULT_CASES}
echo "$CASES" | while IFS= read -r c; do
  [ -z "$c" ] && continue
  name=${c%%:*}; rest=${c#*:}; kern=${rest%%:*}; rest=${rest#*:}; skip=${rest%%:*}; args=${rest#*:}
  eval python scripts/profile_step.py $args > $P/plain_$name.log 2>&1 || { echo "plain $name failed"; continue; }
  eval $NCU --set full --import-source on -k regex:$kern -s $skip -c 1 -f -o $P/$name \
      python scripts/profile_step.py $args > $P/ncu_$name.log 2>&1
  python scripts/ncu_summary.py $P/$name.ncu-rep > $P/$name.md 2>&1
  ncu -i $P/$name.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $P/${name}_sass.csv.gz
  ncu -i $P/$name.ncu-rep --page raw --csv 2>/dev/null | gzip > $P/${name}_raw.csv.gz
  gzip -f $P/$name.ncu-rep
  rm -f $P/$name.ncu-rep.gz  # the summaries above are what travels back (gpurun_out <= 64 MiB)
done
du -sh $P; ls -la $P
