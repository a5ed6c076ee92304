#!/bin/bash
# Round-end evidence on one GPU: revalidation (tests, smoke, both bench arms, K=1000,
# 2-rank path), the sweeps behind DESIGN §3.4, and the profiles of the dominant kernels.
cd "$(dirname "$0")/.."
bash scripts/gpu_revalidate.sh
R=gpurun_out/reval
python scripts/sweep.py --cases bluerov,cfg2,cfg3,cfg5_physics,cfg2_k8 --sizes 4096,65536,262144,1048576,4194304 --steps 50 > $R/sweep.jsonl 2> $R/sweep.err
python scripts/sweep.py --cases task_cfg4,task_cfg5 --sizes 4096,65536,262144,1048576 --steps 20 > $R/sweep_task.jsonl 2>> $R/sweep.err
python scripts/probes/rollout_sizes.py > $R/rollout_sizes.jsonl 2>> $R/sweep.err
python scripts/bench_cem.py --cpu-steps 5 > $R/bench_cem.jsonl 2>> $R/sweep.err
python scripts/probes/rollout_fixed_cost.py > $R/rollout_fixed_cost.json 2>> $R/sweep.err
python scripts/probes/rollout_cold_warm.py > $R/rollout_cold_warm.json 2>> $R/sweep.err
python scripts/probes/event_overhead.py > $R/event_overhead.json 2>> $R/sweep.err
python scripts/probes/rollout_host.py > $R/rollout_host.json 2>> $R/sweep.err
CASES="k_rollout_cfg2_4096:k_rollout:0:--case cfg2 --n 4096 --steps 5 --rollout 20
k_step_cfg2_4096:k_step:2:--case cfg2 --n 4096 --steps 5
k_step_cfg2_1m:k_step:2:--case cfg2 --n 1048576 --steps 5
task_cfg5_1m:k_task_step:2:--case task_cfg5 --n 1048576 --steps 5
task_cfg4_1m:k_task_step:2:--case task_cfg4 --n 1048576 --steps 5
policy_episode_512:k_policy_episode:0:--case policy --n 512 --steps 100" bash scripts/gpu_profile.sh > $R/profile.log 2>&1
ls -la $R gpurun_out/prof
