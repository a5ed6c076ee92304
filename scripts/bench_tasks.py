"""Task-level benchmark for BASELINE.json configs 4 and 5 (one JSON line per config).

cfg4: trajectory tracking, bluerov, level "disturbed" (0.25 m/s current, payload),
      8 fused substeps per control step, 1M envs per GPU.
cfg5: docking, bluerov_heavy, level "disturbed_dr" (train-preset DR), full
      obs/reward/termination/auto-reset, 1M envs per GPU, rollout statistics
      all-reduced across ranks (NCCL) once per rollout of `--rollout` steps.

Each step is one fused ``env.step`` launch; steps are replayed from a CUDA graph
and timed with CUDA events; max over ranks.  Run with torchrun for N > 1:

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \
        scripts/bench_tasks.py --envs-per-gpu 1048576
"""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200.distributed import allreduce_max  # noqa: E402
from paper_2503_09203_b200.tasks import TaskConfig, make_env  # noqa: E402


def run(cfg, n, steps, rollout, dev, rank, world):
    if cfg == "cfg4":
        task = TaskConfig(task="tracking", vehicle="bluerov", level="disturbed")
        sim = E.SimConfig(batch_size=n, substeps=8)
    else:
        task = TaskConfig(task="docking", vehicle="bluerov_heavy", level="disturbed_dr")
        sim = E.SimConfig(batch_size=n)
    env = make_env(task, sim, seed=0, device=dev, env_offset=rank * n)
    env.reset()
    a = env.action_dim
    gen = torch.Generator(device=dev).manual_seed(rank)
    cmds = torch.rand((rollout, n, a), device=dev, generator=gen) * 2 - 1
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for t in range(3):
            env.step(cmds[t])
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for t in range(rollout):
                env.step(cmds[t])
    g.replay()
    torch.cuda.synchronize(dev)
    env.rollout_stats(reset=True)
    n_roll = max(1, steps // rollout)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    e0.record(s)
    stats = None
    for _ in range(n_roll):
        with torch.cuda.stream(s):
            g.replay()
            stats = env.rollout_stats(reset=True)  # device reduction + NCCL all-reduce
    e1.record(s)
    torch.cuda.synchronize(dev)
    el = allreduce_max(e0.elapsed_time(e1) / 1e3, dev)
    frames = world * n * rollout * n_roll
    return {"metric": "env frames/sec (fused task step incl. auto-reset)", "config": cfg,
            "value": frames / el, "unit": "env-frames/s", "n_gpus": world, "envs_per_gpu": n,
            "steps": rollout * n_roll, "ms_per_step": 1e3 * el / (rollout * n_roll),
            "substeps": sim.substeps, "rollout_stats_allreduce_per": rollout,
            "last_rollout": {k: stats[k] for k in ("frames", "finished", "success", "failure")}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg4,cfg5")
    ap.add_argument("--envs-per-gpu", type=int, default=1 << 20)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--rollout", type=int, default=50)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("UUV_BENCH_GPU_OVERRIDE", local)))
    torch.cuda.set_device(dev)
    if world > 1:
        backend = os.environ.get("UUV_DIST_BACKEND", "nccl")
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=dev)
        else:
            torch.distributed.init_process_group(backend)
    for cfg in args.configs.split(","):
        line = run(cfg, args.envs_per_gpu, args.steps, args.rollout, dev, rank, world)
        if rank == 0:
            print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
