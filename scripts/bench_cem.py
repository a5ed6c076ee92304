"""Policy-search throughput: one CEM iteration (= one `_rollout_returns` episode loop).

GPU: ``baseline.cem_train`` with the device episode loop (one CUDA-graph replay
per iteration); timed with CUDA events over ``--iterations`` after one warm-up
iteration (graph capture).  CPU: the oracle's numpy restatement of the same
loop (host affine-tanh policy + ``TaskEnv.step``), one host thread, on a
bounded number of steps — the reference's own execution model.

    python scripts/bench_cem.py [--envs 512] [--population 32] [--iterations 5]
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_09203_b200 import baseline as B  # noqa: E402
from paper_2503_09203_b200.engine import SimConfig  # noqa: E402
from paper_2503_09203_b200.tasks import TaskConfig, make_env  # noqa: E402


def gpu_case(task, envs, population, iterations):
    env = make_env(task, SimConfig(batch_size=envs), seed=0)
    B.cem_train(env, population=population, iterations=1, seed=0)  # capture
    runner = B._runner(env, population, envs // population)
    rng = np.random.default_rng(1)
    thetas = [rng.normal(0, 0.3, (population, runner.n_params)) for _ in range(iterations)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    for th in thetas:
        runner.launch(th)
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    for th in thetas[-1:]:
        runner.run(th)
        steps = runner.steps_run()
    dev_s = e0.elapsed_time(e1) / 1e3 / iterations
    # a full cem_train iteration including the host CEM update and the D2H of returns
    t0 = time.perf_counter()
    B.cem_train(env, population=population, iterations=iterations, seed=1)
    full = (time.perf_counter() - t0) / iterations
    return {"impl": "device", "fused_episode": bool(runner._fused), "envs": envs,
            "population": population,
            "episode_length": task.episode_length, "steps_last_iteration": steps,
            "s_per_iteration_device": dev_s, "s_per_iteration_cem_train": full,
            "env_frames_per_s": envs * steps / dev_s, "enqueue_wall_s": wall / iterations}


def cpu_loop(task, envs, population, max_steps):
    """Oracle episode loop with a host affine-tanh population policy (baseline.py:109-127)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from conftest import product_vehicle
    from oracle import uuv_oracle as O
    from paper_2503_09203_b200.randomization import preset
    from paper_2503_09203_b200.tasks import disturbed_spec

    oe = O.TaskEnv(task, product_vehicle(task.vehicle), envs, seed=0,
                   disturbed_spec=disturbed_spec(), train_spec=preset("train"))
    obs = oe.reset()
    slot = envs // population
    used = slot * population
    od, a = obs.shape[1], oe.A
    th = np.random.default_rng(1).normal(0, 0.3, (population, a * od + a))
    w = th[:, :a * od].reshape(population, a, od)
    b = th[:, a * od:]
    t0 = time.perf_counter()
    for _ in range(max_steps):
        x = obs[:used].reshape(population, slot, od)
        cmd = np.zeros((envs, a))
        cmd[:used] = np.tanh(np.einsum("pso,pao->psa", x, w) + b[:, None, :]).reshape(used, a)
        obs, *_ = oe.step(cmd)
    dt = (time.perf_counter() - t0) / max_steps
    return {"impl": "oracle-cpu", "envs": envs, "population": population,
            "s_per_step": dt, "env_frames_per_s": envs / dt,
            "s_per_iteration_est": dt * task.episode_length, "threads": 1,
            "sample_steps": max_steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", default="512,65536")
    ap.add_argument("--population", type=int, default=32)
    ap.add_argument("--iterations", type=int, default=5)
    ap.add_argument("--cpu-steps", type=int, default=50)
    ap.add_argument("--task", default="station_keeping")
    ap.add_argument("--vehicle", default="bluerov_heavy")
    args = ap.parse_args()
    task = TaskConfig(task=args.task, vehicle=args.vehicle)
    for n in (int(x) for x in args.envs.split(",")):
        print(json.dumps(gpu_case(task, n, args.population, args.iterations)), flush=True)
    print(json.dumps(cpu_loop(task, 512, args.population, args.cpu_steps)), flush=True)


if __name__ == "__main__":
    main()
