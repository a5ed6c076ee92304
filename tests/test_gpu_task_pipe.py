"""The pipelined task kernel (k_task_step_pipe: persistent grid, every warp prefetching its
next 32-env tile with cp.async into a double-buffered shared-memory slab) == the per-env
kernel (k_task_step), bit for bit: the same per-env code (task_env) on staged inputs.  The
pipelined kernel serves float32 batches from UUV_TASK_PIPE_MIN_ENVS envs (default 262,144);
a subprocess with the threshold at 1 runs it on small batches with ragged last tiles,
auto-resets, DR, currents and every task kind."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RUN = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2503_09203_b200 import engine as E
from paper_2503_09203_b200.tasks import TaskConfig, make_env
out = {}
cases = [("docking", "bluerov_heavy", "disturbed_dr", 1, 1000),
         ("tracking", "bluerov", "disturbed", 8, 777),
         ("station_keeping", "lauv", "disturbed_dr", 2, 300),
         ("tracking", "hauv", "standard", 1, 129)]
for kind, veh, level, K, n in cases:
    env = make_env(TaskConfig(task=kind, vehicle=veh, level=level, episode_length=7),
                   E.SimConfig(batch_size=n, substeps=K), seed=5)
    obs = env.reset()
    g = torch.Generator(device="cuda").manual_seed(0)
    for t in range(20):
        u = torch.rand((n, env.action_dim), device="cuda", generator=g) * 2.4 - 1.2
        o, r, te, tr, info = env.step(u)
        key = f"{kind}_{veh}_{t}"
        out[key + "_obs"] = o.cpu().numpy()
        out[key + "_r"] = r.cpu().numpy()
        out[key + "_f"] = np.stack([te.cpu().numpy(), tr.cpu().numpy(),
                                    info["finished"].cpu().numpy()])
    for k in ("p", "q", "nu", "act", "steps", "episodes", "diverged"):
        out[f"{kind}_{veh}_{k}"] = getattr(env.state, k).cpu().numpy()
    s = env.rollout_stats()
    out[f"{kind}_{veh}_frames"] = np.array([s["frames"], s["finished"]])
np.savez(sys.argv[2], **out)
"""


def run(tmp_path, threshold):
    path = tmp_path / f"out_{threshold}.npz"
    env = dict(os.environ, UUV_TASK_PIPE_MIN_ENVS=str(threshold))
    r = subprocess.run([sys.executable, "-c", RUN, ROOT, str(path)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(path)


def test_pipelined_task_kernel_equals_per_env_kernel(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    piped, plain = run(tmp_path, 1), run(tmp_path, 0)
    assert set(piped.files) == set(plain.files)
    for k in plain.files:
        assert np.array_equal(piped[k], plain[k], equal_nan=True), k
    # auto-resets happened (episode_length 7 over 20 steps)
    assert plain["docking_bluerov_heavy_episodes"].max() >= 2
