"""The product's multi-rank path on one GPU: two ranks (torch.distributed.run, gloo, both
on GPU 0) each step their global-index shard through the kernels; the union of the shards
equals one un-sharded batch bit for bit (the reference's worker invariance,
engine.py:471-484) and the all-reduced rollout statistics equal the single-process ones.
On the 8-GPU box the same code runs one rank per GPU over NCCL (bench.py --gpus N)."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_2503_09203_b200 import engine as E
from paper_2503_09203_b200.distributed import free_port
from paper_2503_09203_b200.randomization import preset
from paper_2503_09203_b200.tasks import TaskConfig, make_env
from paper_2503_09203_b200.vehicles import load_vehicle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_two_ranks_of_the_product_equal_one_batch(tmp_path):
    n_global, steps = 3001, 12  # an odd split: 1500 + 1501 rows
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           os.path.join(ROOT, "tests", "multirank_worker.py"), str(tmp_path), str(n_global),
           str(steps)]
    env = dict(os.environ, UUV_DIST_BACKEND="gloo")
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    parts = [np.load(tmp_path / f"rank{k}.npz") for k in range(2)]
    assert [int(p["world"]) for p in parts] == [2, 2]
    assert int(parts[0]["off"]) == 0 and int(parts[1]["off"]) == n_global // 2
    # one process, one batch
    st = E.make_batch(load_vehicle("bluerov_heavy"), E.SimConfig(batch_size=n_global),
                      master_seed=7)
    E.reset_envs(st, np.ones(n_global, bool), E.spec_sampler(preset("train")))
    cmds = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, (steps, n_global, 8))).float()
    for t in range(steps):
        E.step_batch(st, cmds[t].cuda())
    for k in ("p", "q", "nu", "act"):
        whole = getattr(st, k).cpu().numpy()
        assert np.array_equal(np.concatenate([p[k] for p in parts]), whole), k
    envd = make_env(TaskConfig(task="docking", vehicle="bluerov_heavy", level="disturbed_dr",
                               episode_length=20), E.SimConfig(batch_size=n_global), seed=3)
    envd.reset()
    for t in range(3 * steps):
        envd.step(cmds[t % steps].cuda())
    assert np.array_equal(np.concatenate([p["ep"] for p in parts]),
                          envd.state.episodes.cpu().numpy())
    assert np.array_equal(np.concatenate([p["tp"] for p in parts]), envd.state.p.cpu().numpy())
    stats = envd.rollout_stats()
    want = np.array([stats[k] for k in sorted(stats)])
    for p in parts:  # every rank holds the all-reduced sums
        assert np.allclose(p["stats"], want, rtol=1e-12, atol=0), (p["stats"], want)
    assert want[sorted(stats).index("frames")] == 3 * steps * n_global
