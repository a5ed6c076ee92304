"""Multi-process (gloo, world_size 2) coverage of the sharded path on CPU.

Each rank owns a contiguous global env range, keys its Philox streams by the
global index, steps its shard and contributes rollout sums to one all-reduce.
The union of the shards must equal one un-sharded batch bit for bit (the
reference's worker-invariance contract, engine.py:471-484), and the reduced
statistics must equal the single-process sums.  The per-rank compute here is
the CPU oracle; on the GPU box the same host logic drives the kernels.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_09203_b200.distributed import allreduce_max, allreduce_sum, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _sampler(O, spec):
    def s(i, ep, rng):
        return O.Init(p=rng.uniform(-1, 1, 3), nu=rng.uniform(-0.1, 0.1, 6),
                      overlay=O.draw_overlay(spec, rng))
    return s


def _worker(rank, world, port, n_global, out_dir):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle import uuv_oracle as O
    from paper_2503_09203_b200.randomization import preset
    from paper_2503_09203_b200.vehicles import load_vehicle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    off, cnt = shard_range(n_global, rank, world)
    spec = {k: v for k, v in preset("train").items() if not k.startswith("current")}
    b = O.Batch(load_vehicle("bluerov_heavy"), cnt, seed=7, env_offset=off)
    b.reset(np.ones(cnt, bool), _sampler(O, spec))
    cmds = np.random.default_rng(0).uniform(-1, 1, (n_global, 8))[off:off + cnt]
    for _ in range(5):
        b.step(cmds)
    stats = torch.tensor([b.p.sum(), float(cnt), b.nu.__abs__().sum()], dtype=torch.float64)
    allreduce_sum(stats)
    tmax = allreduce_max(float(rank + 1), "cpu")
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), p=b.p, q=b.q, nu=b.nu, off=off,
             stats=stats.numpy(), tmax=tmax)
    dist.destroy_process_group()


def test_shard_range_partitions():
    for n in (1, 7, 4096, 262144):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and sum(c for _, c in parts) == n
            for (o1, c1), (o2, _) in zip(parts, parts[1:]):
                assert o1 + c1 == o2


def test_two_rank_gloo_shards_equal_single_batch(tmp_path):
    from oracle import uuv_oracle as O
    from paper_2503_09203_b200.randomization import preset
    from paper_2503_09203_b200.vehicles import load_vehicle

    n_global, world = 10, 2
    mp.start_processes(_worker, args=(world, _free_port(), n_global, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    spec = {k: v for k, v in preset("train").items() if not k.startswith("current")}
    ref = O.Batch(load_vehicle("bluerov_heavy"), n_global, seed=7)
    ref.reset(np.ones(n_global, bool), _sampler(O, spec))
    cmds = np.random.default_rng(0).uniform(-1, 1, (n_global, 8))
    for _ in range(5):
        ref.step(cmds)
    for k in ("p", "q", "nu"):
        got = np.concatenate([p[k] for p in parts])
        assert got.tobytes() == getattr(ref, k).tobytes(), k
    want = np.array([ref.p[:5].sum() + ref.p[5:].sum(), float(n_global),
                     np.abs(ref.nu[:5]).sum() + np.abs(ref.nu[5:]).sum()])
    for p in parts:
        assert np.allclose(p["stats"], want, rtol=1e-12)
        assert float(p["tmax"]) == 2.0


_LAUNCHED = r"""
import os, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2503_09203_b200 import distributed as D
ctx = D.init("gloo")
t = torch.tensor([float(ctx.rank + 1), 1.0], dtype=torch.float64)
D.allreduce_sum(t)
off, cnt = D.shard_range(11, ctx.rank, ctx.world)
np.savez(os.path.join(sys.argv[2], f"r{ctx.rank}.npz"), sum=t.numpy(), world=ctx.world,
         rank=ctx.rank, off=off, cnt=cnt, dist=ctx.distributed, tmax=D.allreduce_max(
             float(ctx.rank), "cpu"))
D.finalize(ctx)
"""


def test_launch_and_init_two_cpu_ranks(tmp_path):
    """distributed.launch re-executes a script as two ranks (torch.distributed.run on
    127.0.0.1); distributed.init joins the gloo group from the environment -- the path
    bench.py --gpus N takes, on CPU."""
    from paper_2503_09203_b200 import distributed as D

    script = tmp_path / "w.py"
    script.write_text(_LAUNCHED)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {"CUDA_VISIBLE_DEVICES": ""}
    assert D.launch(str(script), [root, str(tmp_path)], 2, env=env) == 0
    r = [np.load(tmp_path / f"r{k}.npz") for k in range(2)]
    for k, p in enumerate(r):
        assert int(p["rank"]) == k and int(p["world"]) == 2 and bool(p["dist"])
        assert p["sum"].tolist() == [3.0, 2.0] and float(p["tmax"]) == 1.0
    assert [(int(p["off"]), int(p["cnt"])) for p in r] == [(0, 5), (5, 6)]
    ctx = D.init()  # no WORLD_SIZE: a single process, no group
    assert not ctx.distributed and ctx.world == 1
