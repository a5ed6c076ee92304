"""Multi-GPU: one process per GPU, env-range shards, the rollout-statistics all-reduce.

Environments are independent, so a job shards by contiguous
global env ranges with no data-path collective: rank r owns
[offset_r, offset_r + n_r) and keys its random streams by the GLOBAL index,
which makes every trajectory independent of the GPU count (the reference's
worker-invariance contract, engine.py:471-484, where ``workers`` threads split
contiguous ranges).  The only collective is one all-reduce of ~8 float64
rollout statistics per rollout (NCCL over NVLink/NVSwitch on the GPU box, gloo
in the CPU tests) -- SURVEY.md §8(e).

    ctx = distributed.init()                     # RANK / WORLD_SIZE / LOCAL_RANK
    batch = distributed.make_shard(vehicle, n_global, sim, ctx, master_seed=0)
    ... step_batch(batch, commands_for_my_rows) ...
    stats = env.rollout_stats()                  # all-reduced over ctx's group

``launch`` re-executes a script under ``torch.distributed.run`` (one rank per
GPU, rendezvous on 127.0.0.1) for callers started as a single process.
"""

from __future__ import annotations

import os
import socket
import subprocess
import sys
from dataclasses import dataclass

import torch


@dataclass
class DistContext:
    rank: int
    world: int
    local_rank: int
    device: torch.device
    backend: str | None  # None: single process, no process group

    @property
    def distributed(self) -> bool:
        return self.backend is not None

    def barrier(self):
        if self.distributed:
            torch.distributed.barrier()


def shard_range(n_global: int, rank: int, world: int) -> tuple:
    """(offset, count) of rank's contiguous slice; same split as np.linspace bounds."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = (n_global * rank) // world
    hi = (n_global * (rank + 1)) // world
    return lo, hi - lo


def init(backend: str | None = None, device_index: int | None = None) -> DistContext:
    """Join the process group described by the torchrun environment variables.

    One process per GPU: rank r uses GPU ``LOCAL_RANK`` (``device_index``
    overrides, e.g. to put several ranks on one GPU in tests).  ``backend``
    defaults to NCCL when CUDA is available, else gloo.  With WORLD_SIZE unset
    or 1 no process group is created.
    """
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cuda = torch.cuda.is_available()
    if cuda:
        idx = local if device_index is None else device_index
        if idx >= torch.cuda.device_count():
            raise RuntimeError(f"rank {rank}: GPU {idx} requested, {torch.cuda.device_count()} "
                               "visible (one process per GPU)")
        dev = torch.device("cuda", idx)
        torch.cuda.set_device(dev)
    else:
        dev = torch.device("cpu")
    if world <= 1:
        return DistContext(rank, world, local, dev, None)
    backend = backend or ("nccl" if cuda else "gloo")
    if not torch.distributed.is_initialized():
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=dev)
        else:
            torch.distributed.init_process_group(backend)
    return DistContext(rank, world, local, dev, backend)


def finalize(ctx: DistContext):
    if ctx.distributed and torch.distributed.is_initialized():
        torch.distributed.destroy_process_group()


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch(script: str, argv: list, nproc: int, env: dict | None = None) -> int:
    """Run ``script argv`` as ``nproc`` ranks of one node (torch.distributed.run, rendezvous
    on 127.0.0.1); returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", script, *argv]
    full = dict(os.environ)
    full.update(env or {})
    return subprocess.run(cmd, env=full).returncode


def make_shard(vehicle, n_global: int, sim, ctx: DistContext, **kw):
    """This rank's batch of a job of ``n_global`` envs: rows [offset, offset + count) of the
    global batch, random streams keyed by the global index (env_offset)."""
    from dataclasses import replace

    from .engine import make_batch

    off, cnt = shard_range(n_global, ctx.rank, ctx.world)
    return make_batch(vehicle, replace(sim, batch_size=cnt), device=ctx.device,
                      env_offset=off, **kw)


def dist_ready(group=None) -> bool:
    return torch.distributed.is_available() and torch.distributed.is_initialized()


def allreduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    """Sum ``t`` over the process group in place (no-op when not distributed);
    stream-ordered on the current stream for NCCL, no host synchronisation.  A CUDA
    tensor under gloo (the multi-rank tests on one GPU) is reduced through the host."""
    if dist_ready(group):
        if t.is_cuda and torch.distributed.get_backend(group) == "gloo":
            h = t.cpu()
            torch.distributed.all_reduce(h, op=torch.distributed.ReduceOp.SUM, group=group)
            t.copy_(h)
        else:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.SUM, group=group)
    return t


def allreduce_max(x: float, device, group=None) -> float:
    """Max of a host scalar over ranks (used for device-timed max-over-ranks)."""
    if not dist_ready(group):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX, group=group)
    return float(t.item())
