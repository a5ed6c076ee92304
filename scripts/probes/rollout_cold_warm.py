"""Why a K-step rollout runs slower per step after the bench's L2 flush than warm
(cfg2, 4096 envs): per-step slope over K for (1) write flush (the bench), (2) write
flush followed by a read pass over another buffer > L2 (L2 left clean), (3) no flush
but fresh ring slots every launch, (4) no flush, the same slots (warm)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200.vehicles import load_vehicle  # noqa: E402

dev = torch.device("cuda", 0)
n = 4096
st = E.make_batch(load_vehicle("bluerov"), E.SimConfig(batch_size=n), master_seed=0, device=dev)
E.reset_envs(st, torch.ones(n, dtype=torch.bool, device=dev), E.spec_sampler(bench.dr_spec()))
ring = bench.command_ring(n, 6, dev, torch.Generator(device=dev).manual_seed(0))
S = ring.shape[0]
stream = torch.cuda.Stream(dev)
timer = bench.DeviceTimer(dev, stream, lambda: None)
clean = torch.ones(256 << 20, dtype=torch.uint8, device=dev)
ks = [5, 20, 50, 100, 200]
out = {}
pos = [0]


def run(mode, k):
    def enq():
        E.rollout(st, ring, k, start=start)
    vals = []
    for _ in range(9):
        if mode == "fresh_slots":
            pos[0] = (pos[0] + k) % S
            start = pos[0]
        else:
            start = 7
        if mode == "write_then_read_flush":
            with torch.cuda.stream(stream):
                timer.flush.fill_(1)
                clean.sum()
            vals.append(timer.run(enq, flush=False))
        else:
            vals.append(timer.run(enq, flush=(mode == "write_flush")))
    return float(np.median(vals[1:])) * 1e6


fits = {}
for mode in ("write_flush", "write_then_read_flush", "fresh_slots", "warm"):
    us = [run(mode, k) for k in ks]
    out[mode] = dict(zip(map(str, ks), us))
    slope, icpt = np.polyfit(ks, us, 1)
    fits[mode] = {"per_step_us": slope, "fixed_us": icpt}
print(json.dumps({"us": out, "fit": fits}))
