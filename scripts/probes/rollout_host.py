"""Host-to-host rollout (engine.rollout with pinned host commands / trace), cfg2 4096 envs:
host-clock time per call over K, for the trace written by the kernel over the host link
(13 + A rows, 13 rows, none) and for the device trace moved by one DMA copy afterwards;
plus plain pinned-memory DMA copy rates for the same byte counts.  Median of 7 calls."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200.vehicles import load_vehicle  # noqa: E402

dev = torch.device("cuda", 0)
n, A = 4096, 6
st = E.make_batch(load_vehicle("bluerov"), E.SimConfig(batch_size=n), master_seed=0, device=dev)
E.reset_envs(st, torch.ones(n, dtype=torch.bool, device=dev), E.spec_sampler(bench.dr_spec()))
cur = torch.cuda.current_stream(dev)


def timed(fn, reps=7):
    fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        fn()
        cur.synchronize()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)) * 1e6


out = {}
for k in (20, 50, 100, 200):
    hc = (torch.rand(k, n, A) * 2 - 1).pin_memory()
    dc = hc.to(dev)
    ht19 = torch.empty((k, 19, n)).pin_memory()
    ht13 = torch.empty((k, 13, n)).pin_memory()
    dt19 = torch.empty((k, 19, n), device=dev)
    out[f"host19_{k}"] = timed(lambda: E.rollout(st, hc, k, trace=ht19))
    out[f"host13_{k}"] = timed(lambda: E.rollout(st, hc, k, trace=ht13))
    out[f"hostcmd_notrace_{k}"] = timed(lambda: E.rollout(st, hc, k))
    out[f"dev_notrace_{k}"] = timed(lambda: E.rollout(st, dc, k))

    def dma():
        dc.copy_(hc, non_blocking=True)
        E.rollout(st, dc, k, trace=dt19)
        ht19.copy_(dt19, non_blocking=True)
    out[f"dma19_{k}"] = timed(dma)
    out[f"memcpy_d2h_19_{k}"] = timed(lambda: ht19.copy_(dt19, non_blocking=True))
    out[f"memcpy_h2d_cmd_{k}"] = timed(lambda: dc.copy_(hc, non_blocking=True))
fits = {}
for key in ("host19", "host13", "hostcmd_notrace", "dev_notrace", "dma19", "memcpy_d2h_19"):
    ks = [20, 50, 100, 200]
    slope, icpt = np.polyfit(ks, [out[f"{key}_{k}"] for k in ks], 1)
    fits[key] = {"us_per_step": slope, "fixed_us": icpt}
fits["d2h_GBps_host19"] = 19 * 4 * n / fits["host19"]["us_per_step"] / 1e3
fits["d2h_GBps_memcpy"] = 19 * 4 * n / fits["memcpy_d2h_19"]["us_per_step"] / 1e3
print(json.dumps({"us": out, "fit": fits}))
