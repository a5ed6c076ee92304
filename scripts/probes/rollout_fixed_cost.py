"""Fixed vs per-step cost of one engine.rollout launch (cfg2, 4096 envs): device time of
a K-step rollout for several K with the bench's gate, L2 flushed before each launch
(cold) or not (warm: state and code left in L2 by the previous launch); a linear fit
gives the per-launch constant and the per-step slope."""
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
stream = torch.cuda.Stream(dev)
timer = bench.DeviceTimer(dev, stream, lambda: None)
ks = [1, 2, 5, 10, 20, 50, 100, 200]
out, fits = {}, {}
for mode in ("cold", "warm"):
    us = []
    for k in ks:
        def enq(k=k):
            E.rollout(st, ring, k, start=7)
        timer.run(enq)
        t = float(np.median([timer.run(enq, flush=(mode == "cold")) for _ in range(7)])) * 1e6
        out[f"{mode}_{k}"] = t
        us.append(t)
    slope, icpt = np.polyfit(ks, us, 1)
    fits[mode] = {"per_step_us": slope, "fixed_us": icpt}
# reference points in the same harness: one step_batch launch, and a 1-element torch fill
# (event + launch overhead of any kernel)
tiny = torch.zeros(1, device=dev)
for name, enq in (("step_batch_1", lambda: E.step_batch(st, ring[3])),
                  ("torch_fill_1", lambda: tiny.fill_(1.0))):
    timer.run(enq)
    out[name] = float(np.mean([timer.run(enq) for _ in range(50)])) * 1e6
for k in (1, 20):  # means over 50 launches (the event clock ticks in ~1 us steps)
    def enq(k=k):
        E.rollout(st, ring, k, start=7)
    out[f"mean50_cold_{k}"] = float(np.mean([timer.run(enq) for _ in range(50)])) * 1e6
print(json.dumps({"us": out, "fit": fits}))
