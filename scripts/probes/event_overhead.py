"""What the bench's event pair costs by itself: device time between e0 and e1 in the
DeviceTimer harness (L2 flush, device-side gate) around nothing, a 1-element fill, a
K-step rollout launched directly and the same launch replayed from a CUDA graph --
with and without the gate.  Means over 50 runs (the event clock ticks in ~1 us)."""
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
tiny = torch.zeros(1, device=dev)

g = torch.cuda.CUDAGraph()
with torch.cuda.stream(stream):
    E.rollout(st, ring, 20, start=3)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=stream), E.no_gc():
        E.rollout(st, ring, 20, start=3)

cases = {
    "empty": lambda: None,
    "fill": lambda: tiny.fill_(1.0),
    "fill_x2": lambda: (tiny.fill_(1.0), tiny.fill_(2.0)),
    "rollout20": lambda: E.rollout(st, ring, 20, start=7),
    "rollout20_graph": lambda: g.replay(),
}
out = {}
for gate in (True, False):
    for name, enq in cases.items():
        timer.run(enq, gate=gate)
        out[f"{name}{'' if gate else '_nogate'}"] = float(
            np.mean([timer.run(enq, gate=gate) for _ in range(50)])) * 1e6
print(json.dumps({"us": out}))
