"""Event + launch overhead of the bench harness (gate spin, L2 flush, start event, work,
end event): a 1-element fill and a 20-step rollout, launched directly or as a one-node
CUDA graph, mean over 50 timed runs each."""
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


def graph_of(fn):
    with torch.cuda.stream(stream):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream), torch.cuda.graph(g, stream=stream), E.no_gc():
        fn()
    return g


cases = {
    "fill_direct": lambda: tiny.fill_(1.0),
    "rollout20_direct": lambda: E.rollout(st, ring, 20, start=3),
}
g_fill = graph_of(cases["fill_direct"])
g_roll = graph_of(cases["rollout20_direct"])
cases["fill_graph"] = g_fill.replay
cases["rollout20_graph"] = g_roll.replay
out = {}
for name, fn in cases.items():
    timer.run(fn)
    out[name] = float(np.mean([timer.run(fn) for _ in range(50)])) * 1e6
print(json.dumps(out))
