"""Helper for test_gpu_api.test_pdl_modes_bitwise: a graph-replayed DR rollout whose
commands come from a ring larger than L2; prints a hash of the final state."""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200.randomization import DRParameter, Uniform  # noqa: E402
from paper_2503_09203_b200.vehicles import load_vehicle  # noqa: E402

n = int(sys.argv[1])
spec = {k: DRParameter(k, Uniform(0.8, 1.2)) for k in ("damping*", "mass*", "thrust_coeff*", "volume*")}
st = E.make_batch(load_vehicle("bluerov"), E.SimConfig(batch_size=n), master_seed=0)
E.reset_envs(st, np.ones(n, bool), E.spec_sampler(spec))
g = torch.Generator(device="cuda").manual_seed(0)
ring = torch.rand((64, n, 6), device="cuda", generator=g) * 2 - 1
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for t in range(3):
        E.step_batch(st, ring[t])
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for t in range(64):
            E.step_batch(st, ring[t])
    for _ in range(4):
        graph.replay()
torch.cuda.synchronize()
h = hashlib.sha256()
for k in ("p", "q", "nu", "act", "steps", "diverged"):
    h.update(getattr(st, k).contiguous().cpu().numpy().tobytes())
print(h.hexdigest())
