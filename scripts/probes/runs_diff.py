import sys
import numpy as np
import torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from conftest import product_vehicle  # noqa: E402
from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200.randomization import preset  # noqa: E402

names = ("bluerov", "bluerov_heavy", "lauv", "iauv", "hauv")
vehs = [product_vehicle(x) for x in names]
n = 140_001
counts = [n // 5 + (1 if i < n % 5 else 0) for i in range(5)]
def make(runs):
    st = E.make_fleet_batch(vehs, counts, E.SimConfig(batch_size=n, substeps=2), master_seed=3)
    E.reset_envs(st, np.ones(n, bool), E.spec_sampler(preset("train")))
    if not runs:
        st._runs, st._cs = None, None
    return st
a, b = make(True), make(False)
g = torch.Generator(device="cuda").manual_seed(0)
for t in range(4):
    c = torch.rand((n, a.a_max), device="cuda", generator=g) * 2 - 1
    E.step_batch(a, c); E.step_batch(b, c)
    d = (a.act - b.act).abs().cpu().numpy()
    A_, B_ = a.act.cpu().numpy(), b.act.cpu().numpy()
    sc = np.abs(B_).max(axis=1); er = d.max(axis=1); r = er / np.maximum(sc, 1e-300)
    k = int(np.argmax(r)); print(t, "worst row", k, "err", er[k], "scale", sc[k], "a", A_[k], "b", B_[k], flush=True)
    starts = np.concatenate([[0], np.cumsum(counts)])
    for ti, name in enumerate(names):
        blk = d[starts[ti]:starts[ti + 1]]
        i = np.unravel_index(np.argmax(blk), blk.shape)
        print(t, name, "max |d act|", blk.max(), "at", i, "a", a.act[starts[ti] + i[0]].cpu().numpy()[:6],
              "b", b.act[starts[ti] + i[0]].cpu().numpy()[:6])
