import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2503_09203_b200 import engine as E
from paper_2503_09203_b200.vehicles import load_vehicle
from paper_2503_09203_b200.randomization import DRParameter, Uniform
n = 3000
vehs = [load_vehicle(v) for v in ("bluerov", "lauv", "hauv")]
spec = {k: DRParameter(k, Uniform(0.8, 1.2)) for k in ("mass*", "volume*")}
def make():
    counts = [n // 3, n // 3, n - 2 * (n // 3)]
    st = E.make_fleet_batch(vehs, counts, E.SimConfig(batch_size=n, substeps=2), master_seed=4, dtype=torch.float32)
    E.reset_envs(st, np.ones(n, bool), E.spec_sampler(spec))
    return st
a, b = make(), make()
w = E._cmd_width(a)
g = torch.Generator().manual_seed(1)
cmds = [(torch.rand((n, w), generator=g, dtype=torch.float64) * 2 - 1).float().pin_memory() for _ in range(6)]
cmds[4][5, 0] = float("nan")
out = torch.empty((13, n)).pin_memory()
torch.equal(out, torch.cat([a.p, a.q, a.nu], dim=1).T.cpu())
def cmp(tag):
    want = torch.cat([a.p, a.q, a.nu], dim=1).T.cpu()
    bad = (out != want).any(0).nonzero().flatten().tolist()
    if bad:
        print(tag, "bad rows", bad[:10], len(bad))
        for r in bad[:3]:
            print(" row", r, "a", want[:, r].tolist()[:7], "\n      b", out[:, r].tolist()[:7], "div", int(a.diverged[r]), int(b.diverged[r]))
with E.serve(b):
    for t in range(6):
        E.step_batch(a, cmds[t].cuda()); E.step_batch(b, cmds[t], pose_out=out)
        cmp(f"t{t}")
    E.step_batch(b, np.asarray(cmds[0])); E.step_batch(a, cmds[0].cuda())
    reuse = torch.empty_like(cmds[0]).pin_memory()
    for t in range(30):
        reuse.copy_(cmds[t % 6] * (1.0 - 0.01 * t))
        E.step_batch(a, reuse.cuda()); E.step_batch(b, reuse, pose_out=out)
        cmp(f"reuse{t}")
print("div a", a.diverged.nonzero().flatten().tolist(), "b", b.diverged.nonzero().flatten().tolist())
