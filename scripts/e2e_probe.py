"""Break down the host-buffer step path (e2e) into its parts on the GPU box."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200.vehicles import load_vehicle  # noqa: E402

n, A, K = 4096, 6, 500
st = E.make_batch(load_vehicle("bluerov"), E.SimConfig(batch_size=n))
E.reset_envs(st, torch.ones(n, dtype=torch.bool, device="cuda"))
hc = (torch.rand(n, A) * 2 - 1).pin_memory()
ho = torch.empty((13, n)).pin_memory()
dc = hc.cuda()
cur = torch.cuda.current_stream()


def timeit(label, fn):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(K):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / K
    print(f"{label:40s} {dt * 1e6:8.1f} us/step  {n / dt:.3e} frames/s", flush=True)


timeit("device step (no sync)", lambda: E.step_batch(st, dc))
timeit("device step + sync", lambda: (E.step_batch(st, dc), cur.synchronize()))
timeit("H2D only + sync", lambda: (dc.copy_(hc, non_blocking=True), cur.synchronize()))
timeit("D2H only + sync", lambda: (ho.copy_(st._soa[:13, :n], non_blocking=True), cur.synchronize()))
timeit("step_batch(host, pose_out)", lambda: E.step_batch(st, hc, pose_out=ho))
timeit("step_batch(host) no pose", lambda: E.step_batch(st, hc))
