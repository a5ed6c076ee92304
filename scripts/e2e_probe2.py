"""Where the host-buffer step's time goes: Python API vs the C call vs the device."""
import ctypes as C
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_09203_b200 import _native as N  # noqa: E402
from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200.randomization import DRParameter, Uniform  # noqa: E402
from paper_2503_09203_b200.vehicles import load_vehicle  # noqa: E402

n, A, K = int(os.environ.get("N", 4096)), 6, 2000
st = E.make_batch(load_vehicle("bluerov"), E.SimConfig(batch_size=n))
spec = {k: DRParameter(k, Uniform(0.8, 1.2)) for k in ("damping*", "mass*", "thrust_coeff*", "volume*")}
E.reset_envs(st, torch.ones(n, dtype=torch.bool, device="cuda"), E.spec_sampler(spec))
hc = (torch.rand(n, A) * 2 - 1).pin_memory()
ho = torch.empty((13, n)).pin_memory()
dc = hc.cuda()
cur = torch.cuda.current_stream()
lib = N.load()


def timeit(label, fn, k=K):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / k
    print(f"{label:44s} {dt * 1e6:8.2f} us/step  {n / dt:.3e} frames/s", flush=True)


cs = st._cstate()
ctx = st._ctx
args_host = (ctx, C.byref(cs), hc.data_ptr(), A, st._dcmd.data_ptr() if st._dcmd is not None else None,
             ho.data_ptr(), 1, 0.02, st._stream(), 1)
E.step_batch(st, hc, pose_out=ho)  # allocates the staging buffers
args_host = (ctx, C.byref(cs), hc.data_ptr(), A, st._dcmd.data_ptr(), ho.data_ptr(), 1, 0.02,
             st._stream(), 1)
args_dev = (ctx, C.byref(cs), dc.data_ptr(), A, 1, 0.02, st._stream())
f_host, f_dev = lib.uuv_step_host, lib.uuv_step
timeit("C uuv_step (device cmds, no sync)", lambda: f_dev(*args_dev))
timeit("C uuv_step + stream sync", lambda: (f_dev(*args_dev), cur.synchronize()))
timeit("C uuv_step_host (H2D, step, D2H, sync)", lambda: f_host(*args_host))
timeit("step_batch(device cmds)", lambda: E.step_batch(st, dc))
timeit("step_batch(host cmds, pose_out)", lambda: E.step_batch(st, hc, pose_out=ho))
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    E.step_batch(st, dc)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        E.step_batch(st, dc)
timeit("graph replay of 1 step + sync", lambda: (g.replay(), torch.cuda.current_stream().synchronize()))
timeit("H2D 98KB + D2H 213KB + sync (torch)", lambda: (dc.copy_(hc, non_blocking=True),
                                                       ho.copy_(st._soa[:13, :n], non_blocking=True),
                                                       cur.synchronize()))
