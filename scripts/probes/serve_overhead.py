"""Served-step cost split: step_batch (Python) vs the bare C call vs GPU-side phases."""
import ctypes
import os
os.environ.setdefault("UUV_SERVE_STAMPS", "1")
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2503_09203_b200 import _native as N  # noqa: E402
from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200.randomization import DRParameter, Uniform  # noqa: E402
from paper_2503_09203_b200.vehicles import load_vehicle  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
K = 3000
spec = {k: DRParameter(k, Uniform(0.8, 1.2)) for k in ("damping*", "mass*", "thrust_coeff*", "volume*")}
st = E.make_batch(load_vehicle("bluerov"), E.SimConfig(batch_size=n), master_seed=0)
E.reset_envs(st, np.ones(n, bool), E.spec_sampler(spec))
cmd = (torch.rand((n, 6)) * 2 - 1).pin_memory()
out = torch.empty((13, n)).pin_memory()
lib = N.load()
with E.serve(st) as srv:
    ring = (torch.rand((1000, n, 6)) * 2 - 1).pin_memory()  # a fresh buffer per step, as bench.py
    t0 = time.perf_counter()
    for k in range(1000):
        E.step_batch(st, ring[k], pose_out=out)
    print(f"n={n} step_batch, 1000-buffer ring {1e6 * (time.perf_counter() - t0) / 1000:7.2f} us/step",
          flush=True)
    import glob
    import os
    libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
        glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                               "libcudart.so*"))
    if libs:
        cr = ctypes.CDLL(libs[0])
        at = (ctypes.c_char * 64)()
        ptrs = [ring[k].data_ptr() for k in range(1000)]
        t0 = time.perf_counter()
        for pt in ptrs:
            cr.cudaPointerGetAttributes(at, ctypes.c_void_p(pt))
        print(f"cudaPointerGetAttributes per new address: {1e6 * (time.perf_counter() - t0) / 1000:.2f} us",
              flush=True)
    t0 = time.perf_counter()
    for k in range(1000):
        E.step_batch(st, ring[k], pose_out=out)
    print(f"n={n} step_batch, ring again {1e6 * (time.perf_counter() - t0) / 1000:7.2f} us/step",
          flush=True)
    for mode in ("step_batch", "C call", "C call, no pose"):
        h, cp, op = srv._h, cmd.data_ptr(), out.data_ptr()
        f = lib.uuv_server_step
        if mode == "step_batch":
            fn = lambda: E.step_batch(st, cmd, pose_out=out)  # noqa: E731
        elif mode == "C call":
            fn = lambda: f(h, cp, 6, op)  # noqa: E731
        else:
            fn = lambda: f(h, cp, 6, None)  # noqa: E731
        for _ in range(100):
            fn()
        t0 = time.perf_counter()
        for _ in range(K):
            fn()
        dt = (time.perf_counter() - t0) / K * 1e6
        print(f"n={n} {mode:18s} {dt:7.2f} us/step", flush=True)
    rows = []
    for _ in range(500):
        lib.uuv_server_step(srv._h, cmd.data_ptr(), 6, out.data_ptr())
        b = (ctypes.c_uint64 * 8)()
        lib.uuv_server_stamps(srv._h, b)
        ring = b[6]
        rows.append([b[0] - ring, b[1] - ring, b[2] - ring, b[3] - ring, b[4] - ring, b[5] - ring,
                     b[7] - ring])
    med = np.median(np.array(rows, dtype=np.int64), axis=0)
    print("ns after host ring: detect, acq fence, cmds read, physics (CTA0), sysfence begin,"
          " end (last CTA), host sees done:", med.tolist(), flush=True)
