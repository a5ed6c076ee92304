"""Step-server probe: per-step latency and failure diagnosis (small, bounded)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200.randomization import DRParameter, Uniform  # noqa: E402
from paper_2503_09203_b200.vehicles import load_vehicle  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
spec = {k: DRParameter(k, Uniform(0.8, 1.2)) for k in ("mass*", "volume*")}
st = E.make_batch(load_vehicle("bluerov"), E.SimConfig(batch_size=n, substeps=2), master_seed=4)
E.reset_envs(st, np.ones(n, bool), E.spec_sampler(spec))
cmd = (torch.rand((n, 6)) * 2 - 1).pin_memory()
out = torch.empty((13, n)).pin_memory()
lat = []
import ctypes
import os
os.environ.setdefault("UUV_SERVE_STAMPS", "1")
from paper_2503_09203_b200 import _native as N
stamps = []
with E.serve(st, idle_timeout_ms=2000) as srv:
    for t in range(steps):
        if t == steps - 1:
            time.sleep(0.001)
        t0 = time.perf_counter()
        try:
            E.step_batch(st, cmd, pose_out=out)
        except Exception as e:
            print("step", t, "failed:", e, "done flags:", flush=True)
            import ctypes
            raise
        lat.append(time.perf_counter() - t0)
        buf = (ctypes.c_uint64 * 6)()
        N.load().uuv_server_stamps(srv._h, buf)
        stamps.append([buf[k] - buf[0] for k in range(5)])
lat = np.array(lat[5:]) * 1e6
sp = np.array(stamps[5:])
print("CTA0 phases (ns from doorbell seen): cmds read, physics, after count-in:", np.median(sp, axis=0)[1:4])
print(f"n={n} steps={steps} median {np.median(lat):.2f} us  p90 {np.percentile(lat, 90):.2f}  max {lat.max():.1f}")
