"""Step-server timeline: host ring (stamp 6) -> doorbell seen on the GPU (0) ->
published (1) -> commands read (2) -> physics done (3) -> count-in (4) -> done
flag released (5) -> host sees done (7).  %globaltimer vs host CLOCK_REALTIME:
the offset is only meaningful if the driver keeps them in step (printed raw)."""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ.setdefault("UUV_SERVE_STAMPS", "1")
sys.path.insert(0, '.')
from paper_2503_09203_b200 import _native as N  # noqa: E402
from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200.vehicles import load_vehicle  # noqa: E402

for n in (256, 4096):
    st = E.make_batch(load_vehicle("bluerov"), E.SimConfig(batch_size=n), master_seed=4)
    E.reset_envs(st, np.ones(n, bool))
    cmd = (torch.rand((n, 6)) * 2 - 1).pin_memory()
    out = E.HostStepOut(st)  # the whole step result (p, q, nu, act, steps, diverged)
    rows = []
    with E.serve(st, idle_timeout_ms=2000) as srv:
        for t in range(300):
            E.step_batch(st, cmd, out=out if t % 2 else None)
            b = (ctypes.c_uint64 * 8)()
            N.load().uuv_server_stamps(srv._h, b)
            rows.append([int(b[k]) for k in range(8)])
    r = np.array(rows[20:], dtype=np.int64)
    for label, sel in (("with result", r[1::2]), ("no result", r[0::2])):
        rel = sel[:, [0, 1, 2, 3, 4, 5, 7]] - sel[:, [6]]
        print(n, label, "median ns from host ring: seen, published, cmds, physics, counted, released, host-done:",
              np.median(rel, axis=0).astype(int).tolist(), "total", int(np.median(sel[:, 7] - sel[:, 6])))
