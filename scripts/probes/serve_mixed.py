import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2503_09203_b200 import _native as N  # noqa: E402
from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200.vehicles import load_vehicle  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
vehs = [load_vehicle(v) for v in ("bluerov", "lauv", "hauv")]
counts = [n // 3, n // 3, n - 2 * (n // 3)]
from paper_2503_09203_b200.randomization import DRParameter, Uniform  # noqa: E402
spec = {k: DRParameter(k, Uniform(0.8, 1.2)) for k in ("mass*", "volume*")}
use_dr = "dr" in sys.argv
other = "other" in sys.argv
st = E.make_fleet_batch(vehs, counts, E.SimConfig(batch_size=n, substeps=2), master_seed=4)
E.reset_envs(st, np.ones(n, bool), E.spec_sampler(spec) if use_dr else E.default_sampler)
if other:
    a = E.make_fleet_batch(vehs, counts, E.SimConfig(batch_size=n, substeps=2), master_seed=4)
    E.reset_envs(a, np.ones(n, bool), E.spec_sampler(spec) if use_dr else E.default_sampler)
cmd = torch.zeros((n, 8)).pin_memory()
srv = E.serve(st, idle_timeout_ms=3000)
srv.__enter__()
time.sleep(0.2)
buf = (ctypes.c_uint64 * 6)()
N.load().uuv_server_stamps(srv._h, buf)
print("after start: idle_ns", buf[4], "start stamp", buf[5], flush=True)
try:
    if other:
        if "side" in sys.argv:
            s2 = torch.cuda.Stream()
            with torch.cuda.stream(s2):
                E.step_batch(a, cmd.cuda())
        else:
            E.step_batch(a, cmd.cuda())
    t0 = time.perf_counter()
    E.step_batch(st, cmd)
    print("step ok", flush=True)
except Exception as e:
    print("step failed after", time.perf_counter() - t0, "s:", e, flush=True)
N.load().uuv_server_stamps(srv._h, buf)
print("stamps", list(buf), flush=True)
time.sleep(0.5)
pass
try:
    srv.__exit__(None, None, None)
except Exception as e:
    print("exit:", e)
