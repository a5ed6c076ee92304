"""engine.rollout per-step time over batch sizes (cfg2 workload, bench harness: gate + L2
flush + CUDA events, fresh command slots from a ring larger than L2).  For A/B builds of
the rollout kernel: UUV_B200_LIB=<variant .so> python scripts/probes/rollout_sizes.py"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200 import roofline as RF  # noqa: E402
from paper_2503_09203_b200.vehicles import load_vehicle  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
timer = bench.DeviceTimer(dev, stream, lambda: None)
lib = os.environ.get("UUV_B200_LIB", "default")
for n in (4096, 65536, 262144, 1 << 20):
    st = E.make_batch(load_vehicle("bluerov"), E.SimConfig(batch_size=n), master_seed=0,
                      device=dev)
    E.reset_envs(st, torch.ones(n, dtype=torch.bool, device=dev), E.spec_sampler(bench.dr_spec()))
    ring = bench.command_ring(n, 6, dev, torch.Generator(device=dev).manual_seed(0))
    for k in ((20, 200) if n <= 65536 else (20,)):
        def enq(k=k):
            E.rollout(st, ring, k, start=1)
        timer.run(enq)
        t = float(np.mean([timer.run(enq) for _ in range(9)]))
        us = t / k * 1e6
        roof = RF.roofline(us, n, RF.rollout_frame_bytes(6, 4, k), RF.substep_flops("bluerov"))
        print(json.dumps({"lib": os.path.basename(lib), "n": n, "steps": k, "us_per_step": us,
                          "frames_per_s": n / (t / k), "frac": roof["frac"],
                          "bound": roof["bound"]}), flush=True)
    del st, ring
    torch.cuda.empty_cache()
