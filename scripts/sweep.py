"""Throughput sweep of the step kernel over batch size and configuration.

Prints one JSON line per case: device-timed (CUDA events around a CUDA-graph
replay of `steps` launches) frames/s, us/launch, algorithmic GB/s and the
fraction of the measured HBM copy bandwidth.  Used for profiles/, not the
driver's bench line.

    python scripts/sweep.py [--cases cfg2,cfg3,bluerov_1m] [--steps 200]
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200.randomization import DRParameter, Uniform, preset  # noqa: E402
from paper_2503_09203_b200.vehicles import BUILTIN_VEHICLES, load_vehicle  # noqa: E402

from paper_2503_09203_b200 import roofline as RF  # noqa: E402

PEAK = RF.hbm_peak()[0]
FP32_TFLOPS, FP32_SOURCE = RF.fp32_peak()
TASK_FLOPS = RF.TASK_FLOPS
substep_flops = RF.substep_flops
frame_bytes = RF.frame_bytes


def roofline(us_per_step, n, bpf, fpf):
    """Per-step roofline: the slower of n*bpf bytes at the HBM copy bandwidth and
    n*fpf flops at the FP32 peak; frac = roofline time / measured time."""
    t_hbm = n * bpf / (PEAK * 1e9) * 1e6
    t_fp = n * fpf / (FP32_TFLOPS * 1e12) * 1e6
    return {"flops_per_frame": fpf, "tflops": n * fpf / us_per_step / 1e6,
            "frac_fp32": t_fp / us_per_step, "roofline_us": max(t_hbm, t_fp),
            "bound": "hbm" if t_hbm >= t_fp else "fp32",
            "frac_roofline": max(t_hbm, t_fp) / us_per_step,
            "fp32_peak_tflops": FP32_TFLOPS, "fp32_peak_source": FP32_SOURCE}


def make_case(name, n):
    dev = torch.device("cuda", 0)
    if name == "cfg3":  # five vehicles mixed, no DR
        vehs = [load_vehicle(v) for v in BUILTIN_VEHICLES]
        counts = [n // 5 + (1 if i < n % 5 else 0) for i in range(5)]
        st = E.make_fleet_batch(vehs, counts, E.SimConfig(batch_size=n), device=dev)
        E.reset_envs(st, torch.ones(n, dtype=torch.bool, device=dev))
        a_mean = sum(v.action_dim * c for v, c in zip(vehs, counts)) / n
        width = st.a_max
        bpf = frame_bytes(a_mean, 0, False, mixed=True)
        fpf = sum(substep_flops(v.name) * c for v, c in zip(vehs, counts)) / n
    elif name.startswith("cfg2") or name.startswith("bluerov"):
        veh = load_vehicle("bluerov")
        substeps = 8 if name.endswith("k8") else 1
        st = E.make_batch(veh, E.SimConfig(batch_size=n, substeps=substeps), device=dev)
        keys = ("damping*", "mass*", "thrust_coeff*", "volume*") if name.startswith("cfg2") else ()
        spec = {k: DRParameter(k, Uniform(0.8, 1.2)) for k in keys}
        E.reset_envs(st, torch.ones(n, dtype=torch.bool, device=dev),
                     E.spec_sampler(spec or None))
        width = 6
        bpf = frame_bytes(6, len(keys), False)
        fpf = substep_flops("bluerov") * substeps
    elif name.startswith("veh:"):  # one vehicle, no DR: veh:<name>
        veh = load_vehicle(name[4:])
        st = E.make_batch(veh, E.SimConfig(batch_size=n), device=dev)
        E.reset_envs(st, torch.ones(n, dtype=torch.bool, device=dev))
        width = veh.action_dim
        bpf = frame_bytes(width, 0, False)
        fpf = substep_flops(name[4:])
    elif name == "cfg5_physics":  # bluerov_heavy + train preset (7 ratios) + current
        veh = load_vehicle("bluerov_heavy")
        st = E.make_batch(veh, E.SimConfig(batch_size=n), device=dev)
        E.reset_envs(st, torch.ones(n, dtype=torch.bool, device=dev),
                     E.spec_sampler(preset("train")))
        width = 8
        bpf = frame_bytes(8, 7, True)
        # payload / cobm draws move r_g: counted with the general formulation
        fpf = substep_flops("bluerov_heavy", current=True, general=True)
    else:
        raise ValueError(name)
    return st, width, bpf, fpf


def measure_task(name, n, steps):
    """Fused task step (physics + obs/reward/termination/auto-reset) per env.step call."""
    from paper_2503_09203_b200.tasks import TaskConfig, make_env

    dev = torch.device("cuda", 0)
    if name == "task_cfg4":  # tracking with ocean current, 8 fused substeps
        task = TaskConfig(task="tracking", vehicle="bluerov", level="disturbed")
        env = make_env(task, E.SimConfig(batch_size=n, substeps=8), seed=0, device=dev)
        a = 6
        # physics 198 B (current) + task: obs 4*(12+6+3), reward 4, term/trunc 2,
        # prev_u 8*6, _dev_sum 8; flops 8 substeps + task layer
        bpf = frame_bytes(6, 0, True) + 4 * (12 + 6 + 3) + 4 + 2 + 8 * 6 + 8
        fpf = 8 * substep_flops("bluerov", current=True) + TASK_FLOPS
    else:  # task_cfg5: docking, train-preset DR, auto-reset on
        task = TaskConfig(task="docking", vehicle="bluerov_heavy", level="disturbed_dr")
        env = make_env(task, E.SimConfig(batch_size=n), seed=0, device=dev)
        a = 8
        # physics 278 B (train DR: 7 ratios + current) + obs 4*(12+8+1), reward 4,
        # term/trunc 2, prev_u 8*8
        bpf = frame_bytes(8, 7, True) + 4 * (12 + 8 + 1) + 4 + 2 + 8 * 8
        fpf = substep_flops("bluerov_heavy", current=True, general=True) + TASK_FLOPS
    env.reset()
    cmds = torch.rand((n, a), device=dev) * 2 - 1
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for _ in range(3):
            env.step(cmds)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(steps):
                env.step(cmds)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(3):
        with torch.cuda.stream(s):
            e0.record(s)
            g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / steps
        best = t if best is None else min(best, t)
    stats = env.rollout_stats()
    gbs = n * bpf / best / 1e9
    return {"case": name, "n": n, "us_per_step": best * 1e6, "frames_per_s": n / best,
            "bytes_per_frame": bpf, "gbs": gbs, "frac_hbm": gbs / PEAK,
            **roofline(best * 1e6, n, bpf, fpf),
            "finished_per_frame": stats["finished"] / max(stats["frames"], 1)}


def measure(name, n, steps):
    if name.startswith("task_"):
        return measure_task(name, n, steps)
    st, width, bpf, fpf = make_case(name, n)
    dev = st.device
    cmds = torch.rand((n, width), device=dev) * 2 - 1
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for _ in range(5):
            E.step_batch(st, cmds)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(steps):
                E.step_batch(st, cmds)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(3):
        with torch.cuda.stream(s):
            e0.record(s)
            g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / steps
        best = t if best is None else min(best, t)
    gbs = n * bpf / best / 1e9
    return {"case": name, "n": n, "us_per_step": best * 1e6, "frames_per_s": n / best,
            "bytes_per_frame": bpf, "gbs": gbs, "frac_hbm": gbs / PEAK,
            **roofline(best * 1e6, n, bpf, fpf),
            "diverged": int(st.diverged.sum().item())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="cfg2,cfg3,bluerov,cfg5_physics,cfg2_k8")
    ap.add_argument("--sizes", default="4096,65536,262144,1048576,4194304")
    ap.add_argument("--steps", type=int, default=100)
    args = ap.parse_args()
    for case in args.cases.split(","):
        for n in (int(x) for x in args.sizes.split(",")):
            print(json.dumps(measure(case, n, args.steps)), flush=True)


if __name__ == "__main__":
    main()
