"""Benchmark: env frames/s of the batched 6-DOF Fossen step (hydro + thruster + integrate).

Workload (BASELINE.json configs[1]): BlueROV2, 4096 envs per GPU, per-env
domain-randomised mass / volume / damping / thruster gain ~ U[0.8, 1.2] drawn
on device from the Philox stream keyed (seed 0, global env, episode 0),
commands U(-1, 1).  A step is one control step (one ``uuv_step`` launch).

* value — device-resident throughput: K steps replayed from a CUDA graph,
  CUDA events on the launching stream, barrier + max over ranks.  Each step
  reads a fresh command buffer from a ring larger than L2 (env state stays
  resident, as in an RL loop); L2 is flushed once before the timed region.
* e2e — the same metric through the public API with HOST buffers:
  ``step_batch(state, pinned_host_commands, pose_out=pinned_host_pose)`` per
  step: the step's commands go host->device and its p, q, nu rows
  device->host, and the call returns when they are in host memory.  Two
  paths are timed and the faster is reported (both in ``e2e.per_path``): one
  launch per step whose kernel reads/writes the mapped pinned buffers over the
  link (CUDA events), and the same calls inside ``engine.serve(state)``, where a
  resident step kernel is driven by a doorbell in mapped pinned memory (no
  launch, no stream sync per step; host clock around exactly K synchronous
  steps).
* roofline — the step kernel's algorithmic bytes per launch / average launch
  duration vs the measured HBM copy bandwidth (MEASURED_PEAKS.json).  At
  4096 envs the step is launch/latency-bound, so ``roofline_at_scale`` also
  reports the same kernel on 1,048,576 envs of the same workload (informational;
  not the bench value).
* cpu_baseline — the CPU oracle (numpy restatement of the reference) on the
  same workload on this box's host cores (rank 0, N = 1 only).

``--impl reference`` runs the reference's CPU algorithm (the oracle port; the
reference is pure numpy and cannot be installed here) on the same workload.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_ENVS = 4096
A_BLUEROV = 6
DR_KEYS = ("damping*", "mass*", "thrust_coeff*", "volume*")
METRIC = "env frames/sec (hydro+thruster+integrate)"
WORKLOAD = ("cfg2: BlueROV2 station-keeping dynamics, 4096 envs/GPU, per-env DR "
            "mass/volume/damping/thrust_coeff ~ U[0.8,1.2] (Philox, device), cmds U(-1,1)")


def algorithmic_bytes_per_frame(a=A_BLUEROV, n_dr=len(DR_KEYS), dtype_bytes=4):
    """state p,q,nu,act read+write, commands read, diverged r/w (1+1 B),
    steps r/w (4+4 B), plus the float64 DR record actually read (8 B per key)."""
    return dtype_bytes * (2 * (13 + a) + a) + 2 + 8 + 8 * n_dr


def dr_spec():
    from paper_2503_09203_b200.randomization import DRParameter, Uniform

    return {k: DRParameter(k, Uniform(0.8, 1.2)) for k in DR_KEYS}


def load_traffic():
    """DRAM bytes per launch of the step kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t["dram_bytes_read"] + t["dram_bytes_write"]
    except Exception:
        return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the GPU is under load."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in getattr(self, "lines", []):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ================================================================ reference (CPU) arm


def cpu_probe(seconds=None, steps=None, warmup=3, workers=None):
    """The oracle on the cfg2 workload: returns (frames/s, steps, elapsed, cores, reset_s)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import uuv_oracle as O
    from paper_2503_09203_b200.vehicles import load_vehicle

    workers = workers or os.cpu_count() or 1
    veh = load_vehicle("bluerov")
    spec = dr_spec()
    b = O.Batch(veh, N_ENVS, 0.02, 1, seed=0, workers=workers)
    t0 = time.perf_counter()
    b.reset(np.ones(N_ENVS, bool), lambda i, ep, r: O.Init(overlay=O.draw_overlay(spec, r)))
    reset_s = time.perf_counter() - t0
    cmds = np.random.default_rng(0).uniform(-1.0, 1.0, (N_ENVS, A_BLUEROV))
    pool = ThreadPoolExecutor(max_workers=workers) if workers > 1 else None
    for _ in range(warmup):
        b.step(cmds, pool)
    k = 0
    t0 = time.perf_counter()
    while True:
        b.step(cmds, pool)
        k += 1
        el = time.perf_counter() - t0
        if (steps is not None and k >= steps) or (seconds is not None and el >= seconds):
            break
    if pool is not None:
        pool.shutdown()
    return N_ENVS * k / el, k, el, workers, reset_s


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    fps, k, el, cores, reset_s = cpu_probe(steps=args.steps, warmup=args.warmup)
    sample = (f"full cfg2 workload ({N_ENVS} envs x {k} steps) on {cores} host threads; "
              f"DR reset of {N_ENVS} envs took {reset_s:.2f} s (excluded)")
    line = {"metric": METRIC, "value": fps, "unit": "env-frames/s", "n_gpus": args.gpus,
            "steps": k, "warmup": args.warmup, "ms_per_step": 1e3 * el / k,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOAD, "global_batch": N_ENVS, "parallelism": "cpu"},
            "cpu_baseline": {"value": fps, "unit": "env-frames/s", "cores": cores,
                             "kind": "port", "sample": sample},
            "e2e": {"value": fps, "unit": "env-frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ================================================================ B200 arm


def run_b200(args, rank, world, local_rank):
    import torch

    from paper_2503_09203_b200 import engine as E
    from paper_2503_09203_b200.distributed import allreduce_max, shard_range
    from paper_2503_09203_b200.vehicles import load_vehicle

    # one process per GPU; UUV_BENCH_GPU_OVERRIDE=0 pins every rank to GPU 0 and
    # UUV_DIST_BACKEND=gloo swaps NCCL for gloo (used to exercise the multi-rank
    # path on a single-GPU box; the driver's runs use one GPU per rank over NCCL)
    dev_index = int(os.environ.get("UUV_BENCH_GPU_OVERRIDE", local_rank))
    dev = torch.device("cuda", dev_index)
    torch.cuda.set_device(dev)
    dist = world > 1
    if dist:
        backend = os.environ.get("UUV_DIST_BACKEND", "nccl")
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=dev)
        else:
            torch.distributed.init_process_group(backend)

    def barrier():
        if dist:
            torch.distributed.barrier()

    veh = load_vehicle("bluerov")
    n = N_ENVS
    offset = rank * n  # weak scaling: each GPU owns 4096 globally-indexed envs
    st = E.make_batch(veh, E.SimConfig(batch_size=n), master_seed=0, device=dev,
                      env_offset=offset)
    E.reset_envs(st, torch.ones(n, dtype=torch.bool, device=dev), E.spec_sampler(dr_spec()))

    # command ring larger than L2 (126 MB): every timed step reads fresh inputs
    ring_bytes = 160 << 20
    per = n * A_BLUEROV * 4
    n_ring = max(2, ring_bytes // per)
    gen = torch.Generator(device=dev).manual_seed(offset)
    ring = torch.rand((n_ring, n, A_BLUEROV), device=dev, generator=gen) * 2 - 1
    stream = torch.cuda.Stream(dev)
    k_total = args.steps

    def capture(k, start):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            with torch.cuda.graph(g, stream=stream):
                for s in range(k):
                    E.step_batch(st, ring[(start + s) % n_ring])
        return g

    torch.cuda.synchronize(dev)
    # warmup (untimed), graph capture of exactly K steps in chunks
    with torch.cuda.stream(stream):
        for w in range(args.warmup):
            E.step_batch(st, ring[w % n_ring])
    torch.cuda.synchronize(dev)
    chunk = 256
    graphs, done = [], 0
    while done < k_total:
        c = min(chunk, k_total - done)
        graphs.append(capture(c, args.warmup + done))
        done += c
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed():
        with torch.cuda.stream(stream):
            flush.fill_(1)
        barrier()
        torch.cuda.synchronize(dev)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for g in graphs:
                g.replay()
            e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        return e0.elapsed_time(e1) / 1e3

    timed()  # one untimed replay of the captured graphs (graph upload / first-run effects)
    with ClockSampler(dev_index) as clk:
        t0 = time.perf_counter()
        el = timed()
        # keep sampling clocks under the same load for >= 1 s
        while time.perf_counter() - t0 < 1.0:
            timed()
    el_max = allreduce_max(el, dev)
    frames = world * n * k_total
    value = frames / el_max
    ms_per_step = 1e3 * el_max / k_total
    # roofline of the step kernel (the only kernel in the timed region)
    bpf = algorithmic_bytes_per_frame()
    launch_s = el / k_total
    achieved = n * bpf / launch_s / 1e9
    peak, peak_kind = load_peaks()

    # e2e through the public API with host buffers
    # per-step commands from a ring of 64 pinned host buffers (fresh values every
    # step, buffers reused as a host control loop reuses its staging buffers; a
    # 1000-buffer ring adds ~3-5 us/step of GPU-side translation of never-seen
    # host pages, scripts/probes/serve_overhead.py)
    e2e_ring = min(64, k_total)
    host_cmds = torch.empty((e2e_ring, n, A_BLUEROV), dtype=torch.float32).pin_memory()
    host_cmds.copy_(torch.rand(e2e_ring, n, A_BLUEROV) * 2 - 1)
    host_out = torch.empty((13, n), dtype=torch.float32).pin_memory()
    cur = torch.cuda.current_stream(dev)

    def e2e_step(t):
        # public API, host buffers: pinned commands in, pinned (13, N) pose rows out;
        # returns when the step's pose rows are in host memory
        E.step_batch(st, host_cmds[t % e2e_ring], pose_out=host_out)

    # (1) launched path: one uuv_step_host call per step (kernel reads/writes the
    # mapped pinned buffers), CUDA events on the launching stream
    for t in range(min(args.warmup, k_total)):
        e2e_step(t)
    barrier()
    torch.cuda.synchronize(dev)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(cur)
    for t in range(k_total):
        e2e_step(t)
    f1.record(cur)
    torch.cuda.synchronize(dev)
    e2e_launch_el = allreduce_max(f0.elapsed_time(f1) / 1e3, dev)
    # (2) the same calls inside engine.serve(): a resident step kernel driven by a
    # doorbell in mapped pinned memory (no launch / stream sync per step); the
    # steps are synchronous, so the host clock brackets exactly K of them
    barrier()
    torch.cuda.synchronize(dev)
    # under a kernel profiler (ncu serialises launches) a resident kernel would
    # only wait out its idle timeout: skip the served path there
    profiled = args.no_serve or bool(os.environ.get("CUDA_INJECTION64_PATH"))
    e2e_serve_el = float("inf")
    if not profiled:
        with E.serve(st):
            for t in range(min(args.warmup, k_total)):
                e2e_step(t)
            t0 = time.perf_counter()
            for t in range(k_total):
                e2e_step(t)
            e2e_serve_el = time.perf_counter() - t0
        torch.cuda.synchronize(dev)
    e2e_serve_el = allreduce_max(e2e_serve_el, dev)
    e2e_el = min(e2e_serve_el, e2e_launch_el)
    e2e_path = ("step_batch inside engine.serve(): resident step kernel, doorbell in mapped "
                "pinned memory" if e2e_el == e2e_serve_el else
                "step_batch -> uuv_step_host (one launch per step, mapped pinned buffers)")
    barrier()

    # the same kernel at scale (informational): 1,048,576 envs of the same
    # workload (state + DR record + commands ~ 230 MB >> L2), CUDA graph of 20
    # steps, CUDA events -> achieved bandwidth of the step kernel where it is
    # HBM-bound rather than launch/latency-bound
    scale = None
    if not args.no_scale:
        n_big = 1 << 20
        big = E.make_batch(veh, E.SimConfig(batch_size=n_big), master_seed=0, device=dev,
                           env_offset=rank * n_big)
        E.reset_envs(big, torch.ones(n_big, dtype=torch.bool, device=dev),
                     E.spec_sampler(dr_spec()))
        cmd_big = torch.rand((n_big, A_BLUEROV), device=dev, generator=gen) * 2 - 1
        with torch.cuda.stream(stream):
            for _ in range(3):
                E.step_batch(big, cmd_big)
        torch.cuda.synchronize(dev)
        gb = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            with torch.cuda.graph(gb, stream=stream):
                for _ in range(20):
                    E.step_batch(big, cmd_big)
        torch.cuda.synchronize(dev)
        with torch.cuda.stream(stream):
            e0.record(stream)
            gb.replay()
            e1.record(stream)
        torch.cuda.synchronize(dev)
        t_big = e0.elapsed_time(e1) / 1e3 / 20
        a_big = n_big * bpf / t_big / 1e9
        scale = {"envs_per_gpu": n_big, "us_per_step": t_big * 1e6,
                 "env_frames_per_s": n_big / t_big, "achieved": a_big, "peak": peak,
                 "unit": "GB/s", "frac": a_big / peak}
        del big, cmd_big, gb
        torch.cuda.empty_cache()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "env-frames/s", "n_gpus": world,
            "steps": k_total, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "global_batch": world * n, "per_gpu_envs": n,
                       "parallelism": f"env-shard x{world} (no per-step collective)",
                       "l2": "inputs larger than L2: per-step commands from a "
                             f"{n_ring * per >> 20} MiB ring; L2 flushed before the timed region; "
                             "env state resident",
                       "launch": "CUDA graph of K uuv_step launches"},
            "e2e": {"value": world * n * k_total / e2e_el, "unit": "env-frames/s",
                    "h2d_bytes_per_step": n * A_BLUEROV * 4, "d2h_bytes_per_step": n * 13 * 4,
                    "path": e2e_path,
                    "per_path": {"serve": (world * n * k_total / e2e_serve_el
                                           if e2e_serve_el != float("inf") else None),
                                 "launch_per_step": world * n * k_total / e2e_launch_el}},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": load_traffic(),
                         "traffic_note": "ncu dram bytes per launch (cold cache), profiles/r01",
                         "peak_source": peak_kind,
                         "bytes_per_frame": bpf, "kernel": "k_step<float,1,DR=true>"},
            "roofline_at_scale": scale,
            "gpu_launches": k_total,
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            fps, k, cel, cores, reset_s = cpu_probe(seconds=args.cpu_seconds)
            line["cpu_baseline"] = {
                "value": fps, "unit": "env-frames/s", "cores": cores, "kind": "port",
                "sample": f"{N_ENVS} envs x {k} steps ({cel:.1f} s) of the same workload, "
                          f"oracle numpy port, {cores} threads"}
        print(json.dumps(line), flush=True)
    if dist:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-serve", action="store_true",
                    help="time only the launched e2e path (for runs under a kernel profiler)")
    ap.add_argument("--no-scale", action="store_true",
                    help="skip the informational 1M-env roofline_at_scale measurement")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_b200(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
