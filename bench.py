"""Benchmark: env frames/s of the batched 6-DOF Fossen step (hydro + thruster + integrate).

Workload (BASELINE.json configs[1], the config quoted "on 1 B200"): BlueROV2,
4096 envs per GPU, per-env domain-randomised mass / volume / damping / thruster
gain ~ U[0.8, 1.2] drawn on device from the Philox stream keyed (seed 0, global
env, episode 0), commands U(-1, 1).  A step is one control step of every env
(``step_batch``: one ``uuv_step_dl`` launch).  N GPUs = N processes, one per
GPU, each owning 4096 globally-indexed envs (weak scaling, no per-step
collective); ``--gpus N`` without torchrun re-executes itself under
``torch.distributed.run`` (NCCL, rendezvous on 127.0.0.1).

* value — device-resident throughput of K control steps through
  ``engine.rollout`` (one ``uuv_rollout_dl`` launch, the state in registers from
  the first step to the last, the state stored every step; bit for bit K
  ``step_batch`` calls), CUDA events on the launching stream, barrier + max over
  ranks.  Each step reads a fresh command slot from a ring larger than L2; L2 is
  flushed before the timed region.  ``per_path.step_batch_graph`` is the same K
  steps as K ``step_batch`` launches replayed from CUDA graphs.  Work is
  enqueued behind a short device-side spin (``torch.cuda._sleep``, before the
  start event), so the GPU does not idle on host submission inside the region;
  the host submission time is reported beside it.
* e2e — the same metric through the public API with HOST buffers; three paths
  are timed and the fastest is reported (all in ``e2e.per_path``):
  ``rollout_host`` -- the `value` path host to host: ONE ``engine.rollout`` call
  with the K steps' commands in pinned host memory and a pinned host trace
  (K, 13 + A, N); the kernel reads each step's command rows and writes each
  step's p, q, nu, act over the host link as it runs, steps / diverged are
  copied back after it (host clock around the call, which returns once the trace
  is in host memory); ``serve`` -- the closed loop:
  ``step_batch(state, pinned_host_commands, out=HostStepOut)`` per step inside
  ``engine.serve(state)`` (a resident step kernel rung by a doorbell in mapped
  pinned memory; host clock around exactly K steps), each step's whole result
  (p, q, nu, act, steps, diverged -- what the reference's step_batch leaves in
  its numpy state) in host memory before the next call; ``launch_per_step`` --
  the same calls outside serve, one launch per step whose kernel reads/writes the
  mapped pinned buffers (CUDA events).
* roofline — the step kernel's algorithmic bytes per launch / average launch
  duration vs the measured HBM copy bandwidth (MEASURED_PEAKS.json).
* at_scale — the other BASELINE configs at their stated per-GPU sizes, each
  device-timed the same way with its own per-step roofline (informational).
* cpu_baseline — the reference's own CPU implementation (the unmodified
  ``uuvsim`` from baseline/_ref when installed, else the oracle numpy port) on
  the same workload on this box's host cores (rank 0, N = 1 only).

``--impl reference`` runs that CPU implementation as the reference arm.
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
RING_BYTES = 160 << 20  # command rings larger than the 126 MB L2


def bench_config(world):
    """The config dict both arms print (identical, so the driver can pair them)."""
    return {"workload": WORKLOAD, "global_batch": world * N_ENVS, "per_gpu_envs": N_ENVS,
            "parallelism": f"env-shard x{world} (no per-step collective)"}


def algorithmic_bytes_per_frame(a=A_BLUEROV, n_dr=len(DR_KEYS)):
    """state p,q,nu,act read+write, commands read, diverged r/w (1+1 B),
    steps r/w (4+4 B), plus the float64 DR record actually read (8 B per key)."""
    from paper_2503_09203_b200.roofline import frame_bytes

    return frame_bytes(a, n_dr)


def dr_spec():
    from paper_2503_09203_b200.randomization import DRParameter, Uniform

    return {k: DRParameter(k, Uniform(0.8, 1.2)) for k in DR_KEYS}


def load_traffic():
    """DRAM bytes per launch of the step kernel from the committed ncu capture."""
    for rnd in ("r02", "r01"):
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "ncu_traffic.json")) as f:
                t = json.load(f)
            return t["dram_bytes_read"] + t["dram_bytes_write"], f"profiles/{rnd}"
        except Exception:
            continue
    return None, None


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


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
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

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


def reference_modules():
    """The unmodified reference (``pip install --target baseline/_ref``), or None."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "uuvsim")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import uuvsim.engine as RE
        import uuvsim.randomization as RD
        import uuvsim.vehicles as RV
        from uuvsim.kinematics import Pose
    except Exception:
        return None
    return RE, RD, RV, Pose


def _reference_batch(workers):
    """cfg2 in the reference itself: its make_batch / reset_envs (its own PCG64 streams,
    sample_overlay draws, apply_overlay) / step_batch (engine.py:298, 487, 465)."""
    RE, RD, RV, Pose = reference_modules()
    veh = RV.load_vehicle("bluerov")
    spec = RD.make_spec([RD.DRParameter(k, RD.Uniform(0.8, 1.2)) for k in DR_KEYS])
    st = RE.make_batch(veh, RE.SimConfig(batch_size=N_ENVS, workers=workers), master_seed=0)
    t0 = time.perf_counter()
    RE.reset_envs(st, np.ones(N_ENVS, bool),
                  lambda i, ep, rng: RE.EnvInit(pose=Pose(), overlay=RD.sample_overlay(spec, rng)))
    return RE, st, time.perf_counter() - t0


def _oracle_batch(workers):
    from oracle import uuv_oracle as O
    from paper_2503_09203_b200.vehicles import load_vehicle

    spec = dr_spec()
    b = O.Batch(load_vehicle("bluerov"), N_ENVS, 0.02, 1, seed=0, workers=workers)
    t0 = time.perf_counter()
    b.reset(np.ones(N_ENVS, bool), lambda i, ep, r: O.Init(overlay=O.draw_overlay(spec, r)))
    return b, time.perf_counter() - t0


def cpu_probe(seconds=None, steps=None, warmup=3):
    """The reference's CPU path on the cfg2 workload, commands held fixed (BASELINE.md §3,
    the throughput_probe protocol).  Worker count: the faster of 1 and all host threads
    (the reference's thread pool gains nothing from more threads on small batches).
    Returns (frames/s, steps, elapsed, workers, reset_s, kind)."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    cmds = np.random.default_rng(0).uniform(-1.0, 1.0, (N_ENVS, A_BLUEROV))
    ncpu = os.cpu_count() or 1
    if reference_modules() is not None:
        kind = "reference"

        def make(w):
            RE, st, rs = _reference_batch(w)
            return (lambda: RE.step_batch(st, cmds)), rs
    else:
        from concurrent.futures import ThreadPoolExecutor

        kind = "port"
        pools = {}

        def make(w):
            b, rs = _oracle_batch(w)
            pool = pools.setdefault(w, ThreadPoolExecutor(max_workers=w) if w > 1 else None)
            return (lambda: b.step(cmds, pool)), rs

    best = None
    for w in sorted({1, ncpu}):  # calibrate the worker count on a few steps
        step, rs = make(w)
        for _ in range(warmup):
            step()
        t0 = time.perf_counter()
        for _ in range(3):
            step()
        rate = 3 / (time.perf_counter() - t0)
        if best is None or rate > best[0]:
            best = (rate, w, step, rs)
    _, workers, step, reset_s = best
    k = 0
    t0 = time.perf_counter()
    while True:
        step()
        k += 1
        el = time.perf_counter() - t0
        if (steps is not None and k >= steps) or (seconds is not None and el >= seconds):
            break
    return N_ENVS * k / el, k, el, workers, reset_s, kind


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    fps, k, el, workers, reset_s, kind = cpu_probe(steps=args.steps, warmup=args.warmup)
    what = ("the unmodified reference uuvsim (baseline/_ref): make_batch / reset_envs / "
            "step_batch" if kind == "reference" else "the oracle numpy port of the reference")
    sample = (f"full cfg2 workload ({N_ENVS} envs x {k} steps, commands held fixed) through "
              f"{what}, {workers} worker thread(s) (faster of 1 and {os.cpu_count()}); DR reset "
              f"of {N_ENVS} envs took {reset_s:.2f} s (excluded)")
    line = {"metric": METRIC, "value": fps, "unit": "env-frames/s", "n_gpus": args.gpus,
            "steps": k, "warmup": args.warmup, "ms_per_step": 1e3 * el / k,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference", "config": bench_config(max(world, 1)),
            "cpu_baseline": {"value": fps, "unit": "env-frames/s", "cores": workers,
                             "host_threads": os.cpu_count(), "cpu_model": cpu_model(),
                             "kind": kind, "sample": sample},
            "e2e": {"value": fps, "unit": "env-frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ================================================================ B200 arm


def command_ring(n, width, dev, gen, dtype=None):
    import torch

    per = n * width * 4
    n_ring = max(2, -(-RING_BYTES // per))
    ring = torch.rand((n_ring, n, width), device=dev, generator=gen) * 2 - 1
    return ring if dtype is None else ring.to(dtype)


class DeviceTimer:
    """CUDA-event timing of graph replays on `stream`: L2 flushed first, the replays
    enqueued behind a device-side spin so host submission is not inside the region."""

    def __init__(self, dev, stream, barrier):
        import torch

        self.torch = torch
        self.dev, self.stream, self.barrier = dev, stream, barrier
        self.flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        self.e0 = torch.cuda.Event(enable_timing=True)
        self.e1 = torch.cuda.Event(enable_timing=True)
        self.gate_us = 200.0
        self.submit_us = None
        self.cycles_per_us = 1965.0  # B200 max SM clock: a spin of >= gate_us at any clock

    def run(self, enqueue, gate=True, flush=True):
        torch = self.torch
        if flush:
            with torch.cuda.stream(self.stream):
                self.flush.fill_(1)
        self.barrier()
        torch.cuda.synchronize(self.dev)
        with torch.cuda.stream(self.stream):
            if gate:
                torch.cuda._sleep(int(self.gate_us * self.cycles_per_us))
            t0 = time.perf_counter()
            self.e0.record(self.stream)
            enqueue()
            self.e1.record(self.stream)
            sub = (time.perf_counter() - t0) * 1e6
        torch.cuda.synchronize(self.dev)
        self.barrier()
        self.submit_us = sub
        # keep the spin longer than the submission it hides (measured, with margin; capped
        # so a slow host -- or a profiler -- cannot stretch it without bound)
        self.gate_us = min(max(self.gate_us, 3.0 * sub + 50.0), 5000.0)
        return self.e0.elapsed_time(self.e1) / 1e3


def capture_steps(step, k_total, stream, chunk=256):
    """CUDA graphs of exactly k_total calls step(t) (chunks of <= chunk launches)."""
    import torch

    from paper_2503_09203_b200 import engine as E

    graphs, done = [], 0
    while done < k_total:
        c = min(chunk, k_total - done)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            with torch.cuda.graph(g, stream=stream), E.no_gc():
                for s in range(c):
                    step(done + s)
        graphs.append(g)
        done += c
    return graphs


def at_scale_blocks(ctx, timer, stream, steps, gen):
    """The other BASELINE configs at their per-GPU sizes (configs[2..4]); each block a
    CUDA graph of `steps` control steps with fresh commands from a ring > L2."""
    import torch

    from paper_2503_09203_b200 import engine as E
    from paper_2503_09203_b200 import roofline as RF
    from paper_2503_09203_b200.distributed import allreduce_max
    from paper_2503_09203_b200.randomization import preset
    from paper_2503_09203_b200.tasks import TaskConfig, make_env
    from paper_2503_09203_b200.vehicles import BUILTIN_VEHICLES, load_vehicle

    dev, rank = ctx.device, ctx.rank
    out = {}

    def measure(name, n, step_fn, warm_fn, bpf, fpf, desc, tail=None):
        for t in range(3):
            warm_fn(t)
        torch.cuda.synchronize(dev)
        graphs = capture_steps(step_fn, steps, stream)

        def enqueue():
            for g in graphs:
                g.replay()
            if tail is not None:
                tail()

        timer.run(enqueue)  # graph upload / first replay
        el = allreduce_max(timer.run(enqueue), dev)
        us = el / steps * 1e6
        out[name] = {"workload": desc, "envs_per_gpu": n, "steps": steps, "us_per_step": us,
                     "env_frames_per_s": ctx.world * n / (el / steps),
                     "roofline": RF.roofline(us, n, bpf, fpf)}
        del graphs
        torch.cuda.empty_cache()

    # cfg2 at 1M envs: the headline kernel where it is bandwidth-bound
    n = 1 << 20
    veh = load_vehicle("bluerov")
    st = E.make_batch(veh, E.SimConfig(batch_size=n), master_seed=0, device=dev,
                      env_offset=rank * n)
    E.reset_envs(st, torch.ones(n, dtype=torch.bool, device=dev), E.spec_sampler(dr_spec()))
    ring = command_ring(n, 6, dev, gen)
    measure("cfg2_1m", n, lambda t: E.step_batch(st, ring[t % len(ring)]),
            lambda t: E.step_batch(st, ring[t]), RF.frame_bytes(6, 4), RF.substep_flops("bluerov"),
            "cfg2 workload at 1,048,576 envs/GPU")
    # the headline kernel (k_rollout) where it is not latency-bound: the same 1M envs,
    # 20 steps in one launch, fresh command slots from the same ring
    def roll():
        E.rollout(st, ring, steps, start=3)

    roll()
    timer.run(roll)
    el = allreduce_max(timer.run(roll), dev)
    us = el / steps * 1e6
    out["cfg2_rollout_1m"] = {
        "workload": "cfg2 workload at 1,048,576 envs/GPU, 20 steps as one engine.rollout launch",
        "envs_per_gpu": n, "steps": steps, "us_per_step": us,
        "env_frames_per_s": ctx.world * n / (el / steps),
        # bytes this kernel must move (commands per step; state, counters and DR record
        # once per launch): FP32-bound; `per_step_model_frac` is the SURVEY per-frame
        # model (state round trip every step) that the rollout beats by construction
        "roofline": dict(RF.roofline(us, n, RF.rollout_frame_bytes(6, 4, steps),
                                     RF.substep_flops("bluerov")),
                         per_step_model_frac=RF.roofline(us, n, RF.frame_bytes(6, 4),
                                                         RF.substep_flops("bluerov"))["frac"])}
    del st, ring

    # configs[2]: all five vehicles mixed, 262,144 envs (contiguous per-type runs)
    n = 262_144
    vehs = [load_vehicle(v) for v in BUILTIN_VEHICLES]
    counts = [n // 5 + (1 if i < n % 5 else 0) for i in range(5)]
    st = E.make_fleet_batch(vehs, counts, E.SimConfig(batch_size=n), device=dev,
                            env_offset=rank * n)
    E.reset_envs(st, torch.ones(n, dtype=torch.bool, device=dev))
    ring = command_ring(n, st.a_max, dev, gen)
    for v, s0, c in zip(vehs, np.concatenate([[0], np.cumsum(counts)[:-1]]), counts):
        ring[:, int(s0):int(s0) + c, v.action_dim:] = 0.0  # padded command columns
    a_mean = sum(v.action_dim * c for v, c in zip(vehs, counts)) / n
    fpf = sum(RF.substep_flops(v.name) * c for v, c in zip(vehs, counts)) / n
    measure("cfg3_mixed_262k", n, lambda t: E.step_batch(st, ring[t % len(ring)]),
            lambda t: E.step_batch(st, ring[t]), RF.frame_bytes(a_mean, 0, mixed=True), fpf,
            "configs[2]: five UUV models mixed (6/8/5/5/8 actuators), 262,144 envs/GPU")
    del st, ring

    # configs[3]: trajectory tracking, ocean current, 8 fused substeps, 1M envs (task step)
    n = 1 << 20
    env = make_env(TaskConfig(task="tracking", vehicle="bluerov", level="disturbed"),
                   E.SimConfig(batch_size=n, substeps=8), seed=0, device=dev,
                   env_offset=rank * n)
    env.reset()
    ring = command_ring(n, 6, dev, gen)
    measure("cfg4_tracking_k8_1m", n, lambda t: env.step(ring[t % len(ring)]),
            lambda t: env.step(ring[t]),
            RF.frame_bytes(6, 0, True) + RF.task_bytes(6, env.obs_dim, True),
            8 * RF.substep_flops("bluerov", current=True) + RF.TASK_FLOPS,
            "configs[3]: tracking task, bluerov, level disturbed (current + payload), K=8, "
            "1,048,576 envs/GPU, fused env.step")
    del env, ring
    torch.cuda.empty_cache()

    # configs[4]: docking, train-preset DR, auto-reset, 1M envs per GPU, NCCL stats
    last_stats = []
    env = make_env(TaskConfig(task="docking", vehicle="bluerov_heavy", level="disturbed_dr"),
                   E.SimConfig(batch_size=n), seed=0, device=dev, env_offset=rank * n)
    env.reset()
    ring = command_ring(n, 8, dev, gen)
    measure("cfg5_docking_1m", n, lambda t: env.step(ring[t % len(ring)]),
            lambda t: env.step(ring[t]),
            RF.frame_bytes(8, len(preset("train")) - 1, True) + RF.task_bytes(8, env.obs_dim,
                                                                                False),
            RF.substep_flops("bluerov_heavy", current=True, general=True) + RF.TASK_FLOPS,
            "configs[4]: docking task, bluerov_heavy, level disturbed_dr (train preset), "
            "auto-reset, 1,048,576 envs/GPU, rollout stats all-reduced once per rollout",
            tail=lambda: last_stats.append(env.rollout_stats_tensor()))
    s5 = dict(zip(("reward_sum", "finished", "success", "failure", "truncated",
                   "metric_sum_finished", "diverged", "frames"), last_stats[-1].tolist()))
    out["cfg5_docking_1m"]["finished_per_frame"] = s5["finished"] / max(s5["frames"], 1)
    del env, ring
    torch.cuda.empty_cache()
    return out


def run_b200(args):
    import torch

    from paper_2503_09203_b200 import distributed as D
    from paper_2503_09203_b200 import engine as E
    from paper_2503_09203_b200 import roofline as RF
    from paper_2503_09203_b200.vehicles import load_vehicle

    # one process per GPU; UUV_BENCH_GPU_OVERRIDE=0 pins every rank to GPU 0 and
    # UUV_DIST_BACKEND=gloo swaps NCCL for gloo (exercises the multi-rank path on a
    # single-GPU box; the driver's runs use one GPU per rank over NCCL)
    override = os.environ.get("UUV_BENCH_GPU_OVERRIDE")
    ctx = D.init(os.environ.get("UUV_DIST_BACKEND"),
                 int(override) if override is not None else None)
    dev, rank, world = ctx.device, ctx.rank, ctx.world
    barrier = ctx.barrier

    veh = load_vehicle("bluerov")
    n = N_ENVS
    offset = rank * n  # weak scaling: each GPU owns 4096 globally-indexed envs
    st = E.make_batch(veh, E.SimConfig(batch_size=n), master_seed=0, device=dev,
                      env_offset=offset)
    E.reset_envs(st, torch.ones(n, dtype=torch.bool, device=dev), E.spec_sampler(dr_spec()))

    gen = torch.Generator(device=dev).manual_seed(offset)
    ring = command_ring(n, A_BLUEROV, dev, gen)
    n_ring = len(ring)
    stream = torch.cuda.Stream(dev)
    k_total = args.steps
    torch.cuda.synchronize(dev)
    with torch.cuda.stream(stream):
        for w in range(args.warmup):
            E.step_batch(st, ring[w % n_ring])
    torch.cuda.synchronize(dev)
    timer = DeviceTimer(dev, stream, barrier)
    # (a) the resident rollout: ONE uuv_rollout_dl launch for the K steps, the state in
    #     registers from the first step to the last, step t reading ring slot
    #     (warmup + t) -- bit for bit K step_batch calls (tests/test_gpu_rollout.py)
    start = args.warmup % n_ring

    def enqueue_rollout():
        E.rollout(st, ring, k_total, start=start)

    # (b) the per-step drop-in call: CUDA graphs of K step_batch launches (uuv_step_dl),
    #     programmatic dependent launch between consecutive steps
    graphs = capture_steps(lambda s: E.step_batch(st, ring[(args.warmup + s) % n_ring]),
                           k_total, stream)

    def enqueue_graphs():
        for g in graphs:
            g.replay()

    timer.run(enqueue_rollout)  # untimed: first launch, gate calibration
    timer.run(enqueue_graphs)  # untimed: graph upload
    with ClockSampler(dev.index) as clk:
        t0 = time.perf_counter()
        el = timer.run(enqueue_rollout)
        submit_us = timer.submit_us
        el_graph = timer.run(enqueue_graphs)
        while time.perf_counter() - t0 < 1.0:  # keep sampling clocks under the same load
            timer.run(enqueue_rollout)
            timer.run(enqueue_graphs)
    el_graph_ungated = timer.run(enqueue_graphs, gate=False)  # host submission inside
    el_max = D.allreduce_max(el, dev)
    el_graph_max = D.allreduce_max(el_graph, dev)
    frames = world * n * k_total
    value = frames / el_max
    ms_per_step = 1e3 * el_max / k_total
    us_step = el / k_total * 1e6
    # the contract's algorithmic bytes: SURVEY.md §8(d)'s per-frame figure (state read +
    # written, commands, counters, the DR record: 218 B for cfg2) x the frames one launch
    # processes -- the same per-frame work as K step_batch calls.  k_rollout moves far
    # less (the state stays in registers between steps): `traffic` (ncu) and
    # `kernel_bytes_per_frame` give what it actually moves.
    roof = RF.roofline(us_step, n, algorithmic_bytes_per_frame(), RF.substep_flops("bluerov"))
    traffic, traffic_src = load_traffic()
    roof.update(traffic=traffic, traffic_note=f"ncu dram bytes read + written by one launch of the "
                f"dominant kernel ({traffic_src}/ncu_traffic.json: 20 steps, cold cache)"
                if traffic_src else None,
                algorithmic_bytes_per_launch=n * k_total * roof["bytes_per_frame"],
                kernel_bytes_per_frame=RF.rollout_frame_bytes(A_BLUEROV, len(DR_KEYS), k_total),
                fp32_frac=n * RF.substep_flops("bluerov") / us_step / 1e6 / RF.fp32_peak()[0],
                kernel="k_rollout<float,1,DR,6,DM>")
    roof_graph = RF.roofline(el_graph / k_total * 1e6, n, algorithmic_bytes_per_frame(),
                             RF.substep_flops("bluerov"))
    roof_graph["kernel"] = "k_step<float,1,DR,6,DM>"

    # e2e through the public API with host buffers: per-step commands from a ring of
    # 64 pinned host buffers (fresh values every step, buffers reused as a host control
    # loop reuses its staging buffers), the whole step result back in pinned buffers
    e2e_ring = min(64, k_total)
    host_cmds = torch.empty((e2e_ring, n, A_BLUEROV), dtype=torch.float32).pin_memory()
    host_cmds.copy_(torch.rand(e2e_ring, n, A_BLUEROV) * 2 - 1)
    res = E.HostStepOut(st)
    cur = torch.cuda.current_stream(dev)

    def e2e_step(t):
        E.step_batch(st, host_cmds[t % e2e_ring], out=res)

    # (1) launched path: one uuv_step_host call per step, CUDA events on its stream
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
    e2e_launch_el = D.allreduce_max(f0.elapsed_time(f1) / 1e3, dev)
    # (2) the same calls inside engine.serve(); synchronous steps, host clock around K
    barrier()
    torch.cuda.synchronize(dev)
    # under a kernel profiler (ncu serialises launches) a resident kernel would only
    # wait out its idle timeout: skip the served path there
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
    e2e_serve_el = D.allreduce_max(e2e_serve_el, dev)
    # (3) the K steps as ONE engine.rollout call host to host (the `value` path with host
    # buffers): K fresh command slots in pinned host memory, every step's p, q, nu, act
    # written into a pinned host trace by the kernel as it runs, then steps / diverged
    # copied back; host clock around the call (it returns once the trace is in host memory)
    rh_cmds = torch.empty((k_total, n, A_BLUEROV), dtype=torch.float32).pin_memory()
    rh_cmds.copy_(torch.rand(k_total, n, A_BLUEROV) * 2 - 1)
    rh_trace = torch.empty((k_total, 13 + A_BLUEROV, n), dtype=torch.float32).pin_memory()
    rh_out = E.HostStepOut(st, fields=("steps", "diverged"))

    def rollout_host():
        E.rollout(st, rh_cmds, k_total, trace=rh_trace, out=rh_out)

    for _ in range(max(1, min(args.warmup, 3))):
        rollout_host()
    barrier()
    torch.cuda.synchronize(dev)
    e2e_rh_el = float("inf")
    for _ in range(10):  # best of ten calls (host clock, like the served path)
        t0 = time.perf_counter()
        rollout_host()
        e2e_rh_el = min(e2e_rh_el, time.perf_counter() - t0)
    e2e_rh_el = D.allreduce_max(e2e_rh_el, dev)
    rh_d2h = (13 + A_BLUEROV) * 4 * n + rh_out.nbytes // k_total
    e2e_paths = {
        "rollout_host": (e2e_rh_el, "engine.rollout(state, pinned host commands (K, N, A), K, "
                         "trace=pinned host (K, 13 + A, N)): one k_rollout launch reading each "
                         "step's commands and writing each step's p, q, nu, act over the host "
                         "link, then steps / diverged copied back", rh_d2h),
        "serve": (e2e_serve_el, "step_batch(host cmds, out=HostStepOut) inside engine.serve(): "
                  "resident step kernel, doorbell in mapped pinned memory (closed loop: each "
                  "step's commands may depend on the previous result)", res.nbytes),
        "launch_per_step": (e2e_launch_el, "step_batch(host cmds, out=HostStepOut) -> "
                            "uuv_step_host (one launch per step, mapped pinned buffers)",
                            res.nbytes),
    }
    e2e_key = min(e2e_paths, key=lambda k: e2e_paths[k][0])
    e2e_el, e2e_path, e2e_d2h = e2e_paths[e2e_key]
    barrier()
    del graphs
    torch.cuda.empty_cache()

    scale = None
    if not args.no_scale:
        scale = at_scale_blocks(ctx, timer, stream, 20, gen)

    if rank == 0:
        cfg = bench_config(world)
        line = {
            "metric": METRIC, "value": value, "unit": "env-frames/s", "n_gpus": world,
            "steps": k_total, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": cfg,
            "timing": {"l2": f"inputs larger than L2: per-step commands from a "
                             f"{n_ring * n * A_BLUEROV * 4 >> 20} MiB ring; L2 flushed before "
                             "the timed region; env state resident",
                       "launch": "value: one engine.rollout launch (k_rollout) for the K steps; "
                                 "per_path.step_batch_graph: CUDA graphs of K step_batch "
                                 "launches (uuv_step_dl, programmatic dependent launch)",
                       "host_submit_us": submit_us, "gate_us": timer.gate_us,
                       "step_batch_graph_us_per_step_submit_inside":
                           el_graph_ungated / k_total * 1e6},
            "per_path": {"rollout": value, "step_batch_graph": frames / el_graph_max,
                         "step_batch_graph_ms_per_step": 1e3 * el_graph_max / k_total,
                         "step_batch_graph_roofline": roof_graph},
            "e2e": {"value": world * n * k_total / e2e_el, "unit": "env-frames/s",
                    "h2d_bytes_per_step": n * A_BLUEROV * 4, "d2h_bytes_per_step": e2e_d2h,
                    "path": e2e_path,
                    "per_path": {k: (world * n * k_total / v[0] if v[0] != float("inf")
                                     else None) for k, v in e2e_paths.items()},
                    "closed_loop": "per_path.serve: one synchronous step per call, the next "
                                   "commands may depend on this step's result"},
            "roofline": roof,
            "at_scale": scale,
            "gpu_launches": 1,  # one k_rollout launch for the K steps
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            fps, k, cel, workers, reset_s, kind = cpu_probe(seconds=args.cpu_seconds)
            what = "unmodified reference uuvsim (baseline/_ref)" if kind == "reference" else \
                "oracle numpy port"
            line["cpu_baseline"] = {
                "value": fps, "unit": "env-frames/s", "cores": workers,
                "host_threads": os.cpu_count(), "cpu_model": cpu_model(), "kind": kind,
                "sample": f"{N_ENVS} envs x {k} steps ({cel:.1f} s) of the same workload, "
                          f"{what}, {workers} worker thread(s)"}
        print(json.dumps(line), flush=True)
    D.finalize(ctx)
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
                    help="skip the informational at-scale blocks of the other configs")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args, rank, world if "WORLD_SIZE" in os.environ else args.gpus)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-execute under torch.distributed.run (NCCL)
        from paper_2503_09203_b200.distributed import launch

        return launch(os.path.abspath(__file__), sys.argv[1:], args.gpus,
                      env={"NCCL_DEBUG": os.environ.get("NCCL_DEBUG", "INFO")})
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
