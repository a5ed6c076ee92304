"""Per-step roofline accounting of the step and task kernels (measurement, not compute).

The north star's roofline: T_roof = max(flops / P_fp32, bytes / BW_hbm) per
control step, fraction = T_roof / T_measured.

* Bytes per frame (one env, one control step) are the ALGORITHMIC bytes the
  kernel must move: state p, q, nu, act read + written, commands read,
  diverged r/w (1+1 B), steps r/w (4+4 B), the float64 DR record actually read
  (8 B per key), current (3 reals) and, for the task layer, observation,
  reward, flags, previous command and the tracking accumulator.
* Flops per substep are counted from the reference formulation (+,-,x,/ = 1,
  FMA = 2, sqrt/sin/cos/atan2 = 1, clamps 0) for the formulation the kernel
  executes: 5A + 16P + 87F + 6(A-1) + C with C = 332 on the diagonal-hull path
  (r_g = 0, diagonal M_A/D: bluerov, bluerov_heavy, lauv) and 638 on the general
  one (iauv, hauv, payload/cobm overlays), + 33 with a current.
* Peaks: HBM = MEASURED_PEAKS.json (driver-written copy bandwidth); FP32 = the
  FFMA-chain measurement of this pool's B200s (profiles/r01/fp32_peak.json),
  else the nominal 148 SM x 128 lanes x 2 x 1.965 GHz.
"""

from __future__ import annotations

import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (A actuators, P props, F fins, diagonal-hull path)
FLEET_SHAPE = {"bluerov": (6, 6, 0, True), "bluerov_heavy": (8, 8, 0, True),
               "lauv": (5, 1, 4, True), "iauv": (5, 1, 4, False), "hauv": (8, 8, 0, False)}
TASK_FLOPS = 250  # obs + reward + termination per frame (SURVEY §8(d) upper estimate)


def hbm_peak():
    """(GB/s, source): the driver-measured copy bandwidth, else the recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def fp32_peak():
    """(TFLOP/s, source): FFMA-chain measurement, else nominal at 1.965 GHz."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01", "fp32_peak.json")) as f:
            return float(json.load(f)["fp32_tflops"]), "measured (profiles/r01/fp32_peak.json)"
    except Exception:
        return 74.4, "nominal"


def substep_flops(vehicle: str, current: bool = False, general: bool = False) -> int:
    a, p, f, dm = FLEET_SHAPE[vehicle]
    c = 332 if (dm and not general) else 638
    return 5 * a + 16 * p + 87 * f + 6 * (a - 1) + c + (33 if current else 0)


def frame_bytes(a: float, n_dr: int = 0, current: bool = False, dtype_bytes: int = 4,
                mixed: bool = False) -> float:
    """Physics step: state r/w, commands, flags/counters, DR record (+current, +type id)."""
    b = dtype_bytes * (2 * (13 + a) + a) + 2 + 8 + 8 * n_dr
    if current:
        b += 3 * dtype_bytes
    if mixed:
        b += 1
    return b


def rollout_frame_bytes(a: int, n_dr: int = 0, steps: int = 1, current: bool = False,
                        dtype_bytes: int = 4) -> float:
    """k_rollout: per step the command row read; per launch (amortised over ``steps``) the
    state, steps/diverged and DR record read and the state, steps, diverged written (the
    states between the first and the last step never leave registers)."""
    per_step = dtype_bytes * a
    state = dtype_bytes * (13 + a) + 4 + 1
    per_launch = 2 * state + 8 * n_dr + (3 * dtype_bytes if current else 0)
    return per_step + per_launch / max(steps, 1)


def task_bytes(a: int, obs_dim: int, tracking: bool, dtype_bytes: int = 4) -> int:
    """Task layer on top of the physics: obs, reward, term/trunc, prev command r/w, dev_sum."""
    return dtype_bytes * obs_dim + dtype_bytes + 2 + 2 * dtype_bytes * a + (8 if tracking else 0)


def roofline(us_per_step: float, n: int, bytes_per_frame: float, flops_per_frame: float) -> dict:
    """The bench line's roofline object for one kernel (per launch = per control step)."""
    bw, bw_src = hbm_peak()
    fp, fp_src = fp32_peak()
    t_hbm = n * bytes_per_frame / (bw * 1e9) * 1e6
    t_fp = n * flops_per_frame / (fp * 1e12) * 1e6
    if t_hbm >= t_fp:
        achieved = n * bytes_per_frame / us_per_step / 1e3  # GB/s
        out = {"bound": "hbm", "achieved": achieved, "peak": bw, "unit": "GB/s",
               "frac": achieved / bw, "peak_source": bw_src}
    else:
        achieved = n * flops_per_frame / us_per_step / 1e6  # TFLOP/s
        out = {"bound": "fp32", "achieved": achieved, "peak": fp, "unit": "TFLOP/s",
               "frac": achieved / fp, "peak_source": fp_src}
    out.update(bytes_per_frame=bytes_per_frame, flops_per_frame=flops_per_frame,
               roofline_us=max(t_hbm, t_fp))
    return out
