"""The roofline accounting behind bench.py's `roofline` objects and DESIGN §3.4 (host
only): SURVEY.md §8(d)'s per-frame bytes and per-substep flops, and the bound / fraction
arithmetic of roofline.roofline()."""

import json

import pytest

import bench
from paper_2503_09203_b200 import roofline as RF


def test_substep_flops_follow_survey_counts():
    # general path bluerov 794, heavy / hauv 848, lauv / iauv 1051; the
    # diagonal-hull fast path drops the constant 638 to 332 (bluerov 488)
    assert RF.substep_flops("bluerov", general=True) == 794
    assert RF.substep_flops("bluerov_heavy", general=True) == 848
    assert RF.substep_flops("hauv") == 848
    assert RF.substep_flops("lauv", general=True) == 1051
    assert RF.substep_flops("iauv") == 1051
    assert RF.substep_flops("bluerov") == 488
    assert RF.substep_flops("bluerov", current=True) == 488 + 33


def test_frame_bytes_follow_survey_formula():
    # B_phys(A) = 4 (26 + 3A) + 10: 186 B at A = 6, 174 at A = 5, 210 at A = 8
    for a, want in ((6, 186), (5, 174), (8, 210)):
        assert RF.frame_bytes(a) == want
    assert RF.frame_bytes(6, current=True) == 186 + 12
    # the bench workload: 4 DR keys read from the float64 record
    assert RF.frame_bytes(6, n_dr=4) == 218 == bench.algorithmic_bytes_per_frame()
    assert RF.frame_bytes(6, mixed=True) == 187


def test_rollout_bytes_amortise_the_state_over_the_launch():
    one = RF.rollout_frame_bytes(6, n_dr=4, steps=1)
    twenty = RF.rollout_frame_bytes(6, n_dr=4, steps=20)
    assert twenty < one
    # per step only the command row remains as the launch grows
    assert RF.rollout_frame_bytes(6, n_dr=4, steps=10**9) == pytest.approx(24.0, abs=1e-6)
    # 20 steps: 24 B of commands + (2 x 81 B of state / counters + 32 B of record) / 20
    assert twenty == pytest.approx(24 + (2 * (4 * 19 + 5) + 32) / 20)


def test_roofline_bound_and_fraction():
    bw, _ = RF.hbm_peak()
    fp, _ = RF.fp32_peak()
    n = 1 << 20
    # a byte-heavy frame: the HBM side bounds it; fraction = achieved / peak
    r = RF.roofline(50.0, n, 218, 488)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert r["achieved"] == pytest.approx(n * 218 / 50.0 / 1e3)
    assert r["frac"] == pytest.approx(r["achieved"] / bw)
    assert r["roofline_us"] == pytest.approx(n * 218 / (bw * 1e9) * 1e6)
    # a flop-heavy frame (K = 8 substeps): the FP32 side bounds it
    r = RF.roofline(130.0, n, 218, 8 * 488)
    assert r["bound"] == "fp32" and r["unit"] == "TFLOP/s"
    assert r["frac"] == pytest.approx(n * 8 * 488 / 130.0 / 1e6 / fp)
    json.dumps(r)  # the bench line embeds it


def test_bench_config_is_weak_scaled_workload():
    # both arms print bench_config(world) (the driver pairs them by it): no model keys,
    # the workload named, 4096 envs per GPU
    cfg = bench.bench_config(2)
    assert set(cfg) == {"workload", "global_batch", "per_gpu_envs", "parallelism"}
    assert cfg["workload"].startswith("cfg2")
    assert cfg["global_batch"] == 2 * cfg["per_gpu_envs"] == 2 * 4096
