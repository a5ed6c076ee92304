"""Gaussian DR on the device: numpy's ziggurat restated (CPU checks).

The device sampler (csrc/uuv_device.cuh ``standard_normal``) is
numpy's ``random_standard_normal`` with the tables in csrc/uuv_ziggurat.cuh and
glibc's ``log1p`` for the tail.  These tests pin both against the host: the
header tables must reproduce numpy's own draws bit for bit, and the
operation-for-operation restatement of glibc's FMA ``log1p`` (the device code's
sequence) must equal libm on the tail's input domain.  The reference's
``Gaussian.sample`` (randomization.py:64-81) is ``clip(rng.normal(mu, sigma))``.
"""

import math
import os
import struct
import sys
from fractions import Fraction

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import gen_ziggurat as Z  # noqa: E402
from paper_2503_09203_b200 import _native as N  # noqa: E402
from paper_2503_09203_b200.engine import DeviceSampler  # noqa: E402
from paper_2503_09203_b200.randomization import DRParameter, Gaussian, Uniform  # noqa: E402

TABLES = Z.parse_header()


def _fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _hi(x):
    return struct.unpack("<q", struct.pack("<d", x))[0] >> 32


def _sethi(x, h):
    b = struct.unpack("<Q", struct.pack("<d", x))[0]
    return struct.unpack("<d", struct.pack("<Q", ((h & 0xFFFFFFFF) << 32) | (b & 0xFFFFFFFF)))[0]


def _i32(v):
    v &= 0xFFFFFFFF
    return v - (1 << 32) if v >= 1 << 31 else v


def log1p_glibc(x):
    """Same operation sequence as csrc/uuv_device.cuh log1p_glibc (x in (-1, 0])."""
    ln2_hi, ln2_lo = 6.93147180369123816490e-01, 1.90821492927058770002e-10
    L1, L2, L3, L4 = (6.666666666666735130e-01, 3.999999999940941908e-01,
                      2.857142874366239149e-01, 2.222219843214978396e-01)
    L5, L6, L7 = 1.818357216161805012e-01, 1.531383769920937332e-01, 1.479819860511658591e-01
    hx = _i32(_hi(x))
    ax = hx & 0x7FFFFFFF
    k, hu, c, f = 1, 0, 0.0, 0.0
    if hx < 0x3FDA827A:
        if ax >= 0x3FF00000:
            return -math.inf if x == -1.0 else math.nan
        if ax < 0x3E200000:
            return x if ax < 0x3C900000 else _fma(-(x * x), 0.5, x)
        if hx > 0 or hx <= _i32(0xBFD2BEC3):
            k, f, hu = 0, x, 1
    if k != 0:
        u = 1.0 + x
        hu = _i32(_hi(u))
        k = (hu >> 20) - 1023
        c = (1.0 - (u - x) if k > 0 else x - (u - 1.0)) / u
        hu &= 0x000FFFFF
        if hu < 0x6A09E:
            u = _sethi(u, hu | 0x3FF00000)
        else:
            k += 1
            u = _sethi(u, hu | 0x3FE00000)
            hu = (0x00100000 - hu) >> 2
        f = u - 1.0
    hfsq = (0.5 * f) * f
    dk = float(k)
    if hu == 0:
        if f == 0.0:
            return 0.0 if k == 0 else _fma(dk, ln2_hi, _fma(dk, ln2_lo, c))
        R = _fma(-f, 0.6666666666666666, 1.0) * hfsq
        return f - R if k == 0 else _fma(dk, ln2_hi, -((R - _fma(dk, ln2_lo, c)) - f))
    s = f / (2.0 + f)
    z = s * s
    R2, R3, R4 = _fma(z, L3, L2), _fma(z, L5, L4), _fma(z, L7, L6)
    z2 = z * z
    z4 = z2 * z2
    z6 = z2 * z4
    R = _fma(z6, R4, _fma(z4, R3, _fma(z, L1, z2 * R2)))
    t = s * (R + hfsq)
    if k == 0:
        return f - (hfsq - t)
    return _fma(dk, ln2_hi, -((hfsq - (_fma(dk, ln2_lo, c) + t)) - f))


def _host_has_fma():
    try:
        return " fma " in open("/proc/cpuinfo").read().replace("\n", " ")
    except OSError:
        return False


def _draws(bitgen_factory, n, log1p=math.log1p):
    want = np.random.Generator(bitgen_factory()).standard_normal(n)
    raw = iter(bitgen_factory().random_raw(4 * n + 64).tolist())
    got = np.array([Z.standard_normal(lambda: next(raw), *TABLES, log1p=log1p) for _ in range(n)])
    return got, want


@pytest.mark.parametrize("bitgen", ["philox", "pcg64"])
def test_header_tables_reproduce_numpy_standard_normal(bitgen):
    mk = {"philox": lambda: np.random.Philox(key=[3, 1 << 40]),
          "pcg64": lambda: np.random.PCG64(np.random.SeedSequence(11, spawn_key=(5, 2)))}[bitgen]
    got, want = _draws(mk, 60_000)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert np.count_nonzero(np.abs(want) > Z.R) > 0  # the tail branch ran


@pytest.mark.skipif(not _host_has_fma(), reason="glibc selects its non-FMA log1p on this CPU")
def test_log1p_restatement_matches_libm_on_tail_domain():
    rng = np.random.default_rng(7)
    us = np.concatenate([
        rng.integers(0, 1 << 53, 40_000, dtype=np.uint64).astype(np.float64) * 2.0 ** -53,
        rng.random(5_000) * 1e-3, rng.random(5_000) * 2e-9, 1 - rng.random(5_000) * 1e-6,
        np.arange(1, 5_001, dtype=np.float64) * 2.0 ** -53, [0.0, 0.5, 0.25, 1 - 2.0 ** -53]])
    bad = [u for u in us if log1p_glibc(-float(u)) != math.log1p(-float(u))]
    assert not bad, bad[:5]


def test_standard_normal_with_restated_log1p_matches_numpy():
    got, want = _draws(lambda: np.random.Philox(key=[99, 7]), 30_000, log1p=log1p_glibc)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_sampler_packs_gaussian_draws():
    spec = {"mass*": DRParameter("mass*", Gaussian(1.0, 0.1, (0.8, 1.2))),
            "volume*": DRParameter("volume*", Uniform(0.9, 1.1)),
            "current_velocity": DRParameter("current_velocity", Gaussian(0.3, 0.05, (0.0, 0.6)))}
    from paper_2503_09203_b200.engine import spec_sampler

    smp = spec_sampler(spec).pack()
    d = smp.overlay[0]
    assert N.OV_KEYS[d.key] == "mass*" and d.dist == N.DIST_GAUSSIAN
    assert (d.mu, d.sigma, d.lo, d.hi) == (1.0, 0.1, 0.8, 1.2)
    assert smp.overlay[1].dist == N.DIST_UNIFORM
    assert smp.current_speed.dist == N.DIST_GAUSSIAN and smp.current_speed.sigma == 0.05
    assert isinstance(DeviceSampler(spec), DeviceSampler)


def test_every_distribution_is_device_encodable():
    from paper_2503_09203_b200.randomization import Piecewise, device_encodable

    spec = {"mass*": DRParameter("mass*", Gaussian(1.0, 0.1, (0.8, 1.2))),
            "volume*": DRParameter("volume*", Uniform(0.9, 1.1)),
            "damping*": DRParameter("damping*", Piecewise([0.5, 1.0, 1.5], [1.0, 3.0]))}
    assert device_encodable(spec) and device_encodable(None)
