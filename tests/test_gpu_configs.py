"""GPU parity at the BASELINE config shapes (BASELINE.json configs[1..3]).

The benchmarked kernels, exactly as the bench launches them, against the
pinned oracle and the reference's own fixtures (tests/golden/make_config_golden.py):

* cfg2 — bluerov, device-drawn DR {damping*, mass*, thrust_coeff*, volume*} ~
  U[0.8, 1.2] (Philox), fresh commands every step.  This is the bench's
  ``k_step<float, 1, DR, 6, DM, PRE>`` (thrust_coeff* in the per-launch PRE
  products).  64 envs against the reference fixture, and the bench's 4096 envs
  against the oracle, both for 100 steps with per-step state re-injection.
* cfg3 — five vehicles mixed at 131,072+ envs: the per-type run dispatch
  (one specialised launch per run on forked streams), a strided sample of rows
  compared with per-vehicle oracle batches.
* Piecewise / Gaussian / vector mount-jitter DR drawn on the device, bit for
  bit against the reference's sample_overlay (Philox and PCG64 streams).
* At the stated full sizes (cfg2, configs[3], configs[4] at 1,048,576 envs):
  rows of the full batch equal small env_offset shards bit for bit, so the
  fixture-checked small-batch behaviour holds at full size.

Tolerances as tests/test_gpu_parity.py: float64 1e-12 per step, float32 1e-5
relative / 1e-6 absolute per step; DR draws and counters bit-exact.
"""

import json

import numpy as np
import pytest
import torch
from conftest import golden, product_vehicle

import make_config_golden_spec as SPEC
from oracle import uuv_oracle as O
from paper_2503_09203_b200 import engine as E
from paper_2503_09203_b200.randomization import DRParameter, Uniform

pytestmark = pytest.mark.gpu

F64_RTOL = 1e-12
FP32_RTOL = 1e-5
FP32_ATOL = 1e-6
CFG2_KEYS = ("damping*", "mass*", "thrust_coeff*", "volume*")


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def host(x):
    return x.detach().double().cpu().numpy()


def rowwise_close(got, want, rtol, atol=0.0, floor=None):
    got = np.asarray(got, dtype=np.float64).reshape(len(want), -1)
    want = np.asarray(want, dtype=np.float64).reshape(len(want), -1)
    err = np.abs(got - want).max(axis=1)
    scale = np.abs(want).max(axis=1)
    if floor is not None:
        scale = np.maximum(scale, floor)
    ok = err <= rtol * scale + atol
    return bool(ok.all()), float((err / np.maximum(scale, 1e-300)).max())


def cfg2_spec():
    return {k: DRParameter(k, Uniform(0.8, 1.2)) for k in CFG2_KEYS}


def set_state(st, p, q, nu, act):
    dt = st.dtype
    st.p[:] = torch.from_numpy(np.asarray(p)).to(st.device, dt)
    st.q[:] = torch.from_numpy(np.asarray(q)).to(st.device, dt)
    st.nu[:] = torch.from_numpy(np.asarray(nu)).to(st.device, dt)
    st.act[:] = torch.from_numpy(np.asarray(act)).to(st.device, dt)


def tol(dtype):
    return (F64_RTOL, 1e-300) if dtype == torch.float64 else (FP32_RTOL, FP32_ATOL)


def cfg2_batch(n, dtype):
    """The bench's batch (bench.py run_b200): seed 0, Philox, device DR draws."""
    st = E.make_batch(product_vehicle("bluerov"), E.SimConfig(batch_size=n), master_seed=0,
                      dtype=dtype)
    E.reset_envs(st, torch.ones(n, dtype=torch.bool, device=st.device),
                 E.spec_sampler(cfg2_spec()))
    return st


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_config2_reference_fixture(dtype):
    """cfg2 at 64 envs vs the reference: device draws bitwise, 100 steps re-injected."""
    g = golden("config2_bluerov_dr64")
    n = 64
    st = cfg2_batch(n, dtype)
    ov = np.array([[st.overlays[i][k] for k in CFG2_KEYS] for i in range(n)])
    assert np.array_equal(ov, g["overlay"])  # the device Philox draws == the reference's
    P = st.params
    for k in ("mass", "volume", "thrust_coeff"):
        assert np.array_equal(host(getattr(P, k)), g[f"param_{k}"]), k
    ok, err = rowwise_close(host(P.M_inv), g["param_M_inv"], F64_RTOL)
    assert ok, ("M_inv", err)
    cmds = np.random.default_rng(0).uniform(-1.0, 1.0, size=(100, n, 6))
    rtol, atol = tol(dtype)
    prev = (g["p0"], g["q0"], g["nu0"], g["act0"])
    for t in range(100):
        set_state(st, *prev)
        E.step_batch(st, torch.from_numpy(cmds[t]).to(st.device, dtype))
        for k, arr in (("p", st.p), ("q", st.q), ("nu", st.nu), ("act", st.act)):
            floor = 100.0 if (k == "act" and dtype == torch.float32) else None
            ok, err = rowwise_close(host(arr), g[f"traj_{k}"][t], rtol, atol, floor)
            assert ok, (t, k, err)
        prev = tuple(g[f"traj_{k}"][t] for k in ("p", "q", "nu", "act"))
    assert np.array_equal(host(st.steps), g["steps"])
    assert not st.diverged.any().item()


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_config2_bench_batch_vs_oracle(dtype):
    """The bench's exact workload (4096 envs) against the oracle for 100 steps, the state
    re-injected every step; the oracle draws its own overlays from numpy's Philox."""
    n = 4096
    st = cfg2_batch(n, dtype)
    spec = cfg2_spec()
    b = O.Batch(product_vehicle("bluerov"), n, seed=0)
    b.reset(np.ones(n, bool), lambda i, ep, r: O.Init(overlay=O.draw_overlay(spec, r)))
    assert st.overlays == b.overlays  # 4 x 4096 device draws, bit for bit
    rng = np.random.default_rng(12)
    rtol, atol = tol(dtype)
    for t in range(100):
        cmd = rng.uniform(-1.0, 1.0, (n, 6))
        # the oracle steps from the product's current state (re-injection)
        b.p[:], b.q[:], b.nu[:], b.act[:] = host(st.p), host(st.q), host(st.nu), host(st.act)
        b.step(cmd)
        E.step_batch(st, torch.from_numpy(cmd).to(st.device, dtype))
        for k in ("p", "q", "nu", "act"):
            floor = 100.0 if (k == "act" and dtype == torch.float32) else None
            ok, err = rowwise_close(host(getattr(st, k)), getattr(b, k), rtol, atol, floor)
            assert ok, (t, k, err)
    assert np.array_equal(host(st.steps), b.steps)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_config3_per_run_dispatch_vs_oracle(dtype):
    """Five vehicles mixed at 131,075 envs (the per-type run path): a strided sample of
    rows against per-vehicle oracle batches, three re-injected steps."""
    names = ("bluerov", "bluerov_heavy", "lauv", "iauv", "hauv")
    vehs = [product_vehicle(x) for x in names]
    n = 131_075
    counts = [n // 5] * 5
    counts[-1] += n - sum(counts)
    st = E.make_fleet_batch(vehs, counts, E.SimConfig(batch_size=n), master_seed=0, dtype=dtype)
    E.reset_envs(st, np.ones(n, bool))
    assert st._cstate().n_runs == 5 and n >= 131_072  # per-run dispatch (uuv_b200.cu)
    rng = np.random.default_rng(5)
    starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
    picks = []
    for s0, c in zip(starts, counts):  # run edges + a stride through each run
        rows = np.unique(np.concatenate([[s0, s0 + 1, s0 + c - 2, s0 + c - 1],
                                         np.arange(s0, s0 + c, 997)]))
        picks.append(rows)
    orc = [O.Batch(v, len(r), seed=0) for v, r in zip(vehs, picks)]
    for b in orc:
        b.reset(np.ones(b.n, bool))
    rtol, atol = tol(dtype)
    for t in range(3):
        cmd = np.zeros((n, st.a_max))
        for v, s0, c in zip(vehs, starts, counts):
            cmd[s0:s0 + c, :v.action_dim] = rng.uniform(-1.0, 1.0, (c, v.action_dim))
        P, Q, NU, ACT = host(st.p), host(st.q), host(st.nu), host(st.act)
        E.step_batch(st, torch.from_numpy(cmd).to(st.device, dtype))
        P1, Q1, NU1, ACT1 = host(st.p), host(st.q), host(st.nu), host(st.act)
        for v, b, rows in zip(vehs, orc, picks):
            A = v.action_dim
            b.p[:], b.q[:], b.nu[:], b.act[:] = P[rows], Q[rows], NU[rows], ACT[rows, :A]
            b.step(cmd[rows, :A])
            for k, got in (("p", P1), ("q", Q1), ("nu", NU1)):
                ok, err = rowwise_close(got[rows], getattr(b, k), rtol, atol)
                assert ok, (v.name, t, k, err)
            floor = 100.0 if dtype == torch.float32 else None
            ok, err = rowwise_close(ACT1[rows, :A], b.act, rtol, atol, floor)
            assert ok, (v.name, t, "act", err)
            assert np.all(ACT1[rows, A:] == 0.0)  # padded command columns never act


@pytest.mark.parametrize("name,rng", [("dr_piecewise_jitter", "philox"),
                                      ("dr_piecewise_jitter_pcg64", "pcg64")])
def test_device_piecewise_gaussian_jitter_draws(name, rng):
    """Piecewise (randomization.py:84-117), Gaussian and the vector mount_position_jitter
    key (vehicles/__init__.py:481-494) drawn in the reset kernel == the reference's
    sample_overlay draws, bit for bit; the jittered mounts and 20 steps at 1e-12."""
    g = golden(name)
    spec = SPEC.build(json.loads(str(g["spec"])))
    n = g["p0"].shape[0]
    st = E.make_batch(product_vehicle("bluerov"), E.SimConfig(batch_size=n, substeps=2),
                      master_seed=9, dtype=torch.float64, rng=rng)
    E.reset_envs(st, np.ones(n, bool), E.spec_sampler(spec))
    ovs = st.overlays
    assert np.array_equal(np.array([o["mass*"] for o in ovs]), g["ov_mass"])
    assert np.array_equal(np.array([o["volume*"] for o in ovs]), g["ov_volume"])
    assert np.array_equal(np.array([o["damping*"] for o in ovs]), g["ov_damping"])
    assert np.array_equal(np.array([o["mount_position_jitter"] for o in ovs]), g["ov_jitter"])
    assert np.array_equal(host(st.params.mounts), g["param_mounts"])
    prev = (g["p0"], g["q0"], g["nu0"], g["act0"])
    for t in range(g["cmds"].shape[0]):
        set_state(st, *prev)
        E.step_batch(st, torch.from_numpy(g["cmds"][t]).cuda())
        for k, arr in (("p", st.p), ("q", st.q), ("nu", st.nu), ("act", st.act)):
            ok, err = rowwise_close(host(arr), g[f"traj_{k}"][t], F64_RTOL, 1e-300)
            assert ok, (t, k, err)
        prev = tuple(g[f"traj_{k}"][t] for k in ("p", "q", "nu", "act"))


# ------------------------------------------------------------------ full-size properties


def _rows_of_big_equal_small(make, n_big, picks, m, steps, cmd_fn, fields):
    """make(size, env_offset) -> object with .step(commands) and .state; the rows
    [k, k + m) of the big batch must equal a small batch at env_offset k."""
    big = make(n_big, 0)
    smalls = [(k, make(m, k)) for k in picks]
    for t in range(steps):
        cmd = cmd_fn(t, n_big)
        big.step(cmd)
        for k, s in smalls:
            s.step(cmd[k:k + m])
    for k, s in smalls:
        for f in fields:
            a = getattr(big.state, f)[k:k + m]
            b = getattr(s.state, f)
            assert torch.equal(a, b), (k, f)


@pytest.mark.parametrize("kind", ["tracking_k8", "docking_dr"])
def test_task_configs_at_full_size_equal_small_shards(kind):
    """BASELINE configs[3] / [4] at their stated 1,048,576 envs per GPU: rows of the full
    batch (random streams keyed by the global env index, auto-resets on) equal the same
    rows stepped as small batches with env_offset -- bit for bit, so the fixture-checked
    small-batch behaviour holds at full size (and under any sharding)."""
    from paper_2503_09203_b200.tasks import TaskConfig, make_env

    if kind == "tracking_k8":
        task = TaskConfig(task="tracking", vehicle="bluerov", level="disturbed",
                          episode_length=6)
        substeps = 8
    else:
        task = TaskConfig(task="docking", vehicle="bluerov_heavy", level="disturbed_dr",
                          episode_length=6)
        substeps = 1
    n = 1 << 20

    def make(size, off):
        env = make_env(task, E.SimConfig(batch_size=size, substeps=substeps), seed=0,
                       env_offset=off)
        env.reset()
        return env

    g = torch.Generator(device="cuda").manual_seed(3)
    cmds = [torch.rand((n, 8 if kind == "docking_dr" else 6), device="cuda", generator=g) * 2 - 1
            for _ in range(9)]
    _rows_of_big_equal_small(make, n, (0, 333_333, n - 500), 500, 9, lambda t, _: cmds[t],
                             ("p", "q", "nu", "act", "steps", "episodes", "diverged"))


def test_config2_at_full_size_equals_small_shards():
    """cfg2 at 1M envs (the 96-register large-batch build, DR record prefetch) == the same
    rows as 4096-env shards (the small-batch build), bit for bit."""
    n, m = 1 << 20, 4096
    spec = cfg2_spec()

    class Shard:
        def __init__(self, size, off):
            self.state = E.make_batch(product_vehicle("bluerov"), E.SimConfig(batch_size=size),
                                      master_seed=0, env_offset=off)
            E.reset_envs(self.state, torch.ones(size, dtype=torch.bool, device="cuda"),
                         E.spec_sampler(spec))

        def step(self, cmd):
            E.step_batch(self.state, cmd)

    g = torch.Generator(device="cuda").manual_seed(4)
    cmds = [torch.rand((n, 6), device="cuda", generator=g) * 2 - 1 for _ in range(5)]
    _rows_of_big_equal_small(Shard, n, (0, 500_000, n - m), m, 5, lambda t, _: cmds[t],
                             ("p", "q", "nu", "act", "steps", "diverged"))
