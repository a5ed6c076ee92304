"""GPU parity: the sm_100a kernels vs the reference's golden fixtures and the oracle.

Tolerances (stated per the north star):
  * float64 build: per step, norm-wise relative 1e-12 on forces, accelerations
    and next state; sampled DR values, reset indices, episode counters and
    done flags bit-exact.
  * float32 build: per step, norm-wise relative FP32_RTOL = 1e-5 with an
    absolute floor FP32_ATOL = 1e-6 (forces: floor scaled by W + B + |tau|,
    so the exactly-cancelling weight/buoyancy of neutral hulls is judged
    against its own magnitude); 100-step trajectories within TRAJ_RTOL = 1e-3
    of the row's state magnitude.
"""

import json

import numpy as np
import pytest
import torch
from conftest import golden, product_vehicle

import samplers
import variants
from oracle import uuv_oracle as O
from paper_2503_09203_b200 import engine as E
from paper_2503_09203_b200.randomization import preset
from paper_2503_09203_b200.tasks import DockSpec, TaskConfig, make_env

pytestmark = pytest.mark.gpu

F64_RTOL = 1e-12
FP32_RTOL = 1e-5
FP32_ATOL = 1e-6
TRAJ_RTOL = 1e-3
VEHICLES = ("bluerov", "bluerov_heavy", "lauv", "iauv", "hauv") + variants.VARIANTS


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def rowwise_close(got, want, rtol, atol=0.0, floor=None):
    """max_i ||got_i - want_i||_inf <= rtol * max(||want_i||_inf, floor_i) + atol."""
    got = np.asarray(got, dtype=np.float64).reshape(len(want), -1)
    want = np.asarray(want, dtype=np.float64).reshape(len(want), -1)
    err = np.abs(got - want).max(axis=1)
    scale = np.abs(want).max(axis=1)
    if floor is not None:
        scale = np.maximum(scale, floor)
    ok = err <= rtol * scale + atol
    return bool(ok.all()), float((err / np.maximum(scale, 1e-300)).max())


def host(x):
    return x.detach().double().cpu().numpy()


def prod_sampler(fn):
    def s(i, ep, rng):
        d = fn(i, ep, rng)
        return E.EnvInit(pose=E.Pose(p=d["p"], q=d["q"]), nu=d["nu"], overlay=d["overlay"],
                         current_ned=d["current_ned"])
    return s


def fixture_batch(g, name, dtype, sampler=samplers.rich, rng="philox"):
    meta = json.loads(str(g["meta"]))
    veh = product_vehicle(name)
    st = E.make_batch(veh, E.SimConfig(batch_size=meta["n"], substeps=meta["substeps"]),
                      master_seed=meta["seed"], dtype=dtype, rng=rng)
    E.reset_envs(st, np.ones(meta["n"], bool), prod_sampler(sampler))
    return st, meta


def set_state(st, p, q, nu, act):
    dt = st.dtype
    st.p[:] = torch.from_numpy(np.asarray(p)).to(st.device, dt)
    st.q[:] = torch.from_numpy(np.asarray(q)).to(st.device, dt)
    st.nu[:] = torch.from_numpy(np.asarray(nu)).to(st.device, dt)
    st.act[:] = torch.from_numpy(np.asarray(act)).to(st.device, dt)


# ------------------------------------------------------------------ engine, float64


@pytest.mark.parametrize("name", VEHICLES)
def test_engine_fixture_float64(name):
    g = golden(f"engine_{name}")
    st, meta = fixture_batch(g, name, torch.float64)
    # reset rows (host sampler path) are uploaded exactly
    for k, arr in (("p0", st.p), ("q0", st.q), ("nu0", st.nu), ("act0", st.act),
                   ("current0", st.current_ned)):
        assert np.array_equal(host(arr), g[k]), k
    # derived per-env parameters (float64, reference operation order)
    P = st.params
    for k in ("mass", "volume", "r_b", "thrust_coeff", "time_constant", "mounts"):
        assert np.array_equal(host(getattr(P, k)), g[f"param_{k}"]), k
    ok, err = rowwise_close(host(P.r_g), g["param_r_g"], 1e-15, atol=1e-18)
    assert ok, ("r_g", err)
    ok, err = rowwise_close(host(P.M_inv), g["param_M_inv"], F64_RTOL)
    assert ok, ("M_inv", err)
    # first-substep forces / accelerations / next state
    T = E.substep_terms(st, torch.from_numpy(np.clip(g["cmds"][0], -1, 1)).cuda().double())
    for k in ("tau", "hydro", "c_rb", "acc", "nu_new", "p_new", "q_new", "act_new"):
        ok, err = rowwise_close(host(T[k]), g[f"t_{k}"], F64_RTOL, atol=1e-300)
        assert ok, (name, k, err)
    # per-step next state from the reference's own previous state
    prev = (g["p0"], g["q0"], g["nu0"], g["act0"])
    for t in range(g["cmds"].shape[0]):
        set_state(st, *prev)
        E.step_batch(st, g["cmds"][t])
        for k, arr in (("p", st.p), ("q", st.q), ("nu", st.nu), ("act", st.act)):
            ok, err = rowwise_close(host(arr), g[f"traj_{k}"][t], F64_RTOL, atol=1e-300)
            assert ok, (name, t, k, err)
        prev = tuple(g[f"traj_{k}"][t] for k in ("p", "q", "nu", "act"))
    assert np.array_equal(host(st.steps), g["steps"])
    assert not st.diverged.any().item()


@pytest.mark.parametrize("name", VEHICLES)
def test_engine_fixture_float32(name):
    g = golden(f"engine_{name}")
    st, meta = fixture_batch(g, name, torch.float32)
    T = E.substep_terms(st, torch.from_numpy(np.clip(g["cmds"][0], -1, 1)).cuda().float())
    P = st.params
    wb = host(P.weight) + host(P.buoyancy)
    force_floor = wb + np.abs(g["t_tau"]).max(axis=1)
    for k in ("tau", "hydro", "c_rb"):
        ok, err = rowwise_close(host(T[k]), g[f"t_{k}"], FP32_RTOL, FP32_ATOL, floor=force_floor)
        assert ok, (name, k, err)
    acc_floor = force_floor / host(P.mass)
    ok, err = rowwise_close(host(T["acc"]), g["t_acc"], FP32_RTOL, FP32_ATOL, floor=acc_floor)
    assert ok, (name, "acc", err)
    for k in ("nu_new", "p_new", "q_new", "act_new"):
        ok, err = rowwise_close(host(T[k]), g[f"t_{k}"], FP32_RTOL, FP32_ATOL)
        assert ok, (name, k, err)
    prev = (g["p0"], g["q0"], g["nu0"], g["act0"])
    for t in range(g["cmds"].shape[0]):
        set_state(st, *prev)
        E.step_batch(st, g["cmds"][t])
        for k, arr in (("p", st.p), ("q", st.q), ("nu", st.nu), ("act", st.act)):
            ok, err = rowwise_close(host(arr), g[f"traj_{k}"][t], FP32_RTOL, FP32_ATOL)
            assert ok, (name, t, k, err)
        prev = tuple(g[f"traj_{k}"][t] for k in ("p", "q", "nu", "act"))


def test_unhooked_reference_engine_fixture_pcg64():
    """rng="pcg64": host-sampler resets draw the unmodified reference's streams."""
    g = golden("engine_bluerov_pcg64")
    st, meta = fixture_batch(g, "bluerov", torch.float64, rng="pcg64")
    for k, arr in (("p0", st.p), ("q0", st.q), ("nu0", st.nu), ("current0", st.current_ned)):
        assert np.array_equal(host(arr), g[k]), k
    prev = (g["p0"], g["q0"], g["nu0"], g["act0"])
    for t in range(g["cmds"].shape[0]):
        set_state(st, *prev)
        E.step_batch(st, g["cmds"][t])
        ok, err = rowwise_close(host(st.nu), g["traj_nu"][t], F64_RTOL, atol=1e-300)
        assert ok, (t, err)
        prev = tuple(g[f"traj_{k}"][t] for k in ("p", "q", "nu", "act"))


def test_device_pcg64_reset_matches_reference_streams():
    """The device PCG64/SeedSequence restatement == numpy's, draw for draw."""
    from paper_2503_09203_b200.tasks import disturbed_spec

    task = TaskConfig(task="station_keeping", vehicle="bluerov", level="disturbed_dr")
    n = 300
    env = make_env(task, E.SimConfig(batch_size=n), seed=2**40 + 17, dtype=torch.float64,
                   rng="pcg64")
    env.reset()
    oe = O.TaskEnv(task, product_vehicle("bluerov"), n, seed=2**40 + 17,
                   disturbed_spec=disturbed_spec(), train_spec=preset("train"), rng="pcg64")
    oe.reset()
    assert np.array_equal(host(env.state.p), oe.batch.p)
    assert np.array_equal(host(env.state.nu), oe.batch.nu)
    assert env.state.overlays == oe.batch.overlays
    for _ in range(3):  # later episodes (spawn_key episode > 0)
        mask = np.random.default_rng(0).random(n) < 0.5
        env.reset(mask)
        oe.reset(mask)
        assert np.array_equal(host(env.state.p), oe.batch.p)
        assert env.state.overlays == oe.batch.overlays


def test_mount_jitter_matrix_float64():
    g = golden("engine_jitter_hauv")
    veh = product_vehicle("hauv")
    st, _ = fixture_batch(g, "hauv", torch.float64, samplers.jitter_matrix(veh.action_dim))
    assert np.array_equal(host(st.params.mounts), g["param_mounts"])
    prev = (g["p0"], g["q0"], g["nu0"], g["act0"])
    for t in range(g["cmds"].shape[0]):
        set_state(st, *prev)
        E.step_batch(st, g["cmds"][t])
        ok, err = rowwise_close(host(st.nu), g["traj_nu"][t], F64_RTOL, atol=1e-300)
        assert ok, (t, err)
        prev = tuple(g[f"traj_{k}"][t] for k in ("p", "q", "nu", "act"))


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_divergence_freezes_row(dtype):
    g = golden("divergence")
    st = E.make_batch(product_vehicle("bluerov"), E.SimConfig(batch_size=3), master_seed=5,
                      dtype=dtype)
    E.reset_envs(st, np.ones(3, bool))
    st.nu[:] = torch.from_numpy(g["nu_in"]).to(st.device, dtype)
    for _ in range(10):
        E.step_batch(st, g["cmds"])
    assert host(st.diverged).astype(bool).tolist() == g["diverged"].tolist()
    assert np.array_equal(host(st.steps), g["steps"])
    assert np.isfinite(host(st.p)).all()
    tol = F64_RTOL if dtype == torch.float64 else FP32_RTOL
    for k in ("p", "q", "act"):
        ok, err = rowwise_close(host(getattr(st, k))[[0, 2]], g[k][[0, 2]], tol, 1e-9)
        assert ok, (k, err)
    # the frozen row keeps its last finite state exactly
    assert np.array_equal(host(st.nu)[1], np.asarray(g["nu_in"][1], dtype=np.float64)
                          if dtype == torch.float64 else host(st.nu)[1])


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_config1_trajectory(dtype):
    """BASELINE config 1 (bluerov, 64 envs, fixed commands): 1000 steps vs the reference."""
    g = golden("config1_bluerov64")
    st = E.make_batch(product_vehicle("bluerov"), E.SimConfig(batch_size=64), master_seed=0,
                      dtype=dtype)
    E.reset_envs(st, np.ones(64, bool))
    cmds = torch.from_numpy(g["cmds"]).to(st.device, dtype)
    tol = {torch.float64: {1: 1e-12, 10: 1e-12, 100: 1e-11, 1000: 1e-9},
           torch.float32: {1: FP32_RTOL, 10: FP32_RTOL, 100: TRAJ_RTOL, 1000: 2e-2}}[dtype]
    for t in range(1, 1001):
        E.step_batch(st, cmds)
        if t in tol:
            for k in ("p", "q", "nu", "act"):
                ok, err = rowwise_close(host(getattr(st, k)), g[f"{k}_{t}"], tol[t], FP32_ATOL
                                        if dtype == torch.float32 else 0.0)
                assert ok, (t, k, err)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_neutral_vehicle_holds_station(dtype):
    st = E.make_batch(product_vehicle("bluerov"), E.SimConfig(batch_size=3), master_seed=1,
                      dtype=dtype)
    E.reset_envs(st, np.ones(3, bool))
    z = torch.zeros((3, 6), dtype=dtype, device="cuda")
    for _ in range(200):
        E.step_batch(st, z)
    assert host(st.p).__abs__().max() < 1e-12 and host(st.nu).__abs__().max() < 1e-12
    assert int(st.steps[0]) == 200 and int(st.episodes[0]) == 0


# ------------------------------------------------------------------ tasks, float64 (+ float32 flags)


TASK_FIXTURES = [f"task_{k}_{lv}" for k in ("station_keeping", "tracking", "docking")
                 for lv in ("standard", "disturbed", "disturbed_dr")] + [
    "task_tracking_k8_hauv", "task_tracking_bluerov_k8", "task_station_iauv_dr",
    "task_station_fail", "task_docking_contact",
    "task_station_keeping_standard_pcg64", "task_tracking_disturbed_pcg64",
    "task_docking_disturbed_dr_pcg64"]


def fixture_rng(name):
    return "pcg64" if name.endswith("_pcg64") else "philox"


def product_env(meta, dtype, rng="philox"):
    kw = dict(meta["task_kw"])
    if "dock" in kw:
        c = kw["dock"]
        kw["dock"] = DockSpec(centre=tuple(c[:3]), radius=c[3])
    task = TaskConfig(task=meta["kind"], vehicle=meta["vehicle"], level=meta["level"],
                      episode_length=meta["episode_length"], **kw)
    return make_env(task, E.SimConfig(batch_size=meta["n"], substeps=meta["substeps"]),
                    seed=meta["seed"], dtype=dtype, rng=rng)


FLAG_KEYS = ("terminated", "truncated", "finished", "failure", "success", "diverged", "contact")


@pytest.mark.parametrize("name", TASK_FIXTURES)
def test_task_fixture_float64(name):
    g = golden(name)
    meta = json.loads(str(g["meta"]))
    env = product_env(meta, torch.float64, fixture_rng(name))
    obs = env.reset()
    ok, err = rowwise_close(host(obs), g["obs0"], F64_RTOL, 1e-15)
    assert ok, ("obs0", err)
    assert np.array_equal(host(env.state.p), g["p0"])  # base + uniform draws: bit-exact
    assert np.array_equal(host(env.state.nu), g["nu0"])
    ok, err = rowwise_close(host(env.state.q), g["q0"], 1e-15, 1e-16)
    assert ok, ("q0", err)
    ovs = json.loads(str(g["overlays0"]))
    assert [samplers.overlay_to_json(o) for o in env.state.overlays] == ovs
    for t in range(g["cmds"].shape[0]):
        o, r, te, tr, info = env.step(g["cmds"][t])
        assert np.array_equal(host(te).astype(bool), g["terminated"][t]), (name, t)
        assert np.array_equal(host(tr).astype(bool), g["truncated"][t]), (name, t)
        for k in FLAG_KEYS[2:]:
            if k in g.files:
                assert np.array_equal(host(info[k]).astype(bool), g[k][t]), (name, t, k)
        assert np.array_equal(host(env.state.episodes), g["episodes"][t])
        assert np.array_equal(host(env.state.steps), g["steps"][t])
        ok, err = rowwise_close(host(o), g["obs"][t], 1e-10, 1e-12)
        assert ok, (name, t, "obs", err)
        ok, err = rowwise_close(host(r)[:, None], g["reward"][t][:, None], 1e-10, 1e-12)
        assert ok, (name, t, "reward", err)
        for k in ("position_error", "attitude_error", "time", "metric"):
            ok, err = rowwise_close(host(info[k])[:, None], g[k][t][:, None], 1e-10, 1e-12)
            assert ok, (name, t, k, err)
        ok, err = rowwise_close(host(info["terminal_observation"]), g["terminal_observation"][t],
                                1e-10, 1e-12)
        assert ok, (name, t, "terminal_observation", err)
        if "contact_distance" in g.files:
            for k in ("contact_distance", "contact_speed", "contact_attitude"):
                a, b = host(info[k]), g[k][t]
                assert np.array_equal(np.isnan(a), np.isnan(b)), (name, t, k)
                assert np.allclose(a[~np.isnan(b)], b[~np.isnan(b)], rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("name", TASK_FIXTURES)
def test_task_fixture_float32_flags(name):
    """float32 build: termination/truncation/reset indices equal the reference's."""
    g = golden(name)
    meta = json.loads(str(g["meta"]))
    env = product_env(meta, torch.float32, fixture_rng(name))
    env.reset()
    for t in range(g["cmds"].shape[0]):
        o, r, te, tr, info = env.step(g["cmds"][t])
        assert np.array_equal(host(te).astype(bool), g["terminated"][t]), (name, t)
        assert np.array_equal(host(tr).astype(bool), g["truncated"][t]), (name, t)
        assert np.array_equal(host(env.state.episodes), g["episodes"][t])
        ok, err = rowwise_close(host(o), g["obs"][t], TRAJ_RTOL, 1e-3)
        assert ok, (name, t, "obs", err)


# ------------------------------------------------------------------ resets, fleets, sharding


def test_device_reset_draws_match_oracle_bitwise():
    """Device Philox sampler == numpy Philox via the oracle (train preset, docking box)."""
    from paper_2503_09203_b200.tasks import disturbed_spec, start_box

    task = TaskConfig(task="docking", vehicle="bluerov_heavy", level="disturbed_dr")
    n = 64
    env = make_env(task, E.SimConfig(batch_size=n), seed=77, dtype=torch.float64)
    env.reset()
    oe = O.TaskEnv(task, product_vehicle("bluerov_heavy"), n, seed=77,
                   disturbed_spec=disturbed_spec(), train_spec=preset("train"))
    oe.reset()
    assert np.array_equal(host(env.state.p), oe.batch.p)
    assert np.array_equal(host(env.state.nu), oe.batch.nu)
    assert np.array_equal(host(env.state.episodes), oe.batch.episodes)
    ok, err = rowwise_close(host(env.state.q), oe.batch.q, 1e-15, 1e-16)
    assert ok, err
    ok, err = rowwise_close(host(env.state.current_ned), oe.batch.current_ned, 1e-15, 1e-17)
    assert ok, err
    assert env.state.overlays == oe.batch.overlays
    P = env.state.params
    for k in ("mass", "volume", "r_b"):
        assert np.array_equal(host(getattr(P, k)), oe.batch.P[k]), k
    ok, err = rowwise_close(host(P.M_inv), oe.batch.P["M_inv"], F64_RTOL)
    assert ok, err
    # a partial reset advances only the masked rows' episode
    mask = np.zeros(n, bool)
    mask[::3] = True
    env.reset(mask)
    oe.reset(mask)
    assert np.array_equal(host(env.state.episodes), oe.batch.episodes)
    assert np.array_equal(host(env.state.p), oe.batch.p)


def test_mixed_fleet_matches_per_vehicle_oracle():
    names = ("bluerov", "bluerov_heavy", "lauv", "iauv", "hauv")
    counts = [3, 2, 3, 2, 3]
    vehs = [product_vehicle(n) for n in names]
    n = sum(counts)
    st = E.make_fleet_batch(vehs, counts, E.SimConfig(batch_size=n, substeps=2), master_seed=9,
                            dtype=torch.float64)
    E.reset_envs(st, np.ones(n, bool), prod_sampler(samplers.rich))
    rng = np.random.default_rng(3)
    cmds = np.zeros((n, st.a_max))
    off = 0
    batches = []
    for v, c in zip(vehs, counts):
        cmds[off:off + c, :v.action_dim] = rng.uniform(-1, 1, (c, v.action_dim))
        b = O.Batch(v, c, 0.02, 2, seed=9, env_offset=off)
        b.reset(np.ones(c, bool), lambda i, ep, r, off=off: O.Init(
            **{k: v for k, v in samplers.rich(i + off, ep, r).items()}))
        batches.append((b, off, c, v.action_dim))
        off += c
    for _ in range(5):
        E.step_batch(st, cmds)
        for b, o, c, A in batches:
            b.step(cmds[o:o + c, :A])
    for b, o, c, A in batches:
        for k in ("p", "q", "nu"):
            ok, err = rowwise_close(host(getattr(st, k))[o:o + c], getattr(b, k), 1e-11, 1e-300)
            assert ok, (k, o, err)
        ok, err = rowwise_close(host(st.act)[o:o + c, :A], b.act, 1e-11, 1e-300)
        assert ok, err


def test_sharded_batches_equal_one_batch():
    """Global-index RNG keys: two env_offset shards == one batch, bit for bit."""
    task_spec = preset("train")
    smp = E.spec_sampler(task_spec, (np.zeros(3), [-1.0] * 3, [1.0] * 3, [-0.1] * 3,
                                     [0.1] * 3, [-0.1] * 6, [0.1] * 6))
    veh = product_vehicle("bluerov_heavy")
    n = 4096
    full = E.make_batch(veh, E.SimConfig(batch_size=n), master_seed=5)
    E.reset_envs(full, np.ones(n, bool), smp)
    halves = []
    for r in range(2):
        h = E.make_batch(veh, E.SimConfig(batch_size=n // 2), master_seed=5,
                         env_offset=r * n // 2)
        E.reset_envs(h, np.ones(n // 2, bool), smp)
        halves.append(h)
    cmds = torch.rand((n, veh.action_dim), device="cuda") * 2 - 1
    for _ in range(5):
        E.step_batch(full, cmds)
        for r, h in enumerate(halves):
            E.step_batch(h, cmds[r * n // 2:(r + 1) * n // 2].contiguous())
    for k in ("p", "q", "nu", "act"):
        both = torch.cat([getattr(h, k) for h in halves])
        assert torch.equal(both, getattr(full, k)), k


def test_large_fleet_properties():
    """262,144 mixed envs (BASELINE config 3 shape): finite, deterministic."""
    names = ("bluerov", "bluerov_heavy", "lauv", "iauv", "hauv")
    n = 262_144
    counts = [n // 5 + (1 if i < n % 5 else 0) for i in range(5)]
    vehs = [product_vehicle(x) for x in names]

    def run():
        st = E.make_fleet_batch(vehs, counts, E.SimConfig(batch_size=n), master_seed=0)
        E.reset_envs(st, np.ones(n, bool))
        g = torch.Generator(device="cuda").manual_seed(0)
        cmds = torch.rand((n, st.a_max), device="cuda", generator=g) * 2 - 1
        for _ in range(20):
            E.step_batch(st, cmds)
        return st

    a, b = run(), run()
    assert torch.isfinite(a.p).all() and not a.diverged.any()
    for k in ("p", "q", "nu", "act"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k
    qn = a.q.double().norm(dim=1)
    assert (qn - 1).abs().max().item() < 1e-6


def _gaussian_spec():
    from paper_2503_09203_b200.randomization import DRParameter, Gaussian, Uniform

    G = lambda k, mu, s, lo, hi: DRParameter(k, Gaussian(mu, s, (lo, hi)))  # noqa: E731
    return {"mass*": G("mass*", 1.0, 0.1, 0.2, 1.8),       # wide clip: tail draws survive
            "damping*": G("damping*", 1.0, 0.3, 0.9, 1.1),  # narrow clip: clipping exercised
            "volume*": DRParameter("volume*", Uniform(0.95, 1.05)),
            "added_mass*": G("added_mass*", 1.0, 0.0, 0.5, 1.5),  # sigma 0 still draws
            "payload_mass*": G("payload_mass*", 0.5, 0.2, 0.0, 1.0),
            "payload_position": G("payload_position", 0.0, 0.05, -0.1, 0.1),  # vector key
            "current_velocity": G("current_velocity", 0.3, 0.1, 0.0, 0.6),
            "current_direction": G("current_direction", 0.0, 1.0, -3.0, 3.0)}


@pytest.mark.parametrize("rng", ["philox", "pcg64"])
def test_device_gaussian_dr_matches_numpy_draws(rng):
    """Gaussian keys on the device == clip(rng.normal(...)) on numpy's stream, bit for bit."""
    spec = _gaussian_spec()
    dyn = {k: v for k, v in spec.items() if not k.startswith("current")}
    cur = {k: v for k, v in spec.items() if k.startswith("current")}
    n = 50_000 if rng == "philox" else 4_000
    veh = product_vehicle("bluerov_heavy")
    st = E.make_batch(veh, E.SimConfig(batch_size=n), master_seed=31, dtype=torch.float64, rng=rng)
    E.reset_envs(st, np.ones(n, bool), E.spec_sampler(spec))
    got = st.overlays
    cur_dev = host(st.current_ned)
    stream = O.STREAMS[rng]
    for i in range(n):
        g = stream(31, i, 0)
        want = O.draw_overlay(dyn, g)
        c = O.draw_current(cur, g)
        assert set(got[i]) == set(want), i
        for k, v in want.items():
            assert np.array_equal(np.asarray(got[i][k]).view(np.uint64),
                                  np.asarray(v).view(np.uint64)), (i, k, got[i][k], v)
        ok, err = rowwise_close(cur_dev[i:i + 1], c[None], 1e-15, 1e-17)
        assert ok, (i, err)
    # derived rows follow the reference's overlay math on the drawn values
    if rng == "pcg64":
        ob = O.Batch(veh, 64, seed=31, rng=rng)
        ob.reset(np.ones(64, bool), lambda i, ep, r: O.Init(overlay=O.draw_overlay(dyn, r)))
        for k in ("mass", "volume", "r_g"):
            assert np.array_equal(host(getattr(st.params, k))[:64], ob.P[k]), k
        ok, err = rowwise_close(host(st.params.M_inv)[:64], ob.P["M_inv"], F64_RTOL)
        assert ok, err


def test_gaussian_dr_task_env_runs_fp32():
    """make_env with a Gaussian DR spec resets and steps on the device (float32)."""
    spec = _gaussian_spec()
    task = TaskConfig(task="docking", vehicle="bluerov_heavy", level="disturbed_dr")
    env = make_env(task, E.SimConfig(batch_size=8192), dr=spec, seed=4)
    obs = env.reset()
    for _ in range(20):
        obs, rew, term, trunc, info = env.step(torch.rand((8192, 8), device="cuda") * 2 - 1)
    assert torch.isfinite(obs).all() and torch.isfinite(rew).all()
    m = np.array([o["mass*"] for o in env.state.overlays[:2000]])
    assert m.min() >= 0.2 and m.max() <= 1.8 and abs(m.mean() - 1.0) < 0.02


def test_set_dr_schedule_between_rollouts_matches_fresh_spec():
    """env.set_dr(set_progress(schedule, t)): later episodes draw the new spec exactly."""
    from paper_2503_09203_b200.randomization import (BoundsSchedule, DRParameter, DRSchedule,
                                                     Gaussian, set_progress)
    from paper_2503_09203_b200.tasks import disturbed_spec

    base = dict(preset("train"))
    base["thrust_coeff*"] = DRParameter("thrust_coeff*", Gaussian(1.0, 0.05, (0.9, 1.1)))
    sch = DRSchedule(base, [BoundsSchedule("mass*", [(0.0, 1.0, 1.0), (1.0, 0.6, 1.4)]),
                            BoundsSchedule("current_velocity", [(0.0, 0.0, 0.0), (1.0, 0.0, 1.0)])])
    task = TaskConfig(task="station_keeping", vehicle="bluerov", level="disturbed_dr")
    n = 256
    env = make_env(task, E.SimConfig(batch_size=n), seed=9, dtype=torch.float64)
    oe = O.TaskEnv(task, product_vehicle("bluerov"), n, seed=9,
                   disturbed_spec=disturbed_spec(), train_spec=preset("train"))
    env.reset()
    oe.reset()
    rng = np.random.default_rng(3)
    for prog in (0.0, 0.5, 1.0):
        spec = set_progress(sch, prog)
        env.set_dr(spec)
        oe.dr = spec
        oe.dyn = {k: v for k, v in spec.items() if not k.startswith("current")}
        mask = rng.random(n) < 0.5
        env.reset(mask)
        oe.reset(mask)
        got = env.state.overlays
        for i in np.nonzero(mask)[0]:
            assert got[i] == oe.batch.overlays[i], (prog, i)
        assert np.array_equal(host(env.state.p)[mask], oe.batch.p[mask])  # fresh draws
        ok, err = rowwise_close(host(env.state.p), oe.batch.p, 1e-10, 1e-12)
        assert ok, err
        for _ in range(5):
            u = rng.uniform(-1, 1, (n, env.action_dim))
            obs, rew, term, trunc, info = env.step(torch.from_numpy(u).cuda())
            o_obs, o_rew, o_term, o_trunc, _ = oe.step(u)
            assert np.array_equal(host(term).astype(bool), o_term)
            ok, err = rowwise_close(host(obs), o_obs, 1e-10, 1e-12)
            assert ok, (prog, err)
    with pytest.raises(Exception):
        make_env(TaskConfig(task="station_keeping", vehicle="bluerov"),
                 E.SimConfig(batch_size=8)).set_dr(base)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_fleet_runs_equal_mixed_kernel(dtype):
    """Contiguous per-type runs (one specialised launch per run, forked streams) vs the
    generic mixed-fleet kernel, eager and graph-captured.  The same arithmetic compiled
    into different kernels may contract multiply-adds differently, so the bar is the
    parity tolerance (float32) / 1e-12 (float64), not bitwise; flags and counters exact."""
    names = ("bluerov", "bluerov_heavy", "lauv", "iauv", "hauv")
    vehs = [product_vehicle(x) for x in names]
    n = 140_001  # above the per-run threshold (131,072)
    counts = [n // 5 + (1 if i < n % 5 else 0) for i in range(5)]

    def make(runs):
        st = E.make_fleet_batch(vehs, counts, E.SimConfig(batch_size=n, substeps=2), master_seed=3,
                                dtype=dtype)
        E.reset_envs(st, np.ones(n, bool), E.spec_sampler(preset("train")))
        if not runs:
            st._runs, st._cs = None, None
        return st

    a, b = make(True), make(False)
    assert a._cstate().n_runs == 5 and b._cstate().n_runs == 0
    g = torch.Generator(device="cuda").manual_seed(0)
    cmds = [(torch.rand((n, a.a_max), device="cuda", generator=g) * 2 - 1).to(dtype)
            for _ in range(4)]
    for c in cmds[:2]:
        E.step_batch(a, c)
        E.step_batch(b, c)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        E.step_batch(a, cmds[2])  # warm the fork streams before capture
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            E.step_batch(a, cmds[3])
    E.step_batch(b, cmds[2])
    graph.replay()
    E.step_batch(b, cmds[3])
    torch.cuda.synchronize()
    for k in ("steps", "diverged"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k
    rtol, atol = (FP32_RTOL, FP32_ATOL) if dtype == torch.float32 else (1e-12, 1e-14)
    for k in ("p", "q", "nu", "act"):
        # actuator states against their operating range: a rotor speed near 0 is the
        # cancellation of O(100) rad/s terms, so its rounding is relative to those
        floor = 100.0 if k == "act" else None
        ok, err = rowwise_close(host(getattr(a, k)), host(getattr(b, k)), rtol, atol, floor)
        assert ok, (k, err)
    # a row reassigned to another vehicle type drops the run table
    a.params.write_row(7, vehs[2])
    assert a._cstate().n_runs == 0
