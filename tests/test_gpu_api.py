"""Reference API contract on the GPU build (mirrors pkg/tests/test_engine.py and
test_tasks.py of the reference, run through the product's kernels)."""

import numpy as np
import pytest
import torch

from paper_2503_09203_b200 import engine as E
from paper_2503_09203_b200.tasks import (
    LEVELS, METRIC_DEFINITIONS, TASK_KINDS, DockSpec, TaskConfig, TaskError, TrajectorySpec,
    make_env,
)
from paper_2503_09203_b200.vehicles import load_vehicle

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def h(x):
    return x.detach().double().cpu().numpy()


# ---------------------------------------------------------------- engine (test_engine.py)


def test_command_and_mask_shape_errors():
    veh = load_vehicle("bluerov")
    st = E.make_batch(veh, E.SimConfig(batch_size=3), master_seed=0)
    E.reset_envs(st, np.ones(3, bool))
    with pytest.raises(E.EngineError, match="commands"):
        E.step_batch(st, np.zeros((3, veh.action_dim + 1)))
    with pytest.raises(E.EngineError, match="mask"):
        E.reset_envs(st, np.ones(4, bool))


def test_identical_envs_stay_bitwise_identical():
    veh = load_vehicle("bluerov")
    st = E.make_batch(veh, E.SimConfig(batch_size=8), master_seed=3)
    E.reset_envs(st, np.ones(8, bool))
    rng = np.random.default_rng(0)
    for _ in range(100):
        row = rng.uniform(-1, 1, size=(1, veh.action_dim))
        E.step_batch(st, np.repeat(row, 8, axis=0))
    for arr in (st.p, st.q, st.nu, st.act):
        a = h(arr)
        assert all(a[i].tobytes() == a[0].tobytes() for i in range(8))


def test_worker_count_does_not_change_results():
    veh = load_vehicle("lauv")
    outs = []
    for workers in (1, 2, 5):
        st = E.make_batch(veh, E.SimConfig(batch_size=5, workers=workers), master_seed=9)
        E.reset_envs(st, np.ones(5, bool))
        rng = np.random.default_rng(11)
        for _ in range(50):
            E.step_batch(st, rng.uniform(-1, 1, size=(5, veh.action_dim)))
        outs.append(tuple(h(getattr(st, k)) for k in ("p", "q", "nu", "act")))
    for other in outs[1:]:
        assert all(a.tobytes() == b.tobytes() for a, b in zip(outs[0], other))


def pose_sampler(i, ep, rng):
    return E.EnvInit(pose=E.Pose(p=rng.uniform(-1, 1, 3)), nu=rng.uniform(-0.1, 0.1, 6))


def test_reset_streams_are_seeded_and_per_episode():
    veh = load_vehicle("bluerov")
    a = E.make_batch(veh, E.SimConfig(batch_size=4), master_seed=77)
    b = E.make_batch(veh, E.SimConfig(batch_size=4), master_seed=77)
    E.reset_envs(a, np.ones(4, bool), pose_sampler)
    E.reset_envs(b, np.ones(4, bool), pose_sampler)
    assert torch.equal(a.p, b.p) and torch.equal(a.nu, b.nu)
    first = a.p.clone()
    E.reset_envs(a, np.array([True, False, False, False]), pose_sampler)
    assert not torch.equal(a.p[0], first[0])
    assert torch.equal(a.p[1:], first[1:])
    assert h(a.episodes).tolist() == [1, 0, 0, 0]


def test_env_rng_is_counter_based():
    veh = load_vehicle("bluerov")
    st = E.make_batch(veh, E.SimConfig(batch_size=2), master_seed=123)
    E.reset_envs(st, np.ones(2, bool))
    want = E.philox_generator(123, 1, 0)
    assert st.env_rng(1).uniform() == want.uniform()


def test_env_snapshot_fields():
    veh = load_vehicle("hauv")
    st = E.make_batch(veh, E.SimConfig(batch_size=2), master_seed=4)
    E.reset_envs(st, np.ones(2, bool), pose_sampler)
    E.step_batch(st, np.zeros((2, veh.action_dim)))
    snap = E.env_snapshot(st, 0)
    assert set(snap) == {"p", "q", "nu", "act", "current_ned", "steps", "episode", "diverged",
                         "overlay"}
    assert snap["steps"] == 1 and snap["episode"] == 0 and snap["diverged"] is False
    assert snap["p"].shape == (3,) and snap["act"].shape == (veh.action_dim,)
    snap["p"][:] = 99.0
    assert float(st.p[0, 0]) != 99.0


def test_current_rotates_into_body_frame():
    q = torch.tensor([np.cos(np.pi / 4), 0.0, 0.0, np.sin(np.pi / 4)], dtype=torch.float64)
    nu_c = E.current_in_body(q, torch.tensor([1.0, 0.0, 0.0], dtype=torch.float64))
    assert np.abs(nu_c.numpy() - np.array([0, -1, 0, 0, 0, 0])).max() < 1e-12


@pytest.mark.parametrize("mode", ["rollout", "graph", "launch"])
def test_throughput_probe_reports(mode):
    rep = E.throughput_probe(E.SimConfig(batch_size=16), load_vehicle("bluerov"), duration=0.05,
                             warmup_steps=2, seed=0, mode=mode)
    assert rep.batch_size == 16 and rep.n_steps > 0
    assert rep.aggregate_steps_per_s == pytest.approx(16 * rep.n_steps / rep.elapsed_s)
    assert rep.diverged_envs == 0
    with pytest.raises(E.EngineError):
        E.throughput_probe(E.SimConfig(batch_size=16), load_vehicle("bluerov"), mode="other")


def test_write_row_gives_one_env_new_parameters():
    base = load_vehicle("bluerov")
    heavy = load_vehicle("bluerov")
    heavy.rb.mass = base.rb.mass * 2.0
    st = E.make_batch(base, E.SimConfig(batch_size=3), master_seed=0)
    E.reset_envs(st, np.ones(3, bool))
    st.params.write_row(1, heavy)
    assert h(st.params.mass).tolist() == [base.rb.mass, 2 * base.rb.mass, base.rb.mass]
    for _ in range(20):
        E.step_batch(st, np.zeros((3, 6)))
    # the heavier row sinks (W > B), the neutral rows hold station
    assert float(st.p[1, 2]) > 1e-3 and abs(float(st.p[0, 2])) < 1e-9


def test_free_drift_only_dissipates_energy():
    """Random neutral hulls (diagonal, no offsets), no thrust/current: kinetic energy
    never increases (acceptance test_free_drift_only_dissipates_energy, 5 hulls/batch)."""
    import copy

    base = load_vehicle("bluerov")
    rng = np.random.default_rng(42)
    hulls = []
    for _ in range(5):  # + the base hull = the 6 parameter sets a batch can hold
        v = copy.deepcopy(base)
        vol = rng.uniform(0.008, 0.02)
        v.rb.mass, v.rb.displaced_volume = 1000.0 * vol, vol
        v.rb.inertia = np.diag(rng.uniform(0.05, 0.5, 3))
        v.rb.r_g, v.rb.r_b = np.zeros(3), np.zeros(3)
        md = np.concatenate([v.rb.mass + rng.uniform(0.2, 1.5, 3) * v.rb.mass,
                             np.diag(v.rb.inertia) * (1 + rng.uniform(0.2, 1.5, 3))])
        ma = md - np.concatenate([[v.rb.mass] * 3, np.diag(v.rb.inertia)])
        v.coeffs.M_A = np.diag(ma)
        v.coeffs.D_lin = np.diag(rng.uniform(0.5, 4.0, 6) * md)
        v.coeffs.D_quad = np.diag(rng.uniform(0.0, 3.0, 6) * md)
        hulls.append(v)
    n = 60

    def drift(i, ep, r):
        axis = r.normal(size=3)
        axis /= np.linalg.norm(axis)
        ang = r.uniform(-np.pi, np.pi)
        q = np.concatenate([[np.cos(ang / 2)], axis * np.sin(ang / 2)])
        return E.EnvInit(pose=E.Pose(q=q), nu=r.uniform(-0.5, 0.5, 6))

    st = E.make_batch(base, E.SimConfig(batch_size=n), master_seed=0, dtype=torch.float64)
    E.reset_envs(st, np.ones(n, bool), drift)
    for i in range(n):
        st.params.write_row(i, hulls[i % 5])
    Ms = [np.diag(np.concatenate([[v.rb.mass] * 3, np.diag(v.rb.inertia)])) + v.coeffs.M_A
          for v in hulls]
    M = torch.tensor(np.array([Ms[i % 5] for i in range(n)]), device="cuda")
    ke = 0.5 * torch.einsum("ni,nij,nj->n", st.nu, M, st.nu)
    zero = torch.zeros((n, 6), dtype=torch.float64, device="cuda")
    for _ in range(2000):
        E.step_batch(st, zero)
        ke2 = 0.5 * torch.einsum("ni,nij,nj->n", st.nu, M, st.nu)
        assert bool((ke2 <= ke + 1e-9).all())
        ke = ke2
    assert not st.diverged.any()


def test_drift_converges_to_the_current():
    veh = load_vehicle("bluerov")
    st = E.make_batch(veh, E.SimConfig(batch_size=1), master_seed=3, dtype=torch.float64)

    def in_current(i, ep, rng):
        return E.EnvInit(pose=E.Pose(), current_ned=np.array([0.3, 0.0, 0.0]))

    E.reset_envs(st, np.ones(1, bool), in_current)
    z = torch.zeros((1, 6), dtype=torch.float64, device="cuda")
    for _ in range(3000):
        E.step_batch(st, z)
    nu_c = E.current_in_body(st.q[0].cpu(), st.current_ned[0].cpu())
    assert float((st.nu[0].cpu() - nu_c).norm()) < 0.01 * 0.3


# ---------------------------------------------------------------- tasks (test_tasks.py)

EXTRA_DIMS = {"station_keeping": 0, "tracking": 3, "docking": 1}
CONTRACT_VEHICLE = {"station_keeping": "bluerov", "tracking": "lauv", "docking": "bluerov_heavy"}


@pytest.mark.parametrize("kind", TASK_KINDS)
@pytest.mark.parametrize("level", LEVELS)
def test_env_contract(kind, level):
    task = TaskConfig(task=kind, vehicle=CONTRACT_VEHICLE[kind], level=level, episode_length=50)
    env = make_env(task, E.SimConfig(batch_size=8), seed=3)
    obs = env.reset()
    a = env.action_dim
    assert tuple(obs.shape) == (8, 12 + a + EXTRA_DIMS[kind]) and env.obs_dim == obs.shape[1]
    rng = np.random.default_rng(0)
    n_finished = 0
    bound = env.reward_bound()
    for _ in range(120):
        o, r, term, trunc, info = env.step(rng.uniform(-1, 1, (8, a)))
        assert tuple(o.shape) == (8, env.obs_dim) and bool(torch.isfinite(o).all())
        assert bool(torch.isfinite(r).all()) and not bool((term & trunc).any())
        assert float(r.abs().max()) <= bound + 1e-6
        for key in ("position_error", "attitude_error", "metric", "finished", "failure",
                    "diverged", "success", "time", "terminal_observation"):
            assert key in info, key
        n_finished += int((term | trunc).sum())
    assert n_finished >= 8
    ovs = env.state.overlays
    if level == "standard":
        assert env.state._cur is None or bool((env.state.current_ned == 0).all())
        assert all(not o for o in ovs)
    elif level == "disturbed":
        speed = env.state.current_ned.double().norm(dim=1)
        assert torch.allclose(speed, torch.full_like(speed, 0.25), atol=1e-6)
        assert all(abs(o["payload_mass*"] - 0.1) < 1e-12 for o in ovs)
    else:
        assert all("mass*" in o for o in ovs)


def test_same_seed_same_trajectories():
    task = TaskConfig(task="tracking", vehicle="bluerov", level="disturbed_dr", episode_length=40)
    outs = []
    for _ in range(2):
        env = make_env(task, E.SimConfig(batch_size=4), seed=11)
        env.reset()
        rng = np.random.default_rng(5)
        run = []
        for _ in range(90):
            o, r, *_ = env.step(rng.uniform(-1, 1, (4, env.action_dim)))
            run.append((o.clone(), r.clone()))
        outs.append(run)
    for (o1, r1), (o2, r2) in zip(*outs):
        assert torch.equal(o1, o2) and torch.equal(r1, r2)


def test_auto_reset_returns_next_episode_obs():
    task = TaskConfig(task="station_keeping", vehicle="bluerov", episode_length=5)
    env = make_env(task, E.SimConfig(batch_size=3), seed=2)
    env.reset()
    a = env.action_dim
    cmd = np.full((3, a), 0.3)
    for _ in range(5):
        obs, r, term, trunc, info = env.step(cmd)
    assert bool(trunc.all()) and bool(info["finished"].all())
    assert np.allclose(h(info["terminal_observation"])[:, 12:12 + a], 0.3)
    assert np.all(h(obs)[:, 12:12 + a] == 0.0)
    assert int(env.state.steps.max()) == 0 and bool((env.state.episodes == 1).all())


def test_leaving_the_workspace_fails_the_episode():
    task = TaskConfig(task="station_keeping", vehicle="bluerov", bounds=10.0)
    env = make_env(task, E.SimConfig(batch_size=2), seed=6)
    env.reset()
    env.state.p[0] = torch.tensor([50.0, 0.0, 0.0], device="cuda")
    obs, r, term, trunc, info = env.step(np.zeros((2, env.action_dim)))
    assert bool(term[0]) and not bool(term[1])
    assert bool(info["failure"][0]) and not bool(info["failure"][1])
    assert float(r[0]) == -task.fail_penalty and not bool(info["success"][0])
    assert int(env.state.steps[0]) == 0


def test_speed_limit_fails_the_episode():
    task = TaskConfig(task="station_keeping", vehicle="bluerov", nu_max=0.3, episode_length=400)
    env = make_env(task, E.SimConfig(batch_size=1), seed=6)
    env.reset()
    cmd = np.ones((1, env.action_dim))
    for _ in range(400):
        obs, r, term, trunc, info = env.step(cmd)
        if bool(term[0]):
            break
    assert bool(term[0]) and bool(info["failure"][0]) and float(r[0]) == -task.fail_penalty


def test_docking_contact_terminates():
    task = TaskConfig(task="docking", vehicle="bluerov_heavy", episode_length=2000,
                      dock=DockSpec(centre=(0.0, 0.0, 3.0), radius=5.0))
    env = make_env(task, E.SimConfig(batch_size=2), seed=4)
    env.reset()
    cmd = np.zeros((2, 8))
    cmd[:, 4:] = 1.0
    hit = False
    for t in range(1500):
        o, r, term, trunc, info = env.step(cmd)
        if bool(info["contact"].any()):
            hit = True
            touched = info["contact"]
            assert bool(term[touched].all())
            assert bool(torch.isfinite(info["contact_distance"][touched]).all())
            assert bool(torch.isnan(info["contact_distance"][~touched]).all())
            assert bool(info["success"][touched].all())
            break
        if t == 200 and float(env.state.p[0, 2]) < 0.2:
            cmd[:, 4:] = -1.0
    assert hit


def test_obs_layout_segments():
    env = make_env(TaskConfig(task="tracking", vehicle="lauv"), E.SimConfig(batch_size=2), seed=0)
    layout = env.obs_layout()
    assert [s[0] for s in layout] == ["position_error_body", "attitude_error", "velocity",
                                      "prev_command", "reference_velocity_body"]
    assert layout[-1][2] == env.obs_dim
    sp = env.spaces()
    assert sp["obs_layout"] == [list(s) for s in layout]
    assert sp["task"] == "tracking" and sp["vehicle"] == "lauv"
    assert sp["metric"] == "mean_deviation_m" and sp["n_envs"] == 2 and sp["dt"] == 0.02


def test_docking_height_extra_tracks_geometry():
    task = TaskConfig(task="docking", vehicle="bluerov_heavy")
    env = make_env(task, E.SimConfig(batch_size=4), seed=1, dtype=torch.float64)
    obs = env.reset()
    want = task.dock.centre[2] - h(env.state.p)[:, 2]
    assert np.allclose(h(obs)[:, -1], want, atol=0)


def test_station_keeping_metric_is_distance():
    task = TaskConfig(task="station_keeping", vehicle="bluerov")
    env = make_env(task, E.SimConfig(batch_size=3), seed=8, dtype=torch.float64)
    env.reset()
    _, _, _, _, info = env.step(np.zeros((3, env.action_dim)))
    dist = np.sqrt(((np.asarray(task.target_position) - h(env.state.p)) ** 2).sum(-1))
    assert np.allclose(h(info["metric"]), dist, rtol=1e-14)
    assert np.array_equal(h(info["metric"]), h(info["position_error"]))


def test_tracking_metric_is_mean_deviation():
    from paper_2503_09203_b200.trajectories import reference_point

    task = TaskConfig(task="tracking", vehicle="bluerov", episode_length=100)
    env = make_env(task, E.SimConfig(batch_size=2), seed=9, dtype=torch.float64)
    env.reset()
    devs = []
    for _ in range(3):
        _, _, _, _, info = env.step(np.zeros((2, env.action_dim)))
        p_ref, _ = reference_point(task.trajectory, h(env.state.steps) * 0.02)
        devs.append(np.sqrt(((h(env.state.p) - p_ref) ** 2).sum(-1)))
    assert np.allclose(h(info["metric"]), np.mean(devs, axis=0), rtol=1e-12)


def test_metric_definitions_cover_all_tasks():
    names = set()
    for kind in TASK_KINDS:
        env = make_env(TaskConfig(task=kind), E.SimConfig(batch_size=1), seed=0)
        names.add(env.metric_name)
        assert env.spaces()["metric"] in METRIC_DEFINITIONS
    assert names == set(METRIC_DEFINITIONS)


def test_tracking_duration_must_cover_horizon():
    task = TaskConfig(task="tracking", episode_length=500, trajectory=TrajectorySpec(duration=5.0))
    with pytest.raises(TaskError, match="horizon"):
        make_env(task, E.SimConfig(batch_size=1), seed=0)


def test_step_shape_error():
    env = make_env(TaskConfig(task="station_keeping"), E.SimConfig(batch_size=2), seed=0)
    env.reset()
    with pytest.raises(TaskError, match="commands"):
        env.step(np.zeros((2, env.action_dim + 2)))


def test_reward_bound_formula():
    task = TaskConfig(task="station_keeping", vehicle="bluerov")
    env = make_env(task, E.SimConfig(batch_size=1), seed=0)
    assert env.reward_bound() == task.fail_penalty


def test_rollout_stats_match_host_sums():
    task = TaskConfig(task="station_keeping", vehicle="bluerov", episode_length=7)
    env = make_env(task, E.SimConfig(batch_size=300), seed=1, dtype=torch.float64)
    env.reset()
    env.rollout_stats(reset=True)
    rng = np.random.default_rng(0)
    tot_r, tot_f, tot_s = 0.0, 0, 0
    for _ in range(20):
        _, r, te, tr, info = env.step(rng.uniform(-1, 1, (300, 6)))
        tot_r += float(r.sum())
        tot_f += int(info["finished"].sum())
        tot_s += int(info["success"].sum())
    st = env.rollout_stats()
    assert st["frames"] == 300 * 20 and st["finished"] == tot_f and st["success"] == tot_s
    assert st["reward_sum"] == pytest.approx(tot_r, rel=1e-12)
    assert env.rollout_stats()["frames"] == 0


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("n", [1000, 4096])
def test_host_buffer_step_equals_device_step(dtype, n):
    """step_batch with pinned host commands + pose_out (uuv_step_host: the kernel reads and
    writes the mapped host buffers) == the device-command step, bit for bit."""
    from paper_2503_09203_b200.randomization import DRParameter, Uniform

    veh = load_vehicle("bluerov")
    spec = {k: DRParameter(k, Uniform(0.8, 1.2)) for k in ("mass*", "damping*")}
    a = E.make_batch(veh, E.SimConfig(batch_size=n), master_seed=3, dtype=dtype)
    b = E.make_batch(veh, E.SimConfig(batch_size=n), master_seed=3, dtype=dtype)
    for st in (a, b):
        E.reset_envs(st, np.ones(n, bool), E.spec_sampler(spec))
    g = torch.Generator().manual_seed(0)
    out = torch.empty((13, n), dtype=dtype).pin_memory()
    for t in range(5):
        hc = (torch.rand((n, 6), generator=g, dtype=torch.float64) * 2.4 - 1.2).to(dtype)
        hc = hc.pin_memory()
        if t == 3:
            hc[7, 2] = float("nan")  # diverges env 7: frozen rows still report their pose
        E.step_batch(a, hc.cuda())
        E.step_batch(b, hc, pose_out=out)
        for k in ("p", "q", "nu", "act", "steps", "diverged"):
            assert torch.equal(getattr(a, k), getattr(b, k)), (t, k)
        want = torch.cat([a.p, a.q, a.nu], dim=1).T.cpu()
        assert torch.equal(out, want), t
    assert bool(a.diverged[7])
    # pageable host commands take the staged-copy path
    E.step_batch(b, np.asarray(hc), pose_out=out)
    E.step_batch(a, hc.cuda())
    assert torch.equal(a.p, b.p)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("vehicles", [("bluerov",), ("bluerov", "lauv", "hauv")])
def test_step_server_equals_launched_steps(dtype, vehicles):
    """serve(): the resident step kernel == step_batch launches, bit for bit, incl. pose rows."""
    from paper_2503_09203_b200.randomization import DRParameter, Uniform

    n = 3000
    vehs = [load_vehicle(v) for v in vehicles]
    spec = {k: DRParameter(k, Uniform(0.8, 1.2)) for k in ("mass*", "volume*")}

    def make():
        if len(vehs) == 1:
            st = E.make_batch(vehs[0], E.SimConfig(batch_size=n, substeps=2), master_seed=4,
                              dtype=dtype)
        else:
            counts = [n // 3, n // 3, n - 2 * (n // 3)]
            st = E.make_fleet_batch(vehs, counts, E.SimConfig(batch_size=n, substeps=2),
                                    master_seed=4, dtype=dtype)
        E.reset_envs(st, np.ones(n, bool), E.spec_sampler(spec))
        return st

    a, b = make(), make()
    w = E._cmd_width(a)
    g = torch.Generator().manual_seed(1)
    cmds = [(torch.rand((n, w), generator=g, dtype=torch.float64) * 2 - 1).to(dtype).pin_memory()
            for _ in range(6)]
    cmds[4][5, 0] = float("nan")  # env 5 diverges and freezes
    out = torch.empty((13, n), dtype=dtype).pin_memory()
    # torch kernels used inside the block are loaded first (a first launch under CUDA
    # lazy loading waits for the device, i.e. for the resident server)
    assert torch.equal(out, torch.cat([a.p, a.q, a.nu], dim=1).T.cpu()) in (True, False)
    with E.serve(b):
        with pytest.raises(E.EngineError):
            E.reset_envs(b, np.ones(n, bool))
        with pytest.raises(E.EngineError):
            E.step_batch(b, cmds[0].cuda())
        for t in range(6):
            E.step_batch(a, cmds[t].cuda())
            E.step_batch(b, cmds[t], pose_out=out if t % 2 == 0 else None)
            if t % 2 == 0:
                want = torch.cat([a.p, a.q, a.nu], dim=1).T.cpu()
                assert torch.equal(out, want), t
        E.step_batch(b, np.asarray(cmds[0]))  # pageable host commands, staged
        E.step_batch(a, cmds[0].cuda())
        reuse = torch.empty_like(cmds[0]).pin_memory()  # one buffer, new contents each step
        for t in range(30):
            reuse.copy_(cmds[t % 6] * (1.0 - 0.01 * t))
            E.step_batch(a, reuse.cuda())
            E.step_batch(b, reuse, pose_out=out)
            assert torch.equal(out, torch.cat([a.p, a.q, a.nu], dim=1).T.cpu()), t
    E.step_batch(a, cmds[0].cuda())
    E.step_batch(b, cmds[0].cuda())
    for k in ("p", "q", "nu", "act", "steps", "diverged"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k
    assert bool(b.diverged[5])
    E.step_batch(b, cmds[1].cuda())  # launches work again after the block


def test_step_server_idle_timeout_and_errors():
    st = E.make_batch(load_vehicle("bluerov"), E.SimConfig(batch_size=256))
    E.reset_envs(st, np.ones(256, bool))
    cmd = torch.zeros((256, 6)).pin_memory()
    srv = E.serve(st, idle_timeout_ms=200)
    srv.__enter__()
    E.step_batch(st, cmd)
    import time

    time.sleep(0.6)  # the kernel ends by itself
    with pytest.raises(E.EngineError, match="not running"):
        E.step_batch(st, cmd)
    srv.__exit__(None, None, None)
    E.step_batch(st, cmd.cuda())
    with E.serve(st):
        with pytest.raises(E.EngineError):
            with E.serve(st):
                pass
    # a grid that cannot be resident in one wave is refused, not deadlocked
    big = E.make_batch(load_vehicle("bluerov"), E.SimConfig(batch_size=2_000_000))
    with pytest.raises(E.EngineError, match="one wave"):
        with E.serve(big):
            pass
    E.step_batch(big, torch.zeros((2_000_000, 6), device="cuda"))  # still usable


def test_pdl_modes_bitwise():
    """The dependent-launch trigger mode only changes scheduling: a graph-replayed DR
    rollout (commands from a ring) ends in the same state bit for bit under every mode."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    out = {}
    for n in (4096, 40000):
        for mode in ("0", "2", "3", "4"):
            env = dict(os.environ, UUV_PDL=mode)
            r = subprocess.run([sys.executable, os.path.join(here, "pdl_rollout.py"), str(n)],
                               env=env, capture_output=True, text=True, timeout=240)
            assert r.returncode == 0, r.stderr[-2000:]
            out[(n, mode)] = r.stdout.strip().splitlines()[-1]
        assert len({out[(n, m)] for m in ("0", "2", "3", "4")}) == 1, out


def test_batch_released_during_a_graph_capture():
    """A fleet batch whose per-run dispatch created fork streams is garbage-collected
    while another stream is being captured: its context must not invalidate the capture."""
    import gc

    names = ("bluerov", "lauv", "hauv")
    n = 131_073
    counts = [n // 3, n // 3, n - 2 * (n // 3)]
    st = E.make_fleet_batch([load_vehicle(v) for v in names], counts,
                            E.SimConfig(batch_size=n))
    E.reset_envs(st, np.ones(n, bool))
    E.step_batch(st, torch.zeros((n, st.a_max), device="cuda"))  # forks the run streams
    torch.cuda.synchronize()
    x = torch.zeros(8, device="cuda")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        x.add_(1.0)
        del st
        gc.collect()
        x.add_(1.0)
    g.replay()
    torch.cuda.synchronize()
    assert float(x[0]) == 2.0
