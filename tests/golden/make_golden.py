"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the unmodified ``uuvsim`` package and installs exactly one hook:
``BatchState.env_rng`` (engine.py:291-295) is replaced by the Philox4x64-10
mapping ``Philox(key=[seed, env], counter=[0, episode, 0, 0])`` that the
GPU reset kernel implements (SURVEY.md §8(c) "RNG parity hook").  Every
other line of the reference runs as shipped.  Outputs are compressed ``.npz``
files next to this script; the tests load them on CPU (oracle pin) and on
the GPU box (kernel parity) without needing the reference.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import samplers  # noqa: E402
import variants  # noqa: E402
from uuvsim import actuation as R_act  # noqa: E402
from uuvsim import engine as R_eng  # noqa: E402
from uuvsim import hydrodynamics as R_hyd  # noqa: E402
from uuvsim import vehicles as R_veh  # noqa: E402
from uuvsim.kinematics import BodyVelocity, Pose, integrate_pose, matvec  # noqa: E402
from uuvsim.tasks import DockSpec, TaskConfig, make_env  # noqa: E402

M64 = (1 << 64) - 1


def _philox_env_rng(self, i):
    return np.random.Generator(np.random.Philox(
        key=np.array([int(self.master_seed) & M64, int(i) & M64], dtype=np.uint64),
        counter=np.array([0, int(self.episodes[i]) & M64, 0, 0], dtype=np.uint64)))


_REFERENCE_ENV_RNG = R_eng.BatchState.env_rng
R_eng.BatchState.env_rng = _philox_env_rng  # the single hook


class unhooked:
    """Run the reference exactly as shipped (PCG64/SeedSequence streams)."""

    def __enter__(self):
        R_eng.BatchState.env_rng = _REFERENCE_ENV_RNG

    def __exit__(self, *exc):
        R_eng.BatchState.env_rng = _philox_env_rng


def vehicle(name):
    if name in variants.VARIANTS:
        return variants.build(name, R_veh, R_act, R_hyd, R_veh.load_vehicle("bluerov"))
    return R_veh.load_vehicle(name)


def wrap(fn):
    def sampler(i, ep, rng):
        d = fn(i, ep, rng)
        return R_eng.EnvInit(pose=Pose(p=d["p"], q=d["q"]), nu=d["nu"], overlay=d["overlay"],
                             current_ned=d["current_ned"])
    return sampler


def snapshot_params(st):
    P = st.params
    return {f"param_{k}": np.array(getattr(P, k)) for k in
            ("mass", "volume", "r_g", "r_b", "M_RB", "M_A", "M_inv", "D_lin", "D_quad",
             "thrust_coeff", "time_constant", "mounts")}


def substep_terms(st, u, dt):
    """Intermediates of the first substep, from the reference's own functions
    in _substeps order (engine.py:425-433)."""
    sl = slice(0, st.sim.batch_size)
    view = R_eng._ParamsView(st.params, st.layout, sl)
    pose = Pose(p=st.p.copy(), q=st.q.copy())
    act_new = R_eng._advance_rotors(st, sl, u, dt)
    nu_c = R_eng.current_in_body(pose, st.current_ned)
    nu_r = st.nu - nu_c
    tau = R_eng._actuator_wrench_batch(st, sl, act_new, nu_r)
    w_h = R_hyd.hydro_wrench(pose, st.nu, nu_c, view, view)
    c_rb = R_hyd.coriolis_force(st.params.M_RB, st.nu)
    acc = matvec(st.params.M_inv, tau + w_h - c_rb)
    nu_new = st.nu + dt * acc
    pn = integrate_pose(pose, BodyVelocity.from_vector(nu_new), dt)
    return dict(t_act_new=act_new, t_tau=tau, t_hydro=w_h, t_c_rb=c_rb, t_acc=acc,
                t_nu_new=nu_new, t_p_new=pn.p, t_q_new=pn.q)


def engine_fixture(name, n=8, steps=30, substeps=2, seed=42, sampler=samplers.rich):
    veh = vehicle(name)
    A = veh.action_dim
    st = R_eng.make_batch(veh, R_eng.SimConfig(batch_size=n, substeps=substeps), master_seed=seed)
    R_eng.reset_envs(st, np.ones(n, bool), wrap(sampler))
    out = dict(p0=st.p.copy(), q0=st.q.copy(), nu0=st.nu.copy(), act0=st.act.copy(),
               current0=st.current_ned.copy(), episodes0=st.episodes.copy())
    out.update(snapshot_params(st))
    out["overlays"] = np.array(json.dumps([samplers.overlay_to_json(o) for o in st.overlays]))
    cmds = np.random.default_rng(7).uniform(-1.2, 1.2, size=(steps, n, A))
    u0 = np.clip(cmds[0], -1.0, 1.0)
    out.update(substep_terms(st, u0, st.sim.dt / substeps))
    traj = {k: [] for k in ("p", "q", "nu", "act")}
    for t in range(steps):
        R_eng.step_batch(st, cmds[t])
        for k in traj:
            traj[k].append(getattr(st, k).copy())
    out.update({f"traj_{k}": np.array(v) for k, v in traj.items()})
    out.update(cmds=cmds, steps=st.steps.copy(), diverged=st.diverged.copy(),
               meta=np.array(json.dumps(dict(vehicle=name, n=n, substeps=substeps, seed=seed,
                                             dt=st.sim.dt))))
    return out


def divergence_fixture():
    veh = vehicle("bluerov")
    st = R_eng.make_batch(veh, R_eng.SimConfig(batch_size=3), master_seed=5)
    R_eng.reset_envs(st, np.ones(3, bool))
    st.nu[1] = 1e200
    nu_in = st.nu.copy()
    cmds = np.random.default_rng(2).uniform(-1, 1, (3, veh.action_dim))
    for _ in range(10):
        R_eng.step_batch(st, cmds)
    return dict(nu_in=nu_in, cmds=cmds, p=st.p, q=st.q, nu=st.nu, act=st.act,
                diverged=st.diverged, steps=st.steps)


def config1_fixture():
    """BASELINE config 1: bluerov, 64 envs, fixed U(-1,1) commands, 1000 steps."""
    veh = vehicle("bluerov")
    st = R_eng.make_batch(veh, R_eng.SimConfig(batch_size=64), master_seed=0)
    R_eng.reset_envs(st, np.ones(64, bool))
    cmds = np.random.default_rng(0).uniform(-1.0, 1.0, size=(64, veh.action_dim))
    keep = {1, 10, 100, 1000}
    out = dict(cmds=cmds)
    for t in range(1, 1001):
        R_eng.step_batch(st, cmds)
        if t in keep:
            for k in ("p", "q", "nu", "act"):
                out[f"{k}_{t}"] = getattr(st, k).copy()
    return out


INFO_KEYS = ("position_error", "attitude_error", "metric", "finished", "failure", "diverged",
             "success", "time", "terminal_observation", "contact", "contact_distance",
             "contact_speed", "contact_attitude")


def task_fixture(kind, vehicle_name, level, n=6, steps=40, episode_length=15, substeps=1,
                 seed=5, cmd_fn=None, **task_kw):
    task = TaskConfig(task=kind, vehicle=vehicle_name, level=level,
                      episode_length=episode_length, **task_kw)
    env = make_env(task, R_eng.SimConfig(batch_size=n, substeps=substeps), seed=seed)
    obs0 = env.reset()
    st = env.state
    out = dict(obs0=obs0, p0=st.p.copy(), q0=st.q.copy(), nu0=st.nu.copy(),
               current0=st.current_ned.copy())
    out["overlays0"] = np.array(json.dumps([samplers.overlay_to_json(o) for o in st.overlays]))
    rng = np.random.default_rng(11)
    rec = {k: [] for k in ("cmds", "obs", "reward", "terminated", "truncated", "p", "q", "nu",
                           "episodes", "steps") + INFO_KEYS}
    for t in range(steps):
        u = cmd_fn(t, rng, env) if cmd_fn else rng.uniform(-1.1, 1.1, (n, env.action_dim))
        o, r, te, tr, info = env.step(u)
        rec["cmds"].append(u)
        rec["obs"].append(o)
        rec["reward"].append(r)
        rec["terminated"].append(te)
        rec["truncated"].append(tr)
        for k in ("p", "q", "nu", "episodes", "steps"):
            rec[k].append(getattr(env.state, k).copy())
        for k in INFO_KEYS:
            if k in info:
                rec[k].append(np.asarray(info[k]))
    for k, v in rec.items():
        if v:
            out[k] = np.array(v)
    out["meta"] = np.array(json.dumps(dict(kind=kind, vehicle=vehicle_name, level=level, n=n,
                                           steps=steps, episode_length=episode_length,
                                           substeps=substeps, seed=seed, task_kw={
                                               k: (list(v.centre) + [v.radius]
                                                   if isinstance(v, DockSpec) else v)
                                               for k, v in task_kw.items()})))
    return out


def save(name, data):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **data)
    print(f"wrote {path} ({os.path.getsize(path) // 1024} KiB)")


def main():
    for name in R_veh.BUILTIN_VEHICLES + variants.VARIANTS:
        save(f"engine_{name}", engine_fixture(name))
    veh_h = vehicle("hauv")
    save("engine_jitter_hauv", engine_fixture("hauv", n=4, steps=10, substeps=1, seed=3,
                                              sampler=samplers.jitter_matrix(veh_h.action_dim)))
    save("divergence", divergence_fixture())
    save("config1_bluerov64", config1_fixture())
    contract = {"station_keeping": "bluerov", "tracking": "lauv", "docking": "bluerov_heavy"}
    for kind, veh in contract.items():
        for level in ("standard", "disturbed", "disturbed_dr"):
            save(f"task_{kind}_{level}", task_fixture(kind, veh, level))
    save("task_tracking_k8_hauv", task_fixture("tracking", "hauv", "disturbed", substeps=8,
                                               episode_length=25))
    save("task_station_iauv_dr", task_fixture("station_keeping", "iauv", "disturbed_dr"))

    def descend(t, rng, env):
        u = rng.uniform(-0.2, 0.2, (env.n_envs, env.action_dim))
        u[:, 4:] = -1.0
        return u

    def full_thrust(t, rng, env):
        return np.clip(1.0 + rng.uniform(-0.3, 0.3, (env.n_envs, env.action_dim)), -1.0, 1.0)

    save("task_station_fail", task_fixture(
        "station_keeping", "bluerov", "disturbed", n=6, steps=80, episode_length=60,
        cmd_fn=full_thrust, nu_max=0.4, bounds=3.0))
    # the unmodified reference (no hook): PCG64(SeedSequence(seed, spawn_key=(i, ep)))
    with unhooked():
        save("engine_bluerov_pcg64", engine_fixture("bluerov"))
        save("task_station_keeping_standard_pcg64",
             task_fixture("station_keeping", "bluerov", "standard"))
        save("task_tracking_disturbed_pcg64", task_fixture("tracking", "lauv", "disturbed"))
        save("task_docking_disturbed_dr_pcg64",
             task_fixture("docking", "bluerov_heavy", "disturbed_dr"))
    save("task_docking_contact", task_fixture(
        "docking", "bluerov_heavy", "standard", n=4, steps=160, episode_length=400,
        cmd_fn=descend, dock=DockSpec(centre=(0.0, 0.0, 3.0), radius=5.0)))


if __name__ == "__main__":
    main()
