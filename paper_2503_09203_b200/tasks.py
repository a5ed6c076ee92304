"""Vectorised station-keeping / tracking / docking tasks on the GPU step.

Same contract as ``uuvsim/tasks/core.py`` (``VecTaskEnv`` 217-383,
``make_env`` 533-538):

    reset(mask) -> obs
    step(commands) -> (obs, reward, terminated, truncated, info)

with auto-reset of finished rows inside ``step`` and the final observation
of the ended episode in ``info["terminal_observation"]``.

Everything per step — physics (K substeps), observation, reward,
fail/terminated/truncated, info metrics, the auto-reset draw (Philox DR
overlay, current, start pose) and the next-episode observation — runs in a
single fused kernel launch (``uuv_task_step_dl``: commands and observations
cross the C ABI as DLPack tensors); the host only enqueues it.
Arrays are torch CUDA tensors in the batch dtype (float32 by default).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .randomization import CURRENT_KEYS, DRParameter, Uniform, make_spec, preset
from .trajectories import TrajectorySpec, reference_point

STATION_KEEPING = "station_keeping"
TRACKING = "tracking"
DOCKING = "docking"
TASK_KINDS = (STATION_KEEPING, TRACKING, DOCKING)
LEVEL_STANDARD = "standard"
LEVEL_DISTURBED = "disturbed"
LEVEL_DISTURBED_DR = "disturbed_dr"
LEVELS = (LEVEL_STANDARD, LEVEL_DISTURBED, LEVEL_DISTURBED_DR)
DISTURBED_CURRENT_SPEED = 0.25
DISTURBED_PAYLOAD_RATIO = 0.1

METRIC_DEFINITIONS = {
    "distance_to_target_m": "Euclidean distance from the vehicle position to the target "
                            "position at the current step.",
    "mean_deviation_m": "Mean Euclidean deviation from the reference trajectory over the "
                        "steps elapsed this episode.",
    "contact_distance_m": "Planar (horizontal) Euclidean distance from the dock centre at "
                          "the contact step; undefined before contact.",
}


class TaskError(ValueError):
    pass


@dataclass
class RewardWeights:
    """Reward shaping constants (tasks/core.py:98-120)."""

    w_p: float = 1.0
    w_a: float = 0.2
    w_v: float = 0.02
    w_u: float = 0.02
    w_b: float = 10.0
    r_tol: float = 0.15
    speed_cap: float = 10.0
    dock_bonus: float = 100.0
    w_dock_dist: float = 100.0
    w_impact: float = 20.0
    w_level: float = 20.0


@dataclass
class DockSpec:
    centre: tuple = (0.0, 0.0, 3.0)
    radius: float = 0.5

    def __post_init__(self):
        if len(self.centre) != 3:
            raise TaskError("dock centre must have 3 entries")
        if not self.radius > 0:
            raise TaskError(f"dock radius must be > 0, got {self.radius}")


@dataclass
class TaskConfig:
    task: str = STATION_KEEPING
    vehicle: str = "bluerov"
    level: str = LEVEL_STANDARD
    episode_length: int = 500
    bounds: float = 10.0
    nu_max: float = 5.0
    fail_penalty: float = 2000.0
    weights: RewardWeights = field(default_factory=RewardWeights)
    target_position: tuple = (0.0, 0.0, 1.0)
    target_yaw: float = 0.0
    start_radius: float = 2.5
    trajectory: TrajectorySpec = field(default_factory=TrajectorySpec)
    success_tol: float = 0.3
    dock: DockSpec = field(default_factory=DockSpec)

    def __post_init__(self):
        if self.task not in TASK_KINDS:
            raise TaskError(f"unknown task '{self.task}', expected one of {TASK_KINDS}")
        if self.level not in LEVELS:
            raise TaskError(f"unknown level '{self.level}', expected one of {LEVELS}")
        if self.episode_length < 1:
            raise TaskError(f"episode_length must be >= 1, got {self.episode_length}")
        if not self.bounds > 0:
            raise TaskError(f"bounds must be > 0, got {self.bounds}")
        if not (self.nu_max > 0 and self.start_radius > 0):
            raise TaskError("nu_max and start_radius must be > 0")


def disturbed_spec() -> dict:
    """The fixed-point disturbance set of level 'disturbed' (tasks/core.py:232-241)."""
    return make_spec([
        DRParameter("payload_mass*", Uniform(DISTURBED_PAYLOAD_RATIO, DISTURBED_PAYLOAD_RATIO)),
        DRParameter("payload_position", Uniform(0.0, 0.0)),
        DRParameter("current_velocity", Uniform(DISTURBED_CURRENT_SPEED,
                                                DISTURBED_CURRENT_SPEED)),
    ])


def level_spec(level: str, dr=None):
    """DR spec implied by a disturbance level (tasks/core.py:228-246)."""
    if level == LEVEL_STANDARD:
        if dr is not None:
            raise TaskError("a DR spec requires level 'disturbed_dr'")
        return None
    if level == LEVEL_DISTURBED:
        if dr is not None:
            raise TaskError("a DR spec requires level 'disturbed_dr'")
        return disturbed_spec()
    return dict(dr) if dr is not None else preset("train")


def start_box(task: TaskConfig):
    """Per-task start distribution as (p_base, p_lo, p_hi, eul_lo, eul_hi, nu_lo, nu_hi).

    Each task's ``_sample_start`` (tasks/core.py:402-407, 454-460, 503-507) is
    ``p = base + U(lo, hi)``, ``euler = U(lo, hi)``, ``nu = U(lo, hi)`` in that
    draw order, so one descriptor drives the device sampler for all three.
    """
    if task.task == STATION_KEEPING:
        r = task.start_radius
        return (np.asarray(task.target_position, float), [-r] * 3, [r] * 3,
                [-0.15, -0.15, -np.pi], [0.15, 0.15, np.pi], [-0.1] * 6, [0.1] * 6)
    if task.task == TRACKING:
        p0, v0 = reference_point(task.trajectory, 0.0)
        yaw0 = float(np.arctan2(v0[1], v0[0]))
        return (p0, [-0.5] * 3, [0.5] * 3, [-0.1, -0.1, yaw0 - 0.3], [0.1, 0.1, yaw0 + 0.3],
                [-0.05] * 6, [0.05] * 6)
    c = np.asarray(task.dock.centre, float)
    return (c, [-1.5, -1.5, -2.5], [1.5, 1.5, -1.5], [-0.1, -0.1, -np.pi], [0.1, 0.1, np.pi],
            [-0.05] * 6, [0.05] * 6)


def target_yaw_quat(yaw: float) -> np.ndarray:
    """euler_to_quat(0, 0, yaw), normalised (kinematics.py:110-127)."""
    cy, sy = np.cos(yaw / 2), np.sin(yaw / 2)
    q = np.array([cy, 0.0, 0.0, sy])
    return q / np.sqrt((q * q).sum())


# ================================================================ environments

import ctypes as _C  # noqa: E402

import torch  # noqa: E402

from . import _native as _N  # noqa: E402
from .engine import (  # noqa: E402
    BatchState, EngineError, SimConfig, make_batch, spec_sampler,
)
from .vehicles import load_vehicle  # noqa: E402

_KIND_CODE = {STATION_KEEPING: _N.TASK_STATION, TRACKING: _N.TASK_TRACKING,
              DOCKING: _N.TASK_DOCKING}
_EXTRA = {STATION_KEEPING: 0, TRACKING: 3, DOCKING: 1}
_METRIC = {STATION_KEEPING: "distance_to_target_m", TRACKING: "mean_deviation_m",
           DOCKING: "contact_distance_m"}


class _Info(dict):
    """info dict whose ``terminal_observation`` is materialised on first access.

    The fused kernel writes the final observation of an ended episode only for
    the rows that finished; every other row's final observation IS the returned
    observation, so the full array is ``where(finished, term_rows, obs)``.
    """

    def __init__(self, *a, obs=None, term=None, finished=None, **kw):
        super().__init__(*a, **kw)
        self._lazy = (obs, term, finished)

    def _materialise(self):
        if not dict.__contains__(self, "terminal_observation") and self._lazy[0] is not None:
            obs, term, fin = self._lazy
            super().__setitem__("terminal_observation", torch.where(fin[:, None], term, obs))

    def __getitem__(self, k):
        if k == "terminal_observation":
            self._materialise()
        return super().__getitem__(k)

    def __contains__(self, k):
        return k == "terminal_observation" or super().__contains__(k)

    def keys(self):
        self._materialise()
        return super().keys()

    def get(self, k, default=None):
        return self[k] if k in self else default

    def items(self):
        self._materialise()
        return super().items()


class VecTaskEnv:
    """Batched task environment over one engine batch (tasks/core.py:217-383)."""

    def __init__(self, task: TaskConfig, sim: SimConfig, dr=None, seed: int = 0, *,
                 device=None, dtype=torch.float32, env_offset: int = 0, rng: str = "philox"):
        self.task = task
        self.sim = sim
        self.vehicle = load_vehicle(task.vehicle)
        self.seed = int(seed)
        self._dr = level_spec(task.level, dr)
        if task.task == TRACKING:
            horizon = task.episode_length * sim.dt
            if task.trajectory.duration < horizon:
                raise TaskError(f"trajectory duration {task.trajectory.duration} s is shorter than "
                                f"the episode horizon {horizon} s")
        self.state: BatchState = make_batch(self.vehicle, sim, master_seed=self.seed,
                                            device=device, dtype=dtype, env_offset=env_offset,
                                            rng=rng)
        self.n_envs = sim.batch_size
        self.action_dim = self.vehicle.action_dim
        self.metric_name = _METRIC[task.task]
        self.extra_dim = _EXTRA[task.task]
        st = self.state
        self._sampler = spec_sampler(self._dr, start_box(task))
        self._sampler_c = self._sampler.pack()
        self._sampler_c.rng_mode = _N.RNG_MODES[rng]
        st._note_sampler(self._sampler)
        ld, dev = st._ld, st.device
        self._prev_u = torch.zeros((self.action_dim, ld), dtype=dtype, device=dev)
        self._dev_sum = torch.zeros(ld, dtype=dtype, device=dev) if task.task == TRACKING else None
        self._stats = torch.zeros((_N.load().uuv_stats_blocks(self.n_envs), len(_N.ST_NAMES)),
                                  dtype=torch.float64, device=dev)
        self._task_c = self._pack_task()
        self._recorder = None

    # -------------------------------------------------------------- layout
    @property
    def obs_dim(self) -> int:
        return 12 + self.action_dim + self.extra_dim

    def obs_layout(self) -> list:
        a = self.action_dim
        out = [("position_error_body", 0, 3), ("attitude_error", 3, 6), ("velocity", 6, 12),
               ("prev_command", 12, 12 + a)]
        if self.task.task == TRACKING:
            out.append(("reference_velocity_body", 12 + a, 15 + a))
        elif self.task.task == DOCKING:
            out.append(("height_above_dock", 12 + a, 13 + a))
        return out

    def spaces(self) -> dict:
        return {"task": self.task.task, "vehicle": self.vehicle.name, "level": self.task.level,
                "n_envs": self.n_envs, "obs_dim": self.obs_dim, "action_dim": self.action_dim,
                "dt": self.sim.dt, "episode_length": self.task.episode_length,
                "metric": self.metric_name, "obs_layout": [list(s) for s in self.obs_layout()]}

    def reward_bound(self) -> float:
        w = self.task.weights
        d = 2.0 * np.sqrt(3.0) * self.task.bounds
        shaped = (w.w_p * d + w.w_a * np.pi + w.w_v * w.speed_cap
                  + w.w_u * 2.0 * np.sqrt(self.action_dim) + w.w_b)
        terminal = abs(w.dock_bonus) + w.w_dock_dist * self.task.dock.radius \
            + w.w_impact * w.speed_cap + w.w_level * np.pi
        return max(shaped + terminal, self.task.fail_penalty)

    @property
    def prev_u(self):
        return self._prev_u[:, :self.n_envs].t()

    # -------------------------------------------------------------- packing
    def _pack_task(self) -> _N.Task:
        t, w = self.task, self.task.weights
        c = _N.Task()
        c.kind = _KIND_CODE[t.task]
        c.episode_length = t.episode_length
        c.obs_dim = self.obs_dim
        c.bounds, c.nu_max, c.fail_penalty = t.bounds, t.nu_max, t.fail_penalty
        for name in ("w_p", "w_a", "w_v", "w_u", "w_b", "r_tol", "speed_cap", "dock_bonus",
                     "w_dock_dist", "w_impact", "w_level"):
            setattr(c, name, getattr(w, name))
        if t.task == STATION_KEEPING:
            tq = target_yaw_quat(t.target_yaw)
            tp = np.asarray(t.target_position, float)
        else:
            tq = np.array([1.0, 0.0, 0.0, 0.0])
            tp = np.zeros(3)
        for k in range(3):
            c.target_p[k] = tp[k]
            c.dock_centre[k] = t.dock.centre[k]
        for k in range(4):
            c.target_q[k] = tq[k]
        c.success_tol = t.success_tol
        c.dock_radius = t.dock.radius
        t.trajectory.pack_into(c)
        return c

    def _io(self, obs, term=None, rout=None, fout=None, stats=True) -> _N.TaskIO:
        io = _N.TaskIO()
        io.prev_u = self._prev_u.data_ptr()
        io.dev_sum = self._dev_sum.data_ptr() if self._dev_sum is not None else None
        io.obs = obs.data_ptr() if obs is not None else None
        io.obs_ld = obs.stride(0) if obs is not None else 0
        io.term_obs = term.data_ptr() if term is not None else None
        io.real_out = rout.data_ptr() if rout is not None else None
        io.flag_out = fout.data_ptr() if fout is not None else None
        io.stats = self._stats.data_ptr() if stats else None
        if rout is not None and self._recorder is not None:
            io.trace, io.trace_ld = self._recorder._next_slot()
        return io

    def _new_obs(self):
        return torch.empty((self.n_envs, self.obs_dim), dtype=self.state.dtype,
                           device=self.state.device)

    # -------------------------------------------------------------- episode start
    def reset(self, mask=None):
        """Reset masked rows (default all) and return the observation of every row."""
        if self.state._server is not None:
            raise TaskError("the batch is being served (leave the serve() block first)")
        st = self.state
        if mask is None:
            m = None
        else:
            if torch.is_tensor(mask):
                m = mask.to(st.device, torch.bool)
            else:
                m = torch.from_numpy(np.asarray(mask, dtype=bool)).to(st.device)
            if tuple(m.shape) != (self.n_envs,):
                raise TaskError(f"mask: expected shape {(self.n_envs,)}, got {tuple(m.shape)}")
            m = m.to(torch.uint8).contiguous()
        obs = self._new_obs()
        lib = _N.load()
        _N.check(lib.uuv_task_reset(st._ctx, _C.byref(st._cstate()), _C.byref(self._task_c),
                                    _C.byref(self._sampler_c), self.seed & ((1 << 64) - 1),
                                    m.data_ptr() if m is not None else None, self.sim.dt,
                                    _C.byref(self._io(obs, stats=False)), st._stream()),
                 TaskError)
        return obs

    @property
    def dr(self):
        """The DR spec later resets draw from (None at level 'standard')."""
        return self._dr

    def set_dr(self, dr) -> None:
        """Swap the DR spec drawn by every later reset and auto-reset.

        For curriculum schedules (randomization.py:238-287): call
        ``env.set_dr(set_progress(schedule, t))`` between rollouts instead of
        rebuilding the env.  Later episodes are then exactly those of
        ``make_env(task, sim, dr=spec, seed=seed)`` (same streams, same
        episode counters).  Steps captured in a CUDA graph before the call keep
        the old spec: re-capture after it.
        """
        if self.task.level != LEVEL_DISTURBED_DR:
            raise TaskError("a DR spec requires level 'disturbed_dr'")
        mode = self._sampler_c.rng_mode
        self._dr = dict(dr)
        self._sampler = spec_sampler(self._dr, start_box(self.task))
        packed = self._sampler.pack()
        packed.rng_mode = mode
        self.state._note_sampler(self._sampler)
        self._sampler_c = packed

    def observe(self):
        st = self.state
        obs = self._new_obs()
        _N.check(_N.load().uuv_observe(st._ctx, _C.byref(st._cstate()), _C.byref(self._task_c),
                                       self.sim.dt, _C.byref(self._io(obs, stats=False)),
                                       st._stream()), TaskError)
        return obs

    # -------------------------------------------------------------- stepping
    def step(self, commands):
        """One fused launch: physics, reward/termination/info, auto-reset, next obs."""
        if self.state._server is not None:
            raise TaskError("the batch is being served (leave the serve() block first)")
        st = self.state
        n, a = self.n_envs, self.action_dim
        if torch.is_tensor(commands):
            u = commands
            if tuple(u.shape) != (n, a):
                raise TaskError(f"commands: expected shape {(n, a)}, got {tuple(u.shape)}")
            u = u.to(st.device, st.dtype)
        else:
            arr = np.asarray(commands, dtype=float)
            if arr.shape != (n, a):
                raise TaskError(f"commands: expected shape {(n, a)}, got {arr.shape}")
            u = torch.from_numpy(arr).to(st.device, st.dtype)
        if u.stride(1) != 1:
            u = u.contiguous()
        dev, dt = st.device, st.dtype
        obs = self._new_obs()
        term = self._new_obs()
        rout = torch.empty((len(_N.TR_NAMES), st._ld), dtype=dt, device=dev)
        fout = torch.empty((len(_N.TF_NAMES), st._ld), dtype=torch.uint8, device=dev)
        # commands in and the next observation out cross the ABI as DLPack tensors
        _N.check(_N.load().uuv_task_step_dl(
            st._ctx, _C.byref(st._cstate()), _C.byref(self._task_c), _C.byref(self._sampler_c),
            self.seed & ((1 << 64) - 1), _N.DLArg(u), self.sim.substeps, self.sim.dt,
            _C.byref(self._io(None, term, rout, fout)), _N.DLArg(obs), st._stream()),
            TaskError)
        R = {k: rout[i, :n] for i, k in enumerate(_N.TR_NAMES)}
        F = {k: fout[i, :n].view(torch.bool) for i, k in enumerate(_N.TF_NAMES)}
        info = _Info(obs=obs, term=term, finished=F["finished"])
        info.update({"position_error": R["position_error"], "attitude_error": R["attitude_error"],
                     "finished": F["finished"], "failure": F["failure"],
                     "diverged": F["diverged"], "time": R["time"], "success": F["success"],
                     "metric": R["metric"]})
        if self.task.task == DOCKING:
            info.update({"contact": F["contact"], "contact_distance": R["contact_distance"],
                         "contact_speed": R["contact_speed"],
                         "contact_attitude": R["contact_attitude"]})
        return obs, R["reward"], F["terminated"], F["truncated"], info

    # -------------------------------------------------------------- rollout statistics
    def rollout_stats_tensor(self, reset: bool = True, group=None) -> torch.Tensor:
        """``rollout_stats`` as a float64 device tensor in ``_N.ST_NAMES`` order, without a
        host synchronisation (the reduction and the NCCL all-reduce are stream-ordered)."""
        out = torch.empty(len(_N.ST_NAMES), dtype=torch.float64, device=self.state.device)
        _N.check(_N.load().uuv_rollout_stats(self._stats.data_ptr(), self._stats.shape[0],
                                             out.data_ptr(), 1 if reset else 0,
                                             self.state._stream()), TaskError)
        from .distributed import allreduce_sum

        return allreduce_sum(out, group)

    def rollout_stats(self, reset: bool = True, group=None) -> dict:
        """Sums since the last call: reward, finished, success, failure, truncated,
        metric over finished rows, diverged, frames — reduced on device in a fixed
        order, then all-reduced over ``group`` (NCCL) when torch.distributed is up."""
        return dict(zip(_N.ST_NAMES, self.rollout_stats_tensor(reset, group).tolist()))


StationKeepingEnv = TrackingEnv = DockingEnv = VecTaskEnv


def make_env(task: TaskConfig, sim: SimConfig, dr=None, seed: int = 0, **kw) -> VecTaskEnv:
    """Build the vectorised environment for a task/vehicle/level (tasks/core.py:533-538)."""
    if task.task not in TASK_KINDS:
        raise TaskError(f"unknown task '{task.task}', expected one of {TASK_KINDS}")
    return VecTaskEnv(task, sim, dr=dr, seed=seed, **kw)
