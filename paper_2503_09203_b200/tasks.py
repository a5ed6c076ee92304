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
single fused kernel launch (``uuv_task_step``); the host only enqueues it.
Arrays are torch CUDA tensors in the batch dtype (float32 by default).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .randomization import CURRENT_KEYS, DRParameter, Uniform, make_spec, preset
from .trajectories import HELIX, TrajectorySpec, reference_point

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
