"""Trajectory export: device-recorded rollouts in the reference's JSONL format.

The record format is the reference's (``uuvsim/records.py:24-94``): a header
line ``{"schema_version": 1, "kind": ..., **meta}`` then one JSON object per
row; keys are sorted, separators are compact, numpy values become plain Python
and non-finite floats become ``null``.  ``rollout()`` reproduces
``cmd_rollout`` (cli.py:261-303) without the CLI.

What differs is where the rows come from.  The reference copies p/q/ν to the
host after every step and builds one dict per env per step in Python.  Here
``TrajectoryRecorder`` hands the fused task kernel a slot of a device ring
buffer each step; the kernel writes the post-step (post-auto-reset) pose,
velocity, reward, time and raw command while they are still in registers
(``uuv_task_io.trace``), and the ring is read back once at the end.
"""

from __future__ import annotations

import json
from pathlib import Path
from typing import Any, Iterable, Iterator

import numpy as np
import torch

from . import _native as N

SCHEMA_VERSION = 1
TRAJECTORY_FIELDS = ("env", "step", "t", "p", "quat", "euler", "nu", "commands", "reward")


class RecordError(ValueError):
    pass


def sanitize(value: Any) -> Any:
    """JSON-safe plain Python; non-finite floats -> None (records.py:35-50)."""
    if isinstance(value, dict):
        return {str(k): sanitize(v) for k, v in value.items()}
    if isinstance(value, (list, tuple)):
        return [sanitize(v) for v in value]
    if isinstance(value, np.ndarray):
        return sanitize(value.tolist())
    if isinstance(value, torch.Tensor):
        return sanitize(value.detach().cpu().numpy())
    if isinstance(value, (float, np.floating)):
        f = float(value)
        return f if np.isfinite(f) else None
    if isinstance(value, np.integer):
        return int(value)
    if isinstance(value, np.bool_):
        return bool(value)
    return value


def dump_line(obj: Any) -> str:
    return json.dumps(sanitize(obj), sort_keys=True, separators=(",", ":"), allow_nan=False)


def format_records(kind: str, rows: Iterable[dict], meta: dict | None = None) -> Iterator[str]:
    head = {"schema_version": SCHEMA_VERSION, "kind": kind}
    head.update(meta or {})
    yield dump_line(head)
    for r in rows:
        yield dump_line(r)


def write_records(path, kind: str, rows: Iterable[dict], meta: dict | None = None) -> int:
    """Write header + rows; returns the number of data rows."""
    count = 0
    with Path(path).open("w", encoding="utf-8") as fh:
        for k, line in enumerate(format_records(kind, rows, meta)):
            fh.write(line + "\n")
            count = k
    return count


def read_records(path) -> tuple[dict, list[dict]]:
    lines = [ln for ln in Path(path).read_text(encoding="utf-8").splitlines() if ln.strip()]
    if not lines:
        raise RecordError(f"{path}: empty records file")
    head = json.loads(lines[0])
    if not isinstance(head, dict) or "schema_version" not in head:
        raise RecordError(f"{path}: first line is not a records header")
    if head["schema_version"] != SCHEMA_VERSION:
        raise RecordError(f"{path}: schema_version {head['schema_version']} "
                          f"(expected {SCHEMA_VERSION})")
    return head, [json.loads(ln) for ln in lines[1:]]


def quat_to_euler(q: np.ndarray) -> np.ndarray:
    """ZYX [phi, theta, psi] from unit quaternions (kinematics.py:130-142)."""
    w, x, y, z = (q[..., k] for k in range(4))
    phi = np.arctan2(2 * (w * x + y * z), 1 - 2 * (x * x + y * y))
    theta = np.arcsin(np.clip(2 * (w * y - z * x), -1.0, 1.0))
    psi = np.arctan2(2 * (w * z + x * y), 1 - 2 * (y * y + z * z))
    return np.stack([phi, theta, psi], axis=-1)


class TrajectoryRecorder:
    """Device ring of per-step trajectory records filled by ``env.step``.

        rec = TrajectoryRecorder(env, steps=T)
        for t in range(T):
            env.step(u_t)
        rows = rec.rows()        # one D2H copy; cmd_rollout's row dicts

    Ring layout: ``[T][15 + A][ld]`` in the batch dtype (UUV_TRACE_* rows).
    Steps beyond ``steps`` raise; ``detach()`` stops recording.
    """

    def __init__(self, env, steps: int):
        if env._recorder is not None:
            raise RecordError("env already has a recorder attached")
        st = env.state
        self.env = env
        self.capacity = int(steps)
        self.width = N.TRACE_CMD + env.action_dim
        self.ring = torch.empty((self.capacity, self.width, st._ld), dtype=st.dtype,
                                device=st.device)
        self.count = 0
        env._recorder = self

    def _next_slot(self):
        if self.count >= self.capacity:
            raise RecordError(f"recorder full ({self.capacity} steps)")
        t = self.count
        self.count += 1
        return self.ring[t].data_ptr(), self.ring.shape[2]

    def detach(self):
        if self.env._recorder is self:
            self.env._recorder = None

    def arrays(self) -> dict:
        """Host float64 arrays of the recorded steps: p (T,N,3), quat, nu, t, reward, commands."""
        n = self.env.n_envs
        r = self.ring[:self.count, :, :n].double().cpu().numpy()
        tr = lambda a, b: np.ascontiguousarray(np.moveaxis(r[:, a:b], 1, 2))  # noqa: E731
        return {"p": tr(N.TRACE_P, N.TRACE_P + 3), "quat": tr(N.TRACE_Q, N.TRACE_Q + 4),
                "nu": tr(N.TRACE_NU, N.TRACE_NU + 6), "reward": r[:, N.TRACE_REWARD],
                "t": r[:, N.TRACE_T], "commands": tr(N.TRACE_CMD, self.width)}

    def rows(self) -> list:
        """cmd_rollout's records (cli.py:277-287): step-major, env-minor."""
        a = self.arrays()
        euler = quat_to_euler(a["quat"])
        out = []
        for s in range(self.count):
            for i in range(self.env.n_envs):
                out.append({"env": i, "step": s, "t": a["t"][s, i], "p": a["p"][s, i],
                            "quat": a["quat"][s, i], "euler": euler[s, i], "nu": a["nu"][s, i],
                            "commands": a["commands"][s, i], "reward": a["reward"][s, i]})
        return out


def rollout(env, steps: int, policy=None, *, seed=None, task_name=None, level=None,
            vehicle=None, policy_file=None):
    """``uuvsim rollout`` without the CLI (cli.py:261-303).

    ``policy``: None (zero commands), a callable ``obs -> commands`` (host or
    device), or a ``policy.DevicePolicy``.  Returns ``(rows, meta, diverged)``;
    write them with ``write_records(path, "trajectory", rows, meta)``.
    """
    from .tasks import METRIC_DEFINITIONS

    obs = env.reset()
    rec = TrajectoryRecorder(env, steps)
    diverged = torch.zeros((), dtype=torch.bool, device=env.state.device)
    zeros = torch.zeros((env.n_envs, env.action_dim), dtype=env.state.dtype,
                        device=env.state.device)
    try:
        for _ in range(steps):
            u = policy(obs) if policy is not None else zeros
            obs, _r, _te, _tr, info = env.step(u)
            diverged |= info["diverged"].any()
        rows = rec.rows()
    finally:
        rec.detach()
    t = env.task
    meta = {"command": "rollout", "task": task_name or t.task, "vehicle": vehicle or t.vehicle,
            "level": level or t.level, "seed": env.seed if seed is None else seed,
            "dt": env.sim.dt, "envs": env.n_envs, "steps": steps, "policy_file": policy_file,
            "metric": {"name": env.metric_name, "unit": "m",
                       "definition": METRIC_DEFINITIONS[env.metric_name]}}
    return rows, meta, bool(diverged.item())
