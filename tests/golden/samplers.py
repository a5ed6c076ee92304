"""Init samplers shared by the golden generator (reference) and the tests.

Each sampler returns a plain dict so the same draw sequence can be wrapped
into the reference's ``EnvInit``, the oracle's ``Init`` or the product's
``EnvInit``.  The draw order is part of the fixture contract.
"""

import numpy as np


def _axis_angle_quat(axis, angle):
    half = angle / 2.0
    return np.concatenate([[np.cos(half)], axis * np.sin(half)])


def rich(i, ep, rng):
    """Varied starts, currents on odd rows, four overlay families by i % 4."""
    ov = {}
    kind = i % 4
    if kind == 1:
        ov = {"mass*": float(rng.uniform(0.9, 1.1)), "damping*": float(rng.uniform(0.9, 1.1)),
              "cobm": float(rng.uniform(0.8, 2.0)), "thrust_coeff*": float(rng.uniform(0.9, 1.1))}
    elif kind == 2:
        ov = {"volume*": float(rng.uniform(0.95, 1.05)),
              "inertia*": float(rng.uniform(0.8, 1.2)),
              "added_mass*": float(rng.uniform(0.8, 1.2)),
              "time_constant*": float(rng.uniform(0.8, 1.2)),
              "payload_mass*": float(rng.uniform(0.05, 0.3)),
              "payload_position": rng.uniform(-0.1, 0.1, 3)}
    elif kind == 3:
        ov = {"mass*": float(rng.uniform(0.95, 1.05)),
              "mount_position_jitter": rng.uniform(-0.01, 0.01, 3)}
    cur = rng.uniform(-0.2, 0.2, 3) if i % 2 else np.zeros(3)
    axis = rng.uniform(-1.0, 1.0, 3)
    axis = axis / np.sqrt((axis * axis).sum())
    q = _axis_angle_quat(axis, float(rng.uniform(-0.4, 0.4)))
    return dict(p=rng.uniform(-1.0, 1.0, 3), q=q, nu=rng.uniform(-0.3, 0.3, 6),
                overlay=ov, current_ned=cur)


def jitter_matrix(a_dim):
    """Per-actuator (A, 3) mount jitter on every row."""

    def sampler(i, ep, rng):
        return dict(p=rng.uniform(-1.0, 1.0, 3), q=np.array([1.0, 0.0, 0.0, 0.0]),
                    nu=rng.uniform(-0.2, 0.2, 6),
                    overlay={"mount_position_jitter": rng.uniform(-0.02, 0.02, (a_dim, 3))},
                    current_ned=np.zeros(3))

    return sampler


def overlay_to_json(ov):
    return {k: (np.asarray(v).tolist() if not isinstance(v, float) else v) for k, v in ov.items()}
