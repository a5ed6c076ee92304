"""Host-side API parity with the reference (no GPU): configs, DR specs, vehicles.

Mirrors the reference's own unit tests for the host data model
(pkg/tests/test_randomization.py, test_vehicles.py, test_tasks.py validation,
test_trajectories.py) on the product's classes.
"""

import math

import numpy as np
import pytest

from paper_2503_09203_b200 import randomization as R
from paper_2503_09203_b200 import vehicles as V
from paper_2503_09203_b200.engine import EngineError, SimConfig, philox_generator
from paper_2503_09203_b200.tasks import (
    DockSpec, TaskConfig, TaskError, disturbed_spec, level_spec, start_box, target_yaw_quat,
)
from paper_2503_09203_b200.trajectories import TrajectoryError, TrajectorySpec, reference_point


def test_sim_config_defaults_and_validation():
    sim = SimConfig(batch_size=4)
    assert sim.dt == 0.02 and sim.substeps == 1 and sim.workers == 1
    for bad in (dict(dt=0.0), dict(dt=-0.1), dict(substeps=0), dict(batch_size=0),
                dict(workers=0)):
        with pytest.raises(EngineError):
            SimConfig(**{"batch_size": 4, **bad})


def test_task_config_validation():
    with pytest.raises(TaskError, match="unknown task"):
        TaskConfig(task="hovering")
    with pytest.raises(TaskError, match="unknown level"):
        TaskConfig(level="extreme")
    with pytest.raises(TaskError, match="episode_length"):
        TaskConfig(episode_length=0)
    with pytest.raises(TaskError, match="bounds"):
        TaskConfig(bounds=-1.0)
    with pytest.raises(TaskError, match="radius"):
        DockSpec(radius=0.0)
    with pytest.raises(TaskError, match="centre"):
        DockSpec(centre=(0.0, 0.0))


def test_dr_spec_requires_dr_level():
    for level in ("standard", "disturbed"):
        with pytest.raises(TaskError, match="disturbed_dr"):
            level_spec(level, R.preset("train"))
    assert level_spec("standard") is None
    assert set(level_spec("disturbed")) == {"payload_mass*", "payload_position",
                                            "current_velocity"}
    assert set(level_spec("disturbed_dr")) == set(R.preset("train"))


EXPECTED_PRESETS = {
    "train": {"mass*": (0.8, 1.2), "volume*": (0.8, 1.2), "cobm": (0.5, 3.0),
              "inertia*": (0.8, 1.2), "added_mass*": (0.8, 1.2), "damping*": (0.8, 1.2),
              "current_velocity": (0.0, 0.5), "payload_mass*": (0.0, 0.3)},
    "test_env1": {"mass*": (1.1, 1.1), "volume*": (1.1, 1.1), "cobm": (2.0, 2.0),
                  "inertia*": (1.1, 1.1), "added_mass*": (1.1, 1.1), "damping*": (1.1, 1.1),
                  "current_velocity": (0.2, 0.2), "payload_mass*": (0.2, 0.2)},
    "test_env2": {"mass*": (1.4, 1.4), "volume*": (1.4, 1.4), "cobm": (4.0, 4.0),
                  "inertia*": (1.4, 1.4), "added_mass*": (1.4, 1.4), "damping*": (1.4, 1.4),
                  "current_velocity": (0.8, 0.8), "payload_mass*": (0.4, 0.4)},
}


def test_presets_match_published_ranges():
    for name, rows in EXPECTED_PRESETS.items():
        spec = R.preset(name)
        assert set(spec) == set(rows)
        for key, (lo, hi) in rows.items():
            assert spec[key].distribution.support() == (lo, hi), (name, key)
    with pytest.raises(R.DRSpecError):
        R.preset("nope")


def test_parameter_validation():
    with pytest.raises(R.DRSpecError):
        R.DRParameter("bogus*", R.Uniform(1, 2))
    with pytest.raises(R.DRSpecError):
        R.DRParameter("mass*", R.Uniform(0.0, 1.0))
    R.DRParameter("payload_mass*", R.Uniform(0.0, 0.3))
    with pytest.raises(R.DRSpecError):
        R.Uniform(2.0, 1.0)
    with pytest.raises(R.DRSpecError):
        R.make_spec([R.DRParameter("mass*", R.Uniform(1, 2)), R.DRParameter("mass*", R.Uniform(1, 2))])
    with pytest.raises(R.DRSpecError):
        R.Piecewise([0.0, 1.0], [0.0])


def test_sample_overlay_sorted_order_matches_philox_draws():
    spec = R.preset("train")
    dyn = {k: v for k, v in spec.items() if k not in R.CURRENT_KEYS}
    rng = philox_generator(3, 11, 2)
    ov = R.sample_overlay(dyn, rng)
    assert list(ov) == sorted(dyn)
    rng2 = philox_generator(3, 11, 2)
    for key in sorted(dyn):
        lo, hi = dyn[key].distribution.support()
        assert ov[key] == rng2.uniform(lo, hi)


def test_sample_current_geometry():
    spec = {"current_velocity": R.DRParameter("current_velocity", R.Uniform(0.3, 0.3))}
    c = R.sample_current(spec, philox_generator(0, 0, 0))
    assert c[2] == 0.0 and abs(math.hypot(c[0], c[1]) - 0.3) < 1e-15
    assert np.all(R.sample_current({}, philox_generator(0, 0, 0)) == 0.0)


def test_piecewise_cdf_inversion_respects_support():
    pw = R.Piecewise([0.0, 1.0, 3.0], [2.0, 0.5])
    x = pw.sample(np.random.default_rng(0), size=20000)
    assert x.min() >= 0.0 and x.max() <= 3.0
    assert abs((x < 1.0).mean() - 2.0 / 3.0) < 0.02


def test_dr_schedule_progress():
    base = R.preset("train")
    sch = R.DRSchedule(base, [R.BoundsSchedule("mass*", [(0.0, 1.0, 1.0), (1.0, 0.8, 1.2)])])
    mid = R.set_progress(sch, 0.5)
    assert mid["mass*"].distribution.support() == pytest.approx((0.9, 1.1))
    with pytest.raises(R.DRSpecError):
        R.set_progress(sch, 1.5)


def test_vehicle_schema_errors_name_the_field(tmp_path):
    import yaml

    doc = {"schema_version": 1, "name": "x", "bounding_radius_m": 0.3,
           "rigid_body": {"mass_kg": "heavy"}}
    p = tmp_path / "v.yaml"
    p.write_text(yaml.safe_dump(doc))
    with pytest.raises(V.ConfigError, match="rigid_body.mass_kg"):
        V.load_vehicle(p)
    with pytest.raises(V.ConfigError, match="schema_version"):
        V.parse_vehicle({"schema_version": 2})


def test_overlay_math_matches_definitions():
    veh = V.load_vehicle("hauv")
    ov = {"mass*": 1.1, "volume*": 0.9, "cobm": 2.0, "damping*": 1.2, "thrust_coeff*": 0.8,
          "time_constant*": 1.5, "payload_mass*": 0.2, "payload_position": [0.1, 0.0, 0.05]}
    out = V.apply_overlay(veh, ov)
    m = veh.rb.mass * 1.1
    assert out.rb.mass == pytest.approx(m * 1.2)
    assert out.rb.displaced_volume == veh.rb.displaced_volume * 0.9
    assert out.rb.r_b[2] == veh.rb.r_g[2] + 2.0 * (veh.rb.r_b[2] - veh.rb.r_g[2])
    assert np.array_equal(out.coeffs.D_lin, veh.coeffs.D_lin * 1.2)
    assert out.actuators[0].thrust_coeff == veh.actuators[0].thrust_coeff * 0.8
    with pytest.raises(V.ConfigError):
        V.apply_overlay(veh, {"mass*": -1.0})
    with pytest.raises(V.ConfigError):
        V.apply_overlay(veh, {"nonsense": 1.0})


def test_trajectory_points_and_validation():
    spec = TrajectorySpec()
    p, v = reference_point(spec, 0.0)
    assert np.allclose(p, [2.0, 0.0, 1.0]) and np.allclose(v, [0.0, 0.5, 0.05])
    with pytest.raises(TrajectoryError):
        reference_point(spec, 61.0)
    with pytest.raises(TrajectoryError):
        TrajectorySpec(kind="spiral")


def test_start_boxes_follow_task_samplers():
    base, plo, phi, elo, ehi, nlo, nhi = start_box(TaskConfig(task="station_keeping"))
    assert list(base) == [0.0, 0.0, 1.0] and plo == [-2.5] * 3 and ehi[2] == np.pi
    base, plo, phi, elo, ehi, nlo, nhi = start_box(TaskConfig(task="tracking"))
    assert np.allclose(base, [2.0, 0.0, 1.0]) and elo[2] == pytest.approx(math.pi / 2 - 0.3)
    base, plo, phi, *_ = start_box(TaskConfig(task="docking"))
    assert list(base) == [0.0, 0.0, 3.0] and plo == [-1.5, -1.5, -2.5]
    q = target_yaw_quat(0.3)
    assert q[0] == pytest.approx(math.cos(0.15)) and q[3] == pytest.approx(math.sin(0.15))


def test_disturbed_spec_is_fixed_point():
    d = disturbed_spec()
    assert d["payload_mass*"].distribution.support() == (0.1, 0.1)
    assert d["current_velocity"].distribution.support() == (0.25, 0.25)


