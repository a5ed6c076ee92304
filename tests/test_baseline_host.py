"""Policy algebra, policy files and evaluation reports (reference tests/test_baseline.py:28-62, 130-151)."""

import numpy as np
import pytest

from paper_2503_09203_b200.baseline import (BaselineError, EvalCell, EvalReport, Policy,
                                            load_policy, save_policy)


def test_policy_shapes_and_squash():
    p = Policy(weights=np.ones((2, 3)), bias=np.zeros(2))
    assert p.obs_dim == 3 and p.action_dim == 2 and p.n_params == 8
    out = p(np.zeros((5, 3)))
    assert out.shape == (5, 2) and np.all(out == 0.0)
    big = p(np.full((1, 3), 100.0))
    assert np.all(np.abs(big) <= 1.0) and np.allclose(big, 1.0)
    with pytest.raises(BaselineError, match="shape"):
        Policy(weights=np.ones((2, 3)), bias=np.zeros(3))


def test_policy_accepts_torch_tensors():
    import torch

    p = Policy(weights=np.arange(6.0).reshape(2, 3) / 10, bias=np.array([0.1, -0.2]))
    x = np.random.default_rng(0).normal(size=(4, 3))
    got = p(torch.from_numpy(x)).numpy()
    np.testing.assert_allclose(got, p(x), rtol=1e-15, atol=1e-15)


def test_policy_theta_round_trip():
    rng = np.random.default_rng(0)
    p = Policy(weights=rng.normal(size=(4, 7)), bias=rng.normal(size=4))
    again = Policy.from_theta(p.theta(), obs_dim=7, action_dim=4)
    assert p.weights.tobytes() == again.weights.tobytes()
    assert p.bias.tobytes() == again.bias.tobytes()
    with pytest.raises(BaselineError, match="theta"):
        Policy.from_theta(p.theta(), obs_dim=7, action_dim=5)


def test_policy_file_round_trip(tmp_path):
    rng = np.random.default_rng(1)
    p = Policy(weights=rng.normal(size=(6, 19)), bias=rng.normal(size=6))
    path = tmp_path / "policy.json"
    save_policy(path, p, meta={"task": "station_keeping"})
    assert load_policy(path).theta().tobytes() == p.theta().tobytes()
    bad = tmp_path / "bad.json"
    bad.write_text('{"schema_version": 1, "theta": [1.0]}\n')
    with pytest.raises(BaselineError, match="not a valid policy file"):
        load_policy(bad)


def test_reference_policy_files_load():
    import os

    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    p = load_policy(os.path.join(gold, "rollout_docking_pcg64_policy.json"))
    assert (p.action_dim, p.obs_dim) == (8, 21)


def test_eval_report_round_trip():
    rep = EvalReport(task="station_keeping", vehicle="bluerov_heavy",
                     metric_name="distance_to_target_m")
    rep.cells = [EvalCell("ndr/test_env1", 500, 1.0771, 0.61, 0.01),
                 EvalCell("dr/test_env1", 500, 0.6948, 0.48, 0.13)]
    rows = rep.to_records()
    assert all(r["unit"] == "m" for r in rows)
    assert EvalReport.from_records(rows) == rep
    assert rep.cell("dr/test_env1").mean_error == 0.6948
    with pytest.raises(KeyError):
        rep.cell("nope")
    with pytest.raises(BaselineError, match="empty"):
        EvalReport.from_records([])
    table = rep.to_table()
    assert "[m]" in table and "ndr/test_env1" in table and "0.6948" in table
