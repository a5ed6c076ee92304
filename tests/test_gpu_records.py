"""Device trajectory export vs the reference's own rollout records (cli.py:261-303)."""

import gzip
import json
import os

import numpy as np
import pytest
import torch

from paper_2503_09203_b200 import records as RC
from paper_2503_09203_b200.engine import SimConfig
from paper_2503_09203_b200.tasks import TaskConfig, make_env

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
# closed-loop float64 rollout (policy feedback, no state re-injection): the
# per-step 1e-12 parity compounds over up to 240 steps
RTOL, ATOL = 1e-8, 1e-9


def _golden(name):
    with gzip.open(os.path.join(GOLD, f"{name}.jsonl.gz"), "rt") as f:
        lines = f.read().splitlines()
    pol = json.load(open(os.path.join(GOLD, f"{name}_policy.json")))
    return lines, pol


def _torch_policy(pol, dtype):
    a, o = pol["action_dim"], pol["obs_dim"]
    th = torch.tensor(pol["theta"], dtype=dtype, device="cuda")
    w, b = th[:a * o].reshape(a, o), th[a * o:]
    return lambda obs: torch.tanh(obs @ w.T + b)


@pytest.mark.parametrize("name", ["rollout_docking_pcg64", "rollout_station_dr_pcg64"])
def test_rollout_records_match_reference(name):
    lines, pol = _golden(name)
    head = json.loads(lines[0])
    env = make_env(TaskConfig(task=head["task"], vehicle=head["vehicle"], level=head["level"]),
                   SimConfig(batch_size=head["envs"]), seed=head["seed"],
                   dtype=torch.float64, rng="pcg64")
    rows, meta, diverged = RC.rollout(env, head["steps"], _torch_policy(pol, torch.float64),
                                      policy_file=head["policy_file"])
    assert not diverged
    out = list(RC.format_records("trajectory", rows, meta))
    assert out[0] == lines[0]  # header byte for byte
    assert len(out) == len(lines)
    for mine, ref in zip(out[1:], lines[1:]):
        m, r = json.loads(mine), json.loads(ref)
        assert (m["env"], m["step"]) == (r["env"], r["step"])
        assert m["t"] == r["t"], (m["env"], m["step"])  # steps * dt after auto-reset
        for k in ("p", "quat", "euler", "nu", "commands", "reward"):
            np.testing.assert_allclose(m[k], r[k], rtol=RTOL, atol=ATOL, err_msg=f"{k} {ref[:60]}")


def test_recorder_float32_ring_and_limits():
    env = make_env(TaskConfig(task="tracking", vehicle="bluerov", level="disturbed"),
                   SimConfig(batch_size=1000), seed=1)
    env.reset()
    rec = RC.TrajectoryRecorder(env, steps=3)
    with pytest.raises(RC.RecordError):
        RC.TrajectoryRecorder(env, steps=3)
    u = torch.rand((1000, 6), device="cuda") * 4 - 2  # recorded unclipped
    for _ in range(3):
        env.step(u)
    with pytest.raises(RC.RecordError):
        env.step(u)
    a = rec.arrays()
    rec.detach()
    env.step(u)  # detached: no recording
    assert a["p"].shape == (3, 1000, 3) and a["commands"].shape == (3, 1000, 6)
    np.testing.assert_array_equal(a["commands"][2], u.cpu().numpy())
    np.testing.assert_allclose(a["t"][2], 3 * 0.02, rtol=1e-7)
    assert np.isfinite(a["p"]).all()
    assert len(rec.rows()) == 3000
