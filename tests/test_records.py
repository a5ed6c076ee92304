"""Record format (records.py mirror of uuvsim/records.py:24-94) on CPU."""

import gzip
import json
import os

import numpy as np
import pytest

from paper_2503_09203_b200 import records as RC

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _lines(name):
    with gzip.open(os.path.join(GOLD, f"{name}.jsonl.gz"), "rt") as f:
        return f.read().splitlines()


@pytest.mark.parametrize("name", ["rollout_docking_pcg64", "rollout_station_dr_pcg64"])
def test_dump_line_reproduces_reference_records_text(name):
    lines = _lines(name)
    head = json.loads(lines[0])
    rows = [json.loads(x) for x in lines[1:]]
    meta = {k: v for k, v in head.items() if k not in ("schema_version", "kind")}
    again = list(RC.format_records("trajectory", rows, meta))
    assert again == lines
    assert all(tuple(sorted(r)) == tuple(sorted(RC.TRAJECTORY_FIELDS)) for r in rows)


def test_sanitize_and_round_trip(tmp_path):
    rows = [{"env": np.int64(1), "p": np.array([1.0, np.nan, np.inf]), "ok": np.bool_(True),
             "reward": np.float32(0.5)}]
    path = tmp_path / "r.jsonl"
    assert RC.write_records(path, "trajectory", rows, {"seed": 3}) == 1
    head, back = RC.read_records(path)
    assert head == {"schema_version": 1, "kind": "trajectory", "seed": 3}
    assert back == [{"env": 1, "p": [1.0, None, None], "ok": True, "reward": 0.5}]
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"schema_version": 2, "kind": "x"}\n')
    with pytest.raises(RC.RecordError):
        RC.read_records(bad)
    (tmp_path / "empty.jsonl").write_text("")
    with pytest.raises(RC.RecordError):
        RC.read_records(tmp_path / "empty.jsonl")


def test_quat_to_euler_matches_reference_rows():
    rows = [json.loads(x) for x in _lines("rollout_station_dr_pcg64")[1:]]
    q = np.array([r["quat"] for r in rows])
    e = np.array([r["euler"] for r in rows])
    assert np.array_equal(RC.quat_to_euler(q), e)
