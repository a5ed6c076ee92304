"""Golden trajectory records from the REFERENCE's own ``cmd_rollout`` (cli.py:261-303).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_rollout_golden.py

Runs the unmodified reference (its PCG64/SeedSequence streams; no hook) through
the CLI function with an affine-tanh policy file and writes the JSONL records it
prints (header + one row per env per step) next to this script, together with
the policy file.  tests/test_gpu_records.py replays the same rollout through
``records.rollout`` on the device (``rng="pcg64"``) and compares.
"""

import argparse
import contextlib
import gzip
import io
import json
import os
import shutil
import tempfile

import numpy as np
from uuvsim import cli
from uuvsim.baseline import Policy, save_policy

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # docking, heave thrusters driven down: contacts -> auto-resets inside the trace
    "rollout_docking_pcg64": dict(task="docking", vehicle="bluerov_heavy", level="standard",
                                  envs=6, steps=240, seed=5, bias=[0, 0, 0, 0, -3, -3, -3, -3]),
    "rollout_station_dr_pcg64": dict(task="station_keeping", vehicle="bluerov",
                                     level="disturbed_dr", envs=3, steps=40, seed=2,
                                     bias=[0.2, -0.1, 0.3, 0.0, 0.1, -0.2]),
}


def policy_for(case, obs_dim):
    a = len(case["bias"])
    w = np.random.default_rng(case["seed"]).uniform(-0.05, 0.05, (a, obs_dim))
    return Policy(weights=w, bias=np.asarray(case["bias"], dtype=float))


def main():
    from uuvsim.tasks import TaskConfig, make_env
    from uuvsim.engine import SimConfig

    tmp = tempfile.mkdtemp()
    try:
        for name, case in CASES.items():
            env = make_env(TaskConfig(task=case["task"], vehicle=case["vehicle"],
                                      level=case["level"]), SimConfig(batch_size=1))
            pol = policy_for(case, env.obs_dim)
            ppath = os.path.join(HERE, f"{name}_policy.json")
            save_policy(ppath, pol)
            args = argparse.Namespace(task=case["task"], vehicle=case["vehicle"],
                                      level=case["level"], envs=case["envs"], workers=1,
                                      seed=case["seed"], steps=case["steps"], policy=ppath,
                                      out=None, format="records")
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                rc = cli.cmd_rollout(args)
            text = buf.getvalue()
            head = json.loads(text.splitlines()[0])
            head["policy_file"] = os.path.basename(ppath)  # path-independent fixture
            lines = [json.dumps(head, sort_keys=True, separators=(",", ":"))]
            lines += text.splitlines()[1:]
            out = os.path.join(HERE, f"{name}.jsonl.gz")
            with gzip.open(out, "wt") as f:
                f.write("\n".join(lines) + "\n")
            resets = sum(1 for ln in lines[1:] if json.loads(ln)["t"] == 0.0)
            print(f"wrote {out}: {len(lines) - 1} rows, rc={rc}, rows at t=0: {resets}")
    finally:
        shutil.rmtree(tmp)


if __name__ == "__main__":
    main()
