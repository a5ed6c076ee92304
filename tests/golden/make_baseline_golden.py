"""Golden CEM / evaluation results from the REFERENCE's ``uuvsim.baseline``.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_baseline_golden.py

The unmodified reference (PCG64/SeedSequence episode streams, host policy
loop) runs the configurations of its own tests/test_baseline.py plus a
docking case whose batch does not divide by the population (padded rows act
with 0).  tests/test_gpu_baseline.py replays them with the device episode loop
(``rng="pcg64"``, float64) and compares.
"""

import json
import os
import time

import numpy as np
from uuvsim.baseline import Policy, cem_train, evaluate
from uuvsim.engine import SimConfig
from uuvsim.tasks import TaskConfig, make_env

HERE = os.path.dirname(os.path.abspath(__file__))


def small_env(seed=5, batch=40):
    task = TaskConfig(task="station_keeping", vehicle="bluerov", episode_length=60)
    return make_env(task, SimConfig(batch_size=batch), seed=seed)


def dock_env(seed=3, batch=43):
    task = TaskConfig(task="docking", vehicle="bluerov_heavy", level="disturbed_dr",
                      episode_length=80)
    return make_env(task, SimConfig(batch_size=batch), seed=seed)


def cem_case(env, **kw):
    res = cem_train(env, **kw)
    return {"kw": kw, "curve": res.curve, "theta": res.policy.theta().tolist(),
            "best_return": res.best_return, "episodes": env.state.episodes.tolist()}


def cell(c):
    return {"label": c.label, "n_trials": c.n_trials, "mean_error": c.mean_error,
            "std_error": c.std_error, "success_rate": c.success_rate}


def main():
    out = {}
    out["cem_station"] = cem_case(small_env(), population=10, iterations=3, seed=5)
    out["cem_dock_padded"] = cem_case(dock_env(), population=10, iterations=2, seed=3,
                                      init_std=0.3)
    env = small_env(seed=9, batch=25)
    out["eval_zero"] = cell(evaluate(Policy.zeros(env.obs_dim, env.action_dim), env,
                                     n_trials=50))
    out["eval_zero"]["episodes"] = env.state.episodes.tolist()
    trained = Policy.from_theta(np.asarray(out["cem_station"]["theta"]), env.obs_dim,
                                env.action_dim)
    env = small_env(seed=7, batch=30)
    out["eval_trained"] = cell(evaluate(trained, env, n_trials=45, label="trained"))
    # the reference's acceptance run (test_acceptance.py:308-319): ~2.5 CPU-minutes
    t0 = time.perf_counter()
    task = TaskConfig(task="station_keeping", vehicle="bluerov_heavy")
    res = cem_train(make_env(task, SimConfig(batch_size=512), seed=0), population=32,
                    elite_frac=0.25, iterations=60, seed=0)
    t1 = time.perf_counter()
    c = evaluate(res.policy, make_env(task, SimConfig(batch_size=250), seed=1), n_trials=500)
    out["acceptance_cem"] = {
        "settings": "TaskConfig(station_keeping, bluerov_heavy), SimConfig(batch_size=512), "
                    "seed 0; cem_train(population=32, elite_frac=0.25, iterations=60, seed=0); "
                    "evaluate(batch 250, seed 1, n_trials=500)",
        "mean_error": c.mean_error, "std_error": c.std_error, "success_rate": c.success_rate,
        "best_return": res.best_return,
        "reference_cpu_seconds": {"train": t1 - t0, "eval": time.perf_counter() - t1}}
    path = os.path.join(HERE, "baseline_reference.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", path)
    for k, v in out.items():
        print(k, {x: v[x] for x in v if x in ("best_return", "mean_error", "success_rate")})


if __name__ == "__main__":
    main()
