"""Numbers behind the acceptance tests: CEM 60 iterations + 500-trial evaluation, and dr_ablation."""
import json
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2503_09203_b200 import baseline as B  # noqa: E402
from paper_2503_09203_b200.engine import SimConfig  # noqa: E402
from paper_2503_09203_b200.tasks import TaskConfig, make_env  # noqa: E402

for kw, name in (({"dtype": torch.float64, "rng": "pcg64"}, "f64-pcg64"), ({}, "f32-philox")):
    task = TaskConfig(task="station_keeping", vehicle="bluerov_heavy")
    t0 = time.perf_counter()
    env = make_env(task, SimConfig(batch_size=512), seed=0, **kw)
    res = B.cem_train(env, population=32, elite_frac=0.25, iterations=60, seed=0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    cell = B.evaluate(res.policy, make_env(task, SimConfig(batch_size=250), seed=1, **kw), n_trials=500)
    t2 = time.perf_counter()
    print(json.dumps({"case": name, "train_s": t1 - t0, "eval_s": t2 - t1,
                      "best_return": res.best_return, "mean_error": cell.mean_error,
                      "std_error": cell.std_error, "success_rate": cell.success_rate}), flush=True)
t0 = time.perf_counter()
rep = B.dr_ablation(seed=0, dtype=torch.float64, rng="pcg64")
print(json.dumps({"case": "dr_ablation f64-pcg64", "s": time.perf_counter() - t0,
                  "cells": rep.to_records()}), flush=True)
