"""Small fixed workload for ncu: a few direct launches of the step kernel.

    python scripts/profile_step.py [--n 4096] [--case cfg2] [--steps 20] [--rollout 20]
"""

import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

from sweep import make_case  # noqa: E402

from paper_2503_09203_b200 import engine as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--case", default="cfg2")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--rollout", type=int, default=0,
                    help="after the launched steps, one engine.rollout launch of this many steps")
    args = ap.parse_args()
    if args.case.startswith("task_") or args.case == "policy":
        return task_case(args)
    st, width = make_case(args.case, args.n)[:2]
    cmds = torch.rand((args.n, width), device=st.device) * 2 - 1
    for _ in range(args.steps):
        E.step_batch(st, cmds)
    if args.rollout:
        ring = torch.rand((args.rollout, args.n, width), device=st.device) * 2 - 1
        E.rollout(st, ring)
    torch.cuda.synchronize()
    print("ok", args.case, args.n, int(st.diverged.sum().item()))


def task_case(args):
    """task_cfg4 / task_cfg5: fused task steps; policy: device CEM episode launches."""
    from paper_2503_09203_b200 import baseline as B
    from paper_2503_09203_b200.tasks import TaskConfig, make_env

    if args.case == "task_cfg4":
        task = TaskConfig(task="tracking", vehicle="bluerov", level="disturbed")
        env = make_env(task, E.SimConfig(batch_size=args.n, substeps=8), seed=0)
    elif args.case == "task_cfg5":
        task = TaskConfig(task="docking", vehicle="bluerov_heavy", level="disturbed_dr")
        env = make_env(task, E.SimConfig(batch_size=args.n), seed=0)
    else:
        task = TaskConfig(task="station_keeping", vehicle="bluerov_heavy", episode_length=args.steps)
        env = make_env(task, E.SimConfig(batch_size=args.n), seed=0)
        r = B.EpisodeRunner(env, 32, args.n // 32, graph=False)
        import numpy as np
        r.run(np.random.default_rng(0).normal(0, 0.3, (32, r.n_params)))
        print("ok policy", args.n)
        return
    env.reset()
    cmds = torch.rand((args.n, env.action_dim), device="cuda") * 2 - 1
    for _ in range(args.steps):
        env.step(cmds)
    torch.cuda.synchronize()
    print("ok", args.case, args.n)


if __name__ == "__main__":
    main()
