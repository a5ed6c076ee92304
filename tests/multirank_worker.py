"""One rank of the multi-rank product test (tests/test_gpu_multirank.py), launched by
torch.distributed.run: the rank's env shard of a job stepped through the B200 kernels,
its docking-task shard's rollout statistics all-reduced over the process group."""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_09203_b200 import distributed as D  # noqa: E402
from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200.randomization import preset  # noqa: E402
from paper_2503_09203_b200.tasks import TaskConfig, make_env  # noqa: E402
from paper_2503_09203_b200.vehicles import load_vehicle  # noqa: E402


def main():
    out_dir, n_global, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    ctx = D.init(os.environ.get("UUV_DIST_BACKEND", "gloo"), device_index=0)
    # physics: the rank's rows of a bluerov_heavy job with the train-preset DR
    st = D.make_shard(load_vehicle("bluerov_heavy"), n_global, E.SimConfig(batch_size=n_global),
                      ctx, master_seed=7)
    E.reset_envs(st, np.ones(st.n_envs, bool), E.spec_sampler(preset("train")))
    off = st.env_offset
    cmds = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, (steps, n_global, 8))).float()
    for t in range(steps):
        E.step_batch(st, cmds[t, off:off + st.n_envs].to(ctx.device))
    # task layer: docking shard, auto-reset, stats all-reduced (the only collective)
    env = make_env(TaskConfig(task="docking", vehicle="bluerov_heavy", level="disturbed_dr",
                              episode_length=20),
                   E.SimConfig(batch_size=st.n_envs), seed=3, device=ctx.device, env_offset=off)
    env.reset()
    for t in range(3 * steps):
        env.step(cmds[t % steps, off:off + st.n_envs].to(ctx.device))
    stats = env.rollout_stats()
    torch.cuda.synchronize()
    np.savez(os.path.join(out_dir, f"rank{ctx.rank}.npz"), off=off, p=st.p.cpu().numpy(),
             q=st.q.cpu().numpy(), nu=st.nu.cpu().numpy(), act=st.act.cpu().numpy(),
             ep=env.state.episodes.cpu().numpy(), tp=env.state.p.cpu().numpy(),
             stats=np.array([stats[k] for k in sorted(stats)]), world=ctx.world)
    D.finalize(ctx)


if __name__ == "__main__":
    main()
