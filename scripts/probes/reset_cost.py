"""Task step latency with and without auto-resets in the window (config 5, small N)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2503_09203_b200 import engine as E  # noqa: E402
from paper_2503_09203_b200.tasks import TaskConfig, make_env  # noqa: E402

for n in (4096, 65536):
    for mode in ("random", "zero"):
        env = make_env(TaskConfig(task="docking", vehicle="bluerov_heavy", level="disturbed_dr"),
                       E.SimConfig(batch_size=n), seed=0)
        env.reset()
        cmds = (torch.rand((n, 8), device="cuda") * 2 - 1) if mode == "random" else \
            torch.zeros((n, 8), device="cuda")
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                env.step(cmds)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(50):
                    env.step(cmds)
            env.rollout_stats(reset=True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); g.replay(); e1.record(s)
        torch.cuda.synchronize()
        st = env.rollout_stats(reset=True)
        print(n, mode, round(e0.elapsed_time(e1) / 50 * 1e3, 2), "us/step", "finished", st["finished"])
