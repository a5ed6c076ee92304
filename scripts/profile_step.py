"""Small fixed workload for ncu: a few direct launches of the step kernel.

    python scripts/profile_step.py [--n 4096] [--case cfg2] [--steps 20]
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
    args = ap.parse_args()
    st, width, _ = make_case(args.case, args.n)
    cmds = torch.rand((args.n, width), device=st.device) * 2 - 1
    for _ in range(args.steps):
        E.step_batch(st, cmds)
    torch.cuda.synchronize()
    print("ok", args.case, args.n, int(st.diverged.sum().item()))


if __name__ == "__main__":
    main()
