"""Profiling driver: set up the bench step (cfg4 shapes) and run a few steps
so that ncu can capture the kernels of one step.

    python tools/prof_step.py [--grid 256] [--steps 2]
"""

import argparse
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=None)
    ap.add_argument("--family", default="cfg4")
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    grid = args.grid or bench.FAMILIES[args.family]["grid"]
    _, op, rs, fact, _ = bench._setup_step(grid, dev, family=args.family)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(args.steps):
        bench._one_step(fact, op, rs)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("prof_step done")


if __name__ == "__main__":
    main()
