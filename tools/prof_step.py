"""Profiling driver: set up the bench step (cfg4 shapes) and run a few steps
so that ncu can capture the kernels of one step.

    python tools/prof_step.py [--grid 256] [--steps 2]
"""

import argparse
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=None)
    ap.add_argument("--family", default="cfg4")
    ap.add_argument("--labels", default=None, help="write the launch labels of the profiled steps here")
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    grid = args.grid or bench.FAMILIES[args.family]["grid"]
    _, op, rs, fact, _ = bench._setup_step(grid, dev, family=args.family)
    torch.cuda.synchronize()
    from paper_1604_01713_b200 import device as D

    D.LaunchLog.reset(timing=True)
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(args.steps):
        bench._one_step(fact, op, rs)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    # launch order of the profiled steps (tools/ncu_traffic.py pairs it with ncu's launch list)
    # one record per library call; a call may launch several kernels (label repeated)
    recs = [{"label": lbl, "bytes": b // max(nl, 1)} for lbl, _, b, _, nl in D.LaunchLog.records()
            for _ in range(max(nl, 1))]
    D.LaunchLog.reset(timing=False)
    if args.labels:
        pathlib.Path(args.labels).write_text(json.dumps(recs, indent=1))
    print("prof_step done")


if __name__ == "__main__":
    main()
