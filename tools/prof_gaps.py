"""Device idle time between library calls in an unsynchronised cfg4 solve
(system 0 at grid^3): librgb200 brackets every call with events
(rg_profile_enable); the gap before each call is the time since the previous
call ended (torch plumbing + the device waiting on the host).  Gaps are
summed by the (previous label -> next label) transition, which locates them
in the cycle.

    python tools/prof_gaps.py [--grid 256] [--cycles 20]
"""
import argparse
import collections
import ctypes
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--cycles", type=int, default=20)
    args = ap.parse_args()
    from paper_1604_01713_b200 import SolverConfig, problems, solver
    from paper_1604_01713_b200 import device as D

    A, B, system, kw = problems.cfg4_sequence(N=args.grid, n_systems=1)
    solver.solve_block_gcrodr(system(0), B, None, SolverConfig(m=2, k=4, max_cycles=1))  # warm-up / upload
    torch.cuda.synchronize()
    D.LaunchLog.reset(timing=True)
    t0 = time.perf_counter()
    _, rep, _ = solver.solve_block_gcrodr(system(0), B, None, SolverConfig(**dict(kw, max_cycles=args.cycles)))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    recs = D.LaunchLog.records()
    L = D.lib()
    gaps = collections.defaultdict(float)
    cnt = collections.Counter()
    total_gap = 0.0
    ms = ctypes.c_double()
    for i in range(1, len(recs)):
        L.rg_profile_gap(i, ctypes.byref(ms))
        key = f"{recs[i - 1][0].split(' ')[0]} {recs[i - 1][0][-22:]} -> {recs[i][0]}"
        gaps[key] += ms.value
        cnt[key] += 1
        total_gap += ms.value
    D.LaunchLog.reset(timing=False)
    busy = sum(r[1] for r in recs)
    out = {"grid": args.grid, "cycles": rep.cycles, "wall_s": wall, "device_busy_s": busy / 1e3,
           "gaps_s": total_gap / 1e3,
           "top_gaps_ms": {k: [round(v, 2), cnt[k]] for k, v in sorted(gaps.items(), key=lambda kv: -kv[1])[:25]}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
