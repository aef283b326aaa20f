"""Where a GCRO-DR cycle's time goes: wraps the solver's phases with
synchronising timers and solves system 0 (and 1) of the config-4 family at
grid^3.

    python tools/prof_cycle.py [--grid 128] [--systems 2]
"""
import argparse
import collections
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=128)
    ap.add_argument("--systems", type=int, default=2)
    ap.add_argument("--kernels", action="store_true", help="also attribute device time per kernel label")
    args = ap.parse_args()
    from paper_1604_01713_b200 import SolverConfig, arnoldi, dense_kernels, problems, recycling, solver

    acc = collections.defaultdict(float)
    cnt = collections.Counter()

    def wrap(mod, name, label):
        fn = getattr(mod, name)

        def w(*a, **k):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = fn(*a, **k)
            torch.cuda.synchronize()
            acc[label] += time.perf_counter() - t0
            cnt[label] += 1
            return r

        setattr(mod, name, w)

    wrap(arnoldi, "step", "arnoldi.step")  # (the solver's cycles run arnoldi.StepPipeline)
    wrap(solver, "_run_cycle", "cycle: start + block steps")
    wrap(arnoldi, "start", "arnoldi.start")
    wrap(solver, "_update_space", "recycle update")
    wrap(solver, "_apply_update", "apply update")
    wrap(solver, "_scrub", "scrub")
    wrap(solver, "prepare_cross_system", "cross-system prep")
    wrap(solver._Operator, "residual_into", "residual replace")
    wrap(dense_kernels.ProgressiveBlockLs, "append_block", "progressive LS")
    wrap(recycling, "harmonic_ritz_augmented", "  harmonic ritz (aug)")
    wrap(recycling, "update_recycle_space", "  update recycle space")
    wrap(recycling, "eig_generalized", "    eig_generalized")
    A, B, system, kw = problems.cfg4_sequence(N=args.grid, n_systems=args.systems)
    cfg = SolverConfig(**kw)
    solver.solve_block_gcrodr(system(0), B[:, :], None, SolverConfig(m=2, k=4, max_cycles=1))  # warm-up
    acc.clear()
    cnt.clear()
    from paper_1604_01713_b200 import device as D

    if args.kernels:
        D.LaunchLog.reset(timing=True)
    rs = None
    t0 = time.perf_counter()
    steps = 0
    cycles = 0
    for i in range(args.systems):
        _, rep, rs = solver.solve_block_gcrodr(system(i), B, None, cfg, rs_in=rs)
        steps += sum(len(h) for h in rep.residual_history)
        cycles += rep.cycles
    total = time.perf_counter() - t0
    out = {"grid": args.grid, "total_s": total, "cycles": cycles, "block_steps": steps,
           "phases_s": {k: round(v, 4) for k, v in sorted(acc.items(), key=lambda kv: -kv[1])},
           "calls": dict(cnt)}
    if args.kernels:
        summ = D.LaunchLog.summary()
        D.LaunchLog.reset(timing=False)
        out["kernels"] = {k: {"calls": v[0], "ms": round(v[1], 2), "GB/s": round(v[2] / max(v[1], 1e-9) / 1e6, 1)}
                          for k, v in sorted(summ.items(), key=lambda kv: -kv[1][1])}
        out["kernel_ms_total"] = round(sum(v[1] for v in summ.values()), 1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__" and "--recycle" not in sys.argv:
    main()


def recycle_breakdown(grid=256):
    """Per-launch device time of one end-of-cycle recycle update (after a
    full cycle of system 0), plus its host time."""
    from paper_1604_01713_b200 import SolverConfig, arnoldi, device as D, problems, solver

    A, B, system, kw = problems.cfg4_sequence(N=grid, n_systems=1)
    cfg = SolverConfig(**dict(kw, max_cycles=2))
    captured = {}
    orig = solver._update_space

    def grab(fact, rs, cfg_, report):
        captured["args"] = (fact, rs, cfg_, report)  # keep the last (augmented) call
        return orig(fact, rs, cfg_, report)

    solver._update_space = grab
    solver.solve_block_gcrodr(system(0), B, None, cfg)
    solver._update_space = orig
    fact, rs, cfg_, report = captured["args"]
    orig(fact, rs, cfg_, report)  # warm
    torch.cuda.synchronize()
    D.LaunchLog.reset(timing=True)
    t0 = time.perf_counter()
    orig(fact, rs, cfg_, report)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    summ = D.LaunchLog.summary()
    D.LaunchLog.reset(timing=False)
    dev_ms = sum(v[1] for v in summ.values())
    print(json.dumps({"augmented_update_wall_ms": wall * 1e3, "device_ms": dev_ms,
                      "launches": {k: [v[0], round(v[1], 3), round(v[2] / max(v[1], 1e-9) / 1e6, 1)]
                                   for k, v in sorted(summ.items(), key=lambda kv: -kv[1][1])}}, indent=1))


if __name__ == "__main__" and "--recycle" in sys.argv:
    recycle_breakdown()
