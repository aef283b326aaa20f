"""Time the device ILU(0): factorisation and one apply_precond (two
wavefront triangular solves) on the 3-D conv-diff grid^3, block width p.

    python tools/prof_ilu.py [--grid 256] [--p 8] [--reps 5]
"""
import argparse
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    from paper_1604_01713_b200 import device as D, problems
    from paper_1604_01713_b200.precond import apply_precond_device, ilu0
    from paper_1604_01713_b200.sparse_core import spmm_device

    A = problems.conv_diff_3d(args.grid, 20.0)
    n, nnz = A.n_rows, A.nnz
    A.device()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    F = ilu0(A)
    torch.cuda.synchronize()
    t_fact_first = time.perf_counter() - t0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lu = F.device_lu()
    zero = torch.full((1,), 2**62, dtype=torch.int64, device="cuda")
    vals0 = lu.vals.clone()
    e0.record()
    for _ in range(args.reps):
        lu.vals.copy_(A.device().values)
        lu.factor(zero)  # device factorisation only (the schedule is built once)
    e1.record()
    torch.cuda.synchronize()
    assert torch.equal(lu.vals, vals0)
    t_fact = e0.elapsed_time(e1) / args.reps
    X = D.empty_block(n, args.p)
    X.copy_(torch.randn(n, args.p, device="cuda", dtype=torch.float64))
    Y = D.empty_block(n, args.p)
    for _ in range(2):
        apply_precond_device(F, X, Y)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.reps):
        apply_precond_device(F, X, Y)
    e1.record()
    torch.cuda.synchronize()
    t_apply = e0.elapsed_time(e1) / args.reps
    solve_ms = []
    for upper in (False, True):
        e0.record()
        for _ in range(args.reps):
            lu.solve(X, Y, upper=upper)
        e1.record()
        torch.cuda.synchronize()
        solve_ms.append(e0.elapsed_time(e1) / args.reps)
    e0.record()
    for _ in range(args.reps):
        spmm_device(A, X, Y)
    e1.record()
    torch.cuda.synchronize()
    t_spmm = e0.elapsed_time(e1) / args.reps
    # algorithmic bytes: factor = read pattern + read/write values; apply = 2 solves x (LU pattern + 2 p n 8)
    fact_bytes = nnz * (4 + 16) + (n + 1) * 4 + n * 4
    apply_bytes = 2 * (nnz * 12 + (n + 1) * 4 + n * 4) + 2 * 2 * args.p * n * 8
    print(json.dumps({"grid": args.grid, "n": n, "nnz": nnz, "p": args.p,
                      "ilu0_ms": t_fact, "ilu0_first_call_s": t_fact_first, "ilu0_GBs": fact_bytes / t_fact / 1e6,
                      "apply_ms": t_apply, "apply_GBs": apply_bytes / t_apply / 1e6, "spmm_ms": t_spmm,
                      "lower_ms": solve_ms[0], "upper_ms": solve_ms[1], "levels": [lu.lower_sched.levels,
                      lu.upper_sched.levels], "chunks": [lu.lower_sched.nchunks, lu.upper_sched.nchunks]}))


if __name__ == "__main__":
    main()
