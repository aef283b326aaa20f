"""Time rg_spmm_csr_c128 at config-5 shape (160^3 complex 27-point stencil)
and print GB/s of the SpMM model bytes; writes the p=16 output checksum so
variant builds (tools/ab_build.py) can be compared bitwise.

    python tools/prof_spmm_c128.py [--grid 160] [--p 16,8] [--reps 10]
"""
import argparse
import hashlib
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=160)
    ap.add_argument("--p", default="16,8")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    from paper_1604_01713_b200 import device as D, problems
    from paper_1604_01713_b200.sparse_core import DeviceCsr

    rp, ci, v, n = problems.stencil27_complex(args.grid)
    dA = DeviceCsr.from_host(n, n, rp, ci, v)
    out = {}
    for p in map(int, args.p.split(",")):
        g = torch.Generator(device="cuda")
        g.manual_seed(p)
        X = D.empty_block(n, p, dtype=torch.complex128)
        X.copy_(torch.randn(n, p, generator=g, device="cuda", dtype=torch.complex128))
        Y = D.empty_block(n, p, dtype=torch.complex128)
        for _ in range(2):
            D.spmm(dA, X, Y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            D.spmm(dA, X, Y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        nnz = len(ci)
        model = nnz * 20 + (n + 1) * 4 + 2 * p * n * 16
        h = hashlib.sha1(D.to_numpy_block(Y).tobytes()).hexdigest()[:16]
        out[p] = dict(ms=ms, gbs=model / ms / 1e6, sha=h)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
