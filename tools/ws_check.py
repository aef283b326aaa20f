"""A/B check of the warp-specialised rg_tall path against v6 on seeded
shapes: run once with RG_TALL_WS=1 and once with 0 (the switch is read once
per process), then compare.

    RG_TALL_WS=1 python tools/ws_check.py --out /tmp/ws1.npz
    RG_TALL_WS=0 python tools/ws_check.py --out /tmp/ws0.npz
    python tools/ws_check.py --compare /tmp/ws1.npz /tmp/ws0.npz
"""

import argparse
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

# (n, p, a1, merge, gmode, alias, zout: none/sep/inplace, zin)
CASES = [
    (1000, 8, 100, False, 1, True, "none", True),
    (1000, 8, 100, True, 2, False, "sep", True),
    (1000, 8, 0, False, 1, False, "none", True),
    (4097, 4, 36, False, 1, True, "inplace", True),
    (4097, 4, 36, True, 2, False, "inplace", True),
    (333, 16, 52, False, 1, True, "none", True),
    (333, 16, 52, True, 2, False, "sep", True),
    (64 * 148 * 3 + 17, 8, 28, False, 1, False, "sep", True),
    (5000, 3, 20, False, 0, False, "inplace", True),
    (5000, 3, 20, False, 2, False, "sep", False),
    (129, 12, 100, False, 1, True, "none", True),
    (1, 8, 8, False, 1, True, "none", True),
]


def run(out):
    import torch

    from paper_1604_01713_b200 import device as D

    dev = torch.device("cuda", 0)
    res = {}
    for ci, (n, p, a1, merge, gmode, alias, zo, zin_on) in enumerate(CASES):
        g = torch.Generator(device="cpu").manual_seed(ci)
        X = D.empty_block(n, max(a1, 1) + 24, dev)
        X.copy_(torch.randn(X.shape, generator=g, dtype=torch.float64).to(dev))
        X = X[:, : max(a1, 1)] if a1 else None
        Z = D.to_device_block(torch.randn(n, p, generator=g, dtype=torch.float64).numpy(), dev)
        S1 = torch.randn(a1, p, generator=g, dtype=torch.float64).to(dev) if a1 else None
        S2 = torch.randn(a1, p, generator=g, dtype=torch.float64).to(dev) if a1 and merge else None
        gb = None
        if gmode == 1:
            if alias:
                gb = X
            else:
                gb = D.empty_block(n, 40, dev)
                gb.copy_(torch.randn(gb.shape, generator=g, dtype=torch.float64).to(dev))
        gc = gb.shape[1] if gmode == 1 else (p if gmode == 2 else 0)
        gout = torch.zeros(gc, p, dtype=torch.float64, device=dev) if gmode else None
        zout = None
        if zo == "sep":
            zout = D.zeros_block(n, p, dev)
        elif zo == "inplace":
            zout = Z
        t1 = (X, S1, -1.0) if a1 else None
        t2 = (X, S2, 0.5) if a1 and merge else None
        D._tall_call(n, p, Z if zin_on else None, zout, t1, t2, None, None, gmode, gb, gout)
        torch.cuda.synchronize()
        if zout is not None:
            res[f"{ci}/z"] = D.to_numpy_block(zout)
        if gout is not None:
            res[f"{ci}/g"] = gout.cpu().numpy()
    np.savez(out, **res)


def compare(a, b):
    A, B = np.load(a), np.load(b)
    bad = 0
    for k in sorted(A.files):
        d = np.abs(A[k] - B[k]).max() if A[k].size else 0.0
        s = max(np.abs(B[k]).max(), 1.0) if B[k].size else 1.0
        flag = "" if d <= 1e-12 * s else "  <-- MISMATCH"
        bad += bool(flag)
        print(f"{k:10s} max|diff| {d:.3e}  scale {s:.3e}{flag}")
    print("MISMATCHES", bad)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    ap.add_argument("--compare", nargs=2)
    a = ap.parse_args()
    if a.compare:
        compare(*a.compare)
    else:
        run(a.out)
