"""Time the joint-schedule pass shapes (P1 Gram, P2 update + aliased Gram,
P3 merged update + store + self-Gram) over basis widths at n = 2^24, p = 8;
run with RG_TALL_WS=1 and 0 to place the ws / v6 crossover.

    RG_TALL_WS=1 python tools/ws_sweep.py
"""
import json
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402


def main():
    from paper_1604_01713_b200 import device as D

    dev = torch.device("cuda", 0)
    n, p = 1 << 24, 8
    X = D.empty_block(n, 128, dev)
    X.normal_()
    Z = D.empty_block(n, p, dev)
    Z.normal_()
    Zo = D.empty_block(n, p, dev)
    out = {}
    for w in (12, 20, 28, 36, 44, 52, 60, 76, 100, 128):
        Xw = X[:, :w]
        G1 = D.small(w, p, dev)
        G2 = D.small(w, p, dev)
        Gs = D.small(p, p, dev)
        S = torch.randn(w, p, dtype=torch.float64, device=dev) * 1e-3
        shapes = {
            "P1": lambda: D._tall_call(n, p, Z, None, None, None, None, None, 1, Xw, G1),
            "P2": lambda: D._tall_call(n, p, Z, None, (Xw, S, -1.0), None, None, None, 1, Xw, G2),
            "P3": lambda: D._tall_call(n, p, Z, Zo, (Xw, S, -1.0), (Xw, S, -1.0), None, None, 2, None, Gs),
        }
        for name, fn in shapes.items():
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(10):
                fn()
            e1.record()
            torch.cuda.synchronize()
            out[f"{name}/w{w}"] = round(e0.elapsed_time(e1) / 10, 4)
    print(json.dumps({"ws": os.environ.get("RG_TALL_WS", "1"), "ms": out}))


if __name__ == "__main__":
    main()
