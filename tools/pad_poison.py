"""Padding-poison check: every device block gets NaN in its leading-dimension
padding rows (n .. ld-1) and beyond; each rg_tall pass shape, the C-ABI CGS2
(sequential and joint) and CholQR2 must still return finite results equal to
numpy's.  A kernel that reads a padding row as data shows up as NaN.

    python tools/pad_poison.py
"""
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402


def poisoned(a, dev, extra_cols=0):
    from paper_1604_01713_b200 import device as D

    a = np.asfortranarray(a, dtype=np.float64)
    n, p = a.shape
    ld = D.round_ld(n)
    store = torch.full((p + extra_cols, ld), float("nan"), dtype=torch.float64, device=dev)
    v = store.t()[:n, :p]
    v.copy_(torch.from_numpy(a.T).t())
    return v


def main():
    from paper_1604_01713_b200 import _lib
    from paper_1604_01713_b200 import device as D

    dev = torch.device("cuda", 0)
    L = _lib.load()
    rng = np.random.default_rng(0)
    bad = 0
    for n in (1000, 4097, 50000, 70001):
        for p in (4, 8, 16):
            for (a1, gmode, alias, merge) in ((100, 1, True, False), (28, 1, False, False), (0, 1, False, False),
                                              (100, 2, False, True), (20, 0, False, False), (36, 2, False, False)):
                X = rng.standard_normal((n, max(a1, 1)))
                Z = rng.standard_normal((n, p))
                Gb = rng.standard_normal((n, 40))
                S1 = rng.standard_normal((max(a1, 1), p))
                S2 = rng.standard_normal((max(a1, 1), p))
                Xd, Zd, Gd = poisoned(X, dev, 8), poisoned(Z, dev, 8), poisoned(Gb, dev, 8)
                Zo = poisoned(np.zeros((n, p)), dev)
                # coefficient blocks as the kernels take them: column-major, ld = rows
                S1d, S2d = D.small(S1.shape[0], p, dev), D.small(S2.shape[0], p, dev)
                S1d.copy_(torch.from_numpy(S1))
                S2d.copy_(torch.from_numpy(S2))
                t1 = (Xd, S1d, -1.0) if a1 else None
                t2 = (Xd, S2d, -1.0) if a1 and merge else None
                gb = (Xd if alias else Gd) if gmode == 1 else None
                gc = gb.shape[1] if gmode == 1 else (p if gmode == 2 else 0)
                G = torch.zeros(gc, p, dtype=torch.float64, device=dev) if gmode else None
                D._tall_call(n, p, Zd, Zo, t1, t2, None, None, gmode, gb, G)
                torch.cuda.synchronize()
                z = Z.copy()
                if a1:
                    z = z - X @ S1
                    if merge:
                        z = z - X @ S2
                zo = D.to_numpy_block(Zo)
                ok = np.isfinite(zo).all() and np.abs(zo - z).max() <= 1e-9 * max(1.0, np.abs(z).max())
                if gmode:
                    g = G.cpu().numpy()
                    ref = (X if alias else Gb).T @ z if gmode == 1 else z.T @ z
                    ok = ok and np.isfinite(g).all() and np.abs(g - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max())
                if not ok:
                    bad += 1
                    print(f"BAD tall n={n} p={p} a1={a1} gmode={gmode} alias={alias} merge={merge}")
        # C-ABI CGS2, sequential (C and W apart) and joint (W follows C)
        for joint in (False, True):
            p, k, w = 8, 20, 40
            # C orthogonal to W (as in the solver), so the sequential and the
            # joint schedule project the same way
            Q = np.linalg.qr(rng.standard_normal((n, k + w)))[0]
            C, W = Q[:, :k], Q[:, k:]
            A = rng.standard_normal((n, p))
            if joint:
                CW = poisoned(np.hstack([C, W]), dev, 8)
                Cd, Wd = CW[:, :k], CW[:, k:]
            else:
                Cd, Wd = poisoned(C, dev, 8), poisoned(W, dev, 8)
            Zd = poisoned(A, dev, 8)
            coef = torch.zeros((2 * k + 2 * w) * p, dtype=torch.float64, device=dev)
            sm = torch.zeros(4 * p * p, dtype=torch.float64, device=dev)
            ws = D.Workspace.get(L.rg_tall_workspace_bytes(n, p, k, w, 1, k + w))
            rc = L.rg_cgs2_f64(n, p, Zd.data_ptr(), D.ld_of(Zd), Cd.data_ptr(), D.ld_of(Cd), k, Wd.data_ptr(),
                               D.ld_of(Wd), w, coef.data_ptr(), sm.data_ptr(), 1 if joint else 0, ws.data_ptr(), ws.numel(),
                               D.stream_ptr())
            torch.cuda.synchronize()
            z = A - C @ (C.T @ A) - W @ (W.T @ A)
            z = z - C @ (C.T @ z) - W @ (W.T @ z)
            got = D.to_numpy_block(Zd)
            if rc or not np.isfinite(got).all() or np.abs(got - z).max() > 1e-9:
                bad += 1
                print(f"BAD cgs2 n={n} joint={joint} rc={rc} err={np.nanmax(np.abs(got - z))}")
            Qd = poisoned(np.zeros((n, p)), dev)
            st = torch.zeros(2, dtype=torch.int32, device=dev)
            rc = L.rg_cholqr2_f64(n, p, Zd.data_ptr(), D.ld_of(Zd), Qd.data_ptr(), D.ld_of(Qd), sm.data_ptr(),
                                  st.data_ptr(), 1, ws.data_ptr(), ws.numel(), D.stream_ptr())
            torch.cuda.synchronize()
            q = D.to_numpy_block(Qd)
            if rc or not np.isfinite(q).all() or np.abs(q.T @ q - np.eye(p)).max() > 1e-12:
                bad += 1
                print(f"BAD cholqr2 n={n} joint={joint} rc={rc}")
    print("POISON BAD", bad)


if __name__ == "__main__":
    main()
