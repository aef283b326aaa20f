"""The k = 20 recycle-update pass shapes at n = 2^24 (C_new = [C W] Q, 108 -> 20
columns; U_new = ([U W_m] T) R^-1, 20 + 80 -> 20): rg_tall (v6, p = 20) against
cuBLAS DGEMM through torch (R^-1 folded into the small matrices)."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1604_01713_b200 import device as D  # noqa: E402

n, k, w, p = 1 << 24, 20, 88, 20
g = torch.Generator(device="cuda")
g.manual_seed(0)


def blk(c):
    b = D.empty_block(n, c)
    b.copy_(torch.randn(n, c, generator=g, device="cuda", dtype=torch.float64))
    return b


CW = blk(k + w)
U = blk(k)
Q = torch.randn(k + w, p, device="cuda", dtype=torch.float64)
T1, T2 = torch.randn(k, p, device="cuda", dtype=torch.float64), torch.randn(w - 8, p, device="cuda", dtype=torch.float64)
R = torch.triu(torch.rand(p, p, device="cuda", dtype=torch.float64)) + 4 * torch.eye(p, device="cuda", dtype=torch.float64)
out = D.empty_block(n, p)


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


Rinv = torch.linalg.inv(R)
res = {
    "C_new rg_tall": timed(lambda: D.tall(None, out, [(CW, Q, 1.0)], n=n, p=p)),
    "C_new cublas": timed(lambda: torch.mm(CW, Q, out=out)),
    "U_new rg_tall (2 terms + solve)": timed(lambda: D.tall(None, out, [(U, T1, 1.0), (CW[:, k:k + w - 8], T2, 1.0)],
                                                             r1=R, n=n, p=p)),
    "U_new cublas (R folded, 2 GEMMs)": timed(lambda: (torch.mm(U, T1 @ Rinv, out=out),
                                                       out.addmm_(CW[:, k:k + w - 8], T2 @ Rinv))),
}
for kname, ms in res.items():
    cols = (k + w + p) if kname.startswith("C_new") else (k + w - 8 + p)
    print(f"{kname:36s} {ms:.3f} ms  {8 * n * cols / ms / 1e6:.0f} GB/s (algorithmic)")
print("C_new out stride", out.stride(), "contiguous-colmajor")
