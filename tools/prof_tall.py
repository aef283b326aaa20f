"""Time one rg_tall configuration in isolation (CUDA events), e.g.
    python tools/prof_tall.py --n 16777216 --p 8 --a1 20 --gc 80
"""
import argparse, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1604_01713_b200 import device as D

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 24)
ap.add_argument("--p", type=int, default=8)
ap.add_argument("--a1", type=int, default=20)
ap.add_argument("--a2", type=int, default=0)
ap.add_argument("--gc", type=int, default=80)
ap.add_argument("--self", action="store_true")
ap.add_argument("--alias", action="store_true", help="Gram basis = the update operand X1 (the joint schedule's P2)")
ap.add_argument("--store", action="store_true")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--trsm1", action="store_true")
ap.add_argument("--trsm2", action="store_true")
ap.add_argument("--noin", action="store_true", help="no Zin operand (z = the update terms only)")
args = ap.parse_args()
n, p = args.n, args.p
g = torch.Generator(device="cuda"); g.manual_seed(0)
def blk(c):
    b = D.empty_block(n, c)
    b.copy_(torch.randn(n, c, generator=g, device="cuda", dtype=torch.float64))
    return b
Z = blk(p); X1 = blk(args.a1) if args.a1 else None; X2 = blk(args.a2) if args.a2 else None
Gb = (X1[:, :args.gc] if args.alias else blk(args.gc)) if args.gc and not args.self else None
S1 = torch.randn(args.a1, p, device="cuda", dtype=torch.float64) if args.a1 else None
S2 = torch.randn(args.a2, p, device="cuda", dtype=torch.float64) if args.a2 else None
Zo = D.empty_block(n, p) if args.store else None
terms = ([(X1, S1, -1.0)] if X1 is not None else []) + ([(X2, S2, -1.0)] if X2 is not None else [])
gram = ("self", D.small(p, p)) if args.self else (("basis", Gb, D.small(args.gc, p)) if Gb is not None else None)
cols = (0 if args.noin else p) + args.a1 + args.a2 + (args.gc if Gb is not None and not args.alias else 0) + (p if Zo is not None else 0)
if args.gc and args.a1 == args.gc and Gb is not None: pass
R1 = torch.triu(torch.rand(p, p, device="cuda", dtype=torch.float64)) + 4 * torch.eye(p, device="cuda", dtype=torch.float64)
r1 = R1 if (args.trsm1 or args.trsm2) else None
r2 = R1 if args.trsm2 else None
for _ in range(2):
    D.tall(None if args.noin else Z, Zo, terms, r1=r1, r2=r2, gram=gram, n=n, p=p)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.reps):
    D.tall(None if args.noin else Z, Zo, terms, r1=r1, r2=r2, gram=gram, n=n, p=p)
e1.record(); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
ms = e0.elapsed_time(e1) / args.reps
print(f"n={n} p={p} a={args.a1}+{args.a2} gc={args.gc} self={args.self} store={args.store}: {ms:.3f} ms  {8*n*cols/ms/1e6:.0f} GB/s")
