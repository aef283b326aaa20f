import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle
from paper_1604_01713_b200 import _lib, device as D
def det():
    rng = np.random.default_rng(3)
    n, p = 1_000_003, 8
    Zd = D.to_device_block(rng.standard_normal((n, p)))
    Wd = D.to_device_block(rng.standard_normal((n, 80)))
    for _ in range(3):
        o = D.small(80, p); D.tall(Zd, None, gram=("basis", Wd, o)); o.cpu()
def cabi():
    L = _lib.load(); rng = np.random.default_rng(21)
    n, p, k, w = 50_000, 8, 20, 40
    C = np.linalg.qr(rng.standard_normal((n, k)))[0]; W = np.linalg.qr(rng.standard_normal((n, w)))[0]
    A = rng.standard_normal((n, p))
    ref, F, H = oracle.cgs2_project(A, C, W)
    Zd, Cd, Wd = D.to_device_block(A), D.to_device_block(C), D.to_device_block(W)
    coef = torch.zeros((2 * k + 2 * w) * p, dtype=torch.float64, device="cuda")
    small = torch.zeros(4 * p * p, dtype=torch.float64, device="cuda")
    ws = D.Workspace.get(L.rg_tall_workspace_bytes(n, p, k, w, 1, max(k, w)))
    rc = L.rg_cgs2_f64(n, p, Zd.data_ptr(), D.ld_of(Zd), Cd.data_ptr(), D.ld_of(Cd), k, Wd.data_ptr(), D.ld_of(Wd), w,
                       coef.data_ptr(), small.data_ptr(), 0, ws.data_ptr(), ws.numel(), D.stream_ptr())
    z = D.to_numpy_block(Zd)
    print("rc", rc, "gpu sum", float(np.abs(z).sum()), "ref sum", float(np.abs(ref).sum()),
          "C sum", float(np.abs(C).sum()), "rel", float(np.abs(z - ref).max() / np.abs(ref).max()))
mode = sys.argv[1]
if mode == "pair":
    det()
elif mode == "pair_empty":
    det(); torch.cuda.synchronize(); torch.cuda.empty_cache()
elif mode == "twice":
    cabi()
elif mode == "alloc":
    x = torch.empty(1_000_003 * 88, dtype=torch.float64, device="cuda"); x.normal_(); del x
elif mode == "alloc_nan":
    x = torch.full((1_000_003 * 88,), float("nan"), dtype=torch.float64, device="cuda"); del x
cabi()
