"""Fixed costs of one cfg4 256^3 solve outside the cycles: matrix upload,
diagonal-layout plan, B upload, X download (host-resident operands, as the
time-to-solution record measures them)."""
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1604_01713_b200 import device as D, problems  # noqa: E402
from paper_1604_01713_b200 import solver  # noqa: E402


def t(fn, sync=True):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    if sync:
        torch.cuda.synchronize()
    return r, time.perf_counter() - t0


grid = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A, B, system, kw = problems.cfg4_sequence(N=grid, n_systems=2)
A1 = system(1)
dev = torch.device("cuda", 0)
torch.zeros(1, device=dev)
out = {}
dA, out["A upload (first)"] = t(lambda: A.device(dev))
dA1, out["A upload (second matrix)"] = t(lambda: A1.device(dev))
_, out["dia plan"] = t(lambda: dA1.dia())
Bd, out["B upload"] = t(lambda: D.to_device_block(B, dev, torch.float64))
Bd2, out["B upload (again)"] = t(lambda: D.to_device_block(B, dev, torch.float64))
_, out["X download"] = t(lambda: D.to_numpy_block(Bd))
_, out["X download (again)"] = t(lambda: D.to_numpy_block(Bd))
cfg = solver.SolverConfig(**dict(kw, max_cycles=1))
_, out["solve, 1 cycle (incl. uploads of a fresh matrix)"] = t(lambda: solver.solve_block_gcrodr(system(1), B, None, cfg))
_, out["_setup only"] = t(lambda: solver._setup(A1, B, None, cfg, None))
out = {k: round(v, 4) for k, v in out.items()}
out["bytes"] = {"A": int(A.nnz * 12 + (A.n_rows + 1) * 4), "B": int(B.nbytes)}
print(json.dumps(out, indent=1))
