"""Time the device-side diagonal-layout build (sparse_core.DiaPlan) of the
config-4 operator at grid^3."""
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1604_01713_b200 import problems  # noqa: E402
from paper_1604_01713_b200.sparse_core import DiaPlan  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = problems.conv_diff_3d(N, 20.0)
dA = A.device(torch.device("cuda", 0))
torch.cuda.synchronize()
for i in range(3):
    t0 = time.perf_counter()
    plan = DiaPlan.build(dA)
    torch.cuda.synchronize()
    print(f"build {i}: {(time.perf_counter() - t0) * 1e3:.1f} ms, offsets {plan.offsets.tolist()}, "
          f"peak mem {torch.cuda.max_memory_allocated() / 1e9:.1f} GB")
