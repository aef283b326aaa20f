"""Time rg_spmm on the config-2 (128^3 Laplacian) and config-4 (256^3 conv-diff) operators."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1604_01713_b200 import device as D, problems
from paper_1604_01713_b200.sparse_core import spmm_device
for name, A in (("cfg2 lap 128^3", problems.laplacian_3d(128)), ("cfg4 cd 256^3", problems.conv_diff_3d(256, 20.0))):
    for p in (1, 2, 4, 8, 16):
        X = D.empty_block(A.n_rows, p); X.normal_()
        Y = D.empty_block(A.n_rows, p)
        for _ in range(2): spmm_device(A, X, Y)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): spmm_device(A, X, Y)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        b = A.nnz * 12 + (A.n_rows + 1) * 4 + 16 * p * A.n_rows
        print(f"{name} p={p:2d}: {ms*1e3:8.1f} us  {b/ms/1e6:7.0f} GB/s")
