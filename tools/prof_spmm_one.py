"""One SpMM launch for ncu: cfg4 operator (256^3 conv-diff), p columns."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1604_01713_b200 import device as D, problems
from paper_1604_01713_b200.sparse_core import spmm_device
p = int(sys.argv[1]) if len(sys.argv) > 1 else 8
N = int(sys.argv[2]) if len(sys.argv) > 2 else 256
A = problems.conv_diff_3d(N, 20.0)
X = D.empty_block(A.n_rows, p); X.normal_()
Y = D.empty_block(A.n_rows, p)
spmm_device(A, X, Y); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
spmm_device(A, X, Y)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
