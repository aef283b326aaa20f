"""B200-native hot path of block GCRO-DR (block recycled GMRES, arXiv 1604.01713).

Drop-in for the reference package ``recgmres`` (/root/reference/pkg/src/
recgmres/__init__.py:4-13): the same public names, backed by hand-written
sm_100a kernels in librgb200.so (CSR SpMM, fused tall-skinny Gram/update
passes on the FP64 tensor cores, CholQR2 + Householder TSQR) reached through
a C ABI (include/rgb200.h) via ctypes.  torch provides device memory and
streams only.  There is no CPU fallback: without a CUDA device the device
entry points raise ``NoDeviceError``.
"""

from .sparse_core import (CsrMatrix, MatrixMarketError, ShapeError, as_block, gen_banded, read_matrix_market,
                          spmm, spmv, write_matrix_market)
from .recycling import RecycleSpace, load_recycle_space, save_recycle_space
from .solver import (HostOperator, SolveReport, SolverConfig, enlarge_block, solve_block_gcrodr, solve_block_gmres,
                     solve_sequence)
from .device import NoDeviceError
from .precond import Ilu0Factors, ZeroPivotError, apply_precond, ilu0

__version__ = "0.1.0"

__all__ = [
    "CsrMatrix",
    "spmm",
    "spmv",
    "read_matrix_market",
    "write_matrix_market",
    "gen_banded",
    "as_block",
    "ShapeError",
    "MatrixMarketError",
    "RecycleSpace",
    "save_recycle_space",
    "load_recycle_space",
    "SolverConfig",
    "SolveReport",
    "solve_block_gmres",
    "solve_block_gcrodr",
    "solve_sequence",
    "enlarge_block",
    "HostOperator",
    "NoDeviceError",
    "Ilu0Factors",
    "ZeroPivotError",
    "ilu0",
    "apply_precond",
]
