"""Shared test setup: repo root on sys.path, the ``gpu`` marker, golden
fixture loading."""

import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")


def load_golden(name):
    return np.load(GOLDEN / name, allow_pickle=False)


def csr_from(d, prefix):
    """(row_ptr, col_idx, values, shape) of a golden CSR."""
    return (d[prefix + "row_ptr"], d[prefix + "col_idx"], d[prefix + "values"], tuple(d[prefix + "shape"]))


def csr_matrix_from(d, prefix):
    from paper_1604_01713_b200.sparse_core import CsrMatrix

    rp, ci, v, shape = csr_from(d, prefix)
    return CsrMatrix(shape[0], shape[1], rp, ci, v)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test needs a CUDA device (the B200 path has no CPU fallback)")
    return torch.device("cuda", 0)
