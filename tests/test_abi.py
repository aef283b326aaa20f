"""The C-ABI library loads without a GPU and exports every entry point
include/rgb200.h declares (no compute calls)."""

import ctypes
import re

from conftest import ROOT


def _declared():
    text = (ROOT / "include" / "rgb200.h").read_text()
    return sorted(set(re.findall(r"\b(rg_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    from paper_1604_01713_b200 import _lib

    lib = _lib.load()
    declared = _declared()
    assert declared, "no declarations parsed"
    missing = [s for s in declared if getattr(lib, s, None) is None]
    assert not missing, f"librgb200.so lacks {missing}"
    assert all(s in _lib.PROTOTYPES for s in declared), "ctypes prototypes out of sync with the header"


def test_version_and_error_calls_work_without_gpu():
    from paper_1604_01713_b200 import _lib

    lib = _lib.load()
    assert lib.rg_version().startswith(b"rgb200")
    assert isinstance(lib.rg_last_error(), bytes)


def test_argument_validation_without_gpu():
    """Bad shapes are rejected before any launch (status 1, message set)."""
    from paper_1604_01713_b200 import _lib

    lib = _lib.load()
    rc = lib.rg_spmm_csr_f64(10, 0, 11, None, None, None, None, 10, 10, None, 1, 2, None, 10, None)
    assert rc == _lib.RG_EBADARG
    assert b"row range" in lib.rg_last_error()
    rc = lib.rg_tall_f64(10, 40, None, 10, None, 10, None, 1, 0, None, 0.0, None, 1, 0, None, 0.0,
                         None, None, 0, None, 1, 0, None, None, 0, None)
    assert rc == _lib.RG_EBADARG
    rc = lib.rg_tsqr_f64(3, 5, None, 3, None, None, 0, None)
    assert rc == _lib.RG_EBADARG and b"n >= p" in lib.rg_last_error()


def test_product_fails_loudly_without_cuda():
    import numpy as np
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_1604_01713_b200 import CsrMatrix, NoDeviceError, spmm

    A = CsrMatrix.from_coo(2, 2, [0, 1], [0, 1], [1.0, 2.0])
    with pytest.raises(NoDeviceError):
        spmm(A, np.ones((2, 1)))
