"""ORACLE — CPU restatement of the reference hot path.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / the timed CPU baseline.  The product package
``paper_1604_01713_b200`` never imports it and has no CPU fallback.

What it restates (reference = /root/reference/pkg/src/recgmres):

* ``spmm``            sparse_core.py:25-40, :132-149  (C, no FMA, ascending
                      storage order -> bitwise equal to the numba kernel)
* ``reduced_qr``      dense_kernels.py:31-48  (LAPACK Householder via numpy,
                      r_jj >= 0 sign fix, rank flags)
* ``cgs2_project``    arnoldi.py:171-180  (two passes, C first then the basis)
* ``mgs_project``     arnoldi.py:159-170  (one C column at a time, then one
                      basis block at a time)
* ``arnoldi_step``    arnoldi.py:139-193  (SpMM + CGS2 + QR; breakdown repair
                      omitted: the timed / checked inputs are full rank)
* ``gram``/``update`` the numpy ``@`` products of arnoldi.py / solver.py
* ``ilu0``            precond.py:33-76  (C, IKJ on the pattern, separately
                      rounded -> bitwise equal to the reference's factors)
* ``apply_precond``   precond.py:79-90  (textbook substitution; the reference
                      uses SuperLU, so equal within rounding only)

Parity pinning: tests/test_oracle_golden.py checks every function here
against golden vectors produced by running the real reference package
(tests/golden/make_golden.py, which imports /root/reference in the build
container and commits the outputs as .npz fixtures).
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liboracle.so"
_lib = None


def build() -> pathlib.Path:
    """Compile the C restatement (make -C oracle)."""
    subprocess.run(["make", "-C", str(_HERE)], check=True, capture_output=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        lib = ctypes.CDLL(str(_LIB_PATH))
        for name in ("oracle_spmm_f64", "oracle_spmm_c128"):
            fn = getattr(lib, name)
            fn.restype = None
            fn.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                           ctypes.c_int64, ctypes.c_int32]
        lib.oracle_ilu0_f64.restype = ctypes.c_int64
        lib.oracle_ilu0_f64.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 5
        lib.oracle_trsv_f64.restype = None
        lib.oracle_trsv_f64.argtypes = ([ctypes.c_int64] + [ctypes.c_void_p] * 4 + [ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64])
        _lib = lib
    return _lib


def host_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def spmm(row_ptr, col_idx, values, X, nthreads: int | None = None) -> np.ndarray:
    """Y = A @ X with the reference kernel's exact operation order.

    ``X`` is an (n_cols, p) block (any layout; converted to Fortran order,
    as ``as_block`` does at sparse_core.py:51-58).  Complex values/blocks use
    the complex restatement (each partial product and sum rounded
    separately)."""
    lib = _load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    cplx = np.iscomplexobj(values) or np.iscomplexobj(X)
    dt = np.complex128 if cplx else np.float64
    v = np.ascontiguousarray(values, dtype=dt)
    X = np.asarray(X, dtype=dt)
    if X.ndim == 1:
        X = X.reshape(-1, 1)
    X = np.asfortranarray(X)
    n = rp.shape[0] - 1
    p = X.shape[1]
    Y = np.zeros((n, p), dtype=dt, order="F")
    if n == 0 or p == 0:
        return Y
    fn = lib.oracle_spmm_c128 if cplx else lib.oracle_spmm_f64
    fn(n, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, X.ctypes.data, X.shape[0], p,
       Y.ctypes.data, n, int(nthreads or host_threads()))
    return Y


def reduced_qr(X, rank_tol: float = 1e-12):
    """(q, r, flagged) as dense_kernels.reduced_qr (dense_kernels.py:31-48)."""
    X = np.atleast_2d(np.asarray(X))
    n, L = X.shape
    if n < L:
        raise ValueError(f"reduced_qr needs n >= L, got {n} < {L}")
    q, r = np.linalg.qr(X, mode="reduced")
    d = np.real(np.diagonal(r)).copy()
    if np.iscomplexobj(r):
        # complex restatement: phase normalisation so that r_jj is real >= 0
        ph = np.diagonal(r) / np.where(np.abs(np.diagonal(r)) == 0, 1, np.abs(np.diagonal(r)))
        ph = np.where(np.abs(np.diagonal(r)) == 0, 1.0, ph)
        q = q * ph
        r = r * np.conj(ph)[:, None]
    else:
        s = np.where(d < 0.0, -1.0, 1.0)
        q = q * s
        r = r * s[:, None]
    normx = np.linalg.norm(X)
    flagged = np.abs(np.diagonal(r)) <= rank_tol * max(normx, np.finfo(float).tiny)
    return np.asfortranarray(q), r, flagged


def gram(X, Y):
    """X^H @ Y (numpy/OpenBLAS, as arnoldi.py:175,178)."""
    return np.conj(X).T @ Y


def update(Y, X, S, alpha=-1.0):
    """Y + alpha * (X @ S) with the product formed first (as ``Y -= X @ S``)."""
    return Y + alpha * (X @ S)


def cgs2_project(Ahat, C, W):
    """Two CGS passes of arnoldi.py:172-180 (C first, then the basis W).

    Returns (Ahat_projected, F_cols, H_cols) where F_cols / H_cols are the
    accumulated coefficients the reference adds into _F and _H."""
    Ahat = np.array(Ahat, order="F", copy=True)
    k = 0 if C is None else C.shape[1]
    F = np.zeros((k, Ahat.shape[1]), dtype=Ahat.dtype)
    H = np.zeros((W.shape[1], Ahat.shape[1]), dtype=Ahat.dtype)
    for _ in range(2):
        if C is not None:
            S = gram(C, Ahat)
            Ahat -= C @ S
            F += S
        coef = gram(W, Ahat)
        Ahat -= W @ coef
        H += coef
    return Ahat, F, H


def mgs_project(Ahat, C, W, L):
    """Block modified Gram-Schmidt of arnoldi.py:159-170: each column c_i of
    C (coef = c_i^T Ahat; Ahat -= c_i coef), then each basis block V_i of
    the L-column blocks of W.  Returns (Ahat_projected, F_cols, H_cols)."""
    Ahat = np.array(Ahat, order="F", copy=True)
    k = 0 if C is None else C.shape[1]
    F = np.zeros((k, Ahat.shape[1]), dtype=Ahat.dtype)
    H = np.zeros((W.shape[1], Ahat.shape[1]), dtype=Ahat.dtype)
    for i in range(k):
        ci = C[:, i]
        coef = np.conj(ci) @ Ahat
        Ahat -= np.outer(ci, coef)
        F[i] += coef
    for i in range(W.shape[1] // L):
        Vi = W[:, i * L:(i + 1) * L]
        Hblk = np.conj(Vi).T @ Ahat
        Ahat -= Vi @ Hblk
        H[i * L:(i + 1) * L] += Hblk
    return Ahat, F, H


def arnoldi_step(row_ptr, col_idx, values, Vm, C, W, rank_tol: float = 1e-12, nthreads=None):
    """One CGS2 block Arnoldi step (arnoldi.py:139-193): returns
    (V_new, F_cols, H_cols, R_new, flagged)."""
    Ahat = spmm(row_ptr, col_idx, values, Vm, nthreads)
    Ahat, F, H = cgs2_project(Ahat, C, W)
    q, r, flagged = reduced_qr(Ahat, rank_tol)
    return q, F, H, r, flagged


# ---------------------------------------------------------------------------
# algorithmic byte counts (the reference's own SpMM model is
# bench.py:44-47)
# ---------------------------------------------------------------------------


def spmm_bytes(n_rows: int, nnz: int, p: int, elem: int = 8) -> int:
    return nnz * (elem + 4) + (n_rows + 1) * 4 + 2 * p * n_rows * elem


# ---------------------------------------------------------------------------
# ILU(0) (precond.py)
# ---------------------------------------------------------------------------


class OracleZeroPivot(ArithmeticError):
    pass


def _diag_pos(rp, ci):
    n = rp.shape[0] - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    hit = np.flatnonzero(ci == rows)
    d = np.full(n, -1, dtype=np.int64)
    d[rows[hit]] = hit
    return d


def ilu0(row_ptr, col_idx, values):
    """(lu_values, diag_pos): combined L\\U values on A's pattern, as the
    reference's ``vals`` after precond.py:60-72.  Raises OracleZeroPivot with
    the reference's message."""
    lib = _load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    v = np.array(values, dtype=np.float64, copy=True)
    n = rp.shape[0] - 1
    d = _diag_pos(rp, ci)
    if np.any(d < 0):
        raise OracleZeroPivot(f"row {int(np.nonzero(d < 0)[0][0])}: no stored diagonal entry")
    scratch = np.full(max(n, 1), -1, dtype=np.int64)
    bad = lib.oracle_ilu0_f64(n, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, d.ctypes.data, scratch.ctypes.data)
    if bad >= 0:
        raise OracleZeroPivot(f"row {bad}: zero pivot in ILU(0)")
    return v, d


def apply_precond(row_ptr, col_idx, lu_values, diag_pos, X):
    """U^-1 (L^-1 X) on the combined pattern (textbook substitution)."""
    lib = _load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    v = np.ascontiguousarray(lu_values, dtype=np.float64)
    d = np.ascontiguousarray(diag_pos, dtype=np.int64)
    X = np.asfortranarray(np.asarray(X, dtype=np.float64).reshape(len(X), -1))
    n, p = X.shape
    Z = np.zeros_like(X, order="F")
    Y = np.zeros_like(X, order="F")
    lib.oracle_trsv_f64(n, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, d.ctypes.data, 0, p, X.ctypes.data, n,
                        Z.ctypes.data, n)
    lib.oracle_trsv_f64(n, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, d.ctypes.data, 1, p, Z.ctypes.data, n,
                        Y.ctypes.data, n)
    return Y
