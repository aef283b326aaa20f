"""ILU(0) preconditioner on the device.

Drop-in for ``recgmres.precond`` (/root/reference/pkg/src/recgmres/
precond.py): ``ZeroPivotError``, ``Ilu0Factors``, ``ilu0`` and
``apply_precond`` with the reference's signatures, error classes and
messages.

* ``ilu0(A)`` runs rg_ilu0_f64: the IKJ sweep of precond.py:50-72 in place
  on a device copy of A's values, one lane per row, rows taken level by
  level from a host-built level schedule (rg_wave_schedule) in a sync-free
  wavefront (lanes wait on the completion flags of the rows they read).
  The factors are bitwise the reference's.  The diagonal-position scan and
  the missing-diagonal check (precond.py:43-50) are a vectorised host pass.
* ``apply_precond(F, X)`` = U^-1 (L^-1 X) with two rg_sptrsv_f64 wavefront
  solves on the combined LU pattern (replaces the two
  ``spsolve_triangular`` calls of precond.py:87-88; equal to them within
  rounding, not bitwise: SuperLU's solve scales by the inverse diagonal).

``Ilu0Factors.lower`` / ``.upper`` are the reference's host ``CsrMatrix``
factors (strict lower with implicit unit diagonal; upper with diagonal),
copied back from the device on first access.  Factors built from host
``CsrMatrix`` objects (the reference constructor) are assembled into the
device layout on first use.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib
from . import device as _dev
from .sparse_core import CsrMatrix, ShapeError, as_block


class ZeroPivotError(ArithmeticError):
    pass


_INT64_MAX = np.iinfo(np.int64).max
# RG_ILU_PERM=0 solves in the original row order (the A/B baseline of tools/prof_ilu.py)
_PERM = os.environ.get("RG_ILU_PERM", "1") != "0"
# rows per wavefront chunk (each lane of a warp takes chunk_rows / 32 rows of one level)
_CHUNK_ROWS = int(os.environ.get("RG_WAVE_CHUNK", "32"))


class _Schedule:
    """Level schedule of one triangle (rg_wave_schedule, host analysis)."""

    def __init__(self, rp_h, ci_h, dpos_h, upper: bool, device):
        L = _dev.lib()
        n = len(rp_h) - 1
        order = np.empty(max(n, 1), dtype=np.int32)
        chunk = np.empty(int(L.rg_wave_max_chunks(n)), dtype=np.int32)
        nl = np.zeros(1, dtype=np.int32)
        wd = np.zeros(1, dtype=np.int32)
        nc = L.rg_wave_schedule(n, rp_h.ctypes.data, ci_h.ctypes.data, dpos_h.ctypes.data, 1 if upper else 0,
                                _CHUNK_ROWS, order.ctypes.data, chunk.ctypes.data, nl.ctypes.data, wd.ctypes.data)
        if nc < 0:
            raise ValueError("rg_wave_schedule failed")
        self.nchunks = int(nc)
        self.levels = int(nl[0])
        self.width = int(wd[0])
        self.upper = upper
        self.order_h = order[:n]
        self.order = torch.from_numpy(order).to(device)
        self.chunk = torch.from_numpy(chunk[: nc + 1].copy()).to(device)
        self.perm = None

    def build_perm(self, rp_h, ci_h, dpos_h, lu_vals: torch.Tensor):
        """Level-ordered copy of this triangle (rg_wave_permute) with its
        values gathered from the factor on the device."""
        L = _dev.lib()
        n = len(rp_h) - 1
        dev = lu_vals.device
        nnz = len(ci_h)
        pos = np.empty(max(n, 1), dtype=np.int32)
        rp_o = np.empty(n + 1, dtype=np.int32)
        ci_o = np.empty(max(nnz, 1), dtype=np.int32)
        emap = np.empty(max(nnz, 1), dtype=np.int64)
        m = int(L.rg_wave_permute(n, rp_h.ctypes.data, ci_h.ctypes.data, dpos_h.ctypes.data, 1 if self.upper else 0,
                                  self.order_h.ctypes.data, pos.ctypes.data, rp_o.ctypes.data, ci_o.ctypes.data,
                                  emap.ctypes.data))
        d_emap = torch.from_numpy(emap[:max(m, 1)].copy()).to(dev)
        vals = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
        _lib.check(L.rg_gather_f64(m, d_emap.data_ptr(), lu_vals.data_ptr(), vals.data_ptr(), _dev.stream_ptr()),
                   "gather")
        dval = None
        if self.upper:
            didx = torch.from_numpy(dpos_h[self.order_h].astype(np.int64)).to(dev)
            dval = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
            _lib.check(L.rg_gather_f64(n, didx.data_ptr(), lu_vals.data_ptr(), dval.data_ptr(), _dev.stream_ptr()),
                       "gather")
        self.perm = dict(pos=torch.from_numpy(pos).to(dev), rp=torch.from_numpy(rp_o).to(dev),
                         ci=torch.from_numpy(ci_o[:max(m, 1)].copy()).to(dev), vals=vals, dval=dval)


class _DeviceLu:
    """Combined L\\U values on A's pattern, resident in HBM, the lower and
    upper level schedules, and the wave workspace (row flags) with its epoch
    counter."""

    def __init__(self, n, rp_h, ci_h, dpos_h, row_ptr, col_idx, vals, device):
        self.n = n
        self.device = device
        self.row_ptr = row_ptr
        self.col_idx = col_idx
        self.vals = vals
        rp_h = np.ascontiguousarray(rp_h, dtype=np.int32)
        ci_h = np.ascontiguousarray(ci_h, dtype=np.int32)
        dpos_h = np.ascontiguousarray(np.maximum(dpos_h, 0), dtype=np.int32)
        self.dpos = torch.from_numpy(dpos_h).to(device)
        self.lower_sched = _Schedule(rp_h, ci_h, dpos_h, False, device)
        self.upper_sched = _Schedule(rp_h, ci_h, dpos_h, True, device)
        self._host_pattern = (rp_h, ci_h, dpos_h)
        self._ws = {}
        L = _dev.lib()
        self.work = torch.zeros(int(L.rg_wave_workspace_bytes(n)), dtype=torch.uint8, device=device)
        self.epoch = 0
        self.singular = False

    def next_epoch(self) -> int:
        self.epoch += 1
        if self.epoch >= 2**31 - 1:  # wrap: clear the flags once
            self.work.zero_()
            self.epoch = 1
        return self.epoch

    def factor(self, zero_row: torch.Tensor) -> None:
        L = _dev.lib()
        sc = self.lower_sched
        rc = L.rg_ilu0_f64(self.n, self.row_ptr.data_ptr(), self.col_idx.data_ptr(), self.vals.data_ptr(),
                           self.dpos.data_ptr(), sc.order.data_ptr(), sc.chunk.data_ptr(), sc.nchunks, sc.width,
                           zero_row.data_ptr(), self.work.data_ptr(), self.work.numel(), self.next_epoch(),
                           _dev.stream_ptr())
        _lib.check(rc, "ilu0")

    def _permuted(self):
        if self.lower_sched.perm is None:
            rp_h, ci_h, dpos_h = self._host_pattern
            self.lower_sched.build_perm(rp_h, ci_h, dpos_h, self.vals)
            self.upper_sched.build_perm(rp_h, ci_h, dpos_h, self.vals)
        return self.lower_sched, self.upper_sched

    def apply(self, B: torch.Tensor, out: torch.Tensor) -> None:
        """out = U^-1 (L^-1 B) through the level-ordered row-major layout:
        scatter B into L's order, solve, re-order into U's, solve, gather back."""
        L = _dev.lib()
        n, p = B.shape
        ls, us = self._permuted()
        key = p
        if key not in self._ws:
            self._ws[key] = (torch.empty(max(n * p, 1), dtype=torch.float64, device=self.device),
                             torch.empty(max(n * p, 1), dtype=torch.float64, device=self.device))
        w1, w2 = self._ws[key]
        st = _dev.stream_ptr()
        lp, up = ls.perm, us.perm

        def perm(src, lds, ps, dst, ldd, pd):
            _lib.check(L.rg_permute_rows_f64(n, p, src.data_ptr(), lds, ps.data_ptr() if ps is not None else None,
                                             dst.data_ptr(), ldd, pd.data_ptr() if pd is not None else None, st),
                       "permute_rows")

        def solve(sc, pm, w):
            rc = L.rg_sptrsv_perm_f64(n, pm["rp"].data_ptr(), pm["ci"].data_ptr(), pm["vals"].data_ptr(),
                                      pm["dval"].data_ptr() if pm["dval"] is not None else None,
                                      sc.chunk.data_ptr(), sc.nchunks, sc.width, p, w.data_ptr(),
                                      self.work.data_ptr(), self.work.numel(), self.next_epoch(), st)
            _lib.check(rc, "sptrsv_perm")

        perm(B, _dev.ld_of(B), None, w1, 0, lp["pos"])
        solve(ls, lp, w1)
        perm(w1, 0, lp["pos"], w2, 0, up["pos"])
        solve(us, up, w2)
        perm(w2, 0, up["pos"], out, _dev.ld_of(out), None)

    def solve(self, B: torch.Tensor, X: torch.Tensor, upper: bool) -> None:
        L = _dev.lib()
        sc = self.upper_sched if upper else self.lower_sched
        for c0 in range(0, B.shape[1], 64):
            c1 = min(B.shape[1], c0 + 64)
            b, x = B[:, c0:c1], X[:, c0:c1]
            rc = L.rg_sptrsv_f64(self.n, self.row_ptr.data_ptr(), self.col_idx.data_ptr(), self.vals.data_ptr(),
                                 self.dpos.data_ptr(), sc.order.data_ptr(), sc.chunk.data_ptr(), sc.nchunks,
                                 sc.width, 1 if upper else 0, c1 - c0, b.data_ptr(), _dev.ld_of(b), x.data_ptr(),
                                 _dev.ld_of(x), self.work.data_ptr(), self.work.numel(), self.next_epoch(),
                                 _dev.stream_ptr())
            _lib.check(rc, "sptrsv")


def _diag_positions(n, rp, ci):
    """Storage position of each row's diagonal, or -1 (precond.py:43-48)."""
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    hit = np.flatnonzero(ci == rows)
    dpos = np.full(n, -1, dtype=np.int64)
    dpos[rows[hit]] = hit
    return dpos


class Ilu0Factors:
    """Unit lower / upper triangular factors sharing the sparsity pattern of
    the input matrix (precond.py:19-30).  The unit diagonal of ``lower`` is
    implicit: it is not stored."""

    def __init__(self, lower: CsrMatrix | None = None, upper: CsrMatrix | None = None, *, _lu: _DeviceLu | None = None):
        if _lu is None and (lower is None or upper is None):
            raise TypeError("Ilu0Factors needs lower and upper factors")
        self._lower = lower
        self._upper = upper
        self._lu = _lu

    @property
    def n(self) -> int:
        return self._lu.n if self._lu is not None else self._lower.n_rows

    # ---- host views (reference fields)
    def _split(self):
        lu = self._lu
        rp = lu.row_ptr.cpu().numpy().astype(np.int64)
        ci = lu.col_idx.cpu().numpy()
        v = lu.vals.cpu().numpy()
        rows = np.repeat(np.arange(lu.n, dtype=np.int64), np.diff(rp))
        low = ci < rows

        def part(mask):
            counts = np.bincount(rows[mask], minlength=lu.n)
            prp = np.zeros(lu.n + 1, dtype=np.int64)
            np.cumsum(counts, out=prp[1:])
            return CsrMatrix(lu.n, lu.n, prp.astype(np.int32), ci[mask].astype(np.int32), v[mask].copy(),
                             _validated=True)

        self._lower, self._upper = part(low), part(~low)

    @property
    def lower(self) -> CsrMatrix:
        if self._lower is None:
            self._split()
        return self._lower

    @property
    def upper(self) -> CsrMatrix:
        if self._upper is None:
            self._split()
        return self._upper

    # ---- device layout
    def device_lu(self, device=None) -> _DeviceLu:
        dev = _dev.require_cuda(device)
        if self._lu is not None and self._lu.device == dev:
            return self._lu
        lo, up = self.lower, self.upper
        n = lo.n_rows
        if lo.n_cols != n or up.n_rows != n or up.n_cols != n:
            raise ShapeError("ILU factors must be square and of equal size")
        lrp, urp = np.asarray(lo.row_ptr, np.int64), np.asarray(up.row_ptr, np.int64)
        counts = np.diff(lrp) + np.diff(urp)
        rp = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=rp[1:])
        ci = np.empty(rp[-1], dtype=np.int32)
        v = np.empty(rp[-1], dtype=np.float64)
        # row i = its lower entries then its upper entries (both sorted, disjoint column ranges)
        lrow = np.repeat(np.arange(n), np.diff(lrp))
        urow = np.repeat(np.arange(n), np.diff(urp))
        lpos = rp[lrow] + (np.arange(len(lrow)) - lrp[lrow])
        upos = rp[urow] + np.diff(lrp)[urow] + (np.arange(len(urow)) - urp[urow])
        ci[lpos], v[lpos] = lo.col_idx, lo.values
        ci[upos], v[upos] = up.col_idx, up.values
        dpos = _diag_positions(n, rp, ci)
        lu = _DeviceLu(n, rp, ci, dpos, torch.from_numpy(rp.astype(np.int32)).to(dev), torch.from_numpy(ci).to(dev),
                       torch.from_numpy(v).to(dev), dev)
        # spsolve_triangular rejects a zero (or absent) diagonal of U
        lu.singular = bool(np.any(dpos < 0) or np.any(v[np.maximum(dpos, 0)] == 0.0))
        self._lu = lu
        return lu


def ilu0(A: CsrMatrix, device=None) -> Ilu0Factors:
    """Incomplete LU with zero fill-in (precond.py:33-76), on the device.

    For matrices whose exact LU incurs no fill, the factors equal the exact
    LU.  No pivoting is performed; a zero pivot raises, naming the row."""
    n = A.n_rows
    if A.n_cols != n:
        raise ShapeError("ilu0 needs a square matrix")
    if np.iscomplexobj(A.values):
        raise TypeError("ilu0 supports real matrices (the reference's precond.py is float64)")
    rp = np.asarray(A.row_ptr, dtype=np.int64)
    ci = np.asarray(A.col_idx)
    dpos = _diag_positions(n, rp, ci)
    if np.any(dpos < 0):
        missing = int(np.nonzero(dpos < 0)[0][0])
        raise ZeroPivotError(f"row {missing}: no stored diagonal entry")
    dev = _dev.require_cuda(device)
    dA = A.device(dev)
    vals = dA.values.clone()
    lu = _DeviceLu(n, rp, ci, dpos, dA.row_ptr, dA.col_idx, vals, dev)
    zero = torch.full((1,), _INT64_MAX, dtype=torch.int64, device=dev)
    lu.factor(zero)
    z = int(zero.item())
    if z != _INT64_MAX:
        raise ZeroPivotError(f"row {z}: zero pivot in ILU(0)")
    return Ilu0Factors(_lu=lu)


def apply_precond_device(F: Ilu0Factors, X: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """out = U^-1 (L^-1 X) for a column-major CUDA block (out may be X)."""
    if X.shape[0] != F.n:
        raise ShapeError(f"block has {X.shape[0]} rows, factors are {F.n}-dimensional")
    lu = F.device_lu(X.device)
    if lu.singular:
        raise np.linalg.LinAlgError("A is singular: zero entry on diagonal.")
    if out is None:
        out = _dev.empty_block(X.shape[0], X.shape[1], X.device, X.dtype)
    if X.shape[1] == 0 or F.n == 0:
        return out
    if _PERM:
        lu.apply(X, out)
    else:
        lu.solve(X, out, upper=False)
        lu.solve(out, out, upper=True)
    return out


def apply_precond(F: Ilu0Factors, X):
    """Return U^{-1} (L^{-1} X) via two sparse triangular block solves
    (precond.py:79-90).  A numpy block returns a Fortran-ordered numpy array;
    a CUDA tensor returns a CUDA tensor."""
    if isinstance(X, torch.Tensor):
        Xd = _dev.to_device_block(X if X.dim() == 2 else X.reshape(-1, 1))
        return apply_precond_device(F, Xd)
    Xh = as_block(X)
    if Xh.shape[0] != F.n:
        raise ShapeError(f"block has {Xh.shape[0]} rows, factors are {F.n}-dimensional")
    Y = apply_precond_device(F, _dev.to_device_block(Xh))
    return _dev.to_numpy_block(Y)
