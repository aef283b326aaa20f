"""Sparse storage and the sparse-times-block product on the B200.

Drop-in for ``recgmres.sparse_core`` (/root/reference/pkg/src/recgmres/
sparse_core.py): same names, same argument meaning, same exceptions.

* ``CsrMatrix`` (sparse_core.py:61-129): immutable host CSR with the same
  validation rules; the per-row Python loop of the reference (:86-89, 15 s
  at n = 2.1M) is replaced by one vectorised pass.  ``device()`` uploads the
  arrays once (int32 indices, float64 values) and caches the device copy.
* ``spmm`` / ``spmv`` (sparse_core.py:132-157): run the rg_spmm_csr_f64
  kernel; numpy in -> numpy out (host<->device copies included), CUDA tensor
  in -> CUDA tensor out.  Bitwise identical to the reference kernel.
* ``as_block`` (sparse_core.py:51-58) keeps its host semantics.
* Matrix Market I/O and ``gen_banded`` are host utilities (sparse_core.py
  :160-287) reproduced with the same formats and seeded streams.
"""

from __future__ import annotations

import weakref

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from . import device as _dev


class ShapeError(ValueError):
    """Incompatible operand shapes."""


class MatrixMarketError(ValueError):
    """Malformed Matrix Market input; message names the offending line."""


def as_block(x) -> np.ndarray:
    """Host: 2-D float64 array with contiguous columns (sparse_core.py:51-58)."""
    a = np.asarray(x, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    if a.ndim != 2:
        raise ShapeError(f"expected a vector or 2-D block, got ndim={a.ndim}")
    return np.asfortranarray(a)


def as_device_block(x, device=None) -> torch.Tensor:
    """Device: column-major CUDA float64 tensor (zero-copy when already one)."""
    if isinstance(x, torch.Tensor):
        if x.dim() == 1:
            x = x.reshape(-1, 1)
        if x.dim() != 2:
            raise ShapeError(f"expected a vector or 2-D block, got ndim={x.dim()}")
        return _dev.to_device_block(x, device)
    return _dev.to_device_block(as_block(x), device)


# (id(row_ptr), id(col_idx), device) -> (weakrefs to the host arrays, device copies)
_STRUCT_CACHE: dict = {}


class DeviceCsr:
    """CSR arrays resident in HBM: int32 row_ptr (n+1), int32 col_idx and
    float64 values (nnz), in the host matrix's storage order."""

    __slots__ = ("n_rows", "n_cols", "nnz", "row_ptr", "col_idx", "values", "device", "host_row_ptr", "_dia",
                 "dia_rows")

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, values, device):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.device = device
        self.row_ptr = row_ptr
        self.col_idx = col_idx
        self.values = values
        self.nnz = int(values.shape[0])
        self.host_row_ptr = None
        self._dia = False  # not yet analysed; None: not a diagonal matrix
        # rows the diagonal layout covers (None: all).  A row-partitioned operator
        # sets its interior range: only those rows reference owned columns alone
        self.dia_rows = None

    def dia(self):
        """The diagonal layout of this matrix (``DiaPlan``), built on the
        device on first use, or None when its nonzeros do not lie on a few
        well-filled diagonals (the CSR kernel then runs)."""
        if self._dia is False:
            r0, r1 = self.dia_rows if self.dia_rows is not None else (0, self.n_rows)
            self._dia = DiaPlan.build(self, int(r0), int(r1))
        return self._dia


    @classmethod
    def from_host(cls, n_rows, n_cols, row_ptr, col_idx, values, device=None):
        dev = _dev.require_cuda(device)
        if len(values) >= 2**31:
            raise ValueError("nnz >= 2^31 needs 64-bit indices (not supported)")
        # matrices of a sequence share their structure arrays (A_i = A + diag):
        # the device copies of row_ptr / col_idx are shared too
        key = (id(row_ptr), id(col_idx), str(dev))
        hit = _STRUCT_CACHE.get(key)
        if hit is not None and hit[0]() is row_ptr and hit[1]() is col_idx:
            rp, ci = hit[2], hit[3]
        else:
            rp = _dev.upload_array(np.ascontiguousarray(row_ptr, dtype=np.int32), dev)
            ci = _dev.upload_array(np.ascontiguousarray(col_idx, dtype=np.int32), dev)
            if isinstance(row_ptr, np.ndarray) and isinstance(col_idx, np.ndarray):
                if len(_STRUCT_CACHE) >= 4:
                    _STRUCT_CACHE.pop(next(iter(_STRUCT_CACHE)))
                _STRUCT_CACHE[key] = (weakref.ref(row_ptr), weakref.ref(col_idx), rp, ci)
        cplx = np.iscomplexobj(values)
        v = _dev.upload_array(np.ascontiguousarray(values, dtype=np.complex128 if cplx else np.float64), dev)
        out = cls(n_rows, n_cols, rp, ci, v, dev)
        out.host_row_ptr = np.asarray(row_ptr)
        return out


class DiaPlan:
    """Diagonal layout of a DeviceCsr for rg_spmm_dia_f64 (the stencil
    matrices of BASELINE configs[0]-[3]): ascending offsets (host int32), the
    values as an n_rows x ndiag column-major block (zero where a row stores no
    entry on that diagonal) and per-row bit masks of the stored entries.
    Summing each row's masked entries in ascending offset order is the CSR
    row's ascending column order, so the product stays bitwise the
    reference's."""

    MAX_DIAG = 32
    MAX_FILL = 1.25  # ndiag * n_rows <= MAX_FILL * nnz

    __slots__ = ("offsets", "dia", "mask", "rows")

    def __init__(self, offsets, dia, mask, rows):
        self.offsets, self.dia, self.mask, self.rows = offsets, dia, mask, rows

    def covers(self, row_begin: int, row_end: int) -> bool:
        return self.rows[0] <= row_begin and row_end <= self.rows[1]

    @classmethod
    def build(cls, A: "DeviceCsr", r0: int = 0, r1: int | None = None):
        r1 = A.n_rows if r1 is None else r1
        if A.values.dtype != torch.float64 or A.nnz == 0 or r1 <= r0:
            return None
        dev = A.device
        L, st = _dev.lib(), _dev.stream_ptr()
        # pass 1 (rg_dia_offsets): the distinct offsets col - row, in a 64-slot table
        empty = np.iinfo(np.int32).min
        table = torch.full((64,), empty, dtype=torch.int32, device=dev)
        over = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.check(L.rg_dia_offsets(A.n_rows, r0, r1, A.row_ptr.data_ptr(), A.col_idx.data_ptr(), table.data_ptr(),
                                    over.data_ptr(), st), "dia offsets")
        tab = torch.cat([table, over]).cpu().numpy()
        if tab[64]:
            return None
        offsets = np.sort(tab[:64][tab[:64] != empty]).astype(np.int32)
        nd = int(offsets.size)
        if nd == 0 or nd > cls.MAX_DIAG or nd * A.n_rows > cls.MAX_FILL * A.nnz:
            return None
        # pass 2 (rg_dia_fill_f64): values and per-row masks
        dia = _dev.zeros_block(A.n_rows, nd, dev)
        mask = torch.zeros(_dev.round_ld(A.n_rows), dtype=torch.int32, device=dev)
        offs_dev = torch.from_numpy(offsets).to(dev)
        _lib.check(L.rg_dia_fill_f64(A.n_rows, r0, r1, A.row_ptr.data_ptr(), A.col_idx.data_ptr(),
                                     A.values.data_ptr(), nd, offs_dev.data_ptr(), dia.data_ptr(), _dev.ld_of(dia),
                                     mask.data_ptr(), st), "dia fill")
        return cls(offsets, dia, mask, (r0, r1))


def _validate(n_rows, n_cols, rp, ci, v):
    if rp.shape != (n_rows + 1,):
        raise ValueError("row_ptr must have length n_rows+1")
    if rp[0] != 0 or rp[-1] != len(ci) or np.any(np.diff(rp) < 0):
        raise ValueError("row_ptr must be nondecreasing with row_ptr[0]=0")
    if len(ci) != len(v):
        raise ValueError("col_idx and values length mismatch")
    if len(ci) and (ci.min() < 0 or ci.max() >= n_cols):
        raise ValueError("column index out of range")
    if len(ci) > 1:
        step = np.diff(ci.astype(np.int64))
        bad = step <= 0
        # a step across a row boundary is not a violation
        starts = np.asarray(rp[1:-1], dtype=np.int64)
        starts = starts[(starts > 0) & (starts < len(ci))]
        bad[starts - 1] = False
        if bad.any():
            t = int(np.argmax(bad)) + 1
            row = int(np.searchsorted(rp, t, side="right") - 1)
            raise ValueError(f"row {row}: column indices not strictly increasing")


class CsrMatrix:
    """Sparse matrix in compressed-sparse-row form (sparse_core.py:61-129).

    Rows are sorted by column index with no duplicates; instances are
    immutable after construction.  ``device()`` returns the cached HBM copy
    the kernels read."""

    __slots__ = ("n_rows", "n_cols", "row_ptr", "col_idx", "values", "_scipy", "_device")

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, values, _scipy=None, *, _validated=False):
        rp = np.asarray(row_ptr)
        ci = np.asarray(col_idx)
        v = np.asarray(values)
        if not _validated:
            _validate(int(n_rows), int(n_cols), rp, ci, v)
        object.__setattr__(self, "n_rows", int(n_rows))
        object.__setattr__(self, "n_cols", int(n_cols))
        object.__setattr__(self, "row_ptr", rp)
        object.__setattr__(self, "col_idx", ci)
        object.__setattr__(self, "values", v)
        object.__setattr__(self, "_scipy", _scipy)
        object.__setattr__(self, "_device", None)

    def __setattr__(self, name, value):
        raise AttributeError("CsrMatrix is immutable")

    def __repr__(self):
        return f"CsrMatrix(n_rows={self.n_rows}, n_cols={self.n_cols}, nnz={self.nnz})"

    @classmethod
    def from_coo(cls, n_rows, n_cols, rows, cols, vals) -> "CsrMatrix":
        v = np.asarray(vals)
        v = v.astype(np.complex128 if np.iscomplexobj(v) else np.float64)  # complex kept (config 5 extension)
        m = sp.coo_matrix((v, (rows, cols)), shape=(n_rows, n_cols)).tocsr()
        m.sort_indices()
        return cls.from_scipy(m)

    @classmethod
    def from_scipy(cls, m) -> "CsrMatrix":
        m = sp.csr_matrix(m)
        m.sort_indices()
        data = np.asarray(m.data, dtype=np.complex128 if np.iscomplexobj(m.data) else np.float64)
        return cls(m.shape[0], m.shape[1], m.indptr.copy(), m.indices.copy(), data.copy())

    def astype_complex(self) -> "CsrMatrix":
        """The same pattern with complex128 values (real matrix, complex blocks)."""
        return CsrMatrix(self.n_rows, self.n_cols, self.row_ptr, self.col_idx,
                         self.values.astype(np.complex128), _validated=True)

    @property
    def nnz(self) -> int:
        return len(self.values)

    def to_scipy(self) -> sp.csr_matrix:
        if self._scipy is None:
            object.__setattr__(self, "_scipy", sp.csr_matrix(
                (self.values, self.col_idx, self.row_ptr), shape=(self.n_rows, self.n_cols)))
        return self._scipy

    def frobenius_norm(self) -> float:
        return float(np.linalg.norm(self.values))

    def diagonal(self) -> np.ndarray:
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
        d = np.zeros(min(self.n_rows, self.n_cols), dtype=self.values.dtype)
        on = self.col_idx == rows
        d[rows[on]] = self.values[on]
        return d

    def device(self, device=None) -> DeviceCsr:
        """Upload once; later calls return the cached HBM copy."""
        dev = _dev.require_cuda(device)
        cached = self._device
        if cached is None or cached.device != dev:
            cached = DeviceCsr.from_host(self.n_rows, self.n_cols, self.row_ptr, self.col_idx, self.values, dev)
            object.__setattr__(self, "_device", cached)
        return cached


def spmm_device(A, X: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Y = A @ X with X a column-major CUDA block; returns (or fills) Y."""
    dA = A.device(X.device) if isinstance(A, CsrMatrix) else A
    if dA.n_cols != X.shape[0]:
        raise ShapeError(f"cannot multiply {dA.n_rows}x{dA.n_cols} by block with {X.shape[0]} rows")
    if out is None:
        out = _dev.empty_block(dA.n_rows, X.shape[1], X.device, X.dtype)
    elif out.shape != (dA.n_rows, X.shape[1]):
        raise ShapeError(f"output block {tuple(out.shape)} != {(dA.n_rows, X.shape[1])}")
    if X.shape[1] == 0 or dA.n_rows == 0:
        return out
    return _dev.spmm(dA, X, out)


def spmm(A: CsrMatrix, X):
    """Sparse matrix times dense block, Y[:, j] = A @ X[:, j] (sparse_core.py:132-149).

    Output entries are bitwise those of the reference kernel.  A numpy block
    returns a Fortran-ordered numpy array; a CUDA tensor returns a CUDA
    tensor."""
    if isinstance(X, torch.Tensor):
        Xd = as_device_block(X)
        return spmm_device(A, Xd)
    Xh = as_block(X)
    if A.n_cols != Xh.shape[0]:
        raise ShapeError(f"cannot multiply {A.n_rows}x{A.n_cols} by block with {Xh.shape[0]} rows")
    Y = spmm_device(A, _dev.to_device_block(Xh))
    return _dev.to_numpy_block(Y)


def spmv(A: CsrMatrix, x):
    """Single-column specialisation of spmm (sparse_core.py:152-157)."""
    if isinstance(x, torch.Tensor):
        xb = as_device_block(x)
    else:
        xb = as_block(x)
    if xb.shape[1] != 1:
        raise ShapeError("spmv expects a single column")
    return spmm(A, xb)


# ---------------------------------------------------------------------------
# Matrix Market I/O and generators (host utilities)
# ---------------------------------------------------------------------------


def _mm_body(lines, start):
    """Yield (lineno, fields) for the non-comment, non-blank lines."""
    for lineno in range(start, len(lines) + 1):
        s = lines[lineno - 1].strip()
        if s and not s.startswith("%"):
            yield lineno, s.split()


def read_matrix_market(path) -> CsrMatrix:
    """Matrix Market coordinate file (real/integer, general/symmetric)
    -> CsrMatrix (sparse_core.py:160-226 semantics and messages)."""
    with open(path, "rt") as fh:
        lines = fh.readlines()
    if not lines:
        raise MatrixMarketError("line 1: empty file")
    head = lines[0].split()
    if len(head) != 5 or head[0] != "%%MatrixMarket" or head[1].lower() != "matrix" \
            or head[2].lower() != "coordinate":
        raise MatrixMarketError("line 1: expected '%%MatrixMarket matrix coordinate ...' header")
    kind, sym = head[3].lower(), head[4].lower()
    if kind not in ("real", "integer"):
        raise MatrixMarketError(f"line 1: unsupported field '{head[3]}' (need real)")
    if sym not in ("general", "symmetric"):
        raise MatrixMarketError(f"line 1: unsupported symmetry '{head[4]}'")
    body = _mm_body(lines, 2)
    size = next(body, None)
    if size is None:
        raise MatrixMarketError(f"line {len(lines)}: missing size line")
    lineno, f = size
    if len(f) != 3:
        raise MatrixMarketError(f"line {lineno}: expected 'rows cols nnz'")
    try:
        n_rows, n_cols, nnz = (int(t) for t in f)
    except ValueError:
        raise MatrixMarketError(f"line {lineno}: non-integer size entry") from None
    rows, cols, vals = [], [], []
    count = 0
    last = lineno
    for lineno, f in body:
        last = lineno
        if len(f) != 3:
            raise MatrixMarketError(f"line {lineno}: expected 'row col value'")
        try:
            i, j, v = int(f[0]), int(f[1]), float(f[2])
        except ValueError:
            raise MatrixMarketError(f"line {lineno}: malformed entry") from None
        if not (1 <= i <= n_rows and 1 <= j <= n_cols):
            raise MatrixMarketError(f"line {lineno}: index ({i},{j}) out of declared range")
        rows.append(i - 1)
        cols.append(j - 1)
        vals.append(v)
        if sym == "symmetric" and i != j:
            rows.append(j - 1)
            cols.append(i - 1)
            vals.append(v)
        count += 1
    if count != nnz:
        raise MatrixMarketError(f"line {last}: declared {nnz} entries, found {count}")
    r = np.asarray(rows, dtype=np.int64)
    c = np.asarray(cols, dtype=np.int64)
    if len(r) and np.unique(r * max(n_cols, 1) + c).size != len(r):
        raise MatrixMarketError("duplicate entries in coordinate data")
    m = sp.coo_matrix((np.asarray(vals, dtype=np.float64), (r, c)), shape=(n_rows, n_cols)).tocsr()
    return CsrMatrix.from_scipy(m)


def read_matrix_market_array(path) -> np.ndarray:
    """Dense Matrix Market array file -> column-major block."""
    with open(path, "rt") as fh:
        lines = fh.readlines()
    if not lines:
        raise MatrixMarketError("line 1: empty file")
    head = lines[0].split()
    if len(head) != 5 or head[0] != "%%MatrixMarket" or head[2].lower() != "array":
        raise MatrixMarketError("line 1: expected '%%MatrixMarket matrix array ...' header")
    if head[3].lower() not in ("real", "integer"):
        raise MatrixMarketError(f"line 1: unsupported field '{head[3]}'")
    body = [f for _, f in _mm_body(lines, 2)]
    n, L = int(body[0][0]), int(body[0][1])
    vals = [float(f[0]) for f in body[1:1 + n * L]]
    if len(vals) != n * L:
        raise MatrixMarketError(f"expected {n * L} array entries, found {len(vals)}")
    return np.asfortranarray(np.asarray(vals).reshape((n, L), order="F"))


def write_matrix_market(A: CsrMatrix, path) -> None:
    """CsrMatrix -> coordinate/general file (exact round trip via repr)."""
    rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_ptr))
    with open(path, "wt") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{A.n_rows} {A.n_cols} {A.nnz}\n")
        fh.writelines(f"{i + 1} {j + 1} {float(v)!r}\n" for i, j, v in zip(rows, A.col_idx, A.values))


def gen_banded(n: int, band: int, seed: int) -> CsrMatrix:
    """2*band+1 diagonals of seeded uniform(0,1) values, +n on the main
    diagonal (sparse_core.py:269-287: same draw order, same values)."""
    if band < 0 or 2 * band + 1 > n:
        raise ValueError(f"half-bandwidth {band} too large for dimension {n}")
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for off in range(-band, band + 1):
        d = rng.uniform(0.0, 1.0, size=n - abs(off))
        if off == 0:
            d = d + n
        r = np.arange(max(0, -off), max(0, -off) + d.size)
        rows.append(r)
        cols.append(r + off)
        vals.append(d)
    m = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    m.sort_indices()
    return CsrMatrix.from_scipy(m)
