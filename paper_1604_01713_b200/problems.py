"""Seeded synthetic problems for the BASELINE configurations.

The paper's UF / Tramonto / sherman5 matrices are not available, so seeded
stencil operators stand in for them.  Each generator builds the CSR arrays
directly (vectorised, rows in ascending column order) and reproduces, bit for
bit, the scipy ``kron``-sum recipe that tests/golden/make_golden.py runs
against the reference: every stored value is formed with the same sequence
of IEEE operations as scipy's sparse sums (entries present in one operand
only are passed through unchanged; the diagonal of the d-dimensional
Laplacian is ((a + a) + a)).

Grid ordering is lexicographic with x fastest: row = (z*N + y)*N + x.
"""

from __future__ import annotations

import numpy as np

from .sparse_core import CsrMatrix


def _stencil_csr(N: int, dim: int, diag_val: float, off_lo: float, off_hi: float) -> CsrMatrix:
    """(2*dim+1)-point operator with constant coefficients: diagonal
    ``diag_val``; neighbour at -1 along an axis gets ``off_lo``, +1 gets
    ``off_hi`` (the same along every axis)."""
    n = N ** dim
    idx = np.arange(n, dtype=np.int64)
    coords = []
    rem = idx
    for _ in range(dim):
        coords.append(rem % N)
        rem = rem // N
    # neighbour slots in ascending column order: -N^(d-1) ... -1, 0, +1 ... +N^(d-1)
    slots = []
    for ax in reversed(range(dim)):
        slots.append((ax, -1))
    slots.append((None, 0))
    for ax in range(dim):
        slots.append((ax, +1))
    k = len(slots)
    cols = np.empty((n, k), dtype=np.int64)
    vals = np.empty((n, k), dtype=np.float64)
    keep = np.ones((n, k), dtype=bool)
    for s, (ax, d) in enumerate(slots):
        if ax is None:
            cols[:, s] = idx
            vals[:, s] = diag_val
            continue
        stride = N ** ax
        cols[:, s] = idx + d * stride
        vals[:, s] = off_lo if d < 0 else off_hi
        keep[:, s] = (coords[ax] > 0) if d < 0 else (coords[ax] < N - 1)
    counts = keep.sum(axis=1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    if row_ptr[-1] >= 2**31:
        raise ValueError("matrix too large for int32 CSR indices")
    col_idx = cols[keep].astype(np.int32)
    values = vals[keep]
    return CsrMatrix(n, n, row_ptr.astype(np.int32), col_idx, values, _validated=True)


def conv_diff_3d_slab(N: int, Nz: int, beta: float, z0: int, z1: int):
    """Rows of z-planes [z0, z1) of the 7-point conv-diff operator on an
    N x N x Nz grid (h = 1/(N+1) in every direction, same coefficients as
    conv_diff_3d), with GLOBAL column indices.  Used by the weak-scaling
    bench: each rank generates only its slab.  Returns (row_ptr, col_idx,
    values, n_global)."""
    h = 1.0 / (N + 1)
    h2 = h**2
    t_off = -1.0 / h2
    t_diag = 2.0 / h2
    d = 1.0 / (2 * h)
    diag = (t_diag + t_diag) + t_diag
    lo, hi = t_off + beta * (-d), t_off + beta * d
    plane = N * N
    n_global = plane * Nz
    idx = np.arange(z0 * plane, z1 * plane, dtype=np.int64)
    x, y, z = idx % N, (idx // N) % N, idx // plane
    offs = [(-plane, z > 0, lo), (-N, y > 0, lo), (-1, x > 0, lo), (0, None, diag),
            (1, x < N - 1, hi), (N, y < N - 1, hi), (plane, z < Nz - 1, hi)]
    nl = idx.size
    cols = np.empty((nl, 7), dtype=np.int64)
    vals = np.empty((nl, 7), dtype=np.float64)
    keep = np.ones((nl, 7), dtype=bool)
    for s, (o, ok, v) in enumerate(offs):
        cols[:, s] = idx + o
        vals[:, s] = v
        if ok is not None:
            keep[:, s] = ok
    counts = keep.sum(axis=1)
    row_ptr = np.zeros(nl + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return row_ptr, cols[keep], vals[keep], n_global


def conv_diff_2d(N: int, beta: float) -> CsrMatrix:
    """-Lap u + beta (u_x + u_y), 5-point central FD on an N x N interior grid,
    h = 1/(N+1), Dirichlet eliminated (BASELINE configs[0]: N=64, beta=10)."""
    h = 1.0 / (N + 1)
    h2 = h**2
    t_off = -1.0 / h2
    t_diag = 2.0 / h2
    d = 1.0 / (2 * h)
    diag = t_diag + t_diag
    return _stencil_csr(N, 2, diag, t_off + beta * (-d), t_off + beta * d)


def conv_diff_3d(N: int, beta: float) -> CsrMatrix:
    """-Lap u + beta (u_x + u_y + u_z), 7-point central FD, h = 1/(N+1)
    (BASELINE configs[3]: N=256, beta=20)."""
    h = 1.0 / (N + 1)
    h2 = h**2
    t_off = -1.0 / h2
    t_diag = 2.0 / h2
    d = 1.0 / (2 * h)
    diag = (t_diag + t_diag) + t_diag
    return _stencil_csr(N, 3, diag, t_off + beta * (-d), t_off + beta * d)


def laplacian_3d(N: int) -> CsrMatrix:
    """Unscaled 7-point Laplacian (6 on the diagonal, -1 off it)
    (BASELINE configs[1]: N=128)."""
    return _stencil_csr(N, 3, (2.0 + 2.0) + 2.0, -1.0, -1.0)


def add_diagonal(A: CsrMatrix, dvals: np.ndarray) -> CsrMatrix:
    """A + diag(dvals) for a matrix whose diagonal is structurally present
    (scipy's ``A + sp.diags(dvals)`` value for value)."""
    rp, ci = A.row_ptr, A.col_idx
    rows = np.repeat(np.arange(A.n_rows, dtype=np.int64), np.diff(rp))
    on_diag = ci == rows
    if on_diag.sum() != min(A.n_rows, A.n_cols):
        raise ValueError("add_diagonal needs a structurally full diagonal")
    vals = A.values.copy()
    vals[on_diag] = vals[on_diag] + np.asarray(dvals, dtype=np.float64)[rows[on_diag]]
    return CsrMatrix(A.n_rows, A.n_cols, rp, ci, vals, _validated=True)


def cfg1_sequence():
    """BASELINE configs[0]: 2-D conv-diff 64x64, p=4 uniform[-1,1] RHS, 3
    systems A_i = A + 0.01*i*diag(d), d ~ U[0,1] (one default_rng(0): B first,
    then d).  Returns ([(A_i, B)], SolverConfig kwargs)."""
    A = conv_diff_2d(64, 10.0)
    rng = np.random.default_rng(0)
    B = np.asfortranarray(rng.uniform(-1.0, 1.0, (A.n_rows, 4)))
    d = rng.uniform(0.0, 1.0, A.n_rows)
    systems = [(add_diagonal(A, 0.01 * i * d), B) for i in range(3)]
    return systems, dict(m=20, k=10, tol=1e-8)


def cfg3_draws(n: int = 2**24, k: int = 20, p: int = 8, wcols: int = 80, seed: int = 0):
    """BASELINE configs[2] (block orthogonalization microbench), the raw
    draws of the reference's recipe in its order (bench.py:110-113,
    SURVEY.md §8d): one default_rng(seed) gives an n x k N(0,1) block whose
    thin-QR factor is C, then V (n x p, N(0,1)), then an n x wcols N(0,1)
    block whose thin-QR factor is the 10-block basis Q.  Returns the three
    Fortran-ordered draws; ``cfg3_inputs`` orthonormalises them."""
    rng = np.random.default_rng(seed)
    Craw = np.asfortranarray(rng.standard_normal((n, k)))
    V = np.asfortranarray(rng.standard_normal((n, p)))
    Qraw = np.asfortranarray(rng.standard_normal((n, wcols)))
    return Craw, V, Qraw


def cfg3_inputs(n: int = 2**24, k: int = 20, p: int = 8, wcols: int = 80, seed: int = 0, device=None):
    """Device-resident cfg3 operands (C, V, Q) as column-major blocks: the
    draws of ``cfg3_draws`` uploaded once, C and Q orthonormalised by the
    device thin QR (reduced_qr semantics: r_jj >= 0).  At n = 2^24 the draws
    take ~20 s on the host and the QRs well under a second on the device."""
    from . import device as _dev
    from .dense_kernels import reduced_qr_device

    Craw, V, Qraw = cfg3_draws(n, k, p, wcols, seed)
    dev = _dev.require_cuda(device)
    Cd = reduced_qr_device(_dev.to_device_block(Craw, dev)).q
    del Craw
    Vd = _dev.to_device_block(V, dev)
    del V
    Qd = reduced_qr_device(_dev.to_device_block(Qraw, dev)).q
    return Cd, Vd, Qd


def cfg4_sequence(N: int = 256, n_systems: int = 5, p: int = 8, beta: float = 20.0):
    """BASELINE configs[3]: 3-D conv-diff N^3 (beta=20), p=8 N(0,1) RHS, m=10,
    k=20, tol 1e-8, n_systems systems A_i = A + diag(0.005*i*u*diag(A)),
    u ~ U[0,1] (builder decisions).  Systems are generated
    lazily (each is ~1.5 GB at N=256)."""
    A = conv_diff_3d(N, beta)
    B = np.asfortranarray(np.random.default_rng(0).standard_normal((A.n_rows, p)))
    u = np.random.default_rng(1).uniform(0.0, 1.0, A.n_rows)
    diagA = A.diagonal()

    def system(i):
        return add_diagonal(A, 0.005 * i * u * diagA) if i else A

    return A, B, system, dict(m=10, k=20, tol=1e-8, max_cycles=200)


def stencil27_complex(N: int, sigma: complex = complex(-0.5, 0.3), seed: int = 0):
    """BASELINE configs[4]: 27-point stencil on N^3, off-diagonals U[-1,0]
    (seeded, per entry), diagonal 26 + sigma.  Returns (row_ptr, col_idx,
    complex values, n).  Builder decision: the off-diagonal draw is one
    default_rng(seed).uniform(-1, 0, nnz_off) in storage order."""
    n = N**3
    idx = np.arange(n, dtype=np.int64)
    x, y, z = idx % N, (idx // N) % N, idx // (N * N)
    offs = [(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    cols = np.empty((n, 27), dtype=np.int64)
    keep = np.ones((n, 27), dtype=bool)
    for s, (dz, dy, dx) in enumerate(offs):
        cols[:, s] = idx + dz * N * N + dy * N + dx
        keep[:, s] = ((x + dx >= 0) & (x + dx < N) & (y + dy >= 0) & (y + dy < N) & (z + dz >= 0) & (z + dz < N))
    is_diag = np.zeros((n, 27), dtype=bool)
    is_diag[:, 13] = True
    counts = keep.sum(axis=1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    col_idx = cols[keep].astype(np.int32)
    dflag = is_diag[keep]
    vals = np.empty(col_idx.shape[0], dtype=np.complex128)
    rng = np.random.default_rng(seed)
    vals[~dflag] = rng.uniform(-1.0, 0.0, int((~dflag).sum()))
    vals[dflag] = 26.0 + sigma
    return row_ptr.astype(np.int32), col_idx, vals, n


def cfg5_sequence(N: int = 160, n_systems: int = 4, p: int = 16):
    """BASELINE configs[4]: complex 27-point stencil N^3 with p=16 complex
    N(0,1) right-hand sides, m=8, k=16.  The 4-shift sequence is a builder
    decision: system i has diagonal 26 + sigma_i with
    sigma_i = (-0.5 - 0.05 i) + (0.3 + 0.05 i) 1j; tol 1e-8 as config 4.
    Returns (system(i) -> CsrMatrix, B, solver kwargs)."""
    rp, ci, v0, n = stencil27_complex(N)
    diag = np.zeros(len(ci), dtype=bool)
    rows = np.repeat(np.arange(n), np.diff(rp))
    diag[ci == rows] = True
    g = np.random.default_rng(0).standard_normal((n, 2 * p))
    B = np.asfortranarray(g[:, :p] + 1j * g[:, p:])

    def system(i):
        v = v0.copy()
        v[diag] = 26.0 + complex(-0.5 - 0.05 * i, 0.3 + 0.05 * i)
        return CsrMatrix(n, n, rp, ci, v, _validated=True)

    return system, B, dict(m=8, k=16, tol=1e-8, max_cycles=200)
