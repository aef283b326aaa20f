"""Thin QR on the device plus the small host-side dense problems.

Drop-in for ``recgmres.dense_kernels`` (/root/reference/pkg/src/recgmres/
dense_kernels.py).

* ``reduced_qr`` (dense_kernels.py:31-48): for an n x L block — CholQR2 on
  the device (Gram on the FP64 tensor cores, tiny Cholesky, two fused
  solve passes) with a Householder TSQR fallback whenever the Cholesky
  declines (ill-conditioned / rank-deficient blocks), so rank flags are
  always decided on a Householder R like LAPACK's.  Sign convention
  r_jj >= 0 and flags |r_jj| <= rank_tol * max(||X||_F, tiny) as in the
  reference.  Small host matrices (the (k+(m+1)L) x k' problems of the
  recycle update) use LAPACK on the host, which is where the north star
  keeps them.
* ``ProgressiveBlockLs`` (dense_kernels.py:116-203), ``solve_triangular``
  (:51-63) and the eigen-solvers (:211-282) are host-side: they work on
  O((k+mL)^2) data.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg
import torch

from . import device as _dev

# CholQR2 is accepted when min_j r_jj^2 >= CHOL_COND_TOL * max_j G_jj, i.e.
# roughly cond(X) < 3e5: far inside CholQR2's stability region
# (cond < eps^-1/2), and far above the rank-flag threshold (1e-12), so every
# block that could carry a rank flag goes to Householder TSQR.
CHOL_COND_TOL = 1e-11


class SingularMatrixError(np.linalg.LinAlgError):
    pass


@dataclass
class QrFactors:
    """Thin QR of an n x L block: q has orthonormal columns (numpy for numpy
    input, a CUDA tensor for device input), r_factor is the L x L upper
    triangular host array with nonnegative diagonal, flagged marks columns
    whose diagonal fell below the rank tolerance."""

    q: object
    r_factor: np.ndarray
    rank: int
    flagged: np.ndarray


def _flags(r: np.ndarray, norm_x: float, rank_tol: float) -> np.ndarray:
    return np.abs(np.diagonal(r)) <= rank_tol * max(norm_x, np.finfo(float).tiny)


def _phase(d: np.ndarray) -> np.ndarray:
    """Unit factors making a diagonal real and >= 0: the sign for real data
    (dense_kernels.py:42-45), the phase for complex data."""
    if np.iscomplexobj(d):
        a = np.abs(d)
        return np.where(a == 0, 1.0 + 0.0j, d / np.where(a == 0, 1.0, a))
    return np.where(d < 0.0, -1.0, 1.0)


def _host_dtype(X):
    return np.complex128 if np.iscomplexobj(X) else np.float64


def host_small_qr(X, rank_tol: float = 1e-12) -> QrFactors:
    """LAPACK thin QR of a SMALL host matrix (recycling.py:157 problems)."""
    X = np.atleast_2d(np.asarray(X, dtype=_host_dtype(X)))
    n, L = X.shape
    if n < L:
        raise ValueError(f"reduced_qr needs n >= L, got {n} < {L}")
    q, r = np.linalg.qr(X, mode="reduced")
    s = _phase(np.diagonal(r))
    q = np.asfortranarray(q * s)
    r = np.conj(s)[:, None] * r
    flagged = _flags(r, float(np.linalg.norm(X)), rank_tol)
    return QrFactors(q=q, r_factor=r, rank=int(L - flagged.sum()), flagged=flagged)


class QrScratch:
    """Device buffers of one CholQR2 / TSQR (reused across calls)."""

    def __init__(self, L: int, device, dtype=torch.float64):
        self.L = L
        self.dtype = dtype
        # packed: G1 | R1 | G2 | R2 | R_tsqr  (each L x L, column-major) + 2 status ints
        self.buf = torch.zeros(5 * L * L, dtype=dtype, device=device)
        self.status = torch.zeros(2, dtype=torch.int32, device=device)

    def mat(self, i: int) -> torch.Tensor:
        L = self.L
        return self.buf[i * L * L:(i + 1) * L * L].view(L, L).t()  # column-major view

    G1 = property(lambda s: s.mat(0))
    R1 = property(lambda s: s.mat(1))
    G2 = property(lambda s: s.mat(2))
    R2 = property(lambda s: s.mat(3))
    RT = property(lambda s: s.mat(4))


def cholqr2_launch(X: torch.Tensor, Q: torch.Tensor, scr: QrScratch, g1_ready: bool = False):
    """Enqueue CholQR2 of X into Q (Q may not alias X: X is kept intact for
    the TSQR fallback).  If ``g1_ready``, scr.G1 already holds X^T X (fused
    into the producing pass)."""
    if _dev.fused_ok() and X.shape[1] <= _dev.MAX_P_FUSED and X.dtype == torch.float64:
        # G1 | R1 | G2 | R2 are the first four blocks of scr.buf, as rg_cholqr2_f64 expects
        _dev.cholqr2(X, Q, scr.buf, scr.status, g1_ready)
        return
    if not g1_ready:
        _dev.tall(X, None, gram=("self", scr.G1))
    _dev.chol(scr.G1, scr.R1, scr.status[0:1], CHOL_COND_TOL)
    _dev.tall(X, None, r1=scr.R1, gram=("self", scr.G2))
    _dev.chol(scr.G2, scr.R2, scr.status[1:2], CHOL_COND_TOL)
    _dev.tall(X, Q, r1=scr.R1, r2=scr.R2)


def cholqr2_finish(host_buf: np.ndarray, host_status: np.ndarray, L: int):
    """Host side after the D2H copy: (ok, R, ||X||_F)."""
    mats = host_buf.reshape(5, L, L).transpose(0, 2, 1)  # column-major -> row-major views
    G1, R1, _, R2 = mats[0], mats[1], mats[2], mats[3]
    norm_x = float(np.sqrt(max(np.trace(G1).real, 0.0)))
    ok = bool(host_status[0] == 0 and host_status[1] == 0)
    R = np.triu(R2 @ R1) if ok else None
    return ok, R, norm_x


def tsqr_into(X: torch.Tensor, Q: torch.Tensor, scr: QrScratch) -> None:
    """Householder TSQR of X into Q (copying first when they differ).

    Row-partitioned: each rank factors its rows, the ranks' R factors are
    all-gathered, the stack is factored on every rank (identical input,
    identical LAPACK result), and each rank applies its block of the small Q
    to its rows (Q_local <- Q_local S_rank, one rg_tall pass)."""
    if X.dtype == torch.complex128:
        _shifted_cholqr3(X, Q, scr)
        return
    if Q.data_ptr() != X.data_ptr():
        Q.copy_(X)
    _dev.tsqr(Q, scr.RT)
    comm = _dev.get_comm()
    if comm is None or comm.world == 1:
        return
    L = Q.shape[1]
    S_rank, rs = tsqr_combine(np.triu(scr.RT.cpu().numpy()), comm)
    S = torch.from_numpy(S_rank).to(Q.device)
    _dev.tall(None, Q, [(Q, S, 1.0)], n=Q.shape[0], p=L)
    scr.RT.copy_(torch.from_numpy(np.asfortranarray(rs)).to(Q.device))


def _shifted_cholqr3(X: torch.Tensor, Q: torch.Tensor, scr: QrScratch) -> None:
    """Robust thin QR without Householder (used for complex blocks, whose
    TSQR is not implemented): shifted CholQR on X, then CholQR2 on the
    result (Fukaya et al.'s shifted CholQR3).  R = R3 R2 R1 lands in scr.RT."""
    n, L = X.shape
    dt = X.dtype
    dev = X.device
    G = _dev.small(L, L, dev, dt)
    _dev.tall(X, None, gram=("self", G))
    Gh = G.cpu().numpy()
    nrm2 = float(np.trace(Gh).real)
    shift = 11.0 * (n * L + L * (L + 1)) * np.finfo(float).eps * max(nrm2, np.finfo(float).tiny)
    Gs = torch.from_numpy(np.asfortranarray(Gh + shift * np.eye(L))).to(dev)
    Rs = []
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    cur = X
    for stage in range(3):
        R = _dev.small(L, L, dev, dt)
        if stage > 0:
            Gs = _dev.small(L, L, dev, dt)
            _dev.tall(cur, None, gram=("self", Gs))
        _dev.chol(Gs, R, st, 0.0)
        _dev.tall(cur, Q, r1=R)
        cur = Q
        Rs.append(np.triu(R.cpu().numpy()))
    Rt = Rs[2] @ Rs[1] @ Rs[0]
    scr.RT.copy_(torch.from_numpy(np.asfortranarray(np.triu(Rt))).to(dev))


def tsqr_combine(R_local: np.ndarray, comm):
    """Top level of the distributed TSQR: QR of the all-gathered R factors
    (identical on every rank), sign-fixed to r_jj >= 0.  Returns this rank's
    L x L block of the small Q and the global R."""
    L = R_local.shape[1]
    stack = np.vstack(comm.allgather_np(R_local))
    qs, rs = np.linalg.qr(stack, mode="reduced")
    s = np.where(np.diagonal(rs) < 0.0, -1.0, 1.0)
    qs = qs * s
    rs = rs * s[:, None]
    return np.asfortranarray(qs[comm.rank * L:(comm.rank + 1) * L]), rs


TSQR_MAX_P = 32


def _wide_qr(X: torch.Tensor, Q: torch.Tensor, rank_tol: float) -> QrFactors:
    """Thin QR of a block wider than TSQR_MAX_P columns: column panels of
    32, each made orthogonal to the previous panels by block CGS2 (fused
    projection passes) and then factored by Householder TSQR.  R collects the
    projection coefficients above the diagonal blocks."""
    n, L = X.shape
    if Q.data_ptr() != X.data_ptr():
        Q.copy_(X)
    ss = torch.zeros(L, dtype=torch.float64, device=X.device)
    _dev.tall(Q, None, gram=("sumsq", ss))
    norm_x = float(np.sqrt(ss.sum().item()))
    cplx = X.dtype == torch.complex128
    R = np.zeros((L, L), dtype=np.complex128 if cplx else np.float64)
    from .ortho import project_chain

    panel = _dev.MAX_P_C if cplx else TSQR_MAX_P
    for b0 in range(0, L, panel):
        b1 = min(L, b0 + panel)
        Qb = Q[:, b0:b1]
        if b0:
            prev = Q[:, :b0]
            c1 = _dev.small(b0, b1 - b0, X.device, X.dtype)
            c2 = _dev.small(b0, b1 - b0, X.device, X.dtype)
            project_chain(Qb, Qb, [prev, prev], [c1, c2])
            R[:b0, b0:b1] = c1.cpu().numpy() + c2.cpu().numpy()
        scr = QrScratch(b1 - b0, X.device, X.dtype)
        tsqr_into(Qb, Qb, scr)
        R[b0:b1, b0:b1] = np.triu(scr.RT.cpu().numpy())
    flagged = _flags(R, norm_x, rank_tol)
    return QrFactors(q=Q, r_factor=R, rank=int(L - flagged.sum()), flagged=flagged)


def reduced_qr_device(X: torch.Tensor, rank_tol: float = 1e-12, Q: torch.Tensor | None = None,
                      scr: QrScratch | None = None) -> QrFactors:
    """Device thin QR; X is not modified (unless Q is X)."""
    n, L = X.shape
    if n < L:
        raise ValueError(f"reduced_qr needs n >= L, got {n} < {L}")
    dev = X.device
    cplx = X.dtype == torch.complex128
    if Q is None:
        Q = _dev.empty_block(n, L, dev, X.dtype)
    if L > (_dev.MAX_P_C if cplx else TSQR_MAX_P):
        return _wide_qr(X, Q, rank_tol)
    if scr is None or scr.L != L or scr.dtype != X.dtype:
        scr = QrScratch(L, dev, X.dtype)
    in_place = Q.data_ptr() == X.data_ptr()
    if L <= (_dev.MAX_P_C if cplx else _dev.MAX_P) and not in_place:
        cholqr2_launch(X, Q, scr)
        hb = scr.buf.cpu().numpy()
        hs = scr.status.cpu().numpy()
        ok, R, norm_x = cholqr2_finish(hb, hs, L)
        if ok:
            flagged = _flags(R, norm_x, rank_tol)
            return QrFactors(q=Q, r_factor=R, rank=int(L - flagged.sum()), flagged=flagged)
    else:
        ss = torch.empty(L, dtype=torch.float64, device=dev)
        _dev.tall(X, None, gram=("sumsq", ss))
        norm_x = float(np.sqrt(ss.sum().item()))
    tsqr_into(X, Q, scr)
    R = np.triu(scr.RT.cpu().numpy())
    flagged = _flags(R, norm_x, rank_tol)
    return QrFactors(q=Q, r_factor=R, rank=int(L - flagged.sum()), flagged=flagged)


def reduced_qr(X, rank_tol: float = 1e-12) -> QrFactors:
    """Thin QR with nonnegative diagonal (dense_kernels.py:31-48).

    A CUDA tensor runs on the device and returns a CUDA ``q``; a numpy
    block is copied to the device and ``q`` comes back as a Fortran-ordered
    numpy array."""
    if isinstance(X, torch.Tensor):
        Xd = _dev.to_device_block(X if X.dim() == 2 else X.reshape(-1, 1))
        return reduced_qr_device(Xd, rank_tol)
    Xh = np.atleast_2d(np.asarray(X, dtype=_host_dtype(X)))
    n, L = Xh.shape
    if n < L:
        raise ValueError(f"reduced_qr needs n >= L, got {n} < {L}")
    f = reduced_qr_device(_dev.to_device_block(Xh), rank_tol)
    return QrFactors(q=_dev.to_numpy_block(f.q), r_factor=f.r_factor, rank=f.rank, flagged=f.flagged)


def solve_triangular(Rf, rhs) -> np.ndarray:
    """Back substitution Rf Y = rhs; a diagonal below 1e-14 * ||Rf|| signals
    breakdown upstream and raises naming the column (dense_kernels.py:51-63)."""
    Rf = np.asarray(Rf, dtype=_host_dtype(Rf))
    d = np.abs(np.diagonal(Rf))
    bad = np.flatnonzero(d <= 1e-14 * max(np.linalg.norm(Rf), np.finfo(float).tiny))
    if bad.size:
        raise SingularMatrixError(f"singular diagonal in column {bad[0]}")
    return scipy.linalg.solve_triangular(Rf, rhs, lower=False)


# ---------------------------------------------------------------------------
# Progressive triangularisation of the block Hessenberg least-squares problem
# ---------------------------------------------------------------------------


class ProgressiveBlockLs:
    """min ||Hbar Y - E1 G0||_F over a block Hessenberg Hbar that grows by
    one block column per Arnoldi step (dense_kernels.py:116-203).

    Each appended block column is first hit by the orthogonal factors of the
    earlier steps, then its trailing 2L x L window is reduced to upper
    triangular form by one 2L x 2L orthogonal factor (Householder QR of the
    window, LAPACK) with the sign of every diagonal entry made nonnegative.
    The transformed right-hand side gives the per-column residual norms
    without solving for Y."""

    def __init__(self, L: int, g0: np.ndarray):
        g0 = np.atleast_2d(np.asarray(g0, dtype=_host_dtype(g0)))
        if g0.shape[0] != L:
            raise ValueError("g0 must have L rows")
        self.L = L
        self.m = 0
        self.n_rhs = g0.shape[1]
        self._factors: list[np.ndarray] = []  # Q^T of each 2L window (signs folded in)
        self._rcols: list[np.ndarray] = []
        self.g = g0.copy()

    def append_block(self, new_cols: np.ndarray) -> np.ndarray:
        L, m = self.L, self.m
        dt = np.complex128 if (np.iscomplexobj(new_cols) or np.iscomplexobj(self.g)) else np.float64
        blk = np.array(new_cols, dtype=dt, copy=True)
        if blk.shape != ((m + 2) * L, L):
            raise ValueError(f"expected new block of shape {((m + 2) * L, L)}, got {blk.shape}")
        if dt == np.complex128:
            self.g = self.g.astype(np.complex128)
        for i, Qt in enumerate(self._factors):
            rows = slice(i * L, (i + 2) * L)
            blk[rows] = Qt @ blk[rows]
        win = blk[m * L:, :]
        Qw, Rw = np.linalg.qr(win, mode="complete")  # Qw 2L x 2L
        s = np.ones(2 * L, dtype=dt)
        s[:L] = _phase(np.diagonal(Rw))
        # Q^H with the first L rows re-phased: the new diagonal is real >= 0
        Qt = np.conj(s)[:, None] * np.conj(Qw).T
        blk[m * L:, :] = 0.0
        blk[m * L:(m + 1) * L, :] = np.conj(s[:L])[:, None] * Rw[:L]
        self._factors.append(Qt)
        self.g = np.vstack([self.g, np.zeros((L, self.n_rhs), dtype=self.g.dtype)])
        self.g[m * L:, :] = Qt @ self.g[m * L:, :]
        for c in range(L):
            self._rcols.append(blk[:(m + 1) * L, c].copy())
        self.m = m + 1
        return self.residual_norms()

    def residual_norms(self) -> np.ndarray:
        return np.linalg.norm(self.g[self.m * self.L:, :], axis=0)

    def r_factor(self) -> np.ndarray:
        k = self.m * self.L
        R = np.zeros((k, k), dtype=self.g.dtype)
        for j, col in enumerate(self._rcols):
            R[: j + 1, j] = col[: j + 1]
        return R

    def solve(self) -> np.ndarray:
        k = self.m * self.L
        return solve_triangular(self.r_factor(), self.g[:k, :])


# ---------------------------------------------------------------------------
# Small dense eigenproblems (host)
# ---------------------------------------------------------------------------


@dataclass
class EigPairs:
    """Eigenpairs with each conjugate pair stored as adjacent (real part,
    imaginary part) columns of a real basis (dense_kernels.py:211-238).

    pairing: 0 real, 1 first member of a pair, 2 second member."""

    values: np.ndarray
    vectors: np.ndarray
    pairing: np.ndarray

    def complex_vector(self, i: int) -> np.ndarray:
        kind = self.pairing[i]
        if kind == 0:
            return self.vectors[:, i].astype(complex)  # (already complex for complex problems)
        if kind == 1:
            return self.vectors[:, i] + 1j * self.vectors[:, i + 1]
        return self.vectors[:, i - 1] - 1j * self.vectors[:, i]


def _real_basis(w, v) -> EigPairs:
    n = len(w)
    vecs = np.zeros((v.shape[0], n))
    pairing = np.zeros(n, dtype=np.int8)
    i = 0
    while i < n:
        if w[i].imag == 0.0:
            vecs[:, i] = v[:, i].real
            i += 1
            continue
        ok = (i + 1 < n and np.isclose(w[i + 1].real, w[i].real) and np.isclose(w[i + 1].imag, -w[i].imag))
        if not ok:
            raise np.linalg.LinAlgError("unpaired complex eigenvalue")
        vecs[:, i], vecs[:, i + 1] = v[:, i].real, v[:, i].imag
        pairing[i], pairing[i + 1] = 1, 2
        i += 2
    return EigPairs(values=np.asarray(w, dtype=complex), vectors=vecs, pairing=pairing)


def eig_standard(M) -> EigPairs:
    """All eigenpairs of a small real square matrix (LAPACK dgeev)."""
    M = np.asarray(M, dtype=_host_dtype(M))
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError("eig_standard needs a square matrix")
    try:
        w, v = np.linalg.eig(M)
    except np.linalg.LinAlgError as e:
        raise np.linalg.LinAlgError(f"eigenvalue iteration failed: {e}") from e
    if np.iscomplexobj(M):
        # complex problems use the eigenvectors directly (no conjugate pairs)
        return EigPairs(values=np.asarray(w, dtype=complex), vectors=v, pairing=np.zeros(len(w), dtype=np.int8))
    return _real_basis(w, v)


def eig_generalized(Ag, Bg) -> EigPairs:
    """Ag t = theta Bg t via Bg^{-1} Ag; raises SingularMatrixError when
    cond(Bg) > 1e14 (dense_kernels.py:267-282)."""
    Ag = np.asarray(Ag, dtype=_host_dtype(Ag) if np.iscomplexobj(Ag) or not np.iscomplexobj(Bg) else np.complex128)
    Bg = np.asarray(Bg, dtype=Ag.dtype)
    if Ag.shape != Bg.shape or Ag.shape[0] != Ag.shape[1]:
        raise ValueError("eig_generalized needs square matrices of equal size")
    if Bg.size and np.linalg.cond(Bg) > 1e14:
        raise SingularMatrixError("degenerate basis: Bg condition above 1e14")
    return eig_standard(np.linalg.solve(Bg, Ag))
