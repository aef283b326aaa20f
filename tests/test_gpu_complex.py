"""complex128 twins (BASELINE configs[4]).  The reference is real-only, so
parity is against the complex restatement of SURVEY.md §8c (oracle.spmm's
complex path, numpy for the dense algebra): parity unpinned by reference
golden vectors."""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def test_spmm_c128_bitwise_vs_complex_oracle(cuda):
    from paper_1604_01713_b200 import device as D, problems
    from paper_1604_01713_b200.sparse_core import DeviceCsr

    rp, ci, v, n = problems.stencil27_complex(14)
    dA = DeviceCsr.from_host(n, n, rp, ci, v)
    rng = np.random.default_rng(0)
    for p in (1, 3, 8, 16):
        X = np.asfortranarray(rng.standard_normal((n, p)) + 1j * rng.standard_normal((n, p)))
        Xd = D.to_device_block(X)
        Y = D.empty_block(n, p, dtype=torch.complex128)
        D.spmm(dA, Xd, Y)
        ref = oracle.spmm(rp, ci, v, X)
        assert np.array_equal(D.to_numpy_block(Y), ref), p


@pytest.mark.parametrize("n", [1, 777, 100003])
@pytest.mark.parametrize("p", [1, 5, 8, 12, 16])
def test_tall_c128(cuda, n, p):
    from paper_1604_01713_b200 import device as D

    rng = np.random.default_rng(n + p)
    cz = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)
    for gc in (3, 20, 60):
        Gb, Z = cz(n, gc), cz(n, p)
        out = D.small(gc, p, dtype=torch.complex128)
        D.tall(D.to_device_block(Z), None, gram=("basis", D.to_device_block(Gb), out))
        assert _rel(out.cpu().numpy(), Gb.conj().T @ Z) <= 1e-12
    X1, S1, X2, S2, Z = cz(n, 12), cz(12, p), cz(n, 30), cz(30, p), cz(n, p)
    Zo = D.empty_block(n, p, dtype=torch.complex128)
    G = D.small(p, p, dtype=torch.complex128)
    D.tall(D.to_device_block(Z), Zo, [(D.to_device_block(X1), torch.from_numpy(S1).to(cuda), -1.0),
                                      (D.to_device_block(X2), torch.from_numpy(S2).to(cuda), -1.0)],
           gram=("self", G))
    ref = (Z - X1 @ S1) - X2 @ S2
    assert _rel(D.to_numpy_block(Zo), ref) <= 1e-12
    assert _rel(G.cpu().numpy(), ref.conj().T @ ref) <= 1e-12
    ss = torch.zeros(p, dtype=torch.float64, device=cuda)
    D.tall(Zo, None, gram=("sumsq", ss))
    assert _rel(ss.cpu().numpy(), (np.abs(ref) ** 2).sum(axis=0)) <= 1e-12
    # fused update + Gram against another basis (the CGS2 pass shape), wide term lists
    for a1, gc in ((16, 40), (130, 24)):
        X1, S1, Gb, Z = cz(n, a1), cz(a1, p), cz(n, gc), cz(n, p)
        Zo = D.empty_block(n, p, dtype=torch.complex128)
        out = D.small(gc, p, dtype=torch.complex128)
        D.tall(D.to_device_block(Z), Zo, [(D.to_device_block(X1), torch.from_numpy(S1).to(cuda), -1.0)],
               gram=("basis", D.to_device_block(Gb), out))
        ref = Z - X1 @ S1
        assert _rel(D.to_numpy_block(Zo), ref) <= 1e-12
        assert _rel(out.cpu().numpy(), Gb.conj().T @ ref) <= 1e-12
    R = np.triu(cz(p, p)) + 4 * np.eye(p)
    np.fill_diagonal(R, np.abs(np.diagonal(R)))  # real positive diagonal, as from Cholesky
    Zo2 = D.empty_block(n, p, dtype=torch.complex128)
    D.tall(D.to_device_block(Z), Zo2, r1=torch.from_numpy(R).to(cuda))
    assert _rel(D.to_numpy_block(Zo2), np.linalg.solve(R.T, Z.T).T) <= 1e-12


def test_chol_c128(cuda):
    from paper_1604_01713_b200 import device as D

    rng = np.random.default_rng(3)
    for p in (1, 8, 16):
        X = rng.standard_normal((200, p)) + 1j * rng.standard_normal((200, p))
        G = X.conj().T @ X
        Gd = torch.from_numpy(np.asfortranarray(G)).to(cuda)
        R = D.small(p, p, dtype=torch.complex128)
        st = torch.zeros(1, dtype=torch.int32, device=cuda)
        D.chol(Gd, R, st, 1e-11)
        Rh = R.cpu().numpy()
        assert st.item() == 0
        assert np.all(np.abs(np.diagonal(Rh).imag) == 0) and np.all(np.diagonal(Rh).real > 0)
        assert _rel(Rh.conj().T @ Rh, G) <= 1e-13


# ---------------------------------------------------------------------------
# complex solver path (config 5): step parity against the complex restatement
# and solve-level properties of the reference's own tests in complex form.
# ---------------------------------------------------------------------------


def _cplx_normal(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.mark.parametrize("L,k", [(4, 6), (16, 16)])
def test_complex_arnoldi_step_vs_oracle(cuda, L, k):
    from paper_1604_01713_b200 import arnoldi, problems
    from paper_1604_01713_b200.recycling import RecycleSpace, prepare_cross_system
    from paper_1604_01713_b200.solver import _Operator

    system, _, _ = problems.cfg5_sequence(N=12, p=L)
    A = system(0)
    n, m = A.n_rows, 3
    rng = np.random.default_rng(L)
    op = _Operator(A, None, "none")
    rs = prepare_cross_system(RecycleSpace(u=np.asfortranarray(_cplx_normal(rng, (n, k))), c=None), op.apply)
    U, C = rs.numpy()
    assert np.linalg.norm(C.conj().T @ C - np.eye(k)) <= 1e-12 * k
    assert np.linalg.norm(A.to_scipy() @ U - C) <= 1e-10 * np.linalg.norm(C)
    R0 = _cplx_normal(rng, (n, L))
    R0 = R0 - C @ (C.conj().T @ R0)
    fact = arnoldi.start(op.apply, R0, m_max=m, recycle=rs, seed=0)
    assert fact.w.dtype == torch.complex128
    for _ in range(m - 1):
        arnoldi.step(fact, op.apply, recycle=rs)
    W = fact.w_numpy()
    Vm = W[:, (m - 1) * L: m * L]
    arnoldi.step(fact, op.apply, recycle=rs)
    q, F, H, r, flagged = oracle.arnoldi_step(A.row_ptr, A.col_idx, A.values, Vm, C, W)
    assert not flagged.any()
    cols = slice((m - 1) * L, m * L)
    scale = max(np.abs(H).max(), 1.0)
    assert np.abs(fact._H[: m * L, cols] - H).max() <= 1e-12 * scale
    assert np.abs(fact._F[:, cols] - F).max() <= 1e-12 * scale
    assert np.abs(fact._H[m * L:(m + 1) * L, cols] - r).max() <= 1e-11 * scale
    assert np.all(np.diagonal(fact._H[m * L:(m + 1) * L, cols]).imag == 0.0)
    assert np.abs(fact.w_numpy()[:, m * L:(m + 1) * L] - q).max() <= 1e-10
    # the reference's invariants in complex form
    Wf = fact.w_numpy()
    assert np.linalg.norm(Wf.conj().T @ Wf - np.eye((m + 1) * L)) <= 1e-12 * (m + 1) * L
    assert np.linalg.norm(C.conj().T @ Wf) <= 1e-10
    AW = A.to_scipy() @ Wf[:, : m * L]
    PAW = AW - C @ (C.conj().T @ AW)
    nA = A.frobenius_norm()
    assert np.linalg.norm(PAW - Wf @ fact.h_bar) <= 1e-10 * nA
    assert np.linalg.norm(fact.f - C.conj().T @ AW) <= 1e-10 * nA


def test_complex_reduced_qr_and_rank_flags(cuda):
    from paper_1604_01713_b200.dense_kernels import reduced_qr

    rng = np.random.default_rng(3)
    for n, L in ((5000, 4), (5000, 8), (3000, 16), (700, 20)):
        X = np.asfortranarray(_cplx_normal(rng, (n, L)))
        f = reduced_qr(X)
        q, r, fl = oracle.reduced_qr(X)
        Q = f.q if isinstance(f.q, np.ndarray) else f.q.cpu().numpy()
        assert np.abs(f.r_factor - r).max() <= 1e-12 * np.abs(r).max(), (n, L)
        assert np.abs(Q - q).max() <= 1e-11, (n, L)
        assert not f.flagged.any()
    # rank-deficient: column 2 = column 0 + column 1 (CholQR fails -> shifted CholQR3)
    X = np.asfortranarray(_cplx_normal(rng, (4000, 6)))
    X[:, 2] = X[:, 0] + 1j * X[:, 1]
    f = reduced_qr(X)
    _, r, fl = oracle.reduced_qr(X)
    assert f.flagged.tolist() == fl.tolist() == [False, False, True, False, False, False]
    assert np.abs(f.r_factor[:, :2] - r[:, :2]).max() <= 1e-10 * np.abs(r).max()
    Q = f.q if isinstance(f.q, np.ndarray) else f.q.cpu().numpy()
    assert np.linalg.norm(Q @ f.r_factor - X) <= 1e-12 * np.linalg.norm(X)


def test_complex_sequence_properties(cuda):
    """Config-5 shaped sequence on a 16^3 grid: every system converges, the
    true residual meets the tolerance, the estimate tracks it, and recycling
    does not cost matvecs on later systems."""
    from paper_1604_01713_b200 import problems
    from paper_1604_01713_b200.solver import SolverConfig, solve_block_gcrodr

    system, B, kw = problems.cfg5_sequence(N=16, p=16)
    cfg = SolverConfig(**kw)
    rs = None
    mv = []
    for i in range(4):
        A = system(i)
        X, rep, rs = solve_block_gcrodr(A, B, None, cfg, rs_in=rs)
        assert rep.converged, i
        assert np.iscomplexobj(X)
        true = np.linalg.norm(B - A.to_scipy() @ X, axis=0)
        assert np.all(true <= 1.01 * cfg.tol * np.linalg.norm(B, axis=0)), i
        est = rep.residual_history[-1][-1]
        assert np.allclose(est, true, rtol=1e-3, atol=1e-6 * cfg.tol * np.linalg.norm(B)), i
        assert rs is not None and rs.k == kw["k"]
        U, C = rs.numpy()
        assert np.linalg.norm(C.conj().T @ C - np.eye(rs.k)) <= 1e-10
        mv.append(rep.matvec_count)
    assert max(mv[1:]) <= mv[0], mv


def test_real_problem_in_complex_arithmetic_matches_real_solve(cuda):
    """A symmetric real system solved with a complex RHS of zero imaginary
    part follows the real solver's cycles (same Krylov and recycle spans)."""
    from paper_1604_01713_b200 import problems
    from paper_1604_01713_b200.solver import SolverConfig, solve_block_gcrodr

    A0 = problems.laplacian_3d(12)
    # a random diagonal splits the Laplacian's repeated eigenvalues
    A = problems.add_diagonal(A0, np.random.default_rng(2).uniform(0.0, 1.0, A0.n_rows))
    B = np.asfortranarray(np.random.default_rng(1).standard_normal((A.n_rows, 4)))
    cfg = SolverConfig(m=6, k=5, tol=1e-9, max_cycles=100)
    Xr, rr, rsr = solve_block_gcrodr(A, B, None, cfg)
    Xc, rc, rsc = solve_block_gcrodr(A, B.astype(np.complex128), None, cfg)
    assert rc.converged and rr.converged
    assert rc.cycles == rr.cycles and rc.matvec_count == rr.matvec_count
    assert np.abs(Xc - Xr).max() <= 1e-7 * np.abs(Xr).max()
    hr = np.concatenate(rr.residual_history)
    hc = np.concatenate(rc.residual_history)
    assert np.abs(hr - hc).max() <= 1e-8 * np.linalg.norm(B)
