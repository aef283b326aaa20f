"""The reference's solver-level behaviours (its tests/test_solver.py groups:
config validation, block GMRES, GCRO-DR, block enlargement, sequences),
re-checked against this package on the GPU with our own seeded problems."""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

pytestmark = pytest.mark.gpu


def _mat(n, density, seed, shift):
    from paper_1604_01713_b200 import CsrMatrix

    g = np.random.default_rng(seed)
    M = sp.random(n, n, density=density, random_state=g, format="csr") + shift * sp.eye(n, format="csr")
    M = sp.csr_matrix(M)
    M.sort_indices()
    return CsrMatrix.from_scipy(M)


def _rhs(n, p, seed):
    return np.asfortranarray(np.random.default_rng(seed).uniform(0.0, 1.0, (n, p)))


def _dense(A):
    return A.to_scipy().toarray()


# ---------------------------------------------------------------- block GMRES


def test_identity_operator_single_step(cuda):
    from paper_1604_01713_b200 import CsrMatrix, SolverConfig, solve_block_gmres

    A = CsrMatrix.from_scipy(sp.eye(12, format="csr"))
    B = _rhs(12, 3, 100)
    X, rep, _ = solve_block_gmres(A, B, cfg=SolverConfig(m=4, tol=1e-12))
    assert rep.converged and rep.cycles == 1 and len(rep.residual_history[0]) == 1
    assert np.abs(X - B).max() <= 1e-12


def test_block_history_dominates_single_columns(cuda):
    from paper_1604_01713_b200 import CsrMatrix, SolverConfig, solve_block_gmres

    n = 24
    A = CsrMatrix.from_coo(n, n, range(n), range(n), np.linspace(1.0, 5.0, n))
    B = _rhs(n, 3, 101)
    cfg = SolverConfig(m=12, tol=1e-14, max_cycles=1, early_exit=False)
    _, rb, _ = solve_block_gmres(A, B, cfg=cfg)
    hb = rb.residual_history[0]
    for j in range(3):
        _, r1, _ = solve_block_gmres(A, B[:, j:j + 1], cfg=cfg)
        h1 = r1.residual_history[0][:, 0]
        s = min(len(hb), len(h1))
        assert np.all(hb[:s, j] <= h1[:s] + 1e-12)


def test_gmres_true_residual_and_monotone_history(cuda):
    from paper_1604_01713_b200 import SolverConfig, solve_block_gmres

    A = _mat(50, 0.2, 102, 5.0)
    B = _rhs(50, 2, 103)
    X, rep, _ = solve_block_gmres(A, B, cfg=SolverConfig(m=14, tol=1e-10, max_cycles=20))
    assert rep.converged
    assert np.linalg.norm(B - _dense(A) @ X) <= 1e-10 * np.linalg.norm(B)
    _, rep, _ = solve_block_gmres(A, B, cfg=SolverConfig(m=10, tol=1e-13, max_cycles=3, early_exit=False))
    for h in rep.residual_history:
        assert np.all(np.diff(h, axis=0) <= 1e-10)


def test_nonconvergence_is_reported(cuda):
    from paper_1604_01713_b200 import SolverConfig, solve_block_gmres

    A = _mat(45, 0.3, 104, 0.1)
    X, rep, _ = solve_block_gmres(A, _rhs(45, 1, 105), cfg=SolverConfig(m=2, tol=1e-14, max_cycles=2))
    assert not rep.converged and rep.error is None and rep.cycles == 2


def test_initial_guess_and_operator_kinds(cuda):
    from paper_1604_01713_b200 import HostOperator, SolverConfig, solve_block_gmres
    from paper_1604_01713_b200.sparse_core import spmm_device

    A = _mat(30, 0.3, 106, 5.0)
    Ad = _dense(A)
    B = _rhs(30, 1, 107)
    cfg = SolverConfig(m=12, tol=1e-10)
    X, rep, _ = solve_block_gmres(A, B, _rhs(30, 1, 108), cfg)
    assert rep.converged and np.linalg.norm(B - Ad @ X) <= 1e-9 * np.linalg.norm(B)
    # a device closure and a numpy closure (HostOperator) give the same solve
    Xd, rd, _ = solve_block_gmres(lambda Z: spmm_device(A, Z), B, cfg=cfg)
    Xh, rh, _ = solve_block_gmres(HostOperator(lambda Z: Ad @ Z), B, cfg=cfg)
    assert rd.converged and rh.converged
    assert np.linalg.norm(Xd - Xh) <= 1e-8 * np.linalg.norm(Xd)


def test_matvec_accounting(cuda):
    from paper_1604_01713_b200 import SolverConfig, solve_block_gmres

    A = _mat(30, 0.3, 109, 5.0)
    cfg = SolverConfig(m=5, tol=1e-14, max_cycles=1, early_exit=False, residual_replace=False)
    _, rep, _ = solve_block_gmres(A, _rhs(30, 3, 110), cfg=cfg)
    assert rep.matvec_count == 3 + 5 * 3  # the initial residual, then m block steps of width p


# ---------------------------------------------------------------- GCRO-DR


def test_full_space_recycle_solves_by_projection(cuda):
    from paper_1604_01713_b200 import SolverConfig, solve_block_gcrodr
    from paper_1604_01713_b200.recycling import RecycleSpace, prepare_cross_system
    from paper_1604_01713_b200.sparse_core import spmm_device

    A = _mat(14, 0.5, 111, 5.0)
    Ad = _dense(A)
    rs = prepare_cross_system(RecycleSpace(u=np.linalg.inv(Ad), c=np.eye(14)), lambda Z: spmm_device(A, Z))
    b = _rhs(14, 1, 112)
    X, rep, _ = solve_block_gcrodr(A, b, None, SolverConfig(m=5, k=14, tol=1e-10), rs_in=rs)
    assert rep.converged and rep.cycles == 0
    assert np.linalg.norm(b - Ad @ X) <= 1e-9 * np.linalg.norm(b)


def test_gcrodr_residual_estimates_and_recycle_invariants(cuda):
    from paper_1604_01713_b200 import SolverConfig, solve_block_gcrodr

    A = _mat(48, 0.25, 113, 2.0)
    Ad = _dense(A)
    B = _rhs(48, 2, 114)
    X, rep, rs = solve_block_gcrodr(A, B, None, SolverConfig(m=8, k=5, tol=1e-10, max_cycles=30, early_exit=False))
    assert rep.converged
    bn = np.linalg.norm(B)
    for h, true in zip(rep.residual_history, rep.cycle_true_residuals):
        assert abs(np.linalg.norm(h[-1]) - np.linalg.norm(true)) <= 1e-8 * bn
    assert abs(rep.final_residual_norm - np.linalg.norm(B - Ad @ X)) <= 1e-8 * bn
    U, C = rs.numpy()
    assert np.linalg.norm(C.T @ C - np.eye(rs.k)) <= 1e-10 * rs.k
    assert np.linalg.norm(Ad @ U - C) <= 1e-10 * np.linalg.norm(Ad) * np.linalg.norm(U)


def test_residual_orthogonal_to_recycle_space(cuda):
    from paper_1604_01713_b200 import SolverConfig, solve_block_gcrodr
    from paper_1604_01713_b200.recycling import RecycleSpace, prepare_cross_system
    from paper_1604_01713_b200.sparse_core import spmm_device

    A = _mat(36, 0.3, 115, 2.0)
    rs = prepare_cross_system(RecycleSpace(u=_rhs(36, 4, 116), c=None), lambda Z: spmm_device(A, Z))
    b = _rhs(36, 1, 117)
    cfg = SolverConfig(m=6, k=4, tol=1e-12, max_cycles=2, early_exit=False, update_recycle=False,
                       residual_replace=False)
    X, rep, _ = solve_block_gcrodr(A, b, None, cfg, rs_in=rs)
    R = b - _dense(A) @ X
    C = rs.numpy()[1]
    assert np.linalg.norm(C.T @ R) <= 1e-8 * np.linalg.norm(R)


def test_k_zero_is_block_gmres(cuda):
    from paper_1604_01713_b200 import SolverConfig, solve_block_gcrodr, solve_block_gmres

    A = _mat(32, 0.3, 118, 4.0)
    B = _rhs(32, 2, 119)
    cfg = SolverConfig(m=8, k=0, tol=1e-10)
    X1, r1, _ = solve_block_gcrodr(A, B, None, cfg)
    X2, r2, _ = solve_block_gmres(A, B, None, cfg)
    assert np.allclose(X1, X2) and r1.matvec_count == r2.matvec_count


def test_enlarged_per_column_and_mgs(cuda):
    from paper_1604_01713_b200 import SolverConfig, solve_block_gcrodr

    A = _mat(44, 0.25, 120, 2.0)
    Ad = _dense(A)
    b = _rhs(44, 1, 121)
    X, rep, _ = solve_block_gcrodr(A, b, None, SolverConfig(m=8, k=4, block_width=3, tol=1e-10, max_cycles=30))
    assert rep.converged and np.linalg.norm(b - Ad @ X) <= 1e-9 * np.linalg.norm(b)
    B = _rhs(44, 2, 122)
    X, rep, _ = solve_block_gcrodr(A, B, None, SolverConfig(m=10, k=4, tol=1e-8, stop_rule="per-column-relative"))
    assert rep.converged
    assert np.all(np.linalg.norm(B - Ad @ X, axis=0) <= 1e-7 * np.linalg.norm(B, axis=0))
    X, rep, _ = solve_block_gcrodr(A, B, None, SolverConfig(m=10, k=4, tol=1e-10, ortho="mgs"))
    assert rep.converged


def test_ilu_preconditioned_banded(cuda):
    from paper_1604_01713_b200 import SolverConfig, gen_banded, ilu0, solve_block_gcrodr

    A = gen_banded(240, 3, 123)
    Ad = _dense(A)
    b = _rhs(240, 1, 124)
    X, rep, _ = solve_block_gcrodr(A, b, None, SolverConfig(m=10, k=5, tol=1e-10, max_cycles=10), precond=ilu0(A))
    assert rep.converged and rep.cycles <= 2
    assert np.linalg.norm(b - Ad @ X) <= 1e-9 * np.linalg.norm(b)
    X, rep, _ = solve_block_gcrodr(A, b, None, SolverConfig(m=10, k=5, tol=1e-10, max_cycles=10,
                                                             precond_side="left"), precond=ilu0(A))
    assert rep.converged and np.linalg.norm(b - Ad @ X) <= 1e-8 * np.linalg.norm(b)


# ---------------------------------------------------------------- enlargement


def test_enlarge_block_rules(cuda):
    from paper_1604_01713_b200 import ShapeError, enlarge_block
    from paper_1604_01713_b200 import device as D

    r = _rhs(16, 1, 125)
    assert enlarge_block(r, 1, 0) is r
    R = enlarge_block(r, 4, 9)
    assert R.shape == (16, 4) and np.array_equal(R[:, 0], r[:, 0])
    assert np.array_equal(enlarge_block(r, 4, 9), R)
    Rd = enlarge_block(D.to_device_block(r), 4, 9)  # device input: the same host draws
    assert np.array_equal(D.to_numpy_block(Rd), R)
    with pytest.raises(ShapeError):
        enlarge_block(np.ones((5, 2)), 3, 0)


# ---------------------------------------------------------------- sequences


def test_sequence_behaviours(cuda):
    from paper_1604_01713_b200 import SolverConfig, gen_banded, ilu0, solve_block_gcrodr, solve_sequence

    A = _mat(70, 0.15, 126, 1.0)
    b = _rhs(70, 1, 127)
    reps = solve_sequence([(A, b), (A, b)], SolverConfig(m=10, k=20, tol=1e-8, max_cycles=40))
    assert all(r.converged for r in reps) and reps[1].matvec_count < reps[0].matvec_count
    cfg = SolverConfig(m=8, k=4, tol=1e-10)
    one = solve_sequence([(A, b)], cfg)[0]
    X, rep, _ = solve_block_gcrodr(A, b, None, cfg)
    assert np.allclose(one.solution, X) and one.matvec_count == rep.matvec_count
    Aw = _mat(30, 0.3, 133, 4.0)
    reps = solve_sequence([(Aw, _rhs(9, 1, 128)), (Aw, _rhs(30, 1, 134))], cfg)
    assert reps[0].error is not None and reps[1].converged
    with pytest.raises(ValueError):
        solve_sequence([])
    Ab = gen_banded(160, 2, 129)
    reps = solve_sequence([(Ab, _rhs(160, 1, 130 + i)) for i in range(2)], SolverConfig(m=10, k=5, tol=1e-10),
                          precond_factory=ilu0)
    assert all(r.converged for r in reps)


def test_device_inputs_and_outputs(cuda):
    """CUDA-tensor right-hand sides are accepted in place of numpy blocks."""
    from paper_1604_01713_b200 import SolverConfig, solve_block_gcrodr

    A = _mat(40, 0.25, 131, 3.0)
    B = _rhs(40, 2, 132)
    X1, r1, _ = solve_block_gcrodr(A, B, None, SolverConfig(m=8, k=4, tol=1e-10))
    X2, r2, _ = solve_block_gcrodr(A, torch.from_numpy(B).to(cuda), None, SolverConfig(m=8, k=4, tol=1e-10))
    assert np.array_equal(X1, X2) and r1.matvec_count == r2.matvec_count


@pytest.mark.parametrize("p", [12, 20, 36])
def test_wide_blocks_solve(cuda, p):
    """Block widths beyond one tall launch (p > 16: wide tiles; p > 32:
    column-blocked passes) through the whole GCRO-DR path."""
    from paper_1604_01713_b200 import SolverConfig, solve_block_gcrodr

    A = _mat(400, 0.02, 140 + p, 3.0)
    B = _rhs(400, p, 141 + p)
    X, rep, rs = solve_block_gcrodr(A, B, None, SolverConfig(m=4, k=6, tol=1e-9, max_cycles=40))
    assert rep.converged
    assert np.linalg.norm(B - _dense(A) @ X) <= 1e-8 * np.linalg.norm(B)
    U, C = rs.numpy()
    assert np.linalg.norm(C.T @ C - np.eye(rs.k)) <= 1e-10 * rs.k


def test_complex_driver_paths(cuda):
    """Complex GMRES, complex enlargement of a single right-hand side, MGS,
    and a real matrix with a complex right-hand side."""
    from paper_1604_01713_b200 import CsrMatrix, SolverConfig, solve_block_gcrodr, solve_block_gmres

    g = np.random.default_rng(150)
    n = 300
    M = sp.random(n, n, density=0.02, random_state=g, format="csr") * (1 + 0.5j) + (4 + 1j) * sp.eye(n)
    A = CsrMatrix.from_scipy(sp.csr_matrix(M))
    Ad = M.toarray()
    B = g.standard_normal((n, 2)) + 1j * g.standard_normal((n, 2))
    X, rep, _ = solve_block_gmres(A, B, cfg=SolverConfig(m=10, tol=1e-10, max_cycles=30))
    assert rep.converged and np.linalg.norm(B - Ad @ X) <= 1e-9 * np.linalg.norm(B)
    b = B[:, :1]
    X, rep, _ = solve_block_gcrodr(A, b, None, SolverConfig(m=6, k=4, block_width=3, tol=1e-10, max_cycles=40))
    assert rep.converged and np.linalg.norm(b - Ad @ X) <= 1e-9 * np.linalg.norm(b)
    X, rep, _ = solve_block_gcrodr(A, B, None, SolverConfig(m=6, k=4, tol=1e-10, ortho="mgs", max_cycles=40))
    assert rep.converged and np.linalg.norm(B - Ad @ X) <= 1e-9 * np.linalg.norm(B)
    Ar = _mat(n, 0.02, 151, 4.0)
    X, rep, _ = solve_block_gcrodr(Ar, B, None, SolverConfig(m=6, k=4, tol=1e-10, max_cycles=40))
    assert np.iscomplexobj(X) and rep.converged
    assert np.linalg.norm(B - _dense(Ar) @ X) <= 1e-9 * np.linalg.norm(B)


@pytest.mark.parametrize("n", [1, 2, 3, 33])
def test_tiny_systems(cuda, n):
    from paper_1604_01713_b200 import SolverConfig, solve_block_gcrodr

    A = _mat(n, 0.5, 160 + n, 3.0)
    B = _rhs(n, 1, 161)
    X, rep, _ = solve_block_gcrodr(A, B, None, SolverConfig(m=4, k=2, tol=1e-12, max_cycles=20))
    assert rep.converged
    assert np.linalg.norm(B - _dense(A) @ X) <= 1e-11 * np.linalg.norm(B)
