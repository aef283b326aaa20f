"""GPU parity of the ILU(0) preconditioner (rg_ilu0_f64 / rg_sptrsv_f64)
against golden runs of the reference's precond.py and its preconditioned
solver paths, plus the reference's own test_precond.py properties."""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

import oracle
from conftest import csr_matrix_from, load_golden

pytestmark = pytest.mark.gpu

CASES = ("cd2d", "rand", "tri", "band")


def test_ilu0_factors_bitwise_vs_reference(cuda):
    from paper_1604_01713_b200.precond import ilu0

    g = load_golden("ilu_cases.npz")
    for name in CASES:
        A = csr_matrix_from(g, f"{name}/A/")
        F = ilu0(A)
        for part, M in (("L", F.lower), ("U", F.upper)):
            assert np.array_equal(np.asarray(M.row_ptr), g[f"{name}/{part}/row_ptr"]), (name, part)
            assert np.array_equal(np.asarray(M.col_idx), g[f"{name}/{part}/col_idx"]), (name, part)
            assert np.array_equal(M.values, g[f"{name}/{part}/values"]), (name, part)


def test_apply_precond_vs_reference(cuda):
    from paper_1604_01713_b200.precond import apply_precond, ilu0

    g = load_golden("ilu_cases.npz")
    for name in CASES:
        F = ilu0(csr_matrix_from(g, f"{name}/A/"))
        Y = apply_precond(F, g[f"{name}/X"])
        ref = g[f"{name}/Y"]
        assert Y.flags.f_contiguous
        assert np.abs(Y - ref).max() <= 1e-12 * np.abs(ref).max(), name
        # device in, device out; column subsets
        Yd = apply_precond(F, torch.from_numpy(np.asfortranarray(g[f"{name}/X"][:, :1])).to(cuda))
        assert Yd.is_cuda
        assert np.abs(Yd.cpu().numpy()[:, 0] - ref[:, 0]).max() <= 1e-12 * np.abs(ref).max()


def test_ilu0_large_vs_oracle(cuda):
    """48^3 7-point conv-diff (110,592 rows, deep wavefront): factors bitwise
    equal to the C restatement; the two solves within rounding."""
    from paper_1604_01713_b200 import problems
    from paper_1604_01713_b200.precond import apply_precond, ilu0

    A = problems.conv_diff_3d(48, 20.0)
    F = ilu0(A)
    lu, dpos = oracle.ilu0(A.row_ptr, A.col_idx, A.values)
    got = F.device_lu().vals.cpu().numpy()
    assert np.array_equal(got, lu)
    X = np.asfortranarray(np.random.default_rng(0).standard_normal((A.n_rows, 8)))
    Y = apply_precond(F, X)
    ref = oracle.apply_precond(A.row_ptr, A.col_idx, lu, dpos, X)
    assert np.abs(Y - ref).max() <= 1e-12 * np.abs(ref).max()


def test_preconditioned_solves_match_reference(cuda):
    from paper_1604_01713_b200.precond import ilu0
    from paper_1604_01713_b200.solver import SolverConfig, solve_block_gcrodr, solve_sequence

    g = load_golden("ilu_cases.npz")
    A = csr_matrix_from(g, "cd2d/A/")
    B = g["solve/B"]
    bn = np.linalg.norm(B)
    for side in ("right", "left"):
        cfg = SolverConfig(m=8, k=4, tol=1e-10, max_cycles=40, precond_side=side)
        X, rep, _ = solve_block_gcrodr(A, B, None, cfg, precond=ilu0(A))
        pre = f"solve/{side}/"
        assert rep.cycles == int(g[pre + "cycles"]), side
        assert [len(h) for h in rep.residual_history] == g[pre + "steps"].tolist(), side
        assert rep.matvec_count == int(g[pre + "matvecs"]), side
        assert rep.converged == bool(g[pre + "converged"])
        hist = np.concatenate(rep.residual_history, axis=0)
        assert np.abs(hist - g[pre + "hist"]).max() <= 1e-9 * bn, side
        assert np.abs(X - g[pre + "X"]).max() <= 1e-8 * np.abs(g[pre + "X"]).max(), side
    systems = [(csr_matrix_from(g, f"seq/A{i}/"), B) for i in range(3)]
    reps = solve_sequence(systems, SolverConfig(m=8, k=4, tol=1e-10), precond_factory=ilu0)
    for i, rep in enumerate(reps):
        pre = f"seq/sys{i}/"
        assert rep.error is None, rep.error
        assert rep.cycles == int(g[pre + "cycles"]) and rep.matvec_count == int(g[pre + "matvecs"]), i
        assert rep.recycle_origin == str(g[pre + "origin"])
        assert np.abs(np.concatenate(rep.residual_history) - g[pre + "hist"]).max() <= 1e-9 * bn, i


def test_zero_pivot_errors_match_reference(cuda):
    from paper_1604_01713_b200.precond import ZeroPivotError, ilu0
    from paper_1604_01713_b200.sparse_core import CsrMatrix

    g = load_golden("ilu_cases.npz")
    for key in ("zero_pivot_mid", "missing_diag"):
        M = sp.csr_matrix(g[f"err/{key}_A/dense"])
        M.eliminate_zeros()
        with pytest.raises(ZeroPivotError) as e:
            ilu0(CsrMatrix.from_scipy(M))
        assert str(e.value) == str(g[f"err/{key}"])


def test_reference_precond_properties(cuda):
    """test_precond.py's cases: identity, no-fill exactness, A-inverse action,
    shape errors."""
    from paper_1604_01713_b200.precond import Ilu0Factors, apply_precond, ilu0
    from paper_1604_01713_b200.sparse_core import CsrMatrix, ShapeError

    F = ilu0(CsrMatrix.from_scipy(sp.eye(4, format="csr")))
    assert F.lower.nnz == 0 and np.array_equal(F.upper.to_scipy().toarray(), np.eye(4))
    X = np.arange(8.0).reshape(4, 2)
    assert np.allclose(apply_precond(F, X), X)
    T = sp.diags([np.full(5, -1.0), np.full(6, 3.0), np.full(5, -1.5)], [-1, 0, 1], format="csr")
    A = CsrMatrix.from_scipy(T)
    F = ilu0(A)
    Lf = F.lower.to_scipy() + sp.eye(6)
    assert np.abs((Lf @ F.upper.to_scipy()).toarray() - T.toarray()).max() <= 1e-14  # no fill -> exact LU
    Xr = np.random.default_rng(1).standard_normal((6, 3))
    assert np.allclose(apply_precond(F, T @ Xr), Xr, atol=1e-12)
    with pytest.raises(ShapeError):
        apply_precond(F, np.ones((4, 1)))
    with pytest.raises(ShapeError):
        ilu0(CsrMatrix.from_scipy(sp.csr_matrix(np.ones((2, 3)))))
    # factors given as host CsrMatrix objects (the reference constructor)
    G = Ilu0Factors(lower=F.lower, upper=F.upper)
    assert np.allclose(apply_precond(G, T @ Xr), Xr, atol=1e-12)


def test_level_ordered_solve_matches_original_order(cuda):
    """The permuted row-major wavefront (apply) and the original-order one
    (solve x2) do the same arithmetic: bitwise equal."""
    from paper_1604_01713_b200 import device as D, problems
    from paper_1604_01713_b200.precond import ilu0

    A = problems.conv_diff_3d(24, 20.0)
    lu = ilu0(A).device_lu()
    X = D.to_device_block(np.random.default_rng(3).standard_normal((A.n_rows, 11)))
    Y1 = D.empty_block(A.n_rows, 11)
    lu.apply(X, Y1)
    Y2 = D.empty_block(A.n_rows, 11)
    lu.solve(X, Y2, upper=False)
    lu.solve(Y2, Y2, upper=True)
    assert torch.equal(Y1, Y2)
