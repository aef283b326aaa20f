"""Golden fixtures for the ILU(0) preconditioner, produced by the REAL
reference (``recgmres.precond`` / ``recgmres.solver``).  Run in the build
container:

    python tests/golden/make_golden_ilu.py

Writes tests/golden/ilu_cases.npz:
  <case>/A/*          input CSR
  <case>/L/*, /U/*    reference ilu0 factors (precond.py:33-76)
  <case>/X, /Y        a seeded block and apply_precond(F, X) (precond.py:79-90)
  solve/<side>/*      preconditioned solve_block_gcrodr reports (right, left)
  seq/sys<i>/*        solve_sequence(..., precond_factory=ilu0) reports
  err/<name>          messages of the reference's ZeroPivotError cases
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from make_golden import OUT, _csr_arrays, _import_reference, _report_arrays, kron_conv_diff_2d


def _random_pattern(n, density, seed, shift):
    rng = np.random.default_rng(seed)
    M = sp.random(n, n, density=density, format="csr", random_state=rng, data_rvs=lambda k: rng.uniform(-1, 1, k))
    return sp.csr_matrix(M + sp.diags(np.full(n, shift)))


def main():
    _import_reference()
    from recgmres.precond import ZeroPivotError, apply_precond, ilu0
    from recgmres.solver import SolverConfig, solve_block_gcrodr, solve_sequence
    from recgmres.sparse_core import CsrMatrix, gen_banded

    out = {}
    cases = {
        "cd2d": kron_conv_diff_2d(24, 10.0),  # 5-point: ILU(0) has dropped fill
        "rand": _random_pattern(400, 0.02, 7, 6.0),  # unstructured, fill dropped
        "tri": sp.diags([np.full(49, -1.0), np.full(50, 2.5), np.full(49, -1.2)], [-1, 0, 1], format="csr"),
    }
    banded = gen_banded(300, 3, seed=11)
    cases["band"] = banded.to_scipy()
    rng = np.random.default_rng(5)
    for name, A in cases.items():
        A = sp.csr_matrix(A)
        A.sort_indices()
        _csr_arrays(f"{name}/A/", A, out)
        F = ilu0(CsrMatrix.from_scipy(A))
        _csr_arrays(f"{name}/L/", F.lower.to_scipy(), out)
        _csr_arrays(f"{name}/U/", F.upper.to_scipy(), out)
        X = np.asfortranarray(rng.standard_normal((A.shape[0], 3)))
        out[f"{name}/X"] = X
        out[f"{name}/Y"] = apply_precond(F, X)

    # preconditioned solves (2-D conv-diff 24x24, p=2)
    A = CsrMatrix.from_scipy(cases["cd2d"])
    B = np.asfortranarray(rng.uniform(-1.0, 1.0, (A.n_rows, 2)))
    out["solve/B"] = B
    for side in ("right", "left"):
        cfg = SolverConfig(m=8, k=4, tol=1e-10, max_cycles=40, precond_side=side)
        _, rep, _ = solve_block_gcrodr(A, B, None, cfg, precond=ilu0(A))
        _report_arrays(f"solve/{side}/", rep, out)
    # sequence with a per-system factorisation (test_acceptance.py:345 style)
    d = rng.uniform(0.0, 1.0, A.n_rows)
    mats = [sp.csr_matrix(cases["cd2d"] + sp.diags(0.05 * i * d)) for i in range(3)]
    for i, M in enumerate(mats):
        _csr_arrays(f"seq/A{i}/", M, out)
    reps = solve_sequence([(CsrMatrix.from_scipy(M), B) for M in mats], SolverConfig(m=8, k=4, tol=1e-10),
                          precond_factory=ilu0)
    for i, rep in enumerate(reps):
        _report_arrays(f"seq/sys{i}/", rep, out)

    # error messages
    def msg(M):
        try:
            ilu0(CsrMatrix.from_scipy(sp.csr_matrix(M)))
        except ZeroPivotError as e:
            return str(e)
        return ""

    out["err/zero_pivot"] = np.array(msg(np.array([[0.0, 1.0], [1.0, 0.0]])))
    z = sp.csr_matrix(np.array([[1.0, 2.0, 0.0], [3.0, 6.0, 1.0], [0.0, 1.0, 4.0]]))
    out["err/zero_pivot_mid"] = np.array(msg(z))
    out["err/zero_pivot_mid_A/dense"] = z.toarray()
    m = sp.csr_matrix(np.array([[1.0, 0.0, 0.0], [1.0, 0.0, 1.0], [0.0, 1.0, 1.0]]))
    m.eliminate_zeros()
    out["err/missing_diag"] = np.array(msg(m))
    out["err/missing_diag_A/dense"] = m.toarray()
    np.savez_compressed(OUT / "ilu_cases.npz", **out)
    print("wrote", OUT / "ilu_cases.npz")


if __name__ == "__main__":
    main()
