"""Round-2 golden fixtures from the REAL reference (run here, where
/root/reference exists):

    python tests/golden/make_golden_r2.py

Writes tests/golden/r2_cases.npz with
  * mgs/<case>      block Arnoldi with ortho="mgs" (arnoldi.py:159-170):
                    W, H, F, z_bar after m steps, with and without C
  * unscrubbed      cgs2 Arnoldi with a recycle space but an R0 that was NOT
                    projected against C first (arnoldi.start does not do it;
                    the joint [C W] schedule must not be used for it)
  * wide/<case>     cgs2 Arnoldi whose basis grows past 128 columns
                    (m = 20, L = 8: w up to 168), with and without C
  * wide_solve      solve_block_gcrodr with m = 20, p = 8, k = 20 (the
                    default-shaped cycle that ran into the 128-column limit)
  * rgmrecyc        the bytes of a file the reference's save_recycle_space
                    wrote (recycling.py:201-209), and the (u, c) it holds
"""

from __future__ import annotations

import pathlib
import sys
import tempfile

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parents[1]))

from make_golden import _csr_arrays, _import_reference, _report_arrays, kron_conv_diff_2d  # noqa: E402


def main():
    _import_reference()
    from recgmres import arnoldi
    from recgmres.recycling import RecycleSpace, prepare_cross_system, save_recycle_space
    from recgmres.solver import SolverConfig, solve_block_gcrodr
    from recgmres.sparse_core import CsrMatrix, spmm
    from conftest import random_csr

    out = {}
    op_of = lambda A: (lambda Z: spmm(A, Z))

    def arnoldi_case(name, A, R0, m, k, seed, ortho, scrub=True):
        rs = None
        if k:
            U0 = np.random.default_rng(seed).standard_normal((A.n_rows, k))
            rs = prepare_cross_system(RecycleSpace(u=U0, c=U0), op_of(A))
            if scrub:
                R0 = R0 - rs.c @ (rs.c.T @ R0)
            out[f"{name}/U"] = rs.u
            out[f"{name}/C"] = rs.c
        fact = arnoldi.start(op_of(A), R0, m_max=m, recycle=rs, seed=seed)
        for _ in range(m):
            arnoldi.step(fact, op_of(A), recycle=rs, ortho=ortho)
        _csr_arrays(f"{name}/", A.to_scipy(), out)
        out[f"{name}/R0"] = np.asfortranarray(R0)
        out[f"{name}/W"] = fact.w
        out[f"{name}/H"] = fact.h_bar
        out[f"{name}/F"] = fact.f
        out[f"{name}/z_bar"] = fact.z_bar
        out[f"{name}/m"] = np.array(m)
        out[f"{name}/k"] = np.array(k)
        out[f"{name}/seed"] = np.array(seed)
        out[f"{name}/events"] = np.array(len(fact.breakdown_events))

    # ---- MGS (arnoldi.py:159-170)
    arnoldi_case("mgs/plain_n300_L3", random_csr(300, 0.03, 21, shift=3.0),
                 np.random.default_rng(22).standard_normal((300, 3)), 6, 0, 2, "mgs")
    arnoldi_case("mgs/recyc_n400_L4_k5", random_csr(400, 0.02, 23, shift=3.0),
                 np.random.default_rng(24).standard_normal((400, 4)), 7, 5, 3, "mgs")
    # ---- unscrubbed R0 with a recycle space (joint schedule gating)
    arnoldi_case("unscrubbed", random_csr(500, 0.02, 25, shift=3.0),
                 np.random.default_rng(26).standard_normal((500, 4)), 6, 6, 4, "cgs2", scrub=False)
    # ---- bases wider than one 128-column Gram launch
    A2 = CsrMatrix.from_scipy(kron_conv_diff_2d(32, 10.0))
    arnoldi_case("wide/plain_L8_m20", A2, np.random.default_rng(27).standard_normal((A2.n_rows, 8)), 20, 0, 5, "cgs2")
    arnoldi_case("wide/recyc_L8_m20_k20", A2, np.random.default_rng(28).standard_normal((A2.n_rows, 8)), 20, 20, 6,
                 "cgs2")
    # ---- a solve whose cycles reach w = 168 with k = 20
    A3 = kron_conv_diff_2d(32, 10.0)
    B3 = np.random.default_rng(29).standard_normal((A3.shape[0], 8))
    X, rep, rs = solve_block_gcrodr(CsrMatrix.from_scipy(A3), B3, None,
                                    SolverConfig(m=20, k=20, tol=1e-9, max_cycles=6))
    _csr_arrays("wide_solve/", A3, out)
    out["wide_solve/B"] = B3
    _report_arrays("wide_solve/", rep, out, with_solution=True)
    # ---- RGMRECYC written by the reference
    with tempfile.TemporaryDirectory() as td:
        path = pathlib.Path(td) / "rs.bin"
        save_recycle_space(rs, path)
        out["rgmrecyc/bytes"] = np.frombuffer(path.read_bytes(), dtype=np.uint8)
    out["rgmrecyc/u"] = np.asfortranarray(rs.u)
    out["rgmrecyc/c"] = np.asfortranarray(rs.c)
    np.savez_compressed(HERE / "r2_cases.npz", **out)
    print("wrote", HERE / "r2_cases.npz", f"(wide_solve: {rep.cycles} cycles, {rep.matvec_count} matvecs, "
          f"converged={rep.converged})")


if __name__ == "__main__":
    main()
