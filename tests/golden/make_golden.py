"""Generate the golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch directory (numba's cache=True would
otherwise write into the read-only reference tree), imports ``recgmres`` from
there, runs the reference's own functions on seeded inputs and writes
``tests/golden/*.npz``.  The GPU box never has /root/reference; tests there
read only these committed fixtures.

Synthetic problem recipes (the paper's UF / Tramonto / sherman5
matrices are not available): they are defined HERE with scipy ``kron`` sums,
and the product's direct CSR generators (paper_1604_01713_b200/problems.py)
must reproduce them bit for bit (tests/test_problems.py).
"""

from __future__ import annotations

import os
import pathlib
import shutil
import sys
import tempfile

import numpy as np
import scipy.sparse as sp

OUT = pathlib.Path(__file__).resolve().parent
REF_PKG = pathlib.Path("/root/reference/pkg")


def _import_reference():
    scratch = pathlib.Path(tempfile.mkdtemp(prefix="refcopy_"))
    shutil.copytree(REF_PKG, scratch / "pkg")
    os.environ.setdefault("NUMBA_CACHE_DIR", str(scratch / "numba_cache"))
    sys.path.insert(0, str(scratch / "pkg" / "src"))
    sys.path.insert(0, str(scratch / "pkg" / "tests"))
    import recgmres  # noqa: F401

    return scratch


# ---------------------------------------------------------------------------
# recipes (kron form)
# ---------------------------------------------------------------------------


def _tri(N, lo, di, up):
    return sp.diags([np.full(N - 1, lo), np.full(N, di), np.full(N - 1, up)], [-1, 0, 1], format="csr")


def kron_conv_diff_2d(N, beta):
    """-Lap u + beta (u_x + u_y), 5-point, h = 1/(N+1), Dirichlet eliminated."""
    h = 1.0 / (N + 1)
    T = _tri(N, -1.0, 2.0, -1.0) / h**2
    D = sp.diags([np.full(N - 1, -1.0), np.full(N - 1, 1.0)], [-1, 1], format="csr") / (2 * h)
    I = sp.eye(N, format="csr")
    A = (sp.kron(I, T) + sp.kron(T, I)) + beta * (sp.kron(I, D) + sp.kron(D, I))
    return sp.csr_matrix(A)


def kron_conv_diff_3d(N, beta):
    h = 1.0 / (N + 1)
    T = _tri(N, -1.0, 2.0, -1.0) / h**2
    D = sp.diags([np.full(N - 1, -1.0), np.full(N - 1, 1.0)], [-1, 1], format="csr") / (2 * h)
    I = sp.eye(N, format="csr")
    K = lambda a, b, c: sp.kron(sp.kron(a, b), c)
    A = ((K(I, I, T) + K(I, T, I)) + K(T, I, I)) + beta * ((K(I, I, D) + K(I, D, I)) + K(D, I, I))
    return sp.csr_matrix(A)


def kron_laplacian_3d(N):
    """Unscaled 7-point Laplacian (diagonal 6, off-diagonals -1)."""
    T = _tri(N, -1.0, 2.0, -1.0)
    I = sp.eye(N, format="csr")
    K = lambda a, b, c: sp.kron(sp.kron(a, b), c)
    return sp.csr_matrix((K(I, I, T) + K(I, T, I)) + K(T, I, I))


def _csr_arrays(prefix, A, out):
    A = sp.csr_matrix(A)
    A.sort_indices()
    out[prefix + "row_ptr"] = A.indptr.astype(np.int32)
    out[prefix + "col_idx"] = A.indices.astype(np.int32)
    out[prefix + "values"] = A.data.astype(np.float64)
    out[prefix + "shape"] = np.array(A.shape, dtype=np.int64)


# ---------------------------------------------------------------------------
# fixtures
# ---------------------------------------------------------------------------


def gen_spmm():
    from recgmres.sparse_core import CsrMatrix, gen_banded, spmm
    from conftest import random_csr

    out = {}
    cases = []

    def add(name, A, X):
        Y = spmm(A, X)
        _csr_arrays(f"{name}/", A.to_scipy(), out)
        out[f"{name}/X"] = np.asfortranarray(X)
        out[f"{name}/Y"] = Y
        cases.append(name)

    add("ref_test_50", random_csr(50, density=0.1, seed=7), np.random.default_rng(7).standard_normal((50, 4)))
    for p in (1, 3, 8, 16, 20):
        add(f"rand200_p{p}", random_csr(200, density=0.05, seed=3, shift=1.0),
            np.random.default_rng(100 + p).standard_normal((200, p)))
    add("convdiff2d_16_p4", CsrMatrix.from_scipy(kron_conv_diff_2d(16, 10.0)),
        np.random.default_rng(1).uniform(-1, 1, (256, 4)))
    add("lap3d_8_p8", CsrMatrix.from_scipy(kron_laplacian_3d(8)), np.random.default_rng(2).standard_normal((512, 8)))
    add("banded_1000_p4", gen_banded(1000, 5, 0), np.random.default_rng(3).uniform(0, 1, (1000, 4)))
    # ragged / edge inputs: empty rows, a long row, rectangular, 1x1
    rng = np.random.default_rng(4)
    M = sp.random(64, 64, density=0.05, random_state=rng, format="lil")
    M[5, :] = 0.0
    M[6, :] = rng.standard_normal(64)  # dense row
    M[63, :] = 0.0
    add("ragged_64_p5", CsrMatrix.from_scipy(sp.csr_matrix(M)), rng.standard_normal((64, 5)))
    R = sp.random(30, 50, density=0.2, random_state=np.random.default_rng(5), format="csr")
    add("rect_30x50_p2", CsrMatrix.from_scipy(R), np.random.default_rng(6).standard_normal((50, 2)))
    add("one_1x1", CsrMatrix.from_coo(1, 1, [0], [0], [3.5]), np.array([[2.0]]))
    # cancellation-heavy values: exposes any FMA contraction
    V = sp.random(300, 300, density=0.04, random_state=np.random.default_rng(8), format="csr")
    V.data = np.random.default_rng(9).standard_normal(V.nnz) * 10.0 ** np.random.default_rng(10).integers(-8, 8, V.nnz)
    add("wide_range_300_p8", CsrMatrix.from_scipy(V), np.random.default_rng(11).standard_normal((300, 8)))
    out["cases"] = np.array(cases)
    np.savez_compressed(OUT / "spmm_cases.npz", **out)


def gen_qr():
    from recgmres.dense_kernels import reduced_qr

    out = {}
    cases = []

    def add(name, X, tol=1e-12):
        f = reduced_qr(X, rank_tol=tol)
        out[f"{name}/X"] = np.asfortranarray(X)
        out[f"{name}/q"] = f.q
        out[f"{name}/r"] = f.r_factor
        out[f"{name}/flagged"] = f.flagged
        out[f"{name}/rank"] = np.array(f.rank)
        cases.append(name)

    add("three_four_five", np.array([[3.0], [4.0]]))
    add("rand_8x3", np.random.default_rng(1).standard_normal((8, 3)))
    for p in (1, 4, 8, 16, 20):
        add(f"rand_2000x{p}", np.random.default_rng(10 + p).standard_normal((2000, p)))
    x = np.random.default_rng(3).standard_normal((6, 1))
    add("rank_def_6x2", np.hstack([x, 2.0 * x]))
    y = np.random.default_rng(4).standard_normal((1500, 8))
    y[:, 5] = y[:, 1] - 0.5 * y[:, 2]
    add("rank_def_1500x8", y)
    add("orthonormal_7x3", np.linalg.qr(np.random.default_rng(0).standard_normal((7, 3)))[0])
    # scaled columns (condition ~1e6) exercise the Cholesky fallback decision
    z = np.random.default_rng(5).standard_normal((1500, 8)) * np.logspace(0, -6, 8)
    add("graded_1500x8", z)
    out["cases"] = np.array(cases)
    np.savez_compressed(OUT / "qr_cases.npz", **out)


def gen_arnoldi():
    from recgmres import arnoldi
    from recgmres.recycling import RecycleSpace, prepare_cross_system
    from recgmres.sparse_core import spmm
    from conftest import random_csr

    out = {}
    cases = []
    op_of = lambda A: (lambda Z: spmm(A, Z))

    def add(name, A, R0, m, k, seed):
        rs = None
        if k:
            U0 = np.random.default_rng(seed).standard_normal((A.n_rows, k))
            rs = prepare_cross_system(RecycleSpace(u=U0, c=U0), op_of(A))
            R0 = R0 - rs.c @ (rs.c.T @ R0)
            out[f"{name}/U"] = rs.u
            out[f"{name}/C"] = rs.c
        fact = arnoldi.start(op_of(A), R0, m_max=m, recycle=rs, seed=seed)
        for _ in range(m):
            arnoldi.step(fact, op_of(A), recycle=rs, ortho="cgs2")
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
        cases.append(name)

    add("plain_n30_L2", random_csr(30, 0.3, 4, shift=2.0), np.random.default_rng(4).standard_normal((30, 2)), 5, 0, 0)
    add("recyc_n30_L2_k3", random_csr(30, 0.3, 5, shift=2.0), np.random.default_rng(6).standard_normal((30, 2)), 5, 3, 6)
    add("recyc_n400_L4_k6", random_csr(400, 0.02, 9, shift=3.0), np.random.default_rng(7).standard_normal((400, 4)), 8, 6, 9)
    add("plain_n500_L8", random_csr(500, 0.02, 11, shift=3.0), np.random.default_rng(12).standard_normal((500, 8)), 6, 0, 1)
    out["cases"] = np.array(cases)
    np.savez_compressed(OUT / "arnoldi_cases.npz", **out)


def gen_pls():
    from recgmres.dense_kernels import ProgressiveBlockLs
    from conftest import random_block_hessenberg

    out = {}
    rng = np.random.default_rng(5)
    n = 0
    for case in range(12):
        L = int(rng.integers(1, 5))
        m = int(rng.integers(2, 7))
        H = random_block_hessenberg(m, L, seed=7000 + case)
        G0 = rng.standard_normal((L, L))
        pls = ProgressiveBlockLs(L, G0)
        res = [pls.append_block(H[: (j + 2) * L, j * L : (j + 1) * L]) for j in range(m)]
        out[f"{case}/H"] = H
        out[f"{case}/G0"] = G0
        out[f"{case}/L"] = np.array(L)
        out[f"{case}/m"] = np.array(m)
        out[f"{case}/res"] = np.array(res)
        out[f"{case}/Y"] = pls.solve()
        out[f"{case}/R"] = pls.r_factor()
        n += 1
    out["n"] = np.array(n)
    np.savez_compressed(OUT / "pls_cases.npz", **out)


def gen_recycling():
    from recgmres import arnoldi
    from recgmres.recycling import (RecycleSpace, harmonic_ritz_augmented, harmonic_ritz_krylov,
                                    prepare_cross_system, update_recycle_space)
    from recgmres.sparse_core import spmm
    from conftest import random_csr

    out = {}
    A = random_csr(60, 0.2, 21, shift=3.0)
    op = lambda Z: spmm(A, Z)
    rng = np.random.default_rng(21)
    # pure Krylov
    fact = arnoldi.start(op, rng.standard_normal((60, 2)), m_max=6, seed=0)
    for _ in range(6):
        arnoldi.step(fact, op)
    sel = harmonic_ritz_krylov(fact, k_target=5)
    rs1 = update_recycle_space(fact, None, sel, 5)
    _csr_arrays("A/", A.to_scipy(), out)
    out["kry/W"] = fact.w
    out["kry/H"] = fact.h_bar
    out["kry/values"] = sel.pairs.values
    out["kry/keep"] = sel.keep
    out["kry/coeffs"] = sel.coeffs
    out["kry/U"] = rs1.u
    out["kry/C"] = rs1.c
    # augmented
    R0 = rng.standard_normal((60, 2))
    R0 = R0 - rs1.c @ (rs1.c.T @ R0)
    fact2 = arnoldi.start(op, R0, m_max=5, recycle=rs1, seed=1)
    for _ in range(5):
        arnoldi.step(fact2, op, recycle=rs1)
    d = 1.0 / np.linalg.norm(rs1.u, axis=0)
    sel2 = harmonic_ritz_augmented(fact2, rs1, d, k_target=5)
    rs2 = update_recycle_space(fact2, rs1, sel2, 5)
    out["aug/R0"] = R0
    out["aug/W"] = fact2.w
    out["aug/H"] = fact2.h_bar
    out["aug/F"] = fact2.f
    out["aug/d"] = d
    out["aug/values"] = sel2.pairs.values
    out["aug/keep"] = sel2.keep
    out["aug/coeffs"] = sel2.coeffs
    out["aug/U"] = rs2.u
    out["aug/C"] = rs2.c
    # cross-system preparation against a perturbed operator
    B2 = random_csr(60, 0.2, 22, shift=3.0)
    rs3 = prepare_cross_system(rs2, lambda Z: spmm(B2, Z))
    _csr_arrays("A2/", B2.to_scipy(), out)
    out["cross/U"] = rs3.u
    out["cross/C"] = rs3.c
    np.savez_compressed(OUT / "recycling_cases.npz", **out)


def _report_arrays(prefix, rep, out, with_solution=True):
    out[prefix + "cycles"] = np.array(rep.cycles)
    out[prefix + "matvecs"] = np.array(rep.matvec_count)
    out[prefix + "converged"] = np.array(rep.converged)
    out[prefix + "final"] = np.array(rep.final_residual_norm)
    out[prefix + "steps"] = np.array([len(h) for h in rep.residual_history], dtype=np.int64)
    out[prefix + "hist"] = (np.concatenate(rep.residual_history, axis=0)
                            if rep.residual_history else np.zeros((0, 1)))
    out[prefix + "true"] = (np.array(rep.cycle_true_residuals) if rep.cycle_true_residuals
                            else np.zeros((0, 1)))
    out[prefix + "origin"] = np.array(rep.recycle_origin)
    out[prefix + "events"] = np.array(len(rep.breakdown_events))
    if with_solution and rep.solution is not None:
        out[prefix + "X"] = rep.solution


def gen_solver():
    from recgmres.solver import SolverConfig, solve_block_gcrodr, solve_block_gmres, solve_sequence
    from recgmres.sparse_core import CsrMatrix
    from conftest import random_csr

    out = {}
    # ---- config 1 (BASELINE configs[0]): 2-D conv-diff 64x64, p=4, m=20, k=10, 3 systems
    A = kron_conv_diff_2d(64, 10.0)
    n = A.shape[0]
    rng = np.random.default_rng(0)
    B = np.asfortranarray(rng.uniform(-1.0, 1.0, (n, 4)))
    d = rng.uniform(0.0, 1.0, n)
    mats = [sp.csr_matrix(A + sp.diags(0.01 * i * d)) for i in range(3)]
    _csr_arrays("cfg1/A/", A, out)
    out["cfg1/B"] = B
    out["cfg1/d"] = d
    for i, M in enumerate(mats):
        _csr_arrays(f"cfg1/A{i}/", M, out)
    cfg = SolverConfig(m=20, k=10, tol=1e-8)
    reps = solve_sequence([(CsrMatrix.from_scipy(M), B) for M in mats], cfg)
    for i, rep in enumerate(reps):
        _report_arrays(f"cfg1/sys{i}/", rep, out)
    # ---- small cases exercising the other driver paths
    As = random_csr(120, 0.08, 31, shift=4.0)
    Bs = np.asfortranarray(np.random.default_rng(31).standard_normal((120, 3)))
    _csr_arrays("small/A/", As.to_scipy(), out)
    out["small/B"] = Bs
    _, rep, _ = solve_block_gmres(As, Bs, None, SolverConfig(m=6, tol=1e-10, max_cycles=30))
    _report_arrays("small/gmres/", rep, out)
    _, rep, rs = solve_block_gcrodr(As, Bs, None, SolverConfig(m=6, k=4, tol=1e-10, max_cycles=30))
    _report_arrays("small/gcrodr/", rep, out)
    out["small/gcrodr/U"] = rs.u
    out["small/gcrodr/C"] = rs.c
    b1 = Bs[:, :1]
    _, rep, _ = solve_block_gcrodr(As, b1, None, SolverConfig(m=6, k=4, block_width=3, tol=1e-10, max_cycles=30))
    _report_arrays("small/enlarged/", rep, out)
    _, rep, _ = solve_block_gcrodr(As, Bs, None, SolverConfig(m=6, k=4, tol=1e-10, max_cycles=30,
                                                             stop_rule="per-column-relative",
                                                             early_exit=False))
    _report_arrays("small/percol/", rep, out)
    np.savez_compressed(OUT / "solver_cases.npz", **out)


def gen_problems():
    out = {}
    _csr_arrays("cd2d_64_10/", kron_conv_diff_2d(64, 10.0), out)
    _csr_arrays("cd2d_7_3/", kron_conv_diff_2d(7, 3.0), out)
    _csr_arrays("cd3d_12_20/", kron_conv_diff_3d(12, 20.0), out)
    _csr_arrays("cd3d_5_1/", kron_conv_diff_3d(5, 1.0), out)
    _csr_arrays("lap3d_10/", kron_laplacian_3d(10), out)
    np.savez_compressed(OUT / "problem_cases.npz", **out)


def gen_bench_model():
    from recgmres import bench

    out = {
        "matvec_bytes_5_7_3": np.array(bench.matvec_bytes(5, 7, 3)),
        "matvec_bytes_cfg2": np.array([bench.matvec_bytes(2097152, 14581760, p) for p in (1, 2, 4, 8, 16)]),
        "projector_bytes_cgs2": np.array(bench.projector_bytes(1000, 10, 4, "cgs2")),
        "projector_bytes_mgs": np.array(bench.projector_bytes(1000, 10, 4, "mgs")),
    }
    np.savez_compressed(OUT / "bench_model.npz", **out)


if __name__ == "__main__":
    _import_reference()
    for fn in (gen_spmm, gen_qr, gen_arnoldi, gen_pls, gen_recycling, gen_solver, gen_problems, gen_bench_model):
        print("generating", fn.__name__, flush=True)
        fn()
    print("done")
