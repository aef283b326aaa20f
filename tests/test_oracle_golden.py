"""Pin the oracle (oracle/) to golden vectors produced by the real
reference (tests/golden/make_golden.py) — CPU only."""

import numpy as np
import pytest
import torch  # noqa: F401

import oracle
from conftest import csr_from, load_golden


def test_oracle_spmm_bitwise_vs_reference():
    g = load_golden("spmm_cases.npz")
    for name in g["cases"]:
        rp, ci, v, shape = csr_from(g, f"{name}/")
        for threads in (1, 3):
            Y = oracle.spmm(rp, ci, v, g[f"{name}/X"], nthreads=threads)
            assert np.array_equal(Y, g[f"{name}/Y"]), name


def test_oracle_reduced_qr_vs_reference():
    g = load_golden("qr_cases.npz")
    for name in g["cases"]:
        q, r, flagged = oracle.reduced_qr(g[f"{name}/X"])
        assert flagged.tolist() == g[f"{name}/flagged"].tolist(), name
        # same LAPACK, same sign fix: identical up to threading noise
        assert np.abs(r - g[f"{name}/r"]).max() <= 1e-13 * max(np.abs(r).max(), 1.0), name
        ok = ~flagged
        assert np.abs(q[:, ok] - g[f"{name}/q"][:, ok]).max() <= 1e-12, name


def test_oracle_arnoldi_step_vs_reference():
    """Replay each golden step: V_j, the basis V_1..V_j and C must give the
    golden H / F columns and V_{j+1} (arnoldi.py:139-193)."""
    g = load_golden("arnoldi_cases.npz")
    for name in g["cases"]:
        rp, ci, v, shape = csr_from(g, f"{name}/")
        W, H, F = g[f"{name}/W"], g[f"{name}/H"], g[f"{name}/F"]
        m, k = int(g[f"{name}/m"]), int(g[f"{name}/k"])
        L = W.shape[1] // (m + 1)
        C = g[f"{name}/C"] if k else None
        scale = np.abs(v).sum()
        for j in range(m):
            Vm = W[:, j * L:(j + 1) * L]
            q, Fc, Hc, r, flagged = oracle.arnoldi_step(rp, ci, v, Vm, C, W[:, :(j + 1) * L])
            cols = slice(j * L, (j + 1) * L)
            assert np.abs(Hc - H[:(j + 1) * L, cols]).max() <= 1e-12 * scale, (name, j)
            assert np.abs(r - H[(j + 1) * L:(j + 2) * L, cols]).max() <= 1e-12 * scale, (name, j)
            if k:
                assert np.abs(Fc - F[:, cols]).max() <= 1e-12 * scale, (name, j)
            if not flagged.any():
                assert np.abs(q - W[:, (j + 1) * L:(j + 2) * L]).max() <= 1e-10, (name, j)


def test_oracle_bytes_model_vs_reference():
    g = load_golden("bench_model.npz")
    assert oracle.spmm_bytes(5, 7, 3) == int(g["matvec_bytes_5_7_3"])
    for p, ref in zip((1, 2, 4, 8, 16), g["matvec_bytes_cfg2"]):
        assert oracle.spmm_bytes(2097152, 14581760, p) == int(ref)


def test_bench_module_bytes_model_and_csv(tmp_path):
    """The device bench module keeps the reference's bytes model and CSV
    schema (bench.py:44-55, :169-186) — host-only checks."""
    from paper_1604_01713_b200 import bench as B

    g = load_golden("bench_model.npz")
    assert B.matvec_bytes(5, 7, 3) == int(g["matvec_bytes_5_7_3"])
    assert B.projector_bytes(1000, 10, 4, "cgs2") == int(g["projector_bytes_cgs2"])
    assert B.projector_bytes(1000, 10, 4, "mgs") == int(g["projector_bytes_mgs"])
    res = [B.BenchResult("m", 10, 30, 2, "all-at-once", "cgs2", 3, 5, 1.5e-3, 1e-3, 2e-4, 999),
           B.BenchResult("m", 10, 30, 2, "one-at-a-time", "cgs2", 3, 5, 4e-3, 3e-3, 1e-4, 1998)]
    p = tmp_path / "r.csv"
    B.emit_csv(res, p)
    text = p.read_bytes()
    assert b"\r" not in text and text.splitlines()[0].decode().split(",") == B.CSV_HEADER
    back = B.read_results_csv(p)
    assert [(b.matrix_id, b.L, b.mode, b.projector, b.dim_c, b.bytes_model) for b in back] == \
        [(r.matrix_id, r.L, r.mode, r.projector, r.dim_c, r.bytes_model) for r in res]
    assert all(abs(b.mean_seconds - r.mean_seconds) <= 1e-6 * r.mean_seconds for b, r in zip(back, res))
    assert B.block_single_ratios(res)[("m", "cgs2", 3)] == [(2, 1.5e-3 / (4e-3 / 2))]


def test_oracle_ilu0_vs_reference():
    """The C restatement of precond.py's IKJ sweep reproduces the reference's
    factors bit for bit, and its substitution matches apply_precond."""
    g = load_golden("ilu_cases.npz")
    for name in ("cd2d", "rand", "tri", "band"):
        rp, ci, v = g[name + "/A/row_ptr"], g[name + "/A/col_idx"], g[name + "/A/values"]
        lu, dpos = oracle.ilu0(rp, ci, v)
        rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
        low = ci < rows
        assert np.array_equal(lu[low], g[name + "/L/values"]), name
        assert np.array_equal(lu[~low], g[name + "/U/values"]), name
        assert np.array_equal(ci[low], g[name + "/L/col_idx"]) and np.array_equal(ci[~low], g[name + "/U/col_idx"])
        Y = oracle.apply_precond(rp, ci, lu, dpos, g[name + "/X"])
        assert np.abs(Y - g[name + "/Y"]).max() <= 1e-13 * np.abs(g[name + "/Y"]).max(), name
    import scipy.sparse as sp

    for key in ("zero_pivot_mid", "missing_diag"):
        A = sp.csr_matrix(g[f"err/{key}_A/dense"])
        A.eliminate_zeros()
        with pytest.raises(oracle.OracleZeroPivot) as e:
            oracle.ilu0(A.indptr, A.indices, A.data)
        assert str(e.value) == str(g[f"err/{key}"])


def test_oracle_mgs_step_vs_reference():
    """Replay each golden block-MGS step (arnoldi.py:159-170) through
    oracle.mgs_project + oracle.reduced_qr (tests/golden/make_golden_r2.py)."""
    g = load_golden("r2_cases.npz")
    for name in ("mgs/plain_n300_L3", "mgs/recyc_n400_L4_k5"):
        rp, ci, v, shape = csr_from(g, f"{name}/")
        W, H, F = g[f"{name}/W"], g[f"{name}/H"], g[f"{name}/F"]
        m, k = int(g[f"{name}/m"]), int(g[f"{name}/k"])
        L = W.shape[1] // (m + 1)
        C = g[f"{name}/C"] if k else None
        scale = np.abs(v).sum()
        for j in range(m):
            Ahat = oracle.spmm(rp, ci, v, W[:, j * L:(j + 1) * L])
            Ahat, Fc, Hc = oracle.mgs_project(Ahat, C, W[:, :(j + 1) * L], L)
            q, r, flagged = oracle.reduced_qr(Ahat)
            cols = slice(j * L, (j + 1) * L)
            assert np.abs(Hc - H[:(j + 1) * L, cols]).max() <= 1e-12 * scale, (name, j)
            assert np.abs(r - H[(j + 1) * L:(j + 2) * L, cols]).max() <= 1e-12 * scale, (name, j)
            if k:
                assert np.abs(Fc - F[:, cols]).max() <= 1e-12 * scale, (name, j)
            assert not flagged.any()
            assert np.abs(q - W[:, (j + 1) * L:(j + 2) * L]).max() <= 1e-10, (name, j)


def test_oracle_wide_and_unscrubbed_steps_vs_reference():
    """The r2 CGS2 cases (bases past 128 columns; a recycle space with an
    R0 that was not projected against C) replay through oracle.arnoldi_step."""
    g = load_golden("r2_cases.npz")
    for name in ("unscrubbed", "wide/plain_L8_m20", "wide/recyc_L8_m20_k20"):
        rp, ci, v, shape = csr_from(g, f"{name}/")
        W, H, F = g[f"{name}/W"], g[f"{name}/H"], g[f"{name}/F"]
        m, k = int(g[f"{name}/m"]), int(g[f"{name}/k"])
        L = W.shape[1] // (m + 1)
        C = g[f"{name}/C"] if k else None
        scale = np.abs(v).sum()
        for j in range(m):
            q, Fc, Hc, r, flagged = oracle.arnoldi_step(rp, ci, v, W[:, j * L:(j + 1) * L], C, W[:, :(j + 1) * L])
            cols = slice(j * L, (j + 1) * L)
            assert np.abs(Hc - H[:(j + 1) * L, cols]).max() <= 1e-12 * scale, (name, j)
            assert np.abs(r - H[(j + 1) * L:(j + 2) * L, cols]).max() <= 1e-12 * scale, (name, j)
            if k:
                assert np.abs(Fc - F[:, cols]).max() <= 1e-12 * scale, (name, j)
