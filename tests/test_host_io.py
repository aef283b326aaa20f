"""Host utilities against the reference (CPU only): Matrix Market reading
and writing, CsrMatrix validation messages, gen_banded, and the synthetic
problem generators (tests/golden/make_golden_io.py, make_golden.py)."""

import json
import pathlib
import sys

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import load_golden

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent / "golden"))
from make_golden_io import ARRAY_CASES, MM_CASES  # noqa: E402  (the same texts the fixtures were made from)


def _err(g, key):
    return tuple(json.loads(str(g[key])))


@pytest.mark.parametrize("name", sorted(MM_CASES))
def test_read_matrix_market_matches_reference(tmp_path, name):
    from paper_1604_01713_b200 import read_matrix_market

    g = load_golden("io_cases.npz")
    f = tmp_path / "m.mtx"
    f.write_text(MM_CASES[name])
    if f"mm/{name}/error" in g:
        cls, msg = _err(g, f"mm/{name}/error")
        with pytest.raises(Exception) as e:
            read_matrix_market(f)
        assert (type(e.value).__name__, str(e.value)) == (cls, msg)
    else:
        A = read_matrix_market(f)
        assert np.array_equal(np.asarray(A.row_ptr), g[f"mm/{name}/row_ptr"])
        assert np.array_equal(np.asarray(A.col_idx), g[f"mm/{name}/col_idx"])
        assert np.array_equal(np.asarray(A.values), g[f"mm/{name}/values"])
        assert (A.n_rows, A.n_cols) == tuple(g[f"mm/{name}/shape"])


@pytest.mark.parametrize("name", sorted(ARRAY_CASES))
def test_read_matrix_market_array_matches_reference(tmp_path, name):
    from paper_1604_01713_b200.sparse_core import read_matrix_market_array

    g = load_golden("io_cases.npz")
    f = tmp_path / "a.mtx"
    f.write_text(ARRAY_CASES[name])
    if f"arr/{name}/error" in g:
        cls, msg = _err(g, f"arr/{name}/error")
        with pytest.raises(Exception) as e:
            read_matrix_market_array(f)
        assert (type(e.value).__name__, str(e.value)) == (cls, msg)
    else:
        X = read_matrix_market_array(f)
        assert X.flags.f_contiguous and np.array_equal(X, g[f"arr/{name}/value"])


def test_write_read_round_trip(tmp_path):
    from paper_1604_01713_b200 import gen_banded, read_matrix_market, write_matrix_market

    A = gen_banded(40, 3, 7)
    write_matrix_market(A, tmp_path / "b.mtx")
    B = read_matrix_market(tmp_path / "b.mtx")
    assert np.array_equal(np.asarray(A.row_ptr), np.asarray(B.row_ptr))
    assert np.array_equal(np.asarray(A.col_idx), np.asarray(B.col_idx))
    assert np.array_equal(A.values, B.values)  # repr-exact floats


def test_gen_banded_matches_reference():
    from paper_1604_01713_b200 import gen_banded

    g = load_golden("io_cases.npz")
    for n, band, seed in ((50, 2, 3), (200, 5, 11)):
        B = gen_banded(n, band, seed)
        pre = f"banded/{n}_{band}_{seed}/"
        assert np.array_equal(np.asarray(B.row_ptr), g[pre + "row_ptr"])
        assert np.array_equal(np.asarray(B.col_idx), g[pre + "col_idx"])
        assert np.array_equal(B.values, g[pre + "values"])


@pytest.mark.parametrize("name,args", [
    ("rp_len", (2, 2, [0, 1], [0], [1.0])),
    ("rp_start", (2, 2, [1, 1, 2], [0], [1.0])),
    ("len_mismatch", (2, 2, [0, 1, 2], [0, 1], [1.0])),
    ("col_range", (2, 2, [0, 1, 2], [0, 2], [1.0, 2.0])),
    ("unsorted", (2, 3, [0, 2, 2], [1, 0], [1.0, 2.0])),
    ("duplicate", (2, 3, [0, 2, 2], [1, 1], [1.0, 2.0])),
])
def test_csr_validation_messages_match_reference(name, args):
    from paper_1604_01713_b200 import CsrMatrix

    g = load_golden("io_cases.npz")
    cls, msg = _err(g, f"csr/{name}/error")
    with pytest.raises(Exception) as e:
        CsrMatrix(*[np.asarray(a) if isinstance(a, list) else a for a in args])
    assert (type(e.value).__name__, str(e.value)) == (cls, msg)


def test_problem_generators_match_kron_recipes():
    """problems.py's direct CSR generators equal the scipy kron recipes the
    reference fixtures were built from, bit for bit."""
    from paper_1604_01713_b200 import problems

    g = load_golden("problem_cases.npz")
    cases = {"cd2d_64_10": problems.conv_diff_2d(64, 10.0), "cd2d_7_3": problems.conv_diff_2d(7, 3.0),
             "cd3d_12_20": problems.conv_diff_3d(12, 20.0), "cd3d_5_1": problems.conv_diff_3d(5, 1.0),
             "lap3d_10": problems.laplacian_3d(10)}
    for name, A in cases.items():
        # scipy's kron takes a dense-block (BSR) path when a factor is more
        # than half full (N=5 tridiagonal), storing explicit zeros: compare
        # against the recipe with those dropped.
        K = sp.csr_matrix((g[name + "/values"], g[name + "/col_idx"], g[name + "/row_ptr"]),
                          shape=tuple(g[name + "/shape"]))
        K.eliminate_zeros()
        assert np.array_equal(np.asarray(A.row_ptr), K.indptr), name
        assert np.array_equal(np.asarray(A.col_idx), K.indices), name
        assert np.array_equal(A.values, K.data), name
        assert (A.n_rows, A.n_cols) == K.shape, name


def test_rgmrecyc_reads_and_writes_reference_files(tmp_path):
    """A file written by the reference's save_recycle_space
    (recycling.py:201-209, tests/golden/make_golden_r2.py) loads to the same
    U and C, and saving them again reproduces the file byte for byte."""
    from paper_1604_01713_b200.recycling import RecycleSpace, load_recycle_space, save_recycle_space

    g = load_golden("r2_cases.npz")
    ref_bytes = g["rgmrecyc/bytes"].tobytes()
    path = tmp_path / "ref.rgm"
    path.write_bytes(ref_bytes)
    rs = load_recycle_space(path)  # device blocks on a GPU box, host arrays here
    u, c = rs.numpy()
    assert rs.origin == "cross-system"
    assert np.array_equal(u, g["rgmrecyc/u"]) and np.array_equal(c, g["rgmrecyc/c"])
    out = tmp_path / "ours.rgm"
    save_recycle_space(RecycleSpace(u=g["rgmrecyc/u"], c=g["rgmrecyc/c"]), out)
    assert out.read_bytes() == ref_bytes
    save_recycle_space(rs, tmp_path / "again.rgm")
    assert (tmp_path / "again.rgm").read_bytes() == ref_bytes
    bad = tmp_path / "bad.rgm"
    bad.write_bytes(b"NOTRECYC" + ref_bytes[8:])
    with pytest.raises(ValueError, match="not a recycle-space file"):
        load_recycle_space(bad)


def test_progressive_block_ls_vs_reference():
    """The host progressive least squares (dense_kernels.py:116-203) against
    the reference's per-step residual norms, Y and R (pls_cases.npz)."""
    from paper_1604_01713_b200.dense_kernels import ProgressiveBlockLs

    g = load_golden("pls_cases.npz")
    for case in range(int(g["n"])):
        H, G0 = g[f"{case}/H"], g[f"{case}/G0"]
        L, m = int(g[f"{case}/L"]), int(g[f"{case}/m"])
        pls = ProgressiveBlockLs(L, G0)
        res = np.array([pls.append_block(H[: (j + 2) * L, j * L:(j + 1) * L]) for j in range(m)])
        scale = np.abs(G0).max()
        assert np.abs(res - g[f"{case}/res"]).max() <= 1e-12 * scale, case
        R = pls.r_factor()
        assert np.abs(R - g[f"{case}/R"]).max() <= 1e-12 * np.abs(H).max(), case
        Y = pls.solve()
        assert np.abs(Y - g[f"{case}/Y"]).max() <= 1e-10 * max(1.0, np.abs(g[f"{case}/Y"]).max()), case
