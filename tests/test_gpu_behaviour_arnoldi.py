"""The reference's Arnoldi and recycling behaviours (its test_arnoldi.py /
test_recycling.py groups) re-checked against the device-resident
factorization, with our own seeded problems."""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

pytestmark = pytest.mark.gpu


def _mat(n, density, seed, shift):
    from paper_1604_01713_b200 import CsrMatrix

    g = np.random.default_rng(seed)
    M = sp.csr_matrix(sp.random(n, n, density=density, random_state=g, format="csr") + shift * sp.eye(n))
    M.sort_indices()
    return CsrMatrix.from_scipy(M)


def _op(A):
    from paper_1604_01713_b200.sparse_core import spmm_device

    return lambda Z: spmm_device(A, Z)


def _run(A, R0, m, rs=None, ortho="cgs2", seed=0):
    from paper_1604_01713_b200 import arnoldi

    f = arnoldi.start(_op(A), R0, m_max=m, recycle=rs, seed=seed)
    for _ in range(m):
        arnoldi.step(f, _op(A), recycle=rs, ortho=ortho)
    return f


def _recycle(A, k, seed):
    from paper_1604_01713_b200.recycling import RecycleSpace, prepare_cross_system

    U0 = np.random.default_rng(seed).standard_normal((A.n_rows, k))
    return prepare_cross_system(RecycleSpace(u=U0, c=None), _op(A))


# ---------------------------------------------------------------- start


def test_start_block_conventions(cuda):
    from paper_1604_01713_b200 import arnoldi

    A = _mat(16, 0.3, 200, 3.0)
    V = np.linalg.qr(np.random.default_rng(200).standard_normal((16, 3)))[0]
    f = arnoldi.start(_op(A), V, m_max=2)
    s = np.sign(np.diagonal(f.z_bar))
    assert np.allclose(f.z_bar, np.diag(s), atol=1e-12)
    assert np.allclose(f.w_numpy(), V * s, atol=1e-12)
    e = np.zeros((16, 1))
    e[3] = 3.5
    assert arnoldi.start(_op(A), e, m_max=2).z_bar[0, 0] == pytest.approx(3.5)
    with pytest.raises(arnoldi.ZeroStartBlock):
        arnoldi.start(_op(A), np.zeros((16, 2)), m_max=2)


def test_rank_deficient_start_is_repaired(cuda):
    from paper_1604_01713_b200 import arnoldi

    A = _mat(20, 0.3, 201, 3.0)
    x = np.random.default_rng(201).standard_normal((20, 1))
    f = arnoldi.start(_op(A), np.hstack([x, -3.0 * x]), m_max=2, seed=4)
    assert any("rank-deficient" in ev for ev in f.breakdown_events)
    W1 = f.w_numpy()[:, :2]
    assert np.linalg.norm(W1.T @ W1 - np.eye(2)) <= 1e-12


# ---------------------------------------------------------------- step


def test_identity_operator_breakdown_is_logged(cuda):
    from paper_1604_01713_b200 import CsrMatrix, arnoldi

    A = CsrMatrix.from_scipy(sp.eye(7, format="csr"))
    e = np.zeros((7, 1))
    e[2] = 1.0
    f = arnoldi.start(_op(A), e, m_max=1)
    arnoldi.step(f, _op(A))
    assert f.h_bar[0, 0] == pytest.approx(1.0)
    assert abs(f.h_bar[1, 0]) <= 1e-14
    assert any("rank-deficient" in ev for ev in f.breakdown_events)


@pytest.mark.parametrize("ortho", ["mgs", "cgs2"])
def test_invariants_plain_and_recycled(cuda, ortho):
    n, L, m, k = 40, 2, 5, 3
    A = _mat(n, 0.3, 202, 2.0)
    Ad = A.to_scipy().toarray()
    f = _run(A, np.random.default_rng(202).standard_normal((n, L)), m, ortho=ortho)
    W = f.w_numpy()
    assert np.linalg.norm(W.T @ W - np.eye((m + 1) * L)) <= 1e-12 * (m + 1) * L
    assert np.linalg.norm(Ad @ W[:, : m * L] - W @ f.h_bar) <= 1e-12 * A.frobenius_norm() * np.sqrt(m * L)
    rs = _recycle(A, k, 203)
    C = rs.numpy()[1]
    R0 = np.random.default_rng(203).standard_normal((n, L))
    R0 -= C @ (C.T @ R0)
    f = _run(A, R0, m, rs=rs, ortho=ortho)
    W = f.w_numpy()
    P = np.eye(n) - C @ C.T
    assert np.linalg.norm(C.T @ W) <= 1e-10
    assert np.linalg.norm(P @ Ad @ W[:, : m * L] - W @ f.h_bar) <= 1e-10 * A.frobenius_norm()
    assert np.linalg.norm(f.f - C.T @ (Ad @ W[:, : m * L])) <= 1e-10


def test_hessenberg_structure(cuda):
    n, L, m = 30, 3, 4
    A = _mat(n, 0.3, 204, 2.0)
    H = _run(A, np.random.default_rng(204).standard_normal((n, L)), m).h_bar
    for j in range(m):
        assert np.all(H[(j + 2) * L:, j * L:(j + 1) * L] == 0.0)
        blk = H[(j + 1) * L:(j + 2) * L, j * L:(j + 1) * L]
        assert np.array_equal(blk, np.triu(blk)) and np.all(np.diagonal(blk) >= 0.0)


def test_mgs_and_cgs2_span_the_same_space(cuda):
    n, L, m = 120, 2, 6
    A = _mat(n, 0.1, 205, 2.0)
    R0 = np.random.default_rng(205).standard_normal((n, L))
    W1 = _run(A, R0.copy(), m, ortho="mgs").w_numpy()
    W2 = _run(A, R0.copy(), m, ortho="cgs2").w_numpy()
    # sine of the largest principal angle (arccos of a cosine near 1 is ill-conditioned)
    assert np.linalg.norm(W2 - W1 @ (W1.T @ W2), 2) <= 1e-8


def test_capacity_and_ortho_checks(cuda):
    from paper_1604_01713_b200 import arnoldi

    A = _mat(12, 0.4, 206, 2.0)
    f = _run(A, np.random.default_rng(206).standard_normal((12, 1)), 2)
    with pytest.raises(ValueError, match="capacity"):
        arnoldi.step(f, _op(A))
    g = arnoldi.start(_op(A), np.ones((12, 1)), m_max=1)
    with pytest.raises(ValueError, match="ortho"):
        arnoldi.step(g, _op(A), ortho="householder")


# ---------------------------------------------------------------- recycling


def test_harmonic_ritz_full_space_symmetric(cuda):
    from paper_1604_01713_b200 import CsrMatrix
    from paper_1604_01713_b200.recycling import harmonic_ritz_krylov

    n = 14
    S = np.random.default_rng(207).standard_normal((n, n))
    S = S + S.T + 9.0 * np.eye(n)
    A = CsrMatrix.from_scipy(sp.csr_matrix(S))
    f = _run(A, np.random.default_rng(208).standard_normal((n, 1)), n)
    vals = np.sort(harmonic_ritz_krylov(f).pairs.values.real)
    assert np.abs(vals - np.sort(np.linalg.eigvalsh(S))).max() <= 1e-8 * np.linalg.norm(S)


def test_harmonic_ritz_petrov_galerkin(cuda):
    from paper_1604_01713_b200.recycling import harmonic_ritz_krylov

    n, m = 24, 6
    A = _mat(n, 0.4, 209, 4.0)
    Ad = A.to_scipy().toarray()
    f = _run(A, np.random.default_rng(209).standard_normal((n, 1)), m)
    sel = harmonic_ritz_krylov(f)
    AW = Ad @ f.w_numpy()[:, :m]
    Ainv = np.linalg.inv(Ad)
    for i in range(len(sel.pairs.values)):
        y = AW @ sel.pairs.complex_vector(i)
        r = AW.conj().T @ (Ainv @ y - y / sel.pairs.values[i])
        assert np.linalg.norm(r) <= 1e-8 * np.linalg.norm(Ad) * np.linalg.norm(y)


def test_recycle_update_invariants_and_errors(cuda):
    from paper_1604_01713_b200 import arnoldi
    from paper_1604_01713_b200.recycling import (RecyclingError, harmonic_ritz_augmented, harmonic_ritz_krylov,
                                                  update_recycle_space)

    n, L, m, k = 40, 2, 5, 4
    A = _mat(n, 0.3, 210, 4.0)
    Ad = A.to_scipy().toarray()
    with pytest.raises(RecyclingError):
        harmonic_ritz_krylov(arnoldi.start(_op(A), np.ones((n, 1)), m_max=2))
    f = _run(A, np.random.default_rng(210).standard_normal((n, L)), m)
    rs = update_recycle_space(f, None, harmonic_ritz_krylov(f, k_target=k), k)
    U, C = rs.numpy()
    assert np.linalg.norm(C.T @ C - np.eye(rs.k)) <= 1e-12 * rs.k
    assert np.linalg.norm(Ad @ U - C) <= 1e-10 * np.linalg.norm(Ad) * np.linalg.norm(U)
    R0 = np.random.default_rng(211).standard_normal((n, L))
    R0 -= C @ (C.T @ R0)
    f2 = _run(A, R0, m, rs=rs)
    d = 1.0 / np.linalg.norm(U, axis=0)
    with pytest.raises(ValueError):
        harmonic_ritz_augmented(f2, rs, d[:-1])
    rs2 = update_recycle_space(f2, rs, harmonic_ritz_augmented(f2, rs, d, k_target=k), k)
    U2, C2 = rs2.numpy()
    assert np.linalg.norm(C2.T @ C2 - np.eye(rs2.k)) <= 1e-12 * rs2.k
    assert np.linalg.norm(Ad @ U2 - C2) <= 1e-10 * np.linalg.norm(Ad) * np.linalg.norm(U2)


def test_recycle_space_file_round_trip(cuda, tmp_path):
    from paper_1604_01713_b200 import load_recycle_space, save_recycle_space

    A = _mat(30, 0.3, 212, 3.0)
    rs = _recycle(A, 5, 212)
    save_recycle_space(rs, tmp_path / "rs.bin")
    back = load_recycle_space(tmp_path / "rs.bin")
    U, C = rs.numpy()
    U2, C2 = back.numpy()
    assert np.array_equal(U, U2) and np.array_equal(C, C2)
    (tmp_path / "bad.bin").write_bytes(b"NOTRECYC" + bytes(24))
    with pytest.raises(ValueError):
        load_recycle_space(tmp_path / "bad.bin")
    raw = bytearray((tmp_path / "rs.bin").read_bytes())
    raw[8] = 9  # version field
    (tmp_path / "v9.bin").write_bytes(bytes(raw))
    with pytest.raises(ValueError):
        load_recycle_space(tmp_path / "v9.bin")
