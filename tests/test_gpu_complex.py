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
@pytest.mark.parametrize("p", [1, 5, 8, 16])
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
