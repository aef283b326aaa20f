"""Parity at the benchmarked size n = 2^24 (BASELINE configs[2] and the
config-4 step the bench times), against the oracle (oracle/, the CPU
restatement of arnoldi.py:171-180 and dense_kernels.py:31-48) run on the
host on the same operands.  Tolerances are the north star's 1e-12 relative
for FP64 kernel outputs."""

import numpy as np
import pytest
import torch

import oracle
from parity_log import record

pytestmark = pytest.mark.gpu

N = 2**24


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _rel_max(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def cfg3(cuda):
    from paper_1604_01713_b200 import device as D
    from paper_1604_01713_b200 import problems

    Cd, Vd, Qd = problems.cfg3_inputs(N, device=cuda)
    return Cd, Vd, Qd, D.to_numpy_block(Cd), D.to_numpy_block(Vd), D.to_numpy_block(Qd)


def test_cfg3_gram_and_update(cfg3):
    """W = C^T V and V - C W (the first two ops of configs[2])."""
    from paper_1604_01713_b200 import device as D

    Cd, Vd, Qd, C, V, Q = cfg3
    k, p = C.shape[1], V.shape[1]
    Wd = D.small(k, p)
    D.tall(Vd, None, gram=("basis", Cd, Wd))
    W = Wd.cpu().numpy()
    Wref = oracle.gram(C, V)
    e_gram = _rel_max(W, Wref)
    Zd = D.empty_block(N, p)
    D.tall(Vd, Zd, [(Cd, torch.from_numpy(np.asfortranarray(Wref)).cuda(), -1.0)])
    Zref = oracle.update(V, C, Wref)
    e_upd = _rel(D.to_numpy_block(Zd), Zref)
    record("cfg3_gram_update", gram_rel=e_gram, update_rel=e_upd)
    assert e_gram <= 1e-12
    assert e_upd <= 1e-12


def test_cfg3_cgs2_and_qr(cfg3):
    """Block CGS2 of V against the 80-column basis Q (2 passes, C omitted, as
    configs[2] defines it), the same against C then Q through the C-ABI
    orchestrator (rg_cgs2_f64, sequential schedule), then the thin QR of the
    projected n x 8 block."""
    from paper_1604_01713_b200 import device as D
    from paper_1604_01713_b200.dense_kernels import reduced_qr_device
    from paper_1604_01713_b200.ortho import project_chain

    Cd, Vd, Qd, C, V, Q = cfg3
    k, p, w = C.shape[1], V.shape[1], Q.shape[1]
    # (a) against Q alone
    Zd = D.empty_block(N, p)
    c1, c2 = D.small(w, p), D.small(w, p)
    project_chain(Vd, Zd, [Qd, Qd], [c1, c2])
    Zref, _, Href = oracle.cgs2_project(V, None, Q)
    e_z = _rel(D.to_numpy_block(Zd), Zref)
    e_h = _rel_max(c1.cpu().numpy() + c2.cpu().numpy(), Href)
    # (b) against C then Q, one C-ABI call
    Z2 = D.empty_block(N, p)
    Z2.copy_(Vd)
    coef = torch.zeros((2 * k + 2 * w) * p, dtype=torch.float64, device=Vd.device)
    D.cgs2(Z2, Cd, Qd, coef, None)
    Z2ref, Fref, H2ref = oracle.cgs2_project(V, C, Q)
    hc = coef.cpu().numpy()
    S = hc[:k * p].reshape(p, k).T + hc[(k + w) * p:(2 * k + w) * p].reshape(p, k).T
    H2 = hc[k * p:(k + w) * p].reshape(p, w).T + hc[(2 * k + w) * p:].reshape(p, w).T
    e_z2 = _rel(D.to_numpy_block(Z2), Z2ref)
    e_f2 = _rel_max(S, Fref)
    e_h2 = _rel_max(H2, H2ref)
    # (c) thin QR of the projected block
    f = reduced_qr_device(Zd)
    q_ref, r_ref, flagged = oracle.reduced_qr(Zref)
    cond = np.linalg.cond(r_ref)
    e_r = _rel_max(f.r_factor, r_ref)
    e_q = float(np.abs(D.to_numpy_block(f.q) - q_ref).max())
    record("cfg3_cgs2_qr", cgs2_Q_rel=e_z, coef_Q_rel=e_h, cgs2_CQ_rel=e_z2, F_rel=e_f2, H_rel=e_h2, R_rel=e_r,
           Q_abs=e_q, cond=cond)
    assert e_z <= 1e-12 and e_h <= 1e-12
    assert e_z2 <= 1e-12 and e_f2 <= 1e-12 and e_h2 <= 1e-12
    assert not flagged.any() and not f.flagged.any()
    assert e_r <= 1e-12 * cond
    assert e_q <= 1e-12 * cond


def test_cfg4_step_at_full_size(cuda):
    """The benchmarked step (256^3 conv-diff, p = 8, k = 20, step 10 of a
    cycle, joint [C W] schedule with the two-level Gram reductions over
    16.7M rows) against oracle.arnoldi_step on the same V_10, C and basis."""
    from paper_1604_01713_b200 import arnoldi, problems
    from paper_1604_01713_b200 import device as D
    from paper_1604_01713_b200.recycling import RecycleSpace, prepare_cross_system
    from paper_1604_01713_b200.solver import _Operator, _scrub

    A = problems.conv_diff_3d(256, 20.0)
    n, L, k, m = A.n_rows, 8, 20, 10
    op = _Operator(A, None, "none")
    g = torch.Generator(device=cuda)
    g.manual_seed(0)
    U0 = D.empty_block(n, k)
    U0.copy_(torch.randn(n, k, generator=g, device=cuda, dtype=torch.float64))
    rs = prepare_cross_system(RecycleSpace(u=U0, c=None), op.apply)
    R0 = D.empty_block(n, L)
    R0.copy_(torch.randn(n, L, generator=g, device=cuda, dtype=torch.float64))
    R0 = _scrub(R0, D.empty_block(n, L), rs.c)
    fact = arnoldi.start(op.apply, R0, m_max=m, recycle=rs, seed=0, c_orthogonal=True)
    for _ in range(m - 1):
        arnoldi.step(fact, op.apply, recycle=rs)
    W = fact.w_numpy()
    C = D.to_numpy_block(rs.c)
    Vm = W[:, (m - 1) * L: m * L]
    arnoldi.step(fact, op.apply, recycle=rs)
    q, F, H, r, flagged = oracle.arnoldi_step(A.row_ptr, A.col_idx, A.values, Vm, C, W)
    cols = slice((m - 1) * L, m * L)
    e_h = _rel_max(fact._H[: m * L, cols], H)
    e_f = _rel_max(fact._F[:, cols], F)
    e_r = _rel_max(fact._H[m * L:(m + 1) * L, cols], r)
    e_q = float(np.abs(D.to_numpy_block(fact.v_block(m)) - q).max())
    cond = np.linalg.cond(r)
    record("cfg4_step_256", H_rel=e_h, F_rel=e_f, R_rel=e_r, Q_abs=e_q, cond=cond)
    assert not flagged.any()
    assert e_h <= 1e-12 and e_f <= 1e-12
    assert e_r <= 1e-12 * cond
    assert e_q <= 1e-12 * cond


def _golden_cfg4_grid(name):
    from conftest import GOLDEN

    path = GOLDEN / name
    if not path.exists():
        pytest.skip(f"{name} not generated (tests/golden/make_golden_cfg4_grid.py)")
    return np.load(path)


def _check_cfg4_record(test, rep, X, g, bnorm, hist_tol=1e-9):
    assert rep.cycles == int(g["sys0/cycles"]), rep.cycles
    assert [len(h) for h in rep.residual_history] == g["sys0/steps"].tolist()
    assert rep.matvec_count == int(g["sys0/matvecs"])
    assert rep.converged == bool(g["sys0/converged"])
    e_hist = float(np.abs(np.concatenate(rep.residual_history) - g["sys0/hist"]).max() / bnorm)
    e_true = float(np.abs(np.array(rep.cycle_true_residuals) - g["sys0/true"]).max() / bnorm)
    e_x = float(np.abs(np.linalg.norm(X, axis=0) - g["sys0/Xnorms"]).max() / np.abs(g["sys0/Xnorms"]).max())
    record(test, hist_rel_B=e_hist, true_rel_B=e_true, Xnorm_rel=e_x)
    assert e_hist <= hist_tol and e_true <= hist_tol
    assert e_x <= 1e-8


def test_cfg4_256_first_cycles_match_reference(cuda):
    """BASELINE configs[3] at full size (256^3, n = 16.7M): system 0's first
    two cycles (20 block steps, 184 matvecs; 634 s for the reference on 8
    CPU cores) -- identical step and matvec counts, per-step residual
    estimates and cycle-end true residuals within 1e-9 ||B||_F."""
    from paper_1604_01713_b200 import SolverConfig, problems, solve_block_gcrodr

    g = _golden_cfg4_grid("cfg4_256_c2.npz")
    A, B, _, kw = problems.cfg4_sequence(N=256, n_systems=1)
    X, rep, _ = solve_block_gcrodr(A, B, None, SolverConfig(**dict(kw, max_cycles=2)))
    _check_cfg4_record("cfg4_256_c2", rep, X, g, np.linalg.norm(B))


def test_cfg4_128_system0_to_convergence_matches_reference(cuda):
    """The same family at 128^3 solved to convergence: the reference's cycle
    count pins the growth between the 64^3 golden (22 cycles) and the 256^3
    device runs."""
    from paper_1604_01713_b200 import SolverConfig, problems, solve_block_gcrodr

    g = _golden_cfg4_grid("cfg4_128_c200.npz")
    A, B, _, kw = problems.cfg4_sequence(N=128, n_systems=1)
    X, rep, _ = solve_block_gcrodr(A, B, None, SolverConfig(**dict(kw, max_cycles=200)))
    _check_cfg4_record("cfg4_128_c200", rep, X, g, np.linalg.norm(B), hist_tol=1e-8)
