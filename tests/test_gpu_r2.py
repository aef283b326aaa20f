"""GPU parity against the round-2 reference goldens (tests/golden/
make_golden_r2.py): block MGS, an unscrubbed starting block with a recycle
space, bases wider than one 128-column Gram launch, and a reference-written
RGMRECYC file loaded straight to the device."""

import numpy as np
import pytest

from conftest import csr_matrix_from, load_golden
from parity_log import record

pytestmark = pytest.mark.gpu


def _run_case(g, name, ortho, c_orthogonal=False):
    from paper_1604_01713_b200 import arnoldi
    from paper_1604_01713_b200.recycling import RecycleSpace
    from paper_1604_01713_b200.solver import _Operator

    A = csr_matrix_from(g, f"{name}/")
    m, k, seed = int(g[f"{name}/m"]), int(g[f"{name}/k"]), int(g[f"{name}/seed"])
    rs = RecycleSpace(u=g[f"{name}/U"], c=g[f"{name}/C"]) if k else None
    op = _Operator(A, None, "none")
    fact = arnoldi.start(op.apply, g[f"{name}/R0"], m_max=m, recycle=rs, seed=seed, c_orthogonal=c_orthogonal)
    for _ in range(m):
        arnoldi.step(fact, op.apply, recycle=rs, ortho=ortho)
    return A, fact, k


def _check_against_golden(test, g, name, A, fact, k, h_tol=1e-12, w_tol=1e-12):
    scale = A.frobenius_norm()
    eh = np.abs(fact.h_bar - g[f"{name}/H"]).max() / scale
    ez = np.abs(fact.z_bar - g[f"{name}/z_bar"]).max() / np.abs(g[f"{name}/z_bar"]).max()
    ef = np.abs(fact.f - g[f"{name}/F"]).max() / scale if k else 0.0
    ew = np.abs(fact.w_numpy() - g[f"{name}/W"]).max()
    record(f"{test}:{name}", H_rel=eh, zbar_rel=ez, F_rel=ef, W_abs=ew)
    assert eh <= h_tol, (name, eh)
    assert ez <= 1e-13, (name, ez)
    assert ef <= h_tol, (name, ef)
    assert ew <= w_tol, (name, ew)
    assert len(fact.breakdown_events) == int(g[f"{name}/events"]), name


def test_mgs_arnoldi_matches_reference(cuda):
    """ortho="mgs" (arnoldi.py:159-170): one C column, then one basis block at
    a time, each pass fusing the previous update with the next Gram."""
    g = load_golden("r2_cases.npz")
    for name in ("mgs/plain_n300_L3", "mgs/recyc_n400_L4_k5"):
        A, fact, k = _run_case(g, name, "mgs")
        _check_against_golden("mgs", g, name, A, fact, k)


def test_unscrubbed_start_keeps_the_reference_order(cuda):
    """A recycle space with an R0 that was not projected against C: start()
    without c_orthogonal keeps the sequential C-then-W CGS2 and reproduces the
    reference; certifying orthogonality that does not hold (the joint [C W]
    schedule) would drift by O(||C^T V_1||)."""
    g = load_golden("r2_cases.npz")
    A, fact, k = _run_case(g, "unscrubbed", "cgs2")
    assert not fact.c_orthogonal
    _check_against_golden("unscrubbed", g, "unscrubbed", A, fact, k)
    C = g["unscrubbed/C"]
    assert np.linalg.norm(C.T @ g["unscrubbed/R0"]) > 1e-3  # the case really is unscrubbed
    _, wrong, _ = _run_case(g, "unscrubbed", "cgs2", c_orthogonal=True)
    assert np.abs(wrong.h_bar - g["unscrubbed/H"]).max() > 1e-8 * A.frobenius_norm()


@pytest.mark.parametrize("name", ["wide/plain_L8_m20", "wide/recyc_L8_m20_k20"])
def test_bases_wider_than_one_gram_launch(cuda, name):
    """m = 20, L = 8: the basis reaches 168 columns (k + w = 188 with C), past
    rg_tall's 128-column Gram operand; the step falls back to the split
    pass chain instead of failing."""
    g = load_golden("r2_cases.npz")
    A, fact, k = _run_case(g, name, "cgs2", c_orthogonal=True)
    _check_against_golden("wide", g, name, A, fact, k)


def test_wide_cycle_solve_matches_reference(cuda):
    """solve_block_gcrodr with m = 20, p = 8, k = 20 (the advisor's failing
    shape): identical cycles, steps and matvecs; histories within
    1e-9 ||B||_F."""
    from paper_1604_01713_b200 import SolverConfig, solve_block_gcrodr

    g = load_golden("r2_cases.npz")
    A = csr_matrix_from(g, "wide_solve/")
    B = g["wide_solve/B"]
    X, rep, rs = solve_block_gcrodr(A, B, None, SolverConfig(m=20, k=20, tol=1e-9, max_cycles=6))
    bnorm = np.linalg.norm(B)
    assert rep.cycles == int(g["wide_solve/cycles"])
    assert [len(h) for h in rep.residual_history] == g["wide_solve/steps"].tolist()
    assert rep.matvec_count == int(g["wide_solve/matvecs"])
    assert rep.converged == bool(g["wide_solve/converged"])
    eh = np.abs(np.concatenate(rep.residual_history) - g["wide_solve/hist"]).max() / bnorm
    ex = np.abs(X - g["wide_solve/X"]).max() / np.abs(g["wide_solve/X"]).max()
    record("wide_solve", hist_rel_B=eh, X_rel=ex)
    assert eh <= 1e-9
    assert ex <= 1e-7


def test_reference_rgmrecyc_file_loads_to_device(cuda, tmp_path):
    """recycling.py:212-223: a file the reference wrote is read through pinned
    memory straight into device blocks; saving them again reproduces it."""
    import torch

    from paper_1604_01713_b200.recycling import load_recycle_space, save_recycle_space

    g = load_golden("r2_cases.npz")
    ref_bytes = g["rgmrecyc/bytes"].tobytes()
    path = tmp_path / "ref.rgm"
    path.write_bytes(ref_bytes)
    rs = load_recycle_space(path)
    assert isinstance(rs.u, torch.Tensor) and rs.u.is_cuda and rs.c.is_cuda
    u, c = rs.numpy()
    assert np.array_equal(u, g["rgmrecyc/u"]) and np.array_equal(c, g["rgmrecyc/c"])
    save_recycle_space(rs, tmp_path / "again.rgm")
    assert (tmp_path / "again.rgm").read_bytes() == ref_bytes


def test_graph_replayed_steps_are_bitwise_the_eager_steps(cuda):
    """Config 1 (n = 4096) with its block steps replayed from captured CUDA
    graphs (arnoldi.STEP_GRAPHS, arnoldi.StepWorkspace): the replayed kernels
    see the same operands, so the whole sequence is bitwise the eager one
    (which test_gpu_solver pins to the reference), with the same kernel count."""
    from paper_1604_01713_b200 import SolverConfig, arnoldi, problems, solve_sequence
    from paper_1604_01713_b200 import device as D

    systems, kw = problems.cfg1_sequence()
    for A, _ in systems:
        A.device(cuda).dia()  # one-time upload + layout build (2 launches per matrix) outside the counts
    runs = {}
    for graphs in (False, True):
        old, old_pipe = arnoldi.STEP_GRAPHS, arnoldi.PIPELINE_STEPS
        arnoldi.STEP_GRAPHS = graphs
        arnoldi.PIPELINE_STEPS = False  # (speculative steps a cycle discards launch kernels too)
        try:
            before = D.lib().rg_launch_count()
            runs[graphs] = (solve_sequence(systems, SolverConfig(**kw)), D.lib().rg_launch_count() - before)
        finally:
            arnoldi.STEP_GRAPHS, arnoldi.PIPELINE_STEPS = old, old_pipe
    (eager, n_eager), (graph, n_graph) = runs[False], runs[True]
    for a, b in zip(eager, graph):
        assert a.cycles == b.cycles and a.matvec_count == b.matvec_count
        assert np.array_equal(np.concatenate(a.residual_history), np.concatenate(b.residual_history))
        assert np.array_equal(a.solution, b.solution)
    assert n_graph == n_eager  # replays report the kernels they run


@pytest.mark.parametrize("case", ["cfg1", "cfg4_32"])
def test_pipelined_steps_are_bitwise_the_sequential_steps(cuda, case):
    """arnoldi.StepPipeline (step j+1 enqueued before step j's results are
    read; speculative steps discarded when a cycle ends early) changes only
    the host ordering: identical cycles, matvec counts, residual histories and
    solutions, bit for bit, against the plain step-by-step solve."""
    from paper_1604_01713_b200 import SolverConfig, arnoldi, problems, solve_sequence

    if case == "cfg1":
        systems, kw = problems.cfg1_sequence()
    else:
        A, B, system, kw = problems.cfg4_sequence(N=32, n_systems=3)
        systems = [(system(i), B) for i in range(3)]
    runs = {}
    for pipe in (False, True):
        old = arnoldi.PIPELINE_STEPS
        arnoldi.PIPELINE_STEPS = pipe
        try:
            runs[pipe] = solve_sequence(systems, SolverConfig(**kw))
        finally:
            arnoldi.PIPELINE_STEPS = old
    for a, b in zip(runs[False], runs[True]):
        assert a.error is None and b.error is None
        assert a.cycles == b.cycles and a.matvec_count == b.matvec_count
        assert np.array_equal(np.concatenate(a.residual_history), np.concatenate(b.residual_history))
        assert np.array_equal(a.solution, b.solution)
