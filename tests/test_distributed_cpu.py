"""Row-partitioned (multi-GPU) logic on CPU: world_size-2 gloo process groups
exercise the partition, the halo plan and exchange, the distributed SpMM
(bitwise against the single-process oracle), the CGS2 projection schedule
with its Gram allreduce, and the distributed TSQR combine."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(world, fn, *args):
    port = _free_port()
    mp.start_processes(_entry, args=(world, port, fn, args), nprocs=world, join=True, start_method="spawn")


def _entry(rank, world, port, fn, args):
    import sys
    import pathlib

    root = pathlib.Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------- partition (no processes)


def test_row_partition_even_and_aligned():
    from paper_1604_01713_b200.distributed import RowPartition

    p = RowPartition.even(10, 3, 1)
    assert p.bounds.tolist() == [0, 3, 6, 10]
    assert (p.r0, p.r1, p.n_local) == (3, 6, 3)
    q = RowPartition.even(64, 4, 2, align=16)  # whole planes of a 4x4x4 grid
    assert q.bounds.tolist() == [0, 16, 32, 48, 64]
    assert q.owner(np.array([0, 15, 16, 63])).tolist() == [0, 0, 1, 3]


def test_halo_plan_single_rank_view():
    """Plan built from a fake exchange: ghosts, renumbering, interior range."""
    from paper_1604_01713_b200 import problems
    from paper_1604_01713_b200.distributed import HaloPlan, RowPartition, csr_row_block

    A = problems.laplacian_3d(4)  # planes of 16 rows
    part = RowPartition.even(A.n_rows, 2, 0, align=16)
    rp, ci, v = csr_row_block(A.row_ptr, A.col_idx, A.values, part.r0, part.r1)
    plan = HaloPlan.from_local_rows(part, rp, ci, v, exchange=lambda part, lists: {1: lists.get(1, [])})
    assert plan.ghost_cols.tolist() == list(range(32, 48))      # the next plane
    assert plan.recv_ranges == {1: (0, 16)}
    assert plan.interior == (0, 16)                            # last plane touches ghosts
    assert plan.col_idx.max() < part.n_local + plan.n_ghost
    # entries keep their order: renumbering is monotone within each row
    rows = np.repeat(np.arange(part.n_local), np.diff(plan.row_ptr))
    glob = np.where(plan.col_idx < part.n_local, plan.col_idx + part.r0,
                    plan.ghost_cols[np.clip(plan.col_idx - part.n_local, 0, None)])
    assert np.array_equal(glob, ci)
    assert np.all(np.diff(glob)[np.diff(rows) == 0] > 0)


# ---------------------------------------------------------------- multi-process


def _dist_spmm_worker(rank, world, grid, p):
    from dist_helpers import oracle_local_spmm
    from paper_1604_01713_b200 import problems
    from paper_1604_01713_b200.distributed import CommContext, DistCsr, HaloPlan, RowPartition, csr_row_block

    A = problems.conv_diff_3d(grid, 20.0)
    X = np.asfortranarray(np.random.default_rng(5).standard_normal((A.n_rows, p)))
    ref = oracle.spmm(A.row_ptr, A.col_idx, A.values, X, nthreads=1)
    comm = CommContext()
    for align in (grid * grid, 1):  # plane-aligned and arbitrary cuts
        part = RowPartition.even(A.n_rows, world, rank, align)
        rp, ci, v = csr_row_block(A.row_ptr, A.col_idx, A.values, part.r0, part.r1)
        plan = HaloPlan.from_local_rows(part, rp, ci, v)
        op = DistCsr(plan, comm, local_spmm=oracle_local_spmm)
        Z = torch.from_numpy(X[part.r0:part.r1].copy())
        out = torch.zeros_like(Z)
        op.apply_into(Z, out)
        assert np.array_equal(out.numpy(), ref[part.r0:part.r1]), (rank, align)


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_spmm_bitwise(world):
    _run(world, _dist_spmm_worker, 6, 3)


def _dist_cgs2_worker(rank, world):
    from dist_helpers import host_tall_factory
    from paper_1604_01713_b200.distributed import CommContext, RowPartition
    from paper_1604_01713_b200.ortho import project_chain

    rng = np.random.default_rng(11)
    n, k, w, p = 1000, 5, 12, 3
    C = np.linalg.qr(rng.standard_normal((n, k)))[0]
    W = np.linalg.qr(rng.standard_normal((n, w)))[0]
    A = rng.standard_normal((n, p))
    ref, F, H = oracle.cgs2_project(A, C, W)
    comm = CommContext()
    part = RowPartition.even(n, world, rank)
    sl = slice(part.r0, part.r1)
    t = lambda M: torch.from_numpy(np.ascontiguousarray(M[sl]))
    Z = t(A)
    coefs = [torch.zeros(k, p, dtype=torch.float64), torch.zeros(w, p, dtype=torch.float64),
             torch.zeros(k, p, dtype=torch.float64), torch.zeros(w, p, dtype=torch.float64)]
    Cl, Wl = t(C), t(W)
    G = torch.zeros(p, p, dtype=torch.float64)
    project_chain(Z, Z, [Cl, Wl, Cl, Wl], coefs, tail_gram=("self", G), tall=host_tall_factory(comm))
    assert np.abs(Z.numpy() - ref[sl]).max() < 1e-12
    assert np.abs((coefs[0] + coefs[2]).numpy() - F).max() < 1e-12
    assert np.abs((coefs[1] + coefs[3]).numpy() - H).max() < 1e-12
    assert np.abs(G.numpy() - ref.T @ ref).max() < 1e-12


def test_distributed_cgs2_schedule_with_gram_allreduce():
    _run(2, _dist_cgs2_worker)


def _dist_tsqr_worker(rank, world):
    from paper_1604_01713_b200.dense_kernels import tsqr_combine
    from paper_1604_01713_b200.distributed import CommContext, RowPartition

    rng = np.random.default_rng(3)
    n, L = 600, 4
    X = rng.standard_normal((n, L))
    q_ref, r_ref, _ = oracle.reduced_qr(X)
    comm = CommContext()
    part = RowPartition.even(n, world, rank)
    Xl = X[part.r0:part.r1]
    ql, rl, _ = oracle.reduced_qr(Xl)  # stands in for the local device TSQR
    S, R = tsqr_combine(np.triu(rl), comm)
    Q_local = ql @ S
    assert np.abs(R - r_ref).max() < 1e-12 * np.abs(r_ref).max()
    assert np.abs(Q_local - q_ref[part.r0:part.r1]).max() < 1e-12


def test_distributed_tsqr_combine():
    _run(2, _dist_tsqr_worker)


# ---------------------------------------------------------------- peer-memory Gram reduction (host logic)


def test_peer_eligibility_rules():
    from paper_1604_01713_b200.distributed import peer_eligible

    assert peer_eligible([("a", 0), ("a", 1)]) == (True, "ok")
    assert peer_eligible([("a", r) for r in range(8)])[0]
    assert not peer_eligible([("a", 0)])[0]                          # nothing to reduce
    assert not peer_eligible([("a", r) for r in range(9)])[0]        # more ranks than slots
    assert not peer_eligible([("a", 0), ("b", 1)])[0]                # two nodes: no IPC mapping
    assert not peer_eligible([("a", 0), ("a", 0)])[0]                # ranks sharing a GPU would wait on each other
    assert not peer_eligible([("a", 0), ("a", None)])[0]


def _peer_off_worker(rank, world):
    """gloo ranks never register a peer group: the Gram sums stay on the
    group's allreduce and the fused C orchestrators stay off."""
    from paper_1604_01713_b200 import device as D
    from paper_1604_01713_b200.distributed import CommContext, RowPartition

    comm = CommContext()
    assert comm.peer is None and not comm.peer_active
    D.set_comm(comm, RowPartition.even(100, world, rank))
    try:
        assert not D.fused_ok()
        t = torch.full((4,), float(rank + 1), dtype=torch.float64)
        comm.allreduce_(t)
        assert torch.equal(t, torch.full((4,), 3.0, dtype=torch.float64))
    finally:
        D.set_comm(None, None)
        comm.close()
    assert D.fused_ok()


def test_peer_group_off_under_gloo():
    _run(2, _peer_off_worker)


def test_halo_neighbours_are_symmetric():
    """Each pair of ranks that exchanges rows in either direction signals
    both ways (the flow control of the peer-store halo exchange)."""
    from paper_1604_01713_b200.distributed import neighbours

    # rank 0 sends to 1 only; rank 2 receives from 1 only; rank 3 isolated
    infos = [{"send": [1], "recv": {}}, {"send": [2], "recv": {0: (0, 4)}}, {"send": [], "recv": {1: (0, 3)}},
             {"send": [], "recv": {}}]
    nb = [neighbours(infos, r) for r in range(4)]
    assert nb == [[1], [0, 2], [1], []]
    for r, qs in enumerate(nb):
        for q in qs:
            assert r in nb[q]
