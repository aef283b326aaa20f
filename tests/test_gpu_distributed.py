"""Row-partitioned solver on the GPU: two ranks share cuda:0 and talk over
gloo (host-staged halos and Gram allreduces, so no kernel ever waits on
another rank's kernel).  The full block GCRO-DR sequence of BASELINE
configs[0] must reproduce the reference's golden run: same cycles, block
steps and matvec counts, residual histories within 1e-9 ||B||_F, and each
rank's slice of X."""

import numpy as np
import pytest

from test_distributed_cpu import _run

pytestmark = pytest.mark.gpu


def _cfg1_worker(rank, world):
    import torch

    from conftest import load_golden
    from paper_1604_01713_b200 import SolverConfig, distributed, problems, solve_sequence

    torch.cuda.set_device(0)
    g = load_golden("solver_cases.npz")
    systems, kw = problems.cfg1_sequence()
    dist_systems = []
    part = None
    for A, B in systems:
        op, part = distributed.setup(A, align=64)
        dist_systems.append((op, B))
    reps = solve_sequence(dist_systems, SolverConfig(**kw))
    bnorm = np.linalg.norm(g["cfg1/B"])
    for i, rep in enumerate(reps):
        pre = f"cfg1/sys{i}/"
        assert rep.error is None, rep.error
        assert rep.cycles == int(g[pre + "cycles"])
        assert [len(h) for h in rep.residual_history] == g[pre + "steps"].tolist()
        assert rep.matvec_count == int(g[pre + "matvecs"])
        assert rep.converged
        hist = np.concatenate(rep.residual_history, axis=0)
        assert np.abs(hist - g[pre + "hist"]).max() <= 1e-9 * bnorm
        Xref = g[pre + "X"][part.r0:part.r1]
        assert rep.solution.shape == Xref.shape
        assert np.abs(rep.solution - Xref).max() <= 1e-6 * np.abs(g[pre + "X"]).max()
    distributed.teardown()


def test_cfg1_sequence_two_ranks_one_gpu(cuda):
    _run(2, _cfg1_worker)


def _nccl_entry(rank, world, port, fn):
    import os
    import pathlib
    import sys

    import torch
    import torch.distributed as dist

    root = pathlib.Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    try:
        fn(rank, world)
    finally:
        dist.destroy_process_group()


def _cfg1_worker_own_gpu(rank, world):
    import torch

    from paper_1604_01713_b200 import device as D

    _orig = torch.cuda.set_device
    torch.cuda.set_device = lambda d: _orig(rank)  # the worker pins cuda:0; here each rank has its own GPU
    try:
        assert D.get_part() is None
        _cfg1_worker(rank, world)
    finally:
        torch.cuda.set_device = _orig


@pytest.mark.skipif("not __import__('torch').cuda.is_available() or __import__('torch').cuda.device_count() < 2",
                    reason="needs two GPUs (one rank per GPU, NCCL halos and Gram allreduces)")
def test_cfg1_sequence_two_gpus_nccl():
    """The NCCL data plane: one rank per GPU, halo columns and Gram
    allreduces over NCCL, the config-1 golden sequence reproduced."""
    import torch.multiprocessing as mp

    from test_distributed_cpu import _free_port

    mp.start_processes(_nccl_entry, args=(2, _free_port(), _cfg1_worker_own_gpu), nprocs=2, join=True,
                       start_method="spawn")


def _cfg5_worker(rank, world):
    """Complex (config-5 shaped) sequence, row-partitioned over two ranks,
    against the same sequence solved by one process."""
    import torch

    from paper_1604_01713_b200 import SolverConfig, distributed, problems, solve_sequence

    torch.cuda.set_device(0)
    system, B, kw = problems.cfg5_sequence(N=10, p=4)
    cfg = SolverConfig(**dict(kw, k=6))
    mats = [system(i) for i in range(2)]
    ref = solve_sequence([(A, B) for A in mats], cfg)  # same process, no partition
    dist_systems = []
    part = None
    for A in mats:
        op, part = distributed.setup(A, align=100)
        dist_systems.append((op, B))
    reps = solve_sequence(dist_systems, cfg)
    bn = np.linalg.norm(B)
    for r, rr in zip(reps, ref):
        assert r.error is None, r.error
        assert r.converged and r.cycles == rr.cycles and r.matvec_count == rr.matvec_count
        h, hr = np.concatenate(r.residual_history), np.concatenate(rr.residual_history)
        assert np.abs(h - hr).max() <= 1e-9 * bn
        assert np.abs(r.solution - rr.solution[part.r0:part.r1]).max() <= 1e-8 * np.abs(rr.solution).max()
    distributed.teardown()


def test_complex_sequence_two_ranks_one_gpu(cuda):
    _run(2, _cfg5_worker)


def _dist_spmm_3d_worker(rank, world):
    """3-D stencil, plane-aligned partition: the interior rows run on the
    diagonal layout built over the interior range only (the renumbered ghost
    columns would otherwise add far diagonals), the boundary rows on the CSR
    kernel; the product is bitwise the single-process one."""
    import torch

    import oracle
    from paper_1604_01713_b200 import device as D, distributed, problems

    torch.cuda.set_device(0)
    grid = 24
    A = problems.conv_diff_3d(grid, 20.0)
    X = np.asfortranarray(np.random.default_rng(3).standard_normal((A.n_rows, 8)))
    ref = oracle.spmm(A.row_ptr, A.col_idx, A.values, X, nthreads=1)
    op, part = distributed.setup(A, align=grid * grid)
    try:
        plan = op.dcsr.dia()
        assert plan is not None and plan.rows == tuple(op.plan.interior) and len(plan.offsets) == 7
        for p in (8, 3):
            Z = D.to_device_block(X[part.r0:part.r1, :p])
            out = D.empty_block(part.n_local, p)
            op.apply_into(Z, out)
            assert np.array_equal(D.to_numpy_block(out), ref[part.r0:part.r1, :p])
    finally:
        distributed.teardown()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_spmm_3d_stencil_ranks_on_one_gpu(cuda, world):
    _run(world, _dist_spmm_3d_worker)


def _peer_plumbing_worker(rank, world):
    """The real multi-process plumbing of the peer-memory paths, with the two
    ranks sharing one GPU: buffers allocated, IPC handles exchanged, peers'
    buffers mapped, the group registered; the halo pushes of a 3-D stencil
    land in the neighbour's ghost block with the epoch flag.  Host barriers
    separate writers from readers -- no kernel here waits on another rank's
    (the waits themselves are covered by the one-process emulations in
    test_gpu_peer.py)."""
    import torch
    import torch.distributed as dist

    from paper_1604_01713_b200 import device as D, distributed as DI, problems

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    L = D.lib()
    comm = DI.CommContext(peer=False)
    pg = DI.PeerGroup.create(comm, force=True, selftest=False)
    assert pg is not None and L.rg_peer_active() == world and len(pg.ptrs) == world
    comm.peer = pg
    try:
        # every rank's exchange buffer is visible through every other rank's mapping
        mine = DI._wrap(pg.ptrs[rank], (4,), torch.float64, dev)
        mine.fill_(float(rank + 1))
        torch.cuda.synchronize()
        dist.barrier()
        for r in range(world):
            assert float(DI._wrap(pg.ptrs[r], (4,), torch.float64, dev)[0].item()) == r + 1
        dist.barrier()
        mine.zero_()
        torch.cuda.synchronize()
        # halo pushes of a plane-partitioned 3-D operator
        grid, p = 12, 5
        A = problems.conv_diff_3d(grid, 20.0)
        X = np.asfortranarray(np.random.default_rng(4).standard_normal((A.n_rows, p)))
        part = DI.RowPartition.even(A.n_rows, world, rank, align=grid * grid)
        rp, ci, v = DI.csr_row_block(A.row_ptr, A.col_idx, A.values, part.r0, part.r1)
        plan = DI.HaloPlan.from_local_rows(part, rp, ci, v)
        op = DI.DistCsr(plan, comm, dev)
        hp = op._halo_peer
        assert hp is not None and hp in pg.halos and hp.peers == [q for q in range(world) if abs(q - rank) == 1]
        Z = D.to_device_block(X[part.r0:part.r1])
        gb = hp.ghost(p, torch.float64)  # collective: ghost blocks allocated, exchanged, mapped
        for epoch in (1, 2):
            par = hp.push_all(Z, op._send_idx, gb)
            torch.cuda.synchronize()
            dist.barrier()
            assert par == epoch & 1
            got = gb.local[par].t()[: plan.n_ghost].cpu().numpy()
            assert np.array_equal(got, X[plan.ghost_cols])  # the neighbours' rows, in ghost order
            flags = DI._wrap(hp.flags_local, (hp.FLAG_WORDS,), torch.int32, dev).cpu().numpy()
            assert all(flags[par * 8 + q] == epoch for q in hp.peers) and flags[16] == 0 and flags[17] == 0
            dist.barrier()
    finally:
        comm.close()
    assert L.rg_peer_active() == 0


def test_peer_memory_plumbing_two_processes_one_gpu(cuda):
    _run(2, _peer_plumbing_worker)
