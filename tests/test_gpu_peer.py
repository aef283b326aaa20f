"""The in-kernel Gram reduction over peer memory (rg_common.cuh
peer_allreduce, rg_peer.cu).  One GPU: the ranks are emulated as one
cooperative grid over local exchange buffers -- the same device code the
row-partitioned run executes in the last CTA of every Gram pass."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _expected(vals, rounds):
    world, ne = vals.shape
    g = vals.copy()
    for it in range(rounds):
        s = np.zeros(ne)
        for r in range(world):  # rank order, starting from 0.0, as the kernel sums
            s = s + g[r]
        for r in range(world):
            g[r] = s * (1.0 + 0.25 * r) + float(it)
    return g


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("ne", [1, 64, 800, 4096])
def test_peer_allreduce_emulated_ranks(cuda, world, ne):
    from paper_1604_01713_b200 import _lib, device as D

    L = D.lib()
    nb = L.rg_peer_buffer_bytes()
    rng = np.random.default_rng(world * 10007 + ne)
    vals = rng.standard_normal((world, ne))
    for rounds, epoch0 in ((1, 1), (5, 2), (6, 7)):
        buf = torch.zeros(world * nb, dtype=torch.uint8, device=cuda)
        d = torch.from_numpy(vals.copy()).to(cuda)
        _lib.check(L.rg_peer_emulate_f64(world, ne, rounds, epoch0, d.data_ptr(), buf.data_ptr(), D.stream_ptr()),
                   "peer emulate")
        torch.cuda.synchronize()
        got = d.cpu().numpy()
        assert np.array_equal(got, _expected(vals, rounds))
        # no rank timed out (error word of every emulated rank's flag block)
        flags = buf.view(world, nb)[:, nb - 24 * 4:].contiguous().view(torch.int32).view(world, 24)
        assert int(flags[:, 16].abs().sum().item()) == 0


def test_peer_group_registration_single_process(cuda):
    """rg_peer_set with world = 1 registers nothing; the Gram passes and the
    standalone allreduce are then plain single-process sums."""
    from paper_1604_01713_b200 import _lib, device as D

    L = D.lib()
    buf, handle = ctypes.c_void_p(), ctypes.create_string_buffer(64)
    _lib.check(L.rg_peer_alloc(ctypes.byref(buf), handle), "peer alloc")
    try:
        assert handle.raw != b"\0" * 64
        arr = (ctypes.c_void_p * 1)(buf.value)
        _lib.check(L.rg_peer_set(1, 0, arr, 1.0), "peer set")
        assert L.rg_peer_active() == 0
        t = torch.arange(8, dtype=torch.float64, device=cuda)
        _lib.check(L.rg_peer_allreduce_f64(t.data_ptr(), 8, D.stream_ptr()), "peer allreduce")
        assert torch.equal(t.cpu(), torch.arange(8, dtype=torch.float64))
        e = ctypes.c_uint32(5)
        _lib.check(L.rg_peer_error(ctypes.byref(e), D.stream_ptr()), "peer error")
        assert e.value == 0
        n, p = 1000, 8
        Z = np.random.default_rng(0).standard_normal((n, p))
        G = D.small(p, p)
        D.tall(D.to_device_block(Z), None, gram=("self", G))
        assert np.abs(G.cpu().numpy() - Z.T @ Z).max() <= 1e-12 * np.abs(Z.T @ Z).max()
        assert L.rg_peer_set(9, 0, arr, 1.0) == _lib.RG_EBADARG
    finally:
        L.rg_peer_clear()
        _lib.check(L.rg_peer_free(buf), "peer free")


class _FakePeer:
    """World of 2 on one GPU without a second kernel: rank 1's contribution
    and epoch flag are written into rank 0's exchange buffer BEFORE the pass
    is launched, so the pass's last CTA finds its peer already arrived (no
    kernel ever waits on another), sums local + peer in rank order, and
    leaves its own values and flag in rank 1's buffer."""

    SLOT, NE, W = 4096, 4096, 8

    def __init__(self, cuda):
        from paper_1604_01713_b200 import device as D

        self.D, self.L = D, D.lib()
        self.nb = self.L.rg_peer_buffer_bytes()
        self.cuda = cuda
        self.bufs = [torch.zeros(self.nb, dtype=torch.uint8, device=cuda) for _ in range(2)]

    def _views(self, b):
        slot_bytes = 2 * self.W * self.NE * 8
        slots = self.bufs[b][:slot_bytes].view(torch.float64).view(2, self.W, self.NE)
        flags = self.bufs[b][slot_bytes:].view(torch.int32)
        return slots, flags

    def arm(self, epochs_vals):
        """Register the group (epoch counter -> 0) and pre-write rank 1's
        values for epochs 1, 2, ... (flat float64 arrays)."""
        from paper_1604_01713_b200 import _lib

        for b in self.bufs:
            b.zero_()
        slots, flags = self._views(0)
        for i, v in enumerate(epochs_vals):
            epoch = i + 1
            par = epoch & 1
            assert i < 2, "two slot sets: at most two reductions can be pre-armed"
            slots[par, 1, : v.size] = torch.from_numpy(v).to(self.cuda)
            flags[par * self.W + 1] = epoch
        torch.cuda.synchronize()
        arr = (ctypes.c_void_p * 2)(self.bufs[0].data_ptr(), self.bufs[1].data_ptr())
        _lib.check(self.L.rg_peer_set(2, 0, arr, 1.0), "peer set")
        assert self.L.rg_peer_active() == 2

    def sent(self, epoch, count):
        """What rank 0 stored into rank 1's buffer for this epoch, and the flag."""
        slots, flags = self._views(1)
        par = epoch & 1
        return slots[par, 0, :count].cpu().numpy(), int(flags[par * self.W + 0].item())

    def error(self):
        e = ctypes.c_uint32(0)
        self.L.rg_peer_error(ctypes.byref(e), self.D.stream_ptr())
        return e.value

    def close(self):
        self.L.rg_peer_clear()


@pytest.mark.parametrize("shape", ["ws_gram", "ws_update_gram", "ws_self", "nr_self", "nr_sumsq", "v5_gram",
                                   "v6_update_gram", "v3_unaligned", "p20_gram", "complex_gram"])
def test_gram_passes_reduce_over_ranks_in_kernel(cuda, shape):
    """Every rg_tall kernel family finishes its Gram with the peer sum: the
    pass's output is (this rank's Gram) + (the peer's pre-armed values), added
    in rank order, and the peer's buffer holds this rank's Gram and epoch."""
    from paper_1604_01713_b200 import device as D

    rng = np.random.default_rng(5)
    n = 4099
    cplx = shape == "complex_gram"
    p = {"p20_gram": 20, "complex_gram": 8}.get(shape, 8)

    def blk(c):
        a = rng.standard_normal((n, c))
        if cplx:
            a = a + 1j * rng.standard_normal((n, c))
        return a

    Z = blk(p)
    terms, gram_kind, ref_local = [], None, None
    if shape in ("ws_gram", "v5_gram", "p20_gram", "complex_gram"):
        gc = {"ws_gram": 100, "v5_gram": 20, "p20_gram": 108, "complex_gram": 24}[shape]
        Gb = blk(gc)
        ref_local = Gb.conj().T @ Z
        args = dict(Zin=Z, gram=("basis", Gb, gc))
    elif shape in ("ws_update_gram", "v6_update_gram"):
        a = 100 if shape == "ws_update_gram" else 12
        X, S = blk(a), rng.standard_normal((a, p))
        z1 = Z - X @ S
        ref_local = X.T @ z1
        args = dict(Zin=Z, terms=[(X, S)], gram=("basis", X, a))
    elif shape == "ws_self":
        X, S = blk(100), rng.standard_normal((100, p))
        z1 = Z - X @ S
        ref_local = z1.T @ z1
        args = dict(Zin=Z, terms=[(X, S)], gram=("self",))
    elif shape in ("nr_self", "v3_unaligned"):
        ref_local = Z.T @ Z
        args = dict(Zin=Z, gram=("self",))
    else:  # nr_sumsq
        ref_local = (Z * Z).sum(axis=0)
        args = dict(Zin=Z, gram=("sumsq",))

    fake = _FakePeer(cuda)
    try:
        flat = np.asfortranarray(ref_local).reshape(-1, order="F")
        peer_vals = [rng.standard_normal(flat.size * (2 if cplx else 1)) for _ in range(2)]
        fake.arm(peer_vals)
        dt = torch.complex128 if cplx else torch.float64
        Zd = D.to_device_block(Z, cuda, dt)
        if shape == "v3_unaligned":
            Zd = D.to_device_block(np.vstack([np.zeros((1, p)), Z]))[1:]  # row-offset view: 8-byte aligned only
        tl = [(D.to_device_block(X, cuda, dt), torch.from_numpy(np.asfortranarray(S)).to(cuda), -1.0)
              for X, S in args.get("terms", [])]
        for epoch in (1, 2):  # both slot sets
            kind = args["gram"][0]
            if kind == "basis":
                gb = tl[0][0] if args["gram"][1] is args.get("terms", [(None,)])[0][0] else \
                    D.to_device_block(args["gram"][1], cuda, dt)
                out = D.small(args["gram"][2], p, cuda, dt)
                D.tall(Zd, None, tl, gram=("basis", gb, out))
            elif kind == "self":
                out = D.small(p, p, cuda, dt)
                D.tall(Zd, None, tl, gram=("self", out))
            else:
                out = torch.zeros(p, dtype=torch.float64, device=cuda)
                D.tall(Zd, None, tl, gram=("sumsq", out))
            torch.cuda.synchronize()
            assert fake.error() == 0
            got = out.cpu().numpy().reshape(-1, order="F")
            got = got.view(np.float64) if cplx else got
            sent, flag = fake.sent(epoch, got.size)
            assert flag == epoch
            loc = flat.view(np.float64) if cplx else flat
            scale = max(np.abs(loc).max(), 1.0)
            assert np.abs(sent - loc).max() <= 1e-12 * scale          # rank 0's own Gram went to the peer
            assert np.array_equal(got, (0.0 + sent) + peer_vals[epoch - 1])  # rank-order sum, bitwise
    finally:
        fake.close()


@pytest.mark.parametrize("p", [1, 8])
@pytest.mark.parametrize("me", [0, 1, 2])
def test_halo_push_with_prearmed_neighbours(cuda, me, p):
    """The transport-free halo exchange of DistCsr (rg_halo_push /
    rg_halo_wait) for one rank of a 3-rank partition: the neighbours' rows and
    flags are written into this rank's ghost blocks before each product, so no
    kernel waits on another.  The product equals the single-process SpMM
    bitwise; the stand-ins for the neighbours' ghost blocks receive this rank's
    boundary rows at the right offsets with the epoch flag, on both parities."""
    import oracle
    from paper_1604_01713_b200 import device as D, problems
    from paper_1604_01713_b200 import distributed as DI

    world, grid = 3, 9
    A = problems.conv_diff_3d(grid, 20.0)
    rng = np.random.default_rng(11 + me)
    plans, lists = [], {}
    parts = [DI.RowPartition.even(A.n_rows, world, r, align=grid * grid) for r in range(world)]
    blocks = [DI.csr_row_block(A.row_ptr, A.col_idx, A.values, pt.r0, pt.r1) for pt in parts]
    # first pass collects every rank's recv lists, second builds the plans with a local "exchange"
    for r in range(world):
        DI.HaloPlan.from_local_rows(parts[r], *blocks[r], exchange=lambda part, rl: lists.setdefault(part.rank, rl) and {})
    ex = lambda part, rl: {q: lists[q][part.rank] for q in range(world) if q != part.rank and part.rank in lists[q]}  # noqa: E731
    plans = [DI.HaloPlan.from_local_rows(parts[r], *blocks[r], exchange=ex) for r in range(world)]
    plan, part = plans[me], parts[me]
    infos = [{"send": sorted(pl.send_rows), "recv": dict(pl.recv_ranges)} for pl in plans]
    peers = DI.neighbours(infos, me)
    assert peers == {0: [1], 1: [0, 2], 2: [1]}[me]

    flags_local = torch.zeros(64, dtype=torch.int32, device=cuda)
    flags_peer_t = {q: torch.zeros(64, dtype=torch.int32, device=cuda) for q in peers}
    ghost_local = torch.zeros((2, p, max(plan.n_ghost, 1)), dtype=torch.float64, device=cuda)
    ghost_peer_t = {q: torch.full((2, p, max(plans[q].n_ghost, 1)), float("nan"), dtype=torch.float64, device=cuda)
                    for q in peers}
    dst = {q: (plans[q].recv_ranges[me][0], max(plans[q].n_ghost, 1)) for q in peers}
    hp = DI.HaloPeer(me, peers, dst, flags_local.data_ptr(), {q: t.data_ptr() for q, t in flags_peer_t.items()},
                     plan.n_ghost, cuda)
    hp._opener = lambda p_, dt, nb: DI._GhostBlocks(ghost_local.data_ptr(), ghost_local,
                                                    {q: t.data_ptr() for q, t in ghost_peer_t.items()})
    op = DI.DistCsr(plan, None, cuda)
    op._halo_peer = hp
    for epoch in (1, 2, 3):
        X = np.asfortranarray(rng.standard_normal((A.n_rows, p)))
        ref = oracle.spmm(A.row_ptr, A.col_idx, A.values, X, nthreads=1)
        par = epoch & 1
        # pre-arm: the neighbours' rows of X in this rank's ghost block of that parity, and their flags
        ghost_local[par] = torch.from_numpy(np.ascontiguousarray(X[plan.ghost_cols].T)).to(cuda)
        for q in peers:
            flags_local[par * 8 + q] = epoch
        torch.cuda.synchronize()
        Z = D.to_device_block(X[part.r0:part.r1])
        out = D.empty_block(part.n_local, p)
        op.apply_into(Z, out)
        torch.cuda.synchronize()
        hp.check()
        assert hp.epoch == epoch
        assert np.array_equal(D.to_numpy_block(out), ref[part.r0:part.r1])
        for q in peers:
            s0, s1 = plans[q].recv_ranges[me]
            got = ghost_peer_t[q][par, :, s0:s1].cpu().numpy().T
            want = X[plans[q].ghost_cols[s0:s1]]
            assert np.array_equal(got, want)
            assert int(flags_peer_t[q][par * 8 + me].item()) == epoch
            # nothing outside this rank's segment was touched
            rest = torch.cat([ghost_peer_t[q][par, :, :s0].flatten(), ghost_peer_t[q][par, :, s1:].flatten()])
            assert bool(torch.isnan(rest).all().item())
        assert int(flags_local[16].item()) == 0  # ticket re-armed


def test_solver_with_a_silent_peer_is_bitwise_the_single_process_solve(cuda):
    """End to end on one GPU: a peer group of 2 whose other rank has
    'already arrived' at every epoch (its flags pre-set far ahead) and
    contributes zeros.  Every Gram / norm pass of a full GCRO-DR sequence --
    through the fused orchestrators rg_cgs2_f64 / rg_cholqr2_f64 -- then runs
    the in-kernel reduction, and adding the peer's zeros must leave cycles,
    matvec counts, residual histories and solutions bit for bit those of the
    plain run."""
    from paper_1604_01713_b200 import SolverConfig, _lib, device as D, problems, solve_sequence

    L = D.lib()
    systems, kw = problems.cfg1_sequence()
    plain = solve_sequence(systems, SolverConfig(**kw))
    nb = L.rg_peer_buffer_bytes()
    bufs = [torch.zeros(nb, dtype=torch.uint8, device=cuda) for _ in range(2)]
    slot_bytes = 2 * 8 * 4096 * 8
    flags = bufs[0][slot_bytes:].view(torch.int32)
    flags[0 * 8 + 1] = 0x7FFFFFFF  # rank 1, both parities: ahead of every epoch
    flags[1 * 8 + 1] = 0x7FFFFFFF
    torch.cuda.synchronize()
    arr = (ctypes.c_void_p * 2)(bufs[0].data_ptr(), bufs[1].data_ptr())
    _lib.check(L.rg_peer_set(2, 0, arr, 2.0), "peer set")
    try:
        before = L.rg_launch_count()
        peer = solve_sequence(systems, SolverConfig(**kw))
        assert L.rg_launch_count() > before
        e = ctypes.c_uint32(0)
        _lib.check(L.rg_peer_error(ctypes.byref(e), D.stream_ptr()), "peer error")
        assert e.value == 0
    finally:
        L.rg_peer_clear()
    # rank 0 really exchanged: its last Grams and epochs sit in the stand-in for rank 1's buffer
    sent_flags = bufs[1][slot_bytes:].view(torch.int32)
    assert int(sent_flags[0].item()) > 1000 and int(sent_flags[8].item()) > 1000
    for a, b in zip(plain, peer):
        assert a.error is None and b.error is None
        assert a.cycles == b.cycles and a.matvec_count == b.matvec_count
        assert np.array_equal(np.concatenate(a.residual_history), np.concatenate(b.residual_history))
        assert np.array_equal(a.solution, b.solution)
