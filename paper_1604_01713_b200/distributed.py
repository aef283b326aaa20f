"""Row-partitioned multi-GPU execution (one process per GPU).

The reference is single-process; this is the B200 build's
scaling layer:

* ``RowPartition``   contiguous row blocks [r0, r1) of A, B, X, R, W, C, U
                     (optionally aligned to whole grid planes).
* ``HaloPlan``       for the local rows of A: the columns owned by other
                     ranks ("ghosts"), grouped by owner in ascending global
                     order, and the rows this rank must send to each peer
                     (recv lists exchanged once with all_gather_object).
                     The local CSR keeps every row's entries in their
                     original (ascending global column) order and only
                     renumbers the column indices: owned j -> j - r0, ghost
                     j -> n_local + slot.  The SpMM therefore performs the
                     reference's exact per-row operation sequence and stays
                     bitwise equal to the single-GPU product.
* ``DistCsr``        the operator: per application, pack the send rows,
                     exchange them (NCCL isend/irecv, or host-staged for
                     gloo), run the interior rows (no ghost columns) while
                     the exchange is in flight, then the boundary rows.
* ``CommContext``    the sum-allreduce applied to every Gram / norm that
                     rg_tall produces (device.set_comm); the (k+mp) x p
                     Grams are a few KB, i.e. latency-bound.
* ``PeerGroup``      the ranks of one node map each other's exchange buffers
                     (CUDA IPC over NVLink); the Gram passes then finish the
                     sum over the ranks inside their own kernels
                     (rg_common.cuh peer_allreduce): no NCCL call per Gram,
                     and the C orchestrators (rg_cgs2_f64 / rg_cholqr2_f64)
                     run unchanged on a row partition.

Host-side small problems (progressive LS, harmonic Ritz) are replicated on
every rank from bitwise-identical allreduced inputs.  Seeded random vectors
(breakdown repair, block enlargement) are drawn at the global size on every
rank and sliced, so they equal the single-process draws.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from . import device as _dev


# ---------------------------------------------------------------------------
# partition
# ---------------------------------------------------------------------------


@dataclass
class RowPartition:
    n: int
    world: int
    rank: int
    bounds: np.ndarray  # world + 1 row offsets

    @classmethod
    def even(cls, n: int, world: int, rank: int, align: int = 1) -> "RowPartition":
        """Contiguous blocks of (as nearly as possible) equal size, cut at
        multiples of ``align`` rows (e.g. one z-plane of a stencil)."""
        units = (n + align - 1) // align
        cuts = [min(n, (units * q // world) * align) for q in range(world + 1)]
        cuts[-1] = n
        return cls(n, world, rank, np.asarray(cuts, dtype=np.int64))

    @property
    def r0(self) -> int:
        return int(self.bounds[self.rank])

    @property
    def r1(self) -> int:
        return int(self.bounds[self.rank + 1])

    @property
    def n_local(self) -> int:
        return self.r1 - self.r0

    def owner(self, cols: np.ndarray) -> np.ndarray:
        return np.searchsorted(self.bounds, cols, side="right") - 1


# ---------------------------------------------------------------------------
# halo plan
# ---------------------------------------------------------------------------


@dataclass
class HaloPlan:
    part: RowPartition
    row_ptr: np.ndarray           # local CSR (n_local + 1)
    col_idx: np.ndarray           # renumbered columns
    values: np.ndarray
    ghost_cols: np.ndarray        # global ids of ghost slots, ascending
    recv_ranges: dict             # peer -> (slot0, slot1)
    send_rows: dict = field(default_factory=dict)  # peer -> local row ids to send
    interior: tuple = (0, 0)      # [i0, i1): rows without ghost columns

    @property
    def n_ghost(self) -> int:
        return int(self.ghost_cols.size)

    @classmethod
    def from_local_rows(cls, part: RowPartition, row_ptr, col_idx, values, exchange=None) -> "HaloPlan":
        """Build from the local rows (global column indices, ascending per
        row).  ``exchange(recv_lists) -> {peer: rows peer needs from me}``
        defaults to all_gather_object over the default process group."""
        rp = np.asarray(row_ptr, dtype=np.int64)
        ci = np.asarray(col_idx, dtype=np.int64)
        r0, r1 = part.r0, part.r1
        owned = (ci >= r0) & (ci < r1)
        ghosts = np.unique(ci[~owned])
        slot = np.searchsorted(ghosts, ci[~owned])
        new_ci = ci.copy()
        new_ci[owned] -= r0
        new_ci[~owned] = part.n_local + slot
        owners = part.owner(ghosts)
        recv_ranges = {}
        recv_lists = {}
        for q in np.unique(owners):
            idx = np.flatnonzero(owners == q)
            recv_ranges[int(q)] = (int(idx[0]), int(idx[-1]) + 1)
            recv_lists[int(q)] = ghosts[idx]
        # interior rows: the longest middle range whose rows touch no ghost
        nl = part.n_local
        row_has_ghost = np.zeros(nl, dtype=bool)
        if (~owned).any():
            rows = np.repeat(np.arange(nl), np.diff(rp))
            row_has_ghost[np.unique(rows[~owned])] = True
        if row_has_ghost.any():
            g = np.flatnonzero(row_has_ghost)
            # boundary rows form a prefix and a suffix for slab partitions
            first_gap = np.flatnonzero(np.diff(g) > 1)
            if first_gap.size:
                i0 = int(g[first_gap[0]]) + 1
                i1 = int(g[first_gap[0] + 1])
            elif g[0] == 0:
                i0, i1 = int(g[-1]) + 1, nl
            elif g[-1] == nl - 1:
                i0, i1 = 0, int(g[0])
            else:
                i0 = i1 = 0
        else:
            i0, i1 = 0, nl
        plan = cls(part, rp.astype(np.int32), new_ci.astype(np.int32), np.asarray(values),
                   ghosts, recv_ranges, {}, (i0, i1))
        ex = exchange if exchange is not None else _exchange_recv_lists
        needed_from_me = ex(part, recv_lists)
        plan.send_rows = {q: (np.asarray(g_ids, dtype=np.int64) - r0) for q, g_ids in needed_from_me.items()}
        return plan


def _exchange_recv_lists(part: RowPartition, recv_lists: dict) -> dict:
    gathered = [None] * part.world
    dist.all_gather_object(gathered, {q: v.tolist() for q, v in recv_lists.items()})
    out = {}
    for q, lists in enumerate(gathered):
        if q == part.rank or lists is None:
            continue
        mine = lists.get(part.rank)
        if mine:
            out[q] = np.asarray(mine, dtype=np.int64)
    return out


# ---------------------------------------------------------------------------
# communicator context (Gram allreduce + halo exchange transport)
# ---------------------------------------------------------------------------


def peer_eligible(infos, max_world: int = 8):
    """Can these ranks reduce through peer memory?  ``infos`` is every
    rank's (hostname, GPU UUID or device index, None without a GPU).  Returns (ok, reason):
    one node, one distinct GPU per rank, 2..max_world ranks."""
    world = len(infos)
    if world < 2:
        return False, "single rank"
    if world > max_world:
        return False, f"{world} ranks > {max_world}"
    hosts = {h for h, _ in infos}
    if len(hosts) != 1:
        return False, f"ranks span {len(hosts)} hosts"
    devs = [d for _, d in infos]
    if any(d is None for d in devs):
        return False, "a rank has no CUDA device"
    if len(set(devs)) != world:
        return False, "ranks share a GPU (kernels of different ranks must run concurrently)"
    return True, "ok"


class PeerGroup:
    """Exchange buffers of the node's ranks, mapped into each other with
    CUDA IPC, registered with librgb200 (rg_peer_set): from then on every
    Gram / norm pass sums over the ranks inside its own kernel.  ``create``
    returns None (with the reason on stderr) when the ranks are not eligible
    or the self-test fails; the NCCL allreduce then stays in charge."""

    SELFTEST_TIMEOUT_S = 5.0

    def __init__(self, comm, local, mapped, timeout_s):
        self.comm, self.local, self.mapped, self.timeout_s = comm, local, mapped, timeout_s
        self.halos = []  # HaloPeer objects of the operators built on this group
        self.ptrs = []

    @classmethod
    def create(cls, comm: "CommContext", timeout_s: float = 20.0, *, force: bool = False, selftest: bool = True):
        """``force`` / ``selftest=False`` (tests): map the buffers whatever the
        backend and GPU placement, and skip the known-answer reduction -- two
        processes sharing one GPU can check the IPC plumbing with host
        barriers, but must not launch kernels that wait on each other."""
        import ctypes
        import os
        import socket
        import sys

        if not torch.cuda.is_available():
            return None
        if not force and (os.environ.get("RG_PEER_GRAM", "1") == "0" or not comm.nccl):
            return None
        infos = [None] * comm.world
        # the GPU's UUID, not its index: ranks may each see their GPU as device 0 (CUDA_VISIBLE_DEVICES)
        props = torch.cuda.get_device_properties(torch.cuda.current_device())
        gpu = str(getattr(props, "uuid", "")) or torch.cuda.current_device()
        dist.all_gather_object(infos, (socket.gethostname(), gpu), group=comm.group)
        ok, why = peer_eligible(infos)
        if not ok and not force:
            if comm.rank == 0 and comm.world > 1:
                print(f"[rgb200] peer-memory Gram reduction off: {why}", file=sys.stderr)
            return None
        L = _dev.lib()
        buf, handle = ctypes.c_void_p(), ctypes.create_string_buffer(64)
        _lib.check(L.rg_peer_alloc(ctypes.byref(buf), handle), "peer alloc")
        handles = [None] * comm.world
        dist.all_gather_object(handles, handle.raw, group=comm.group)
        ptrs, mapped, failed = [], [], False
        for r, h in enumerate(handles):
            if r == comm.rank:
                ptrs.append(buf.value)
                continue
            q = ctypes.c_void_p()
            if L.rg_peer_open(h, ctypes.byref(q)) != _lib.RG_OK:
                failed = True
                break
            ptrs.append(q.value)
            mapped.append(q.value)
        # all ranks agree on the outcome before anything is registered
        flag = torch.tensor([1 if failed else 0], device="cuda" if comm.nccl else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=comm.group)
        self = cls(comm, buf.value, mapped, timeout_s)
        self.ptrs = list(ptrs)  # rank r's buffer as mapped here (ptrs[rank] = the local one)
        if int(flag.item()):
            self._release()
            if comm.rank == 0:
                print("[rgb200] peer-memory Gram reduction off: cudaIpcOpenMemHandle failed", file=sys.stderr)
            return None
        arr = (ctypes.c_void_p * comm.world)(*ptrs)
        dist.barrier(group=comm.group)
        if not selftest:
            _lib.check(L.rg_peer_set(comm.world, comm.rank, arr, timeout_s), "peer set")
            return self
        _lib.check(L.rg_peer_set(comm.world, comm.rank, arr, cls.SELFTEST_TIMEOUT_S), "peer set")
        # self-test: one reduction of known values, bounded wait
        t = torch.full((8,), float(comm.rank + 1), dtype=torch.float64, device="cuda")
        _lib.check(L.rg_peer_allreduce_f64(t.data_ptr(), 8, _dev.stream_ptr()), "peer allreduce")
        bad = self.error_epoch() != 0 or not bool((t == comm.world * (comm.world + 1) / 2).all().item())
        flag = torch.tensor([1 if bad else 0], device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=comm.group)
        if int(flag.item()):
            L.rg_peer_clear()
            self._release()
            if comm.rank == 0:
                print("[rgb200] peer-memory Gram reduction off: self-test failed", file=sys.stderr)
            return None
        dist.barrier(group=comm.group)
        _lib.check(L.rg_peer_set(comm.world, comm.rank, arr, timeout_s), "peer set")
        return self

    def error_epoch(self) -> int:
        import ctypes

        e = ctypes.c_uint32(0)
        _lib.check(_dev.lib().rg_peer_error(ctypes.byref(e), _dev.stream_ptr()), "peer error")
        return int(e.value)

    def check(self) -> None:
        e = self.error_epoch()
        if e:
            raise _lib.KernelError(f"peer-memory Gram reduction {e}: a rank did not arrive within {self.timeout_s} s")
        for h in self.halos:
            h.check()

    def _release(self):
        L = _dev.lib()
        for h in self.halos:
            h.release()
        self.halos = []
        for q in self.mapped:
            L.rg_peer_close(q)
        self.mapped = []
        if self.local:
            L.rg_peer_free(self.local)
            self.local = None

    def close(self):
        torch.cuda.synchronize()
        dist.barrier(group=self.comm.group)
        _dev.lib().rg_peer_clear()
        self._release()


class _DevView:
    """A raw device allocation as a CUDA-array-interface object."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _wrap(ptr: int, shape, dtype, device) -> torch.Tensor:
    typestr = {torch.float64: "<f8", torch.complex128: "<c16", torch.int32: "<i4"}[dtype]
    return torch.as_tensor(_DevView(ptr, shape, typestr), device=device)


class _GhostBlocks:
    """Two ghost blocks (epoch parity) of one (p, dtype) in an IPC
    allocation, and the neighbours' mappings of theirs."""

    def __init__(self, local_ptr, tensor, peer_ptr):
        self.local_ptr, self.local, self.peer_ptr = local_ptr, tensor, peer_ptr  # tensor: (2, p, n_ghost)


class HaloPeer:
    """Halo exchange of one DistCsr without a transport library: each rank
    stores the rows a neighbour needs straight into that neighbour's ghost
    block (rg_halo_push: NVLink peer stores + an epoch flag) and waits for its
    own neighbours' flags ahead of the boundary rows (rg_halo_wait).  Ghost
    blocks alternate with the epoch's parity and every pair of neighbours
    signals both ways, so a rank is never more than one product ahead of a
    neighbour.  All products of the operator go to one stream, in the same
    order on every rank.

    flags (uint32, one IPC allocation per rank): [par * 8 + src] epochs,
    [16] push ticket, [17] error word."""

    FLAG_WORDS = 64
    TIMEOUT_S = 20.0

    def __init__(self, rank, peers, dst, flags_local, flags_peer, n_ghost, device, opener=None, mapped=None):
        self.rank, self.peers, self.dst = rank, list(peers), dict(dst)
        self.flags_local, self.flags_peer = flags_local, dict(flags_peer)
        self.n_ghost, self.device = n_ghost, device
        self.epoch = 0
        self._ghosts = {}
        self._opener = opener      # (p, dtype, nbytes) -> _GhostBlocks (collective); tests inject pointers
        self._mapped = list(mapped or [])
        self._owned = [flags_local] if opener is not None else []
        import ctypes

        self._peer_arr = (ctypes.c_int32 * max(len(self.peers), 1))(*self.peers)

    @classmethod
    def create(cls, plan: "HaloPlan", comm: "CommContext", device):
        """Collective over the group: exchange the flag handles, each rank's
        ghost layout (who lands where) and neighbour sets."""
        import ctypes

        L = _dev.lib()
        buf, handle = ctypes.c_void_p(), ctypes.create_string_buffer(64)
        _lib.check(L.rg_ipc_alloc(4 * cls.FLAG_WORDS, ctypes.byref(buf), handle), "ipc alloc")
        mine = {"recv": dict(plan.recv_ranges), "send": sorted(plan.send_rows), "n_ghost": plan.n_ghost,
                "flags": handle.raw}
        infos = [None] * comm.world
        dist.all_gather_object(infos, mine, group=comm.group)
        me = comm.rank
        peers = neighbours(infos, me)
        dst = {q: (infos[q]["recv"][me][0], max(infos[q]["n_ghost"], 1)) for q in peers if me in infos[q]["recv"]}
        flags_peer, mapped = {}, []
        for q in peers:
            ptr = ctypes.c_void_p()
            _lib.check(L.rg_peer_open(infos[q]["flags"], ctypes.byref(ptr)), "peer open")
            flags_peer[q] = ptr.value
            mapped.append(ptr.value)

        def opener(p, dtype, nbytes):
            b, h = ctypes.c_void_p(), ctypes.create_string_buffer(64)
            _lib.check(L.rg_ipc_alloc(nbytes, ctypes.byref(b), h), "ipc alloc")
            hs = [None] * comm.world
            dist.all_gather_object(hs, h.raw, group=comm.group)
            peer_ptr = {}
            for q in peers:
                ptr = ctypes.c_void_p()
                _lib.check(L.rg_peer_open(hs[q], ctypes.byref(ptr)), "peer open")
                peer_ptr[q] = ptr.value
                self._mapped.append(ptr.value)
            self._owned.append(b.value)
            dist.barrier(group=comm.group)
            return _GhostBlocks(b.value, _wrap(b.value, (2, p, max(plan.n_ghost, 1)), dtype, device), peer_ptr)

        self = cls(me, peers, dst, buf.value, flags_peer, plan.n_ghost, device, opener, mapped)
        dist.barrier(group=comm.group)
        return self

    def ghost(self, p: int, dtype) -> _GhostBlocks:
        key = (p, dtype)
        if key not in self._ghosts:
            esz = 16 if dtype == torch.complex128 else 8
            self._ghosts[key] = self._opener(p, dtype, 2 * p * max(self.n_ghost, 1) * esz)
        return self._ghosts[key]

    def push_all(self, Z: torch.Tensor, send_idx: dict, gb: _GhostBlocks) -> int:
        """Next epoch: store this rank's rows into every neighbour's ghost
        block of that parity and publish the flag (k = 0: the flag only)."""
        L, st = _dev.lib(), _dev.stream_ptr()
        self.epoch += 1
        par = self.epoch & 1
        p = Z.shape[1]
        esz = 16 if Z.dtype == torch.complex128 else 8
        for q in self.peers:
            idx = send_idx.get(q)
            k = 0 if idx is None else idx.numel()
            s0, ldq = self.dst.get(q, (0, 1))
            out = gb.peer_ptr[q] + (par * p * ldq + s0) * esz if k else None
            _lib.check(L.rg_halo_push(k, p, esz, idx.data_ptr() if k else None, Z.data_ptr(), _dev.ld_of(Z), out, ldq,
                                      self.flags_peer[q] + 4 * (par * 8 + self.rank), self.epoch,
                                      self.flags_local + 4 * 16, st), "halo push")
        return par

    def wait_all(self) -> None:
        if not self.peers:
            return
        par = self.epoch & 1
        _lib.check(_dev.lib().rg_halo_wait(self.flags_local + 4 * (par * 8), self._peer_arr, len(self.peers),
                                           self.epoch, self.TIMEOUT_S, self.flags_local + 4 * 17,
                                           _dev.stream_ptr()), "halo wait")

    def check(self) -> None:
        e = int(_wrap(self.flags_local, (self.FLAG_WORDS,), torch.int32, self.device)[17].item())
        if e:
            raise _lib.KernelError(f"halo exchange {e}: a neighbour's rows did not arrive within {self.TIMEOUT_S} s")

    def release(self) -> None:
        L = _dev.lib()
        for q in self._mapped:
            L.rg_peer_close(q)
        for b in self._owned:
            L.rg_peer_free(b)
        self._mapped, self._owned, self._ghosts = [], [], {}


def neighbours(infos, me: int):
    """Ranks this rank exchanges flags with: everyone it sends rows to or
    receives rows from, made symmetric (q lists me => I list q), so that each
    pair signals both ways every product."""
    mine = set(infos[me]["send"]) | set(infos[me]["recv"])
    for q, inf in enumerate(infos):
        if q != me and (me in inf["send"] or me in inf["recv"]):
            mine.add(q)
    mine.discard(me)
    return sorted(int(q) for q in mine)


class CommContext:
    """Sum-allreduce of Grams and point-to-point halo transport over a
    torch.distributed group.  NCCL moves CUDA buffers directly (NVLink);
    other backends (gloo, used by the CPU tests) stage through host memory.
    With NCCL on one node the Gram sums move into the producing kernels
    (``PeerGroup``); ``allreduce_`` then serves only the buffers no rg_tall
    pass produced."""

    def __init__(self, group=None, peer: bool = True):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nccl = dist.get_backend(group) == "nccl"
        self.peer = PeerGroup.create(self) if (peer and self.world > 1) else None

    @property
    def peer_active(self) -> bool:
        return self.peer is not None

    def close(self):
        if self.peer is not None:
            self.peer.close()
            self.peer = None

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return t
        if self.nccl or not t.is_cuda:
            buf = t if t.is_contiguous() else t.contiguous()
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)
            if buf is not t:
                t.copy_(buf)
            return t
        h = t.detach().cpu().contiguous()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
        t.copy_(h)
        return t

    def exchange(self, sends: dict, recvs: dict):
        """Post all sends/recvs; returns a list of works (wait() on each).
        Keys are peer ranks or (peer, tag) tuples; messages to one peer are
        matched in key order on both sides."""
        ops = []
        staged = []
        peer = lambda key: key[0] if isinstance(key, tuple) else key  # noqa: E731
        sends = dict(sorted(sends.items()))
        recvs = dict(sorted(recvs.items()))
        for key, buf in recvs.items():
            q = peer(key)
            if self.nccl or not buf.is_cuda:
                ops.append(dist.P2POp(dist.irecv, buf, q, self.group))
            else:
                h = torch.empty(buf.shape, dtype=buf.dtype)
                staged.append((buf, h))
                ops.append(dist.P2POp(dist.irecv, h, q, self.group))
        for key, buf in sends.items():
            q = peer(key)
            if self.nccl or not buf.is_cuda:
                ops.append(dist.P2POp(dist.isend, buf, q, self.group))
            else:
                ops.append(dist.P2POp(dist.isend, buf.cpu(), q, self.group))
        works = dist.batch_isend_irecv(ops) if ops else []
        return works, staged

    def allgather_np(self, arr: np.ndarray) -> list:
        """All ranks' copies of a small host array (same shape everywhere)."""
        t = torch.from_numpy(np.ascontiguousarray(arr))
        if self.nccl:
            t = t.cuda()
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return [o.cpu().numpy() for o in out]

    @staticmethod
    def finish(works, staged):
        for w in works:
            w.wait()
        for dst, h in staged:
            dst.copy_(h)


# ---------------------------------------------------------------------------
# distributed operator
# ---------------------------------------------------------------------------


class DistCsr:
    """Row block of A on this rank + its halo plan; ``apply_into`` is the
    distributed A @ Z for column-major local blocks Z (n_local x p)."""

    def __init__(self, plan: HaloPlan, comm: CommContext, device=None, local_spmm=None):
        self.plan = plan
        self.part = plan.part
        self.comm = comm
        self.n_rows = self.part.n_local
        self.n_cols = self.part.n_local
        self.n_global = self.part.n
        self.device = device
        self._local_spmm = local_spmm
        if local_spmm is None:
            from .sparse_core import DeviceCsr

            self.dcsr = DeviceCsr.from_host(self.n_rows, self.n_rows + plan.n_ghost, plan.row_ptr, plan.col_idx,
                                            plan.values, device)
            # the diagonal-layout SpMM serves the interior rows (owned columns only:
            # the stencil's own diagonals); boundary rows read ghosts through the CSR kernel
            self.dcsr.dia_rows = plan.interior
            dev = self.dcsr.device
        else:
            self.dcsr = None
            dev = torch.device("cpu") if device is None else torch.device(device)
        self.dev = dev
        self._send_idx = {q: torch.from_numpy(np.ascontiguousarray(v, dtype=np.int32)).to(dev)
                          for q, v in plan.send_rows.items()}
        self._ghost = {}
        self._sendbuf = {}
        # ranks of one node under NCCL: neighbours store into each other's ghost blocks
        self._halo_peer = None
        if local_spmm is None and comm is not None and getattr(comm, "peer_active", False):
            self._halo_peer = HaloPeer.create(plan, comm, dev)
            comm.peer.halos.append(self._halo_peer)

    def _ghost_block(self, p, dtype):
        key = (p, dtype)
        if key not in self._ghost:
            ng = max(self.plan.n_ghost, 1)
            # (p, n_ghost) contiguous == column-major (n_ghost, p), ld = n_ghost
            self._ghost[key] = torch.zeros((p, ng), dtype=dtype, device=self.dev)
        return self._ghost[key]

    def _pack(self, Z: torch.Tensor, q: int, idx: torch.Tensor) -> torch.Tensor:
        """Rows ``idx`` of Z as a (p, k) contiguous buffer (column c = row c):
        one rg_halo_pack launch on the device, index_select on the CPU path
        of the gloo tests (local_spmm given)."""
        p, k = Z.shape[1], idx.numel()
        if not Z.is_cuda:
            return Z.index_select(0, idx.long()).t().contiguous()
        key = (q, p, Z.dtype)
        buf = self._sendbuf.get(key)
        if buf is None:
            buf = self._sendbuf[key] = torch.empty((p, k), dtype=Z.dtype, device=Z.device)
        esz = 16 if Z.dtype == torch.complex128 else 8
        _lib.check(_dev.lib().rg_halo_pack(k, p, esz, idx.data_ptr(), Z.data_ptr(), _dev.ld_of(Z), buf.data_ptr(),
                                           k, _dev.stream_ptr()), "halo pack")
        return buf

    def apply_into(self, Z: torch.Tensor, out: torch.Tensor) -> None:
        plan = self.plan
        p = Z.shape[1]
        i0, i1 = plan.interior
        if self._halo_peer is not None and Z.is_cuda:
            # peer stores into the neighbours' ghost blocks, the interior rows
            # while they travel, one wait kernel, then the boundary rows
            hp = self._halo_peer
            gb = hp.ghost(p, Z.dtype)
            par = hp.push_all(Z, self._send_idx, gb)
            if i1 > i0:
                self._spmm(Z, out, i0, i1, None)
            hp.wait_all()
            Xg = gb.local[par].t()[: plan.n_ghost] if plan.n_ghost else None
            if i0 > 0:
                self._spmm(Z, out, 0, i0, Xg)
            if i1 < self.n_rows:
                self._spmm(Z, out, max(i1, i0), self.n_rows, Xg)
            return
        G = self._ghost_block(p, Z.dtype)
        # pack the rows each peer needs (one kernel per peer); every column of
        # a send buffer is one message, received straight into the matching
        # contiguous column segment G[c, s0:s1] of the ghost block
        sends, recvs = {}, {}
        for q, idx in self._send_idx.items():
            buf = self._pack(Z, q, idx)
            for c in range(p):
                sends[(q, c)] = buf[c]
        for q, (s0, s1) in plan.recv_ranges.items():
            for c in range(p):
                recvs[(q, c)] = G[c, s0:s1]
        works, staged = self.comm.exchange(sends, recvs) if self.comm is not None else ([], [])
        # interior rows need no ghost column: overlap them with the exchange
        if i1 > i0:
            self._spmm(Z, out, i0, i1, None)
        CommContext.finish(works, staged)
        Xg = G.t()[: plan.n_ghost] if plan.n_ghost else None
        if i0 > 0:
            self._spmm(Z, out, 0, i0, Xg)
        if i1 < self.n_rows:
            self._spmm(Z, out, max(i1, i0), self.n_rows, Xg)

    def _spmm(self, Z, out, rb, re, Xg):
        if self._local_spmm is not None:
            self._local_spmm(self.plan, Z, out, rb, re, Xg)
            return
        _dev.spmm(self.dcsr, Z, out, rb, re, n_local=self.n_rows, Xg=Xg)

    # solver integration
    def __call__(self, Z):
        out = _dev.empty_block(Z.shape[0], Z.shape[1], Z.device, Z.dtype)
        self.apply_into(Z, out)
        return out


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


def local_rows(part: RowPartition, M):
    """Rows [r0, r1) of a host block / CsrMatrix-like array."""
    return M[part.r0: part.r1]


def csr_row_block(row_ptr, col_idx, values, r0, r1):
    """CSR arrays of rows [r0, r1) (global column indices)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    a, b = rp[r0], rp[r1]
    return rp[r0: r1 + 1] - a, np.asarray(col_idx)[a:b], np.asarray(values)[a:b]


def setup(A, group=None, align: int = 1, device=None):
    """Partition a host CsrMatrix across the ranks of ``group`` and register
    the Gram allreduce.  Returns (DistCsr, RowPartition)."""
    comm = CommContext(group)
    part = RowPartition.even(A.n_rows, comm.world, comm.rank, align)
    rp, ci, v = csr_row_block(A.row_ptr, A.col_idx, A.values, part.r0, part.r1)
    plan = HaloPlan.from_local_rows(part, rp, ci, v)
    op = DistCsr(plan, comm, device)
    _dev.set_comm(comm, part)
    return op, part


def teardown():
    comm = _dev.get_comm()
    _dev.set_comm(None, None)
    if comm is not None:
        comm.close()
