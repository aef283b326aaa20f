"""Device-side plumbing: column-major blocks in HBM, workspace, and the thin
wrappers that launch librgb200 kernels on torch's current CUDA stream.

Layout: every n x p block is column-major (Fortran order,
like the reference's ``as_block``, sparse_core.py:51-58) with a leading
dimension ``ld`` rounded up to a multiple of 32 doubles (256 B), so every
column starts on a 256-byte boundary and warp accesses are full segments.
torch is used only as the allocator / stream provider.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import threading

import numpy as np
import torch

from . import _lib

LD_ALIGN = 32
MAX_P = 32        # block width one rg_tall launch handles (p > 16: v6 kernel only)
MAX_P_FUSED = 16  # widest block of the rg_cgs2_f64 / rg_cholqr2_f64 orchestrators
MAX_GC = 128      # Gram basis columns per launch (p <= 16)


def _r_limits(p: int):
    """(max Gram basis columns, max staged term columns) of one real launch."""
    if p <= 16:
        return MAX_GC, MAX_TERM_COLS
    return (32 if p <= 24 else 16), 128
MAX_TERM_COLS = 512
MAX_P_C = 16      # complex128 limits (rg_tall_c128); blocks wider than 8 allow
MAX_GC_C = 48     # a 32-column Gram basis and 128 staged term columns per launch
MAX_TERM_COLS_C = 256


def _c_limits(p: int, has_terms: bool = True):
    """(max Gram basis columns, max staged term columns) of one complex launch."""
    if p > 8:
        return (32 if has_terms else 64), 128
    return MAX_GC_C, MAX_TERM_COLS_C


_COMM = None   # distributed.CommContext when row-partitioned (Gram allreduce)
_PART = None   # distributed.RowPartition of this rank


def set_comm(comm, part) -> None:
    """Register the row-partition context: every Gram / norm rg_tall
    produces is then summed across ranks."""
    global _COMM, _PART
    _COMM, _PART = comm, part


def get_comm():
    return _COMM


def get_part():
    return _PART


class NoDeviceError(RuntimeError):
    """The B200 path needs a CUDA device; there is no CPU fallback."""


_CUDA_OK = None


def require_cuda(device=None) -> torch.device:
    global _CUDA_OK
    if _CUDA_OK is None:
        _CUDA_OK = torch.cuda.is_available()
    if not _CUDA_OK:
        raise NoDeviceError("paper_1604_01713_b200 needs a CUDA device (sm_100a); no CPU fallback exists")
    if device is None:
        return torch.device("cuda", torch._C._cuda_getDevice())
    dev = device if isinstance(device, torch.device) else torch.device(device)
    if dev.type != "cuda":
        raise NoDeviceError(f"device {dev} is not a CUDA device")
    return dev


def lib():
    return _lib._lib if _lib._lib is not None else _lib.load()


def stream_ptr() -> int:
    """Raw handle of torch's current stream on the current device (the
    launch stream of every rg_* call)."""
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def round_ld(n: int) -> int:
    return max(LD_ALIGN, (int(n) + LD_ALIGN - 1) // LD_ALIGN * LD_ALIGN)


def empty_block(n: int, p: int, device=None, dtype=torch.float64, ld: int | None = None) -> torch.Tensor:
    """Column-major (n, p) tensor with padded leading dimension."""
    dev = require_cuda(device)
    ld = round_ld(n) if ld is None else ld
    store = torch.empty((max(p, 1), ld), dtype=dtype, device=dev)
    return store.t()[:n, :p]


def zeros_block(n: int, p: int, device=None, dtype=torch.float64) -> torch.Tensor:
    b = empty_block(n, p, device, dtype)
    b.zero_()
    return b


def small(rows: int, cols: int, device=None, dtype=torch.float64) -> torch.Tensor:
    """Dense column-major rows x cols with ld = rows (coefficient matrices)."""
    dev = require_cuda(device)
    return torch.empty((max(cols, 1), max(rows, 1)), dtype=dtype, device=dev).t()[:rows, :cols]


def upload_small(a: np.ndarray, device=None) -> torch.Tensor:
    """A small host matrix (coefficients) on the device without stalling the
    stream: staged through pinned memory and copied asynchronously, so the
    host does not wait for the queued kernels to drain (a pageable
    ``torch.from_numpy(a).to(dev)`` synchronises the stream first).  The
    result is column-major with ld = rows, like ``small``."""
    dev = require_cuda(device)
    a = np.asarray(a)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    host = torch.empty((a.shape[1], a.shape[0]), dtype=torch.complex128 if np.iscomplexobj(a) else torch.float64,
                       pin_memory=True)
    host.numpy()[...] = a.T
    return host.to(dev, non_blocking=True).t()


def ld_of(t: torch.Tensor) -> int:
    n = t.shape[0]
    if t.dim() == 1:
        return max(n, 1)
    if t.shape[1] <= 1:
        s = t.stride(1)
        return s if s >= n else max(n, 1)
    return t.stride(1)


def is_col_major(t: torch.Tensor) -> bool:
    if t.dim() != 2:
        return False
    if t.shape[0] > 1 and t.stride(0) != 1:
        return False
    return t.shape[1] <= 1 or t.stride(1) >= t.shape[0]


def to_device_block(x, device=None, dtype=torch.float64) -> torch.Tensor:
    """numpy / torch 2-D input -> column-major CUDA tensor (copies if needed)."""
    dev = require_cuda(device)
    if isinstance(x, torch.Tensor):
        t = x
        if t.dim() == 1:
            t = t.reshape(-1, 1)
        if t.is_complex():
            dtype = torch.complex128
        if t.device == dev and t.dtype == dtype and is_col_major(t):
            return t
        out = empty_block(t.shape[0], t.shape[1], dev, dtype)
        out.copy_(t)
        return out
    a = np.asarray(x)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    if np.iscomplexobj(a):
        dtype = torch.complex128
    np_dtype = np.complex128 if dtype == torch.complex128 else np.float64
    a = np.asfortranarray(a, dtype=np_dtype)
    out = empty_block(a.shape[0], a.shape[1], dev, dtype)
    # a is F-ordered: its transpose is a C-contiguous (p, n) array
    host = torch.from_numpy(a.T)
    if a.nbytes >= Staging.MIN_BYTES:
        Staging.upload([(_bytes_view(out[:, c]), _bytes_view(host[c])) for c in range(a.shape[1])])
    else:
        out.copy_(host.t())
    return out


class Staging:
    """Large host <-> device copies through two persistent page-locked
    chunks: the DMA of one chunk overlaps the (multi-threaded) host copy of
    the other between the chunk and the caller's pageable array.  The
    driver's own pageable path moves ~11 GB/s up and, into a freshly
    allocated array, 2.3 GB/s down (page faults inside the copy); a 1 GB
    solution came back in 0.47 s (tools/prof_setup.py)."""

    CHUNK = 64 << 20
    MIN_BYTES = 8 << 20
    _bufs = None
    _events = None
    _lock = threading.Lock()  # one transfer at a time owns the two chunks
    # host-copy threads for the duration of a transfer (launchers such as torchrun
    # export OMP_NUM_THREADS=1, which would leave the chunk copies single-threaded)
    THREADS = max(1, min(16, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)))

    @classmethod
    @contextlib.contextmanager
    def _host_threads(cls):
        old = torch.get_num_threads()
        if old < cls.THREADS:
            torch.set_num_threads(cls.THREADS)
        try:
            yield
        finally:
            if old < cls.THREADS:
                torch.set_num_threads(old)

    @classmethod
    def _get(cls):
        if cls._bufs is None:
            cls._bufs = [torch.empty(cls.CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
            cls._events = [torch.cuda.Event() for _ in range(2)]
        return cls._bufs, cls._events

    @classmethod
    def _segments(cls, dev_flat: torch.Tensor, host_flat: torch.Tensor):
        n = dev_flat.numel()
        return [(dev_flat[o: o + cls.CHUNK], host_flat[o: o + cls.CHUNK]) for o in range(0, n, cls.CHUNK)]

    @classmethod
    def download(cls, pairs) -> None:
        """pairs: [(contiguous CUDA uint8 view, contiguous CPU uint8 view)], same lengths."""
        with cls._lock, cls._host_threads():
            cls._download(pairs)

    @classmethod
    def _download(cls, pairs) -> None:
        bufs, evs = cls._get()
        segs = [sg for d, h in pairs for sg in cls._segments(d, h)]
        stream = torch.cuda.current_stream()
        prev = None
        for j, (d, h) in enumerate(segs):
            b = j & 1
            bufs[b][: d.numel()].copy_(d, non_blocking=True)
            evs[b].record(stream)
            if prev is not None:
                pb, ph = prev
                evs[pb].synchronize()
                ph.copy_(bufs[pb][: ph.numel()])
            prev = (b, h)
        if prev is not None:
            pb, ph = prev
            evs[pb].synchronize()
            ph.copy_(bufs[pb][: ph.numel()])

    @classmethod
    def upload(cls, pairs) -> None:
        """pairs: [(contiguous CUDA uint8 view, contiguous CPU uint8 view)]; returns once
        every chunk is enqueued (the host array may be reused: it has been read)."""
        with cls._lock, cls._host_threads():
            cls._upload(pairs)

    @classmethod
    def _upload(cls, pairs) -> None:
        bufs, evs = cls._get()
        segs = [sg for d, h in pairs for sg in cls._segments(d, h)]
        stream = torch.cuda.current_stream()
        for j, (d, h) in enumerate(segs):
            b = j & 1
            if j >= 2:
                evs[b].synchronize()  # the DMA that last read this chunk has finished
            bufs[b][: h.numel()].copy_(h)
            d.copy_(bufs[b][: h.numel()], non_blocking=True)
            evs[b].record(stream)
        for e in evs[: min(2, len(segs))]:
            e.synchronize()  # the chunks are free for the next call


def _bytes_view(t: torch.Tensor) -> torch.Tensor:
    return t.reshape(-1).view(torch.uint8)


def upload_array(a: np.ndarray, device) -> torch.Tensor:
    """1-D contiguous host array -> CUDA tensor (staged when large)."""
    h = torch.from_numpy(a)
    if h.numel() * h.element_size() < Staging.MIN_BYTES:
        return h.to(device)
    out = torch.empty(h.shape, dtype=h.dtype, device=device)
    Staging.upload([(_bytes_view(out), _bytes_view(h))])
    return out


def to_numpy_block(t: torch.Tensor) -> np.ndarray:
    """Column-major CUDA block -> Fortran-ordered numpy array (D2H; large
    blocks through the page-locked staging chunks)."""
    nbytes = t.numel() * t.element_size()
    if t.is_cuda and t.dim() == 2 and nbytes >= Staging.MIN_BYTES and is_col_major(t):
        n, p = t.shape
        host = torch.empty((p, n), dtype=t.dtype)  # (p, n) C-order == (n, p) F-order
        Staging.download([(_bytes_view(t[:, c]), _bytes_view(host[c])) for c in range(p)])
        return host.numpy().T
    host = t.t().contiguous().cpu().numpy()  # (p, n) C-order
    return np.asfortranarray(host.T)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _aligned16(t: torch.Tensor | None) -> bool:
    """16-byte aligned base and an even leading dimension (what a tensor map needs)."""
    return t is not None and t.data_ptr() % 16 == 0 and ld_of(t) % 2 == 0


class Workspace:
    """Per-device scratch buffer; the leading 256 bytes hold the ticket
    counter of rg_tall's last-CTA reduction (zeroed once, re-armed by the
    kernels).

    RG_WS_GUARD=<bytes> (debug): every request gets a fresh buffer of exactly
    the requested size followed by a guard region; ``check`` after each
    launch raises if a kernel wrote past its workspace."""

    _pools: dict = {}
    _guard = int(os.environ.get("RG_WS_GUARD", "0"))
    _last = None
    _override = None  # fixed slot-0 buffer while a CUDA graph is captured (see ``fixed``)

    @classmethod
    @contextlib.contextmanager
    def fixed(cls, buf: torch.Tensor):
        """Serve every slot-0 request from ``buf`` inside the block: a captured
        CUDA graph keeps the pointers it saw, so its workspace must not be the
        pool buffer that later, larger requests replace."""
        prev, cls._override = cls._override, buf
        try:
            yield
        finally:
            cls._override = prev

    @classmethod
    def check(cls, label: str) -> None:
        if not cls._guard or cls._last is None:
            return
        buf, nb = cls._last
        torch.cuda.synchronize(buf.device)
        if not bool((buf[nb:] == 0xA5).all()):
            bad = int((buf[nb:] != 0xA5).nonzero()[-1].item()) + 1
            raise RuntimeError(f"workspace overflow after {label}: {bad} bytes past the {nb}-byte request")

    @classmethod
    def get(cls, nbytes: int, device=None, slot: int = 0) -> torch.Tensor:
        dev = require_cuda(device)
        if cls._override is not None and slot == 0:
            if cls._override.numel() < nbytes:
                raise RuntimeError(f"fixed workspace of {cls._override.numel()} bytes < {nbytes} requested")
            return cls._override
        if cls._guard:
            nb = max(int(nbytes), 256)
            buf = torch.zeros(nb + cls._guard, dtype=torch.uint8, device=dev)
            buf[nb:] = 0xA5
            cls._last = (buf, nb)
            return buf[:nb]
        key = (dev.index, slot)
        buf = cls._pools.get(key)
        if buf is None or buf.numel() < nbytes:
            size = max(int(nbytes), 1 << 20)
            if buf is not None:
                size = max(size, 2 * buf.numel())
                torch.cuda.current_stream(dev).synchronize()
            buf = torch.zeros(size, dtype=torch.uint8, device=dev)
            cls._pools[key] = buf
        return buf


# ---------------------------------------------------------------------------
# launch accounting (bench / smoke evidence), kept natively by librgb200
# (rg_prof.cu): every kernel-launching entry point counts its launches, and
# with ``timing`` on brackets itself with CUDA events on its own stream and
# records its algorithmic bytes and tensor-core flops -- including the calls
# the C orchestrators make, so the timed path is the production path.
# ---------------------------------------------------------------------------


class LaunchLog:
    timing = False
    _base = 0

    @classmethod
    def reset(cls, timing: bool = False):
        L = lib()
        L.rg_profile_enable(1 if timing else 0)
        cls._base = L.rg_launch_count()
        cls.timing = timing

    @classmethod
    def launches(cls) -> int:
        """Kernels launched since the last reset."""
        return int(lib().rg_launch_count() - cls._base)

    @classmethod
    def records(cls):
        """[(label, ms, bytes, flops, launches)] of the calls recorded since
        the last reset(timing=True) (synchronises)."""
        L = lib()
        out = []
        buf = ctypes.create_string_buffer(128)
        ms, nb, fl, nl = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double(), ctypes.c_int32()
        for i in range(L.rg_profile_count()):
            _lib.check(L.rg_profile_record(i, buf, 128, ctypes.byref(ms), ctypes.byref(nb), ctypes.byref(fl),
                                           ctypes.byref(nl)), "profile")
            out.append((buf.value.decode(), ms.value, nb.value, fl.value, nl.value))
        return out

    @classmethod
    def summary(cls):
        """{label: (calls, total_ms, total_bytes, flops_per_call, launches)}."""
        out = {}
        for label, ms, nb, fl, nl in cls.records():
            c, t, b, _, l = out.get(label, (0, 0.0, 0, 0.0, 0))
            out[label] = (c + 1, t + ms, b + nb, fl, l + nl)
        return out


# ---------------------------------------------------------------------------
# kernel wrappers
# ---------------------------------------------------------------------------


# stencil-like matrices run on the diagonal-layout SpMM (rg_spmm_dia_f64);
# False keeps every product on the CSR kernel (tests compare the two)
SPMM_DIA = True


def spmm(dcsr, X: torch.Tensor, Y: torch.Tensor, row_begin: int = 0, row_end: int | None = None,
         n_local: int | None = None, Xg: torch.Tensor | None = None) -> torch.Tensor:
    """Y[rows] = A[rows] @ X (bitwise the reference kernel's arithmetic)."""
    L = lib()
    n_rows = dcsr.n_rows
    row_end = n_rows if row_end is None else row_end
    p = X.shape[1]
    n_local = dcsr.n_cols if n_local is None else n_local
    cplx = X.dtype == torch.complex128
    if cplx != (dcsr.values.dtype == torch.complex128) or Y.dtype != X.dtype:
        raise TypeError(f"spmm: matrix values {dcsr.values.dtype}, block {X.dtype}, output {Y.dtype} must agree")
    plan = dcsr.dia() if (not cplx and Xg is None and SPMM_DIA and hasattr(dcsr, "dia")) else None
    if (plan is not None and plan.covers(row_begin, row_end) and X.numel() and is_col_major(X)
            and ld_of(X) % 2 == 0 and X.data_ptr() % 16 == 0):
        # stencil-like matrix: the diagonal-layout kernel (same arithmetic, bitwise)
        offs = plan.offsets
        rc = L.rg_spmm_dia_f64(n_rows, row_begin, row_end, len(offs), offs.ctypes.data, plan.dia.data_ptr(),
                               ld_of(plan.dia), plan.mask.data_ptr(), n_local, X.data_ptr(), ld_of(X), p,
                               Y.data_ptr(), ld_of(Y), dcsr.row_ptr.data_ptr(), stream_ptr())
        _lib.check(rc, "spmm (dia)")
        return Y
    fn = L.rg_spmm_csr_c128 if cplx else L.rg_spmm_csr_f64
    rc = fn(n_rows, row_begin, row_end, dcsr.row_ptr.data_ptr(), dcsr.col_idx.data_ptr(),
            dcsr.values.data_ptr(), X.data_ptr() if X.numel() else None, ld_of(X), n_local,
            ptr(Xg), ld_of(Xg) if Xg is not None else 1, p, Y.data_ptr(), ld_of(Y), stream_ptr())
    _lib.check(rc, "spmm")
    return Y


def _tall_call(n, p, zin, zout, t1, t2, r1, r2, gmode, gb, gout, cplx=False):
    L = lib()
    x1, s1, al1 = t1 if t1 is not None else (None, None, 0.0)
    x2, s2, al2 = t2 if t2 is not None else (None, None, 0.0)
    a1 = 0 if x1 is None else x1.shape[1]
    a2 = 0 if x2 is None else x2.shape[1]
    gc = 0
    if gmode == 1:
        gc = gb.shape[1]
    elif gmode == 2:
        gc = p
    elif gmode == 3:
        gc = 1
    gout_k = gout
    if gout is not None and not _dense_f(gout):
        gout_k = small(gout.shape[0], gout.shape[1] if gout.dim() > 1 else 1, gout.device, gout.dtype)
        if gout.dim() == 1:
            gout_k = gout_k[:, 0]
    wsfn = L.rg_tall_c128_workspace_bytes if cplx else L.rg_tall_workspace_bytes
    wsb = wsfn(n, p, a1, a2, gmode, gc) if gmode else 0
    ws = Workspace.get(wsb) if gmode else None
    fn = L.rg_tall_c128 if cplx else L.rg_tall_f64
    rc = fn(n, p,
            ptr(zin), ld_of(zin) if zin is not None else 1,
            ptr(zout), ld_of(zout) if zout is not None else 1,
            ptr(x1), ld_of(x1) if x1 is not None else 1, a1, ptr(s1), float(al1),
            ptr(x2), ld_of(x2) if x2 is not None else 1, a2, ptr(s2), float(al2),
            ptr(r1), ptr(r2), gmode,
            ptr(gb), ld_of(gb) if gb is not None else 1, gc, ptr(gout_k),
            ptr(ws), ws.numel() if ws is not None else 0, stream_ptr())
    _lib.check(rc, "tall")
    Workspace.check(f"rg_tall n={n} p={p} a={a1}+{a2} gmode={gmode} gc={gc} cplx={cplx}")
    if gout_k is not gout:
        gout.copy_(gout_k)
    if gmode and _COMM is not None and not _COMM.peer_active:
        _COMM.allreduce_(gout)  # (peer group: the kernel's last CTA summed over the ranks)


def _dense_f(t: torch.Tensor) -> bool:
    if t.dim() == 1:
        return t.stride(0) == 1 or t.shape[0] <= 1
    return (t.shape[0] <= 1 or t.stride(0) == 1) and (t.shape[1] <= 1 or t.stride(1) == t.shape[0])


def _coef(S: torch.Tensor) -> torch.Tensor:
    """Coefficient matrices must be dense column-major with ld = rows."""
    if S.dim() == 1:
        S = S.reshape(-1, 1)
    a, p = S.shape
    if S.stride(0) == 1 and (p <= 1 or S.stride(1) == a):
        return S
    out = small(a, p, S.device, S.dtype)
    out.copy_(S)
    return out


def _split_terms(terms, max_cols=None):
    """Split wide terms so that each launch stages <= max_cols columns."""
    max_cols = MAX_TERM_COLS if max_cols is None else max_cols
    pieces = []
    for X, S, alpha in terms:
        a = X.shape[1]
        if a == 0:
            continue
        for a0 in range(0, a, max_cols):
            a1 = min(a, a0 + max_cols)
            pieces.append((X[:, a0:a1], _coef(S[a0:a1, :]), alpha))
    return pieces


def tall(Z_in: torch.Tensor | None, Z_out: torch.Tensor | None, terms=(), r1=None, r2=None,
         gram=None, n: int | None = None, p: int | None = None):
    """Fused pass ``z = Zin + sum alpha_t X_t S_t; z = z R1^-1 R2^-1;
    Zout = z; Gram``.  ``gram`` is None, ("basis", Gb, Gout), ("self", Gout)
    or ("sumsq", out).  Shapes beyond one launch are split into several
    passes (wide term lists, Gram bases wider than 128 columns, block widths
    above 16); the split changes only the rounding order.
    """
    if n is None:
        n = (Z_in if Z_in is not None else Z_out).shape[0]
    if p is None:
        p = (Z_in if Z_in is not None else Z_out).shape[1]
    if n == 0 and gram is not None:
        _zero_gram(gram)
        if _COMM is not None and _COMM.peer_active:
            # every rank must launch the same sequence of reducing passes
            raise _lib.KernelError("row partition with an empty rank: the in-kernel Gram reduction needs rows on "
                                   "every rank")
        return
    cplx = any(t is not None and t.dtype == torch.complex128 for t in (Z_in, Z_out))
    if (not cplx and p > 8 and gram is not None and gram[0] == "sumsq" and not terms and r1 is None and r2 is None
            and Z_out is None and Z_in is not None and _aligned16(Z_in) and gram[1].dim() == 1):
        # column norms of a wide block (the k = 20 recycle space): 8 columns at a
        # time on the 256-row TMA ring (0.89 -> 0.45 ms at n = 2^24, p = 20)
        for c0 in range(0, p, 8):
            c1 = min(p, c0 + 8)
            tall(Z_in[:, c0:c1], None, gram=("sumsq", gram[1][c0:c1]), n=n, p=c1 - c0)
        return
    maxp, maxgc = (MAX_P_C, _c_limits(p, bool(terms))[0]) if cplx else (MAX_P, _r_limits(p)[0])
    if (not cplx and 16 < p <= 24 and gram is not None and gram[0] == "basis" and not terms and r1 is None
            and r2 is None and Z_out is None and _aligned16(Z_in) and _aligned16(gram[1])):
        maxgc = MAX_GC  # a pure Gram of a 17..24-column block: the three-tile ws kernel takes 128 columns
    tcols = _c_limits(p)[1] if cplx else _r_limits(p)[1]
    terms = _split_terms(terms, tcols)
    r1 = _coef(r1) if r1 is not None else None
    r2 = _coef(r2) if r2 is not None else None
    if p > maxp:
        _tall_wide(Z_in, Z_out, terms, r1, r2, gram, n, p, cplx)
        return
    if gram is not None and gram[0] == "self" and p > maxgc:
        # a self Gram wider than one launch's Gram tiles: form z, then
        # G[g0:g1, :] = z[:, g0:g1]^T z in basis-Gram chunks
        dev = (Z_in if Z_in is not None else Z_out).device
        zb = Z_out if Z_out is not None else empty_block(n, p, dev, torch.complex128 if cplx else torch.float64)
        tall(Z_in, zb, terms, r1=r1, r2=r2, n=n, p=p)
        for g0 in range(0, p, maxgc):
            g1 = min(p, g0 + maxgc)
            tall(zb, None, gram=("basis", zb[:, g0:g1], gram[1][g0:g1, :]), n=n, p=p)
        return
    gmode, gb, gout = 0, None, None
    if gram is not None:
        kind = gram[0]
        if kind == "basis":
            gmode, gb, gout = 1, gram[1], gram[2]
        elif kind == "self":
            gmode, gout = 2, gram[1]
        elif kind == "sumsq":
            gmode, gout = 3, gram[1]
        else:
            raise ValueError(f"unknown gram kind {kind!r}")
    # passes over the term list (<= 2 terms and <= MAX_TERM_COLS staged columns each)
    groups, cur_g, cur_cols = [], [], 0
    for t in terms:
        a = t[0].shape[1]
        if cur_g and (len(cur_g) == 2 or cur_cols + a > tcols):
            groups.append(cur_g)
            cur_g, cur_cols = [], 0
        cur_g.append(t)
        cur_cols += a
    if cur_g or not groups:
        groups.append(cur_g)
    needs_multi = len(groups) > 1 or (gmode == 1 and gb.shape[1] > maxgc)
    pure_gram = not terms and r1 is None and r2 is None and Z_out is None
    zbuf = Z_out
    if needs_multi and zbuf is None and not pure_gram:
        zbuf = empty_block(n, p, Z_in.device if Z_in is not None else None,
                           torch.complex128 if cplx else torch.float64)
    cur_in = Z_in
    for gi, grp in enumerate(groups):
        last = gi == len(groups) - 1
        t1 = grp[0] if len(grp) > 0 else None
        t2 = grp[1] if len(grp) > 1 else None
        if not last:
            _tall_call(n, p, cur_in, zbuf, t1, t2, None, None, 0, None, None, cplx)
            cur_in = zbuf
            continue
        if gmode == 1 and gb.shape[1] > maxgc:
            gc = gb.shape[1]
            if pure_gram:
                g0 = 0  # every chunk reads the input block directly
                zsrc = cur_in
            else:
                _tall_call(n, p, cur_in, zbuf, t1, t2, r1, r2, 1, gb[:, :maxgc], gout[:maxgc, :], cplx)
                g0 = maxgc
                zsrc = zbuf
            step = _c_limits(p, False)[0] if cplx else maxgc
            while g0 < gc:
                g1 = min(gc, g0 + step)
                _tall_call(n, p, zsrc, None, None, None, None, None, 1, gb[:, g0:g1], gout[g0:g1, :], cplx)
                g0 = g1
        else:
            _tall_call(n, p, cur_in, zbuf if needs_multi else Z_out, t1, t2, r1, r2, gmode, gb, gout, cplx)


def _zero_gram(gram):
    kind = gram[0]
    out = gram[2] if kind == "basis" else gram[1]
    out.zero_()


def _tall_wide(Z_in, Z_out, terms, r1, r2, gram, n, p, cplx):
    """p > 16: column-blocked passes (materialise z, blocked triangular
    solves, blocked Grams)."""
    dev = (Z_in if Z_in is not None else Z_out).device
    dt = torch.complex128 if cplx else torch.float64
    Z = Z_out if Z_out is not None else empty_block(n, p, dev, dt)
    mp = MAX_P_C if cplx else MAX_P
    blocks = [(c0, min(p, c0 + mp)) for c0 in range(0, p, mp)]
    # 1) z = Zin + terms, column block by column block
    for c0, c1 in blocks:
        sub_terms = [(X, S[:, c0:c1], al) for X, S, al in terms]
        tall(Z_in[:, c0:c1] if Z_in is not None else None, Z[:, c0:c1], sub_terms, n=n, p=c1 - c0)
    # 2) right triangular solves, block forward substitution
    for R in (r1, r2):
        if R is None:
            continue
        for bi, (c0, c1) in enumerate(blocks):
            prev = [(Z[:, b0:b1], R[b0:b1, c0:c1], -1.0) for b0, b1 in blocks[:bi]]
            tall(Z[:, c0:c1], Z[:, c0:c1], prev, r1=R[c0:c1, c0:c1], n=n, p=c1 - c0)
    # 3) Gram
    if gram is None:
        return
    kind = gram[0]
    for c0, c1 in blocks:
        zc = Z[:, c0:c1]
        if kind == "basis":
            gb, gout = gram[1], gram[2]
            tall(zc, None, gram=("basis", gb, gout[:, c0:c1]), n=n, p=c1 - c0)
        elif kind == "self":
            gout = gram[1]
            tall(zc, None, gram=("basis", Z, gout[:, c0:c1]), n=n, p=c1 - c0)
        else:
            tall(zc, None, gram=("sumsq", gram[1][c0:c1]), n=n, p=c1 - c0)


def max_p(t: torch.Tensor) -> int:
    """Widest block one rg_tall launch handles for this dtype."""
    return MAX_P_C if t.dtype == torch.complex128 else MAX_P


def fused_ok() -> bool:
    """The C orchestrators (rg_cgs2_f64 / rg_cholqr2_f64) replace the Python
    pass chain on one GPU, and on a row partition whose Gram passes sum over
    the ranks in-kernel (distributed.PeerGroup); with NCCL allreduces between
    the passes the Python chain runs."""
    return _COMM is None or _COMM.peer_active


def cgs2(Z: torch.Tensor, C, W: torch.Tensor, coef: torch.Tensor, G1, joint: bool = False) -> None:
    """One call: CGS2 of Z against C then W (twice) in place; coef receives
    S1|c1|S2|c2; G1 (optional) receives Z^T Z of the result.  ``joint``:
    W follows C in one allocation and C is orthogonal to W -- three passes
    against [C W], coef = G1|G2 (rg_cgs2_f64)."""
    L = lib()
    n, p = Z.shape
    k = 0 if C is None else C.shape[1]
    w = W.shape[1]
    ws = Workspace.get(L.rg_tall_workspace_bytes(n, p, k, w, 1, max(k + w, p)))
    rc = L.rg_cgs2_f64(n, p, Z.data_ptr(), ld_of(Z), ptr(C), ld_of(C) if C is not None else 1, k,
                       W.data_ptr(), ld_of(W), w, coef.data_ptr(), ptr(G1), 1 if joint else 0, ws.data_ptr(),
                       ws.numel(), stream_ptr())
    _lib.check(rc, "cgs2")
    Workspace.check(f"rg_cgs2 n={n} p={p} k={k} w={w}")


def cholqr2(X: torch.Tensor, Q: torch.Tensor, small: torch.Tensor, status: torch.Tensor, gram_ready: bool) -> None:
    L = lib()
    n, p = X.shape
    ws = Workspace.get(L.rg_tall_workspace_bytes(n, p, 0, 0, 2, p))
    rc = L.rg_cholqr2_f64(n, p, X.data_ptr(), ld_of(X), Q.data_ptr(), ld_of(Q), small.data_ptr(), status.data_ptr(),
                          1 if gram_ready else 0, ws.data_ptr(), ws.numel(), stream_ptr())
    _lib.check(rc, "cholqr2")
    Workspace.check(f"rg_cholqr2 n={n} p={p}")


def chol(G: torch.Tensor, R: torch.Tensor, status: torch.Tensor, cond_tol: float):
    p = G.shape[0]
    fn = lib().rg_chol_c128 if G.dtype == torch.complex128 else lib().rg_chol_f64
    rc = fn(p, _coef(G).data_ptr(), R.data_ptr(), status.data_ptr(), float(cond_tol), stream_ptr())
    _lib.check(rc, "chol")


def tsqr(X: torch.Tensor, R: torch.Tensor):
    """In-place Householder TSQR: X <- Q, R <- R (r_jj >= 0)."""
    n, p = X.shape
    L = lib()
    wsb = L.rg_tsqr_workspace_bytes(n, p)
    ws = Workspace.get(wsb, slot=1)
    rc = L.rg_tsqr_f64(n, p, X.data_ptr(), ld_of(X), R.data_ptr(), ws.data_ptr(), ws.numel(), stream_ptr())
    _lib.check(rc, "tsqr")
