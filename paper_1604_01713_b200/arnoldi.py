"""Block Arnoldi with the recycle-space projection, device resident.

Drop-in for ``recgmres.arnoldi`` (/root/reference/pkg/src/recgmres/
arnoldi.py): ``ArnoldiFactorization``, ``start``, ``step``,
``ZeroStartBlock`` with the reference's signatures and semantics.

State placement: the basis W = [V_1 ... V_{m_max+1}] is one
column-major n x (m_max+1)L block in HBM; the small H, F and z_bar stay on
the host (the progressive least-squares problem and the harmonic Ritz
problem read them there).  One step is

    Ahat = A V_m                       rg_spmm_csr_f64 (or the user closure)
    CGS2 vs C then W, twice            ortho.project_chain -> 5 rg_tall passes
    Ahat = V_{m+1} R                   CholQR2 (Gram fused into the last CGS2
                                       pass) or Householder TSQR fallback
    one D2H of all small coefficients  (the only host sync of the step)

and the host accumulates F, H exactly as arnoldi.py:177,180,183 do.
"""

from __future__ import annotations

import numpy as np
import torch

from . import device as _dev
from .dense_kernels import (TSQR_MAX_P, QrScratch, _flags, cholqr2_finish, cholqr2_launch, reduced_qr_device,
                            tsqr_into)
from .ortho import project_chain
from .sparse_core import ShapeError


# CGS2 against [C W] as one basis (three passes) when the caller certified
# that the starting block is C-orthogonal (``start(..., c_orthogonal=True)``:
# the solver scrubs R0 against C first, solver.py:149-155); False forces the
# reference's sequential C-then-W order (five passes) -- tests compare the two
JOINT_PROJECTION = True


# steps of factorizations with at most this many rows are replayed from a
# captured CUDA graph (one per block-step index) when the caller provides a
# StepWorkspace with graphs on: at these sizes a step is launch- and
# sync-bound.  Measured on B200 for config 1 (n = 4096, tools/prof_cfg1_step.py,
# profiles/cfg1_graph_r02.json): a replayed step takes 0.147 ms against 0.195
# ms eager, but one solve uses each (step index, k) shape only a few times, so
# capture + instantiation outweigh the saving (3-system sequence 0.267 s with
# graphs vs 0.250 s eager) -- hence off by default (STEP_GRAPHS).
GRAPH_MAX_ROWS = 1 << 18
STEP_GRAPHS = False

# the solver enqueues block step j+1 before reading step j's results
# (StepPipeline); False runs the plain step-by-step order (tests compare them)
PIPELINE_STEPS = True


class StepWorkspace:
    """Device buffers of the factorizations of one solve, reused from cycle
    to cycle, and the CUDA graphs of their steps.

    A solve creates one and passes it to every ``start``; the factorization
    of cycle c+1 then lives in the buffers of cycle c (the solver is done
    with cycle c's basis when it starts the next), so the pointers a captured
    step graph holds stay valid.  Each step shape runs eagerly
    ``capture_after`` times, is then captured, and replayed from then on
    (capture + instantiation cost a few eager steps, so shapes used only a
    couple of times per solve never pay for a graph)."""

    def __init__(self, graphs: bool | None = None, capture_after: int = 1):
        self._bufs = {}
        self.graphs = {} if (STEP_GRAPHS if graphs is None else graphs) else None
        self._seen = {}
        self.capture_after = capture_after  # eager runs of a step shape before it is captured
        self.scratch = None  # the captured steps' own rg_tall workspace
        self.stream = None   # capture stream

    def buffers(self, key, make):
        b = self._bufs.get(key)
        if b is None:
            b = self._bufs[key] = make()
        return b


class _HostSlot:
    """Pinned host copies of one step's small results: the packed CGS2
    coefficients, the CholQR2 factors and its status words."""

    __slots__ = ("coef", "qr", "st")

    def __init__(self, coef, qr, st):
        self.coef, self.qr, self.st = coef, qr, st


class ZeroStartBlock(ValueError):
    """The starting block is numerically zero (already converged)."""


class ArnoldiFactorization:
    """State of the block Arnoldi iteration (arnoldi.py:22-95).

    w        : basis blocks V_1..V_{m+1}, a CUDA n x (m+1)L column-major view
    h_bar    : block upper-Hessenberg (m+1)L x mL (host)
    f        : C-projection coefficients k x mL (host)
    z_bar    : L x L R-factor of the starting block (host)
    m        : completed block steps
    """

    def __init__(self, n: int, L: int, m_max: int, k: int, rank_tol: float, seed: int, device=None,
                 dtype=torch.float64, workspace: StepWorkspace | None = None):
        self.n = n
        self.dtype = dtype
        npdt = np.complex128 if dtype == torch.complex128 else np.float64
        self.L = L
        self.m_max = m_max
        self.k = k
        self.rank_tol = rank_tol
        self.m = 0
        dev = _dev.require_cuda(device)
        self.device = dev
        self._ws = workspace

        def make():
            wmax = (m_max + 1) * L
            coef = torch.zeros((2 * k + 2 * wmax) * L, dtype=dtype, device=dev)
            # [C | W] in one allocation: C (copied in by start) directly precedes
            # the basis, so the CGS2 projection can treat [C W] as one basis
            # host results of a step in two slots: the solver enqueues step j+1
            # before it reads step j's (StepPipeline)
            host = [_HostSlot(torch.zeros_like(coef, device="cpu").pin_memory(),
                              torch.zeros(5 * L * L, dtype=dtype).pin_memory(),
                              torch.zeros(2, dtype=torch.int32).pin_memory()) for _ in range(2)]
            return dict(CW=_dev.empty_block(n, k + wmax, dev, dtype), ahat=_dev.empty_block(n, L, dev, dtype),
                        coef=coef, host=host, qr=QrScratch(L, dev, dtype))

        bufs = make() if workspace is None else workspace.buffers((n, L, m_max, k, dtype, dev), make)
        self._CW = bufs["CW"]
        self._W = self._CW[:, k:]
        self._c_src = None  # the recycle space C copied into _CW[:, :k] (identity check in step)
        # the caller certified that R0 (hence V_1, and every later block by
        # construction) is orthogonal to C: the joint [C W] schedule applies
        self.c_orthogonal = False
        self._H = np.zeros(((m_max + 1) * L, m_max * L), dtype=npdt)
        self._F = np.zeros((k, m_max * L), dtype=npdt)
        self.z_bar = np.zeros((L, L), dtype=npdt)
        self.breakdown_events: list[str] = []
        self._rng = np.random.default_rng(seed)
        self._ahat = bufs["ahat"]
        # packed small coefficients of one step: S1 | c1 | S2 | c2 (column-major
        # blocks), or G1 | G2 for the joint schedule
        self._coef = bufs["coef"]
        self._host = bufs["host"]
        self._hb = self._host[0]  # the host slot plain step() / start() use
        self._qr = bufs["qr"]
        self.launches = 0  # rg_* kernel launches issued by start/step (diagnostics)
        self._qr_fallback = False  # the last step's Q came from the host-side fallback path

    # ---- views (arnoldi.py:47-76)
    @property
    def w(self) -> torch.Tensor:
        return self._W[:, : (self.m + 1) * self.L]

    @property
    def h_bar(self) -> np.ndarray:
        return self._H[: (self.m + 1) * self.L, : self.m * self.L]

    @property
    def f(self) -> np.ndarray:
        return self._F[:, : self.m * self.L]

    def h_square(self) -> np.ndarray:
        return self._H[: self.m * self.L, : self.m * self.L]

    def h_last_block(self) -> np.ndarray:
        mL = self.m * self.L
        return self._H[mL: mL + self.L, mL - self.L: mL]

    def v_block(self, i: int) -> torch.Tensor:
        return self._W[:, i * self.L: (i + 1) * self.L]

    def new_hbar_columns(self) -> np.ndarray:
        mL = self.m * self.L
        return self._H[: mL + self.L, mL - self.L: mL]

    def w_numpy(self) -> np.ndarray:
        """Host copy of the active basis (D2H; for tests / small problems)."""
        return _dev.to_numpy_block(self.w)

    def _coef_views(self, m: int):
        k, L, w = self.k, self.L, (m + 1) * self.L
        sizes = [k * L, w * L, k * L, w * L]
        rows = [k, w, k, w]
        out, off = [], 0
        for s, r in zip(sizes, rows):
            out.append(self._coef[off: off + s].view(L, r).t() if r else self._coef[off:off].view(L, 0).t())
            off += s
        return out

    def _unit_vector_into(self, col: torch.Tensor, v: torch.Tensor, nrm: float):
        """col = v / nrm (division on the device, as the reference's v / nrm)."""
        r = torch.full((1, 1), nrm, dtype=self.dtype, device=self.device)
        _dev.tall(v, col, r1=r)

    def _random_direction(self, bases, tries=3):
        """Seeded replacement direction: host PCG64 normals (same stream as the
        reference), CGS twice against ``bases`` on the device.  Returns
        (vector, norm) or (None, 0)."""
        scratch = [torch.zeros(b.shape[1], dtype=self.dtype, device=self.device).view(-1, 1) for b in bases]
        part = _dev.get_part()
        cplx = self.dtype == torch.complex128
        for _ in range(tries):
            n_glob = self.n if part is None else part.n
            if cplx:  # complex normal: (re, im) pairs from the same stream
                g = self._rng.standard_normal((n_glob, 2))
                draw = g[:, 0] + 1j * g[:, 1]
            else:
                draw = self._rng.standard_normal(n_glob)
            if part is not None:  # same global stream as one process, sliced to this rank's rows
                draw = draw[part.r0:part.r1]
            v = _dev.to_device_block(draw.reshape(-1, 1))
            for _pass in range(2):
                project_chain(v, v, bases, [s[: b.shape[1]] for s, b in zip(scratch, bases)])
            ss = torch.zeros(1, dtype=torch.float64, device=self.device)
            _dev.tall(v, None, gram=("sumsq", ss))
            nrm = float(np.sqrt(ss.item()))
            if nrm > 1e-8:
                return v, nrm
        return None, 0.0


def _as_block_on(x, dev):
    if isinstance(x, torch.Tensor):
        if x.dim() == 1:
            x = x.reshape(-1, 1)
        if x.dim() != 2:
            raise ShapeError(f"expected a vector or 2-D block, got ndim={x.dim()}")
        return _dev.to_device_block(x, dev)
    a = np.asarray(x, dtype=np.complex128 if np.iscomplexobj(x) else np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    if a.ndim != 2:
        raise ShapeError(f"expected a vector or 2-D block, got ndim={a.ndim}")
    return _dev.to_device_block(a, dev)


def _apply_operator(opA, Z: torch.Tensor, out: torch.Tensor):
    """out = opA(Z); operators exposing ``apply_into`` write in place."""
    into = getattr(opA, "apply_into", None)
    if into is None:
        owner = getattr(opA, "__self__", None)
        into = getattr(owner, "apply_into", None) if owner is not None and getattr(opA, "__name__", "") == "apply" else None
    if into is not None:
        into(Z, out)
        return
    Y = opA(Z)
    if not isinstance(Y, torch.Tensor):
        Y = _dev.to_device_block(np.asarray(Y), Z.device)
    if Y.dim() == 1:
        Y = Y.reshape(-1, 1)
    if tuple(Y.shape) != tuple(out.shape):
        raise ValueError("operator closure returned a block of wrong shape")
    out.copy_(Y)


def start(opA, R0, rank_tol: float = 1e-12, *, m_max: int, recycle=None, seed: int = 0,
          device=None, c_orthogonal: bool = False, workspace: StepWorkspace | None = None) -> ArnoldiFactorization:
    """Initialise from the starting block R0 (arnoldi.py:98-136): V_1, z_bar
    from its thin QR; rank-deficient columns replaced by seeded random
    directions (C- and V_1-orthogonalised twice) and logged.

    ``c_orthogonal`` (keyword, not in the reference): the caller certifies
    that R0 was already projected against the recycle space C (the solver
    scrubs it, solver.py:149-155).  Only then may ``step`` project against
    [C W] as one basis; the default keeps the reference's C-then-W order.
    ``workspace`` (keyword, not in the reference): a StepWorkspace whose
    buffers (and captured step graphs) the factorization reuses."""
    dev = _dev.require_cuda(device if device is not None else
                            (R0.device if isinstance(R0, torch.Tensor) and R0.is_cuda else None))
    R0d = _as_block_on(R0, dev)
    n, L = R0d.shape
    ss = torch.zeros(L, dtype=torch.float64, device=dev)
    _dev.tall(R0d, None, gram=("sumsq", ss))
    norm0 = float(np.sqrt(ss.sum().item()))
    if norm0 == 0.0 or not np.isfinite(norm0):
        raise ZeroStartBlock("starting block is numerically zero")
    k = recycle.k if recycle is not None else 0
    if recycle is not None and recycle.c_device().dtype != R0d.dtype:
        R0d = R0d.to(recycle.c_device().dtype) if R0d.dtype == torch.float64 else R0d
    fact = ArnoldiFactorization(n, L, m_max, k, rank_tol, seed, dev, R0d.dtype, workspace=workspace)
    if recycle is not None and k:
        fact._CW[:, :k].copy_(recycle.c_device())
        fact._c_src = recycle.c_device()
        fact.c_orthogonal = bool(c_orthogonal)
    V1 = fact.v_block(0)
    qr = _block_qr(fact, R0d, V1)
    fact.z_bar = qr[0]
    flagged = qr[1]
    C = recycle.c_device() if recycle is not None else None
    for j in np.flatnonzero(flagged):
        # the reference projects against C, then V1 without column j (arnoldi.py:115-123)
        others = [c for c in range(L) if c != j]
        bases = ([C] if C is not None else []) + ([_dev.to_device_block(V1[:, others])] if others else [])
        v, nrm = fact._random_direction(bases)
        if v is not None:
            fact._unit_vector_into(V1[:, j: j + 1], v, nrm)
        else:
            V1[:, j].zero_()
        fact.breakdown_events.append(f"start: replaced rank-deficient column {j}"
                                     + ("" if v is not None else " (space exhausted, column zeroed)"))
    return fact


def _qr_enqueue(fact: ArnoldiFactorization, X: torch.Tensor, Q: torch.Tensor, g1_ready: bool = False,
                hb: _HostSlot | None = None) -> bool:
    """Enqueue CholQR2 of X into Q and the D2H copies of its small results
    (no host sync).  False when the block is too wide for one CholQR2 launch
    (``_qr_collect`` then runs the TSQR / panelled path)."""
    if X.shape[1] > _dev.max_p(X):
        return False
    hb = hb or fact._hb
    scr = fact._qr
    cholqr2_launch(X, Q, scr, g1_ready=g1_ready)
    hb.qr.copy_(scr.buf, non_blocking=True)
    hb.st.copy_(scr.status, non_blocking=True)
    return True


def _qr_collect(fact: ArnoldiFactorization, X: torch.Tensor, Q: torch.Tensor, enqueued: bool,
                hb: _HostSlot | None = None):
    """After the stream has synchronised: (R, flagged) of the CholQR2, or the
    Householder TSQR fallback when CholQR2 was not attempted or failed its
    conditioning check (dense_kernels.py:31-48 semantics either way)."""
    L = X.shape[1]
    scr = fact._qr
    hb = hb or fact._hb
    fact._qr_fallback = True  # Q is (re)computed below: a speculative next step is stale
    if enqueued:
        ok, R, norm_x = cholqr2_finish(hb.qr.numpy(), hb.st.numpy(), L)
        if ok:
            fact._qr_fallback = False
            return R, _flags(R, norm_x, fact.rank_tol)
    else:
        if L > (_dev.MAX_P_C if X.dtype == torch.complex128 else TSQR_MAX_P):
            # wider than one TSQR: column panels (dense_kernels._wide_qr)
            f = reduced_qr_device(X, fact.rank_tol, Q=Q)
            return f.r_factor, f.flagged
        ss = torch.empty(L, dtype=torch.float64, device=X.device)
        _dev.tall(X, None, gram=("sumsq", ss))
        norm_x = float(np.sqrt(ss.sum().item()))
    tsqr_into(X, Q, scr)
    R = np.triu(scr.RT.cpu().numpy())
    return R, _flags(R, norm_x, fact.rank_tol)


def _block_qr(fact: ArnoldiFactorization, X: torch.Tensor, Q: torch.Tensor, g1_ready: bool = False):
    """Thin QR X -> Q (Q must not alias X).  Returns (R, flagged)."""
    enq = _qr_enqueue(fact, X, Q, g1_ready)
    torch.cuda.current_stream().synchronize()
    return _qr_collect(fact, X, Q, enq)


def _capturable(opA):
    """The solver's operator object behind ``opA`` when its application is
    pure device work that a CUDA graph can hold (a CsrMatrix, no
    preconditioner -- the ILU wave solves carry a per-call epoch -- and no
    row partition), else None."""
    owner = getattr(opA, "__self__", None)
    if owner is None or getattr(opA, "__name__", "") != "apply":
        return None
    if getattr(owner, "_csr", None) is None or getattr(owner, "precond", None) is not None:
        return None
    return owner


def _cgs2_enqueue(fact, opA, owner, C, m, joint, fused, count=True, hb: _HostSlot | None = None):
    """The device work of one CGS2 step up to the QR: A V_m, the projection,
    the coefficient D2H and the CholQR2 (+ its D2H).  Returns whether the QR
    was enqueued."""
    L = fact.L
    Vm, Ahat, Vnew = fact.v_block(m), fact._ahat, fact.v_block(m + 1)
    if owner is not None and not count:
        owner._base_into(Vm, Ahat)  # graph capture: each replay accounts its matvecs
    else:
        _apply_operator(opA, Vm, Ahat)
    active = fact._W[:, : (m + 1) * L]
    scr = fact._qr
    k_, w_ = fact.k, (m + 1) * L
    g1 = L <= _dev.max_p(Ahat)
    if joint:
        CW = fact._CW[:, : k_ + w_]
        if fused:
            # rg_cgs2_f64 runs the same three passes on the adjacent [C W]
            _dev.cgs2(Ahat, fact._CW[:, :k_], active, fact._coef, scr.G1, joint=True)
        else:
            kw = k_ + w_
            G1 = fact._coef[: kw * L].view(L, kw).t()
            G2 = fact._coef[kw * L: 2 * kw * L].view(L, kw).t()
            _dev.tall(Ahat, None, gram=("basis", CW, G1))
            _dev.tall(Ahat, None, [(CW, G1, -1.0)], gram=("basis", CW, G2))
            _dev.tall(Ahat, Ahat, [(CW, G1, -1.0), (CW, G2, -1.0)], gram=("self", scr.G1) if g1 else None)
        ncoef = 2 * (k_ + w_) * L
    else:
        if fused:
            # one C-ABI call runs the same fused pass schedule (rg_cgs2_f64);
            # C is passed from its own allocation here, so the five-pass
            # sequential schedule applies
            _dev.cgs2(Ahat, C, active, fact._coef, scr.G1)
        else:
            S1, c1, S2, c2 = fact._coef_views(m)
            if C is not None:
                bases, coefs = [C, active, C, active], [S1, c1, S2, c2]
            else:
                bases, coefs = [active, active], [c1, c2]
            project_chain(Ahat, Ahat, bases, coefs, tail_gram=("self", scr.G1) if g1 else None)
        ncoef = (2 * fact.k + 2 * (m + 1) * L) * L
    hb = hb or fact._hb
    hb.coef[:ncoef].copy_(fact._coef[:ncoef], non_blocking=True)
    return _qr_enqueue(fact, Ahat, Vnew, g1_ready=g1, hb=hb)


def _replay_step(fact, opA, owner, C, m, joint):
    """Graph path of one step: the device work of ``_cgs2_enqueue`` captured
    once per (step index, schedule, operator, buffers, C) and replayed.  Returns
    whether the QR was enqueued, or None when this shape runs eagerly."""
    ws = fact._ws
    # the factorization's buffers differ per (k, L, ...) shape: key on them too
    key = (m, joint, id(owner), fact._CW.data_ptr(), fact.k, 0 if (joint or C is None) else C.data_ptr())
    hit = ws.graphs.get(key)
    if hit is None:
        seen = ws._seen.get(key, 0)
        if seen < ws.capture_after:  # eager first (warms every launch path and buffer)
            ws._seen[key] = seen + 1
            return None
        g = torch.cuda.CUDAGraph()
        lib = _dev.lib()
        if ws.scratch is None:
            # every Gram of the step: <= 128 basis columns per launch, <= 256
            # requested by the sequential orchestrator call
            ws.scratch = torch.zeros(lib.rg_tall_workspace_bytes(fact.n, max(fact.L, 16), 0, 0, 1, 256),
                                     dtype=torch.uint8, device=fact.device)
        if ws.stream is None:
            ws.stream = torch.cuda.Stream(fact.device)
        before = lib.rg_launch_count()
        # capture on a side stream with the low-level API (torch.cuda.graph's
        # context manager also runs gc.collect() and empty_cache() per capture)
        ws.stream.wait_stream(torch.cuda.current_stream())
        with _dev.Workspace.fixed(ws.scratch), torch.cuda.stream(ws.stream):
            g.capture_begin(capture_error_mode="thread_local")
            try:
                enq = _cgs2_enqueue(fact, opA, owner, C, m, joint, True, count=False)
            finally:
                g.capture_end()
        torch.cuda.current_stream().wait_stream(ws.stream)
        nl = int(lib.rg_launch_count() - before)
        lib.rg_count_launches(-nl)  # captured, not run: each replay reports its kernels
        hit = ws.graphs[key] = (g, enq, nl)
    g, enq, nlaunch = hit
    g.replay()
    owner.count += fact.L
    _dev.lib().rg_count_launches(nlaunch)
    return enq


class _PendingStep:
    """A CGS2 block step whose device work is enqueued: its step index, the
    schedule, the host slot its small results land in, the Ahat buffer it
    projected, and an event after its last D2H copy."""

    __slots__ = ("m", "joint", "enq", "hb", "ahat", "event", "C")

    def __init__(self, m, joint, enq, hb, ahat, event, C):
        self.m, self.joint, self.enq, self.hb, self.ahat, self.event, self.C = m, joint, enq, hb, ahat, event, C


def _enqueue_cgs2(fact, opA, recycle, m, hb, ahat, graphs=False) -> _PendingStep:
    """Enqueue block step m's device work (A V_m, CGS2 against C and the
    basis, CholQR2 of the result into V_{m+1}, the D2H copies of its small
    results into ``hb``) without reading any host result of step m-1."""
    L = fact.L
    C = recycle.c_device() if recycle is not None else None
    k_, w_ = fact.k, (m + 1) * L
    # [C W] as one basis when the caller certified C-orthogonality at start
    # and C is the recycle space copied in front of W (real data; the
    # complex tall pass has no aliased-term merge): 3 passes instead of 5
    joint = (JOINT_PROJECTION and C is not None and k_ > 0 and fact.c_orthogonal and fact._c_src is C
             and fact.dtype == torch.float64 and k_ + w_ <= _dev.MAX_GC and L <= _dev.MAX_P)
    fused = (_dev.fused_ok() and fact.dtype == torch.float64 and L <= _dev.MAX_P_FUSED
             and (joint or (k_ <= _dev.MAX_GC and w_ <= _dev.MAX_GC)))
    owner = _capturable(opA)
    enq = None
    # (a row-partitioned step is never replayed: a captured Gram pass would carry
    # the epoch of its capture into every replay of the in-kernel reduction)
    if (graphs and fused and owner is not None and fact._ws is not None and fact._ws.graphs is not None
            and fact.n <= GRAPH_MAX_ROWS and not _dev.LaunchLog.timing and hb is fact._hb and ahat is fact._ahat
            and _dev.get_comm() is None):
        enq = _replay_step(fact, opA, owner, C, m, joint)
    if enq is None:
        saved = fact._ahat
        fact._ahat = ahat
        try:
            enq = _cgs2_enqueue(fact, opA, owner, C, m, joint, fused, hb=hb)
        finally:
            fact._ahat = saved
    ev = torch.cuda.Event()
    ev.record()
    return _PendingStep(m, joint, enq, hb, ahat, ev, C)


def _collect_cgs2(fact, pend: _PendingStep):
    """Host half of a CGS2 step once its event has completed: the R factor
    and rank flags of the QR, and F, H accumulated as arnoldi.py:177,180,183."""
    m, L = pend.m, fact.L
    cols = slice(m * L, (m + 1) * L)
    k_, w_ = fact.k, (m + 1) * L
    R, flagged = _qr_collect(fact, pend.ahat, fact.v_block(m + 1), pend.enq, hb=pend.hb)
    hc = pend.hb.coef.numpy()
    if pend.joint:
        kw = k_ + w_
        hG1 = hc[: kw * L].reshape(L, kw).T
        hG2 = hc[kw * L: 2 * kw * L].reshape(L, kw).T
        fact._F[:, cols] += hG1[:k_]
        fact._F[:, cols] += hG2[:k_]
        fact._H[: (m + 1) * L, cols] += hG1[k_:]
        fact._H[: (m + 1) * L, cols] += hG2[k_:]
    else:
        off = 0
        blocks = []
        for rows in (k_, w_, k_, w_):
            blocks.append(hc[off: off + rows * L].reshape(L, rows).T)
            off += rows * L
        hS1, hc1, hS2, hc2 = blocks
        if pend.C is not None:
            fact._F[:, cols] += hS1
            fact._F[:, cols] += hS2
        fact._H[: (m + 1) * L, cols] += hc1
        fact._H[: (m + 1) * L, cols] += hc2
    return R, flagged


class StepPipeline:
    """Block steps of one cycle with the next step's device work enqueued
    before the current step's small results are read on the host, so the
    device never idles through the host half of a step (the D2H wait, F / H
    accumulation, the progressive least squares and the stop test).

    Each step is the same arithmetic as ``step``; only the host ordering
    changes.  A speculative step is discarded -- its matvecs uncounted, its
    basis block rewritten later -- when the current step ends the cycle or
    changes V_{m+1} on the host side (a rank-deficient column replaced, or
    the CholQR2 conditioning fallback).  Used for CGS2 on the solver's own
    operator (``_Operator.apply``); other cases run ``step`` unchanged."""

    def __init__(self, fact: ArnoldiFactorization, opA, recycle=None, ortho: str = "cgs2"):
        self.fact, self.opA, self.recycle, self.ortho = fact, opA, recycle, ortho
        owner = getattr(opA, "__self__", None)
        self.owner = owner if owner is not None and hasattr(owner, "count") else None
        self.on = (PIPELINE_STEPS and ortho == "cgs2" and self.owner is not None and fact.L <= _dev.max_p(fact._ahat)
                   and not (fact._ws is not None and fact._ws.graphs is not None))
        self.pending = None
        self._turn = 0
        if self.on:
            spare = fact._ws.buffers(("ahat2",) + tuple(fact._ahat.shape) + (fact.dtype,),
                                     lambda: _dev.empty_block(fact.n, fact.L, fact.device, fact.dtype)) \
                if fact._ws is not None else _dev.empty_block(fact.n, fact.L, fact.device, fact.dtype)
            self._ahat = [fact._ahat, spare]

    def _enqueue(self, m):
        t = self._turn
        self._turn ^= 1
        return _enqueue_cgs2(self.fact, self.opA, self.recycle, m, self.fact._host[t], self._ahat[t])

    def _discard(self, pend):
        self.owner.count -= self.fact.L

    def step(self, speculate_next: bool = True):
        """Commit the next block step; with ``speculate_next`` the step after
        it is enqueued first."""
        fact = self.fact
        if not self.on:
            step(fact, self.opA, recycle=self.recycle, ortho=self.ortho)
            return
        if fact.m >= fact.m_max:
            raise ValueError(f"factorization at capacity m_max={fact.m_max}")
        if self.pending is None:
            self.pending = self._enqueue(fact.m)
        pend = self.pending
        nxt = self._enqueue(fact.m + 1) if speculate_next and fact.m + 1 < fact.m_max else None
        pend.event.synchronize()
        R, flagged = _collect_cgs2(fact, pend)
        _finish_step(fact, pend.m, R, flagged, pend.C)
        if nxt is not None and (flagged.any() or fact._qr_fallback):
            self._discard(nxt)  # it projected the V_{m+1} the host just replaced
            nxt = None
        self.pending = nxt

    def close(self):
        """Drop a speculative step the cycle did not use."""
        if self.on and self.pending is not None:
            self._discard(self.pending)
            self.pending = None


def step(fact: ArnoldiFactorization, opA, recycle=None, ortho: str = "cgs2") -> ArnoldiFactorization:
    """Advance by one block step (arnoldi.py:139-193)."""
    if fact.m >= fact.m_max:
        raise ValueError(f"factorization at capacity m_max={fact.m_max}")
    if ortho not in ("mgs", "cgs2"):
        raise ValueError(f"unknown orthogonalization '{ortho}'")
    m, L = fact.m, fact.L
    cols = slice(m * L, (m + 1) * L)
    C = recycle.c_device() if recycle is not None else None
    Vnew = fact.v_block(m + 1)

    if ortho == "mgs":
        _apply_operator(opA, fact.v_block(m), fact._ahat)
        _mgs_project(fact, fact._ahat, C, m, cols)
        R, flagged = _block_qr(fact, fact._ahat, Vnew)
    else:
        pend = _enqueue_cgs2(fact, opA, recycle, m, fact._hb, fact._ahat, graphs=True)
        torch.cuda.current_stream().synchronize()  # the step's one host sync
        R, flagged = _collect_cgs2(fact, pend)

    _finish_step(fact, m, R, flagged, C)
    return fact


def _finish_step(fact, m, R, flagged, C):
    """R into H, seeded replacement of rank-deficient columns of V_{m+1}
    (arnoldi.py:183-190), m += 1."""
    L = fact.L
    cols = slice(m * L, (m + 1) * L)
    active = fact._W[:, : (m + 1) * L]
    Vnew = fact.v_block(m + 1)
    fact._H[(m + 1) * L: (m + 2) * L, cols] = R
    for j in np.flatnonzero(flagged):
        bases = ([C] if C is not None else []) + [active, Vnew]
        v, nrm = fact._random_direction(bases)
        if v is not None:
            fact._unit_vector_into(Vnew[:, j: j + 1], v, nrm)
        else:
            Vnew[:, j].zero_()
        fact.breakdown_events.append(f"step {m + 1}: replaced rank-deficient basis column {j}"
                                     + ("" if v is not None else " (space exhausted, column zeroed)"))
    fact.m = m + 1


def _mgs_project(fact, Ahat, C, m, cols):
    """Block modified Gram-Schmidt (arnoldi.py:159-170): one vector of C at a
    time, then one basis block at a time; each pass fuses the previous
    update with the next Gram."""
    L = fact.L
    bases = []
    if C is not None:
        bases += [C[:, i: i + 1] for i in range(C.shape[1])]
    bases += [fact.v_block(i) for i in range(m + 1)]
    coef = torch.zeros(sum(b.shape[1] for b in bases) * L, dtype=fact.dtype, device=fact.device)
    views, off = [], 0
    for b in bases:
        a = b.shape[1]
        views.append(coef[off: off + a * L].view(L, a).t())
        off += a * L
    project_chain(Ahat, Ahat, bases, views)
    hc = coef.cpu().numpy()
    off = 0
    kk = C.shape[1] if C is not None else 0
    for i, b in enumerate(bases):
        a = b.shape[1]
        blk = hc[off: off + a * L].reshape(L, a).T
        off += a * L
        if i < kk:
            fact._F[i, cols] += blk[0]
        else:
            bi = i - kk
            fact._H[bi * L: (bi + 1) * L, cols] += blk
