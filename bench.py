#!/usr/bin/env python
"""Benchmark of the block GCRO-DR hot path on B200 (driver contract).

Default workload ("step", BASELINE configs[3] operator with configs[2]
shapes): one block Arnoldi step of the 256^3 3-D convection-diffusion
operator (n = 16,777,216 = 2^24, nnz = 117,047,296, beta = 20) at its widest
point of a cycle (m = 10, step 10):

    Ahat = A V_10                     CSR SpMM, p = 8            (configs[1] kernel)
    CGS2 of Ahat vs C (n x 20) and the 10-block basis (n x 80), 2 passes
    thin QR of the n x 8 result                                   (configs[2] shapes)

one "step" = that whole arnoldi.step call, through the production path (the
C-ABI orchestrators rg_cgs2_f64 / rg_cholqr2_f64).

    value  = reference-model bytes of the step / device time per step.  The
             model is SURVEY.md §8d's per-op compulsory traffic of the
             REFERENCE algorithm (SpMM nnz*12 + (n+1)*4 + 16*p*n; sequential
             CGS2 8n(4k + 4w + 12p); QR 24np): it is the same numerator for
             both arms, so value ratios are time ratios.  The device runs
             the 3-pass joint [C W] schedule, which moves fewer bytes; those
             executed bytes are reported beside it (executed_bytes_per_step,
             roofline.step_frac) and are what the roofline fractions use.
    e2e    = the same metric through arnoldi.step with the step's inputs
             (basis n x 80 and C n x 20) uploaded from pinned host memory and
             the new block V_11 downloaded, every step.
    time_to_solution (N = 1): the full 5-system cfg4 256^3 sequence.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload step|solve|ortho|spmm] [--grid N]

--impl reference times the oracle (oracle/: the CPU restatement of the
reference path -- C SpMM with the reference's arithmetic, numpy/OpenBLAS
CGS2, LAPACK QR) on the host cores, on the same 256^3 operator, p, k and
basis width: each timed step is one of 8 row windows of the step (32 of the
256 z-planes, rotating), so 8 consecutive steps cover the whole operator.
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

P_BLOCK, K_RECYCLE, M_STEPS = 8, 20, 10
CPU_WINDOWS = 8  # row windows of the CPU arm's step sample
DMMA_PEAK_TFLOPS = 36.7  # measured FP64 tensor (DMMA) throughput, profiles/microbench_r01.txt

# operator families of the step workload: cfg4 (real conv-diff, BASELINE
# configs[3]) and cfg5 (complex 27-point stencil, BASELINE configs[4])
FAMILIES = {
    "cfg4": dict(p=8, k=20, m=10, grid=256, esz=8),
    "cfg5": dict(p=16, k=16, m=8, grid=160, esz=16),
}
STEP_METRIC = {
    "cfg4": "SpMM+block-orthog GB/s (reference-model bytes / step time; block Arnoldi step, cfg4 256^3 p=8 k=20 m=10)",
    "cfg5": "SpMM+block-orthog GB/s (reference-model bytes / step time; complex block Arnoldi step, cfg5 160^3 "
            "p=16 k=16 m=8)",
}


def step_model_bytes(n, nnz, p=P_BLOCK, k=K_RECYCLE, j=M_STEPS - 1, esz=8):
    w = (j + 1) * p
    spmm = nnz * (esz + 4) + (n + 1) * 4 + 2 * p * n * esz
    cgs2 = esz * n * (4 * k + 4 * w + 12 * p)
    qr = 3 * esz * n * p
    return spmm + cgs2 + qr, dict(spmm=spmm, cgs2=cgs2, qr=qr)


def step_config(family, grid, world):
    fam = FAMILIES[family]
    n = grid ** 3
    if family == "cfg4":
        desc = (f"cfg4-step: arnoldi.step #10 of a cycle on the {grid}^3 3-D conv-diff operator (beta=20) per GPU, "
                f"p=8, k=20, basis 80 cols (configs[2] shapes)")
    else:
        desc = f"cfg5-step: arnoldi.step #8 of a cycle, {grid}^3 complex 27-point stencil, p=16, k=16, basis 128 cols"
    return {"workload": desc, "grid": grid, "n_per_gpu": n, "p": fam["p"], "k": fam["k"],
            "basis_cols": fam["m"] * fam["p"], "parallelism": f"row-partition x{world}" if world > 1 else "1 GPU",
            "l2": "step operands (>14 GB) far larger than the 126 MB L2; no flush needed"}


def _ncu_traffic(label, family):
    """DRAM bytes (read + write) per launch of the kernel with this launch
    label, from the committed ncu --set full capture of the same step
    (profiles/ncu_traffic_r0*.json, written by tools/ncu_traffic.py)."""
    names = (["ncu_traffic_r02.json", "ncu_traffic_r01.json"] if family == "cfg4"
             else [f"ncu_traffic_r02_{family}.json", f"ncu_traffic_r01_{family}.json"])
    for name in names:
        f = ROOT / "profiles" / name
        if not f.exists():
            continue
        for rec in json.loads(f.read_text())["launches"]:
            if rec["label"] == label:
                return rec["traffic_bytes"], f"profiles/{name}"
    return None, None


def _peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [s.strip() for s in out.stdout.strip().split(",")]
                if len(parts) >= 7:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU arm (oracle): row windows of the same 256^3 step
# ---------------------------------------------------------------------------


class CpuStepSample:
    """The step of the step workload, restated on the host (oracle.arnoldi_step:
    SpMM with the reference's arithmetic on all host threads, numpy/OpenBLAS
    CGS2 against C then the basis, LAPACK QR), on row window w of the 256^3
    operator: rows [w n/8, (w+1) n/8) of A (their SpMM reads the full V_10),
    with C and the basis restricted to those rows.  Timing does not depend on
    the values, so C and the basis are seeded N(0,1) window blocks."""

    def __init__(self, grid=256, windows=CPU_WINDOWS, seed=0):
        import oracle
        from paper_1604_01713_b200 import problems

        self.oracle = oracle
        A = problems.conv_diff_3d(grid, 20.0)
        n = A.n_rows
        self.windows = windows
        rows = n // windows
        rng = np.random.default_rng(seed)
        self.V = np.asfortranarray(rng.standard_normal((n, P_BLOCK)))
        self.C = np.asfortranarray(rng.standard_normal((rows, K_RECYCLE)))
        self.W = np.asfortranarray(rng.standard_normal((rows, M_STEPS * P_BLOCK)))
        rp = np.asarray(A.row_ptr, dtype=np.int64)
        self.win = []
        for w in range(windows):
            r0, r1 = w * rows, (w + 1) * rows
            e0, e1 = int(rp[r0]), int(rp[r1])
            wrp = (rp[r0:r1 + 1] - e0).astype(np.int32)
            self.win.append((wrp, np.asarray(A.col_idx[e0:e1]), np.asarray(A.values[e0:e1]), rows, e1 - e0))
        self.threads = oracle.host_threads()
        self.n, self.nnz, self.grid = n, A.nnz, grid

    def run(self, w):
        """One window step; returns (seconds, model bytes of the window)."""
        rp, ci, v, rows, nnz = self.win[w % self.windows]
        t0 = time.perf_counter()
        self.oracle.arnoldi_step(rp, ci, v, self.V, self.C, self.W, nthreads=self.threads)
        t = time.perf_counter() - t0
        return t, step_model_bytes(rows, nnz)[0]

    def describe(self, steps, warmup):
        return (f"oracle arnoldi_step (C SpMM with the reference's arithmetic on {self.threads} threads + "
                f"numpy/OpenBLAS CGS2 against C then the basis + LAPACK QR) on row windows of the {self.grid}^3 cfg4 "
                f"operator: each step = 1/{self.windows} of the rows ({self.n // self.windows} rows, "
                f"{self.grid // self.windows} z-planes, rotating; "
                f"{self.windows} steps cover the whole operator), p=8, k=20, basis 80 cols; "
                f"{steps} timed after {warmup} warm-up")


def cpu_step_rate(steps, warmup, sample=None):
    s = sample or CpuStepSample()
    # the dense part uses every host thread the SpMM does, whatever OMP_NUM_THREADS
    # says (torchrun exports OMP_NUM_THREADS=1 to its ranks)
    try:
        from threadpoolctl import threadpool_limits

        blas = threadpool_limits(limits=s.threads, user_api="blas")
    except Exception:  # pragma: no cover - threadpoolctl is in the image
        import contextlib

        blas = contextlib.nullcontext()
    ts, bs = [], []
    with blas:
        for i in range(warmup):
            s.run(i)
        for i in range(steps):
            t, b = s.run(warmup + i)
            ts.append(t)
            bs.append(b)
    rate = sum(bs) / sum(ts) / 1e9
    info = {"kind": "port", "cores": s.threads, "sample": s.describe(steps, warmup),
            "window_s_mean": statistics.mean(ts),
            "full_step_s_estimate": statistics.mean(ts) * s.windows}
    return rate, statistics.mean(ts), info


def run_reference(args, rank, world):
    if rank != 0:
        return
    if args.workload != "step":
        print(json.dumps({"impl": "reference", "unavailable": f"the CPU arm covers the step workload only "
                                                             f"(asked: {args.workload})"}), flush=True)
        return
    rate, t, info = cpu_step_rate(args.steps, args.warmup)
    line = {"metric": STEP_METRIC["cfg4"], "value": rate, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": step_config("cfg4", 256, world),
            "cpu_baseline": dict(info, value=rate, unit="GB/s"),
            "e2e": {"value": rate, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def _setup_step(grid, dev, seed=0, world=1, rank=0, family="cfg4"):
    """Operator, recycle space and a 9-step factorisation resident on `dev`.

    world > 1: weak scaling -- rank r owns z-planes [r*grid, (r+1)*grid) of a
    grid x grid x (grid*world) conv-diff operator (2^24 rows per rank at
    grid=256), with the halo exchange and Gram allreduces of the row
    partition (paper_1604_01713_b200.distributed)."""
    import torch

    from paper_1604_01713_b200 import arnoldi, problems
    from paper_1604_01713_b200 import device as D
    from paper_1604_01713_b200.recycling import RecycleSpace, prepare_cross_system
    from paper_1604_01713_b200.solver import _Operator, _scrub

    t0 = time.perf_counter()
    fam = FAMILIES[family]
    P, K, M = fam["p"], fam["k"], fam["m"]
    dt = torch.complex128 if family == "cfg5" else torch.float64
    if family == "cfg5":
        if world != 1:
            raise SystemExit("the cfg5 step workload is single-GPU (weak-scaling runs use cfg4)")
        system, _, _ = problems.cfg5_sequence(N=grid, p=P)
        A = system(0)
        op = _Operator(A, None, "none")
        n, nnz = A.n_rows, A.nnz
    elif world == 1:
        A = problems.conv_diff_3d(grid, 20.0)
        op = _Operator(A, None, "none")
        n, nnz = A.n_rows, A.nnz
    else:
        from paper_1604_01713_b200 import distributed as DI

        rp, ci, v, n_glob = problems.conv_diff_3d_slab(grid, grid * world, 20.0, rank * grid, (rank + 1) * grid)
        comm = DI.CommContext()
        part = DI.RowPartition.even(n_glob, world, rank, align=grid * grid)
        plan = DI.HaloPlan.from_local_rows(part, rp, ci, v)
        dop = DI.DistCsr(plan, comm, dev)
        D.set_comm(comm, part)
        op = _Operator(dop, None, "none")
        n, nnz = part.n_local, len(v)
    t_gen = time.perf_counter() - t0
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    U0 = D.empty_block(n, K, dev, dt)
    U0.copy_(torch.randn(n, K, generator=g, device=dev, dtype=dt))
    rs = prepare_cross_system(RecycleSpace(u=U0, c=None), op.apply)
    R0 = D.empty_block(n, P, dev, dt)
    R0.copy_(torch.randn(n, P, generator=g, device=dev, dtype=dt))
    R0 = _scrub(R0, D.empty_block(n, P, dev, dt), rs.c)
    fact = arnoldi.start(op.apply, R0, m_max=M, recycle=rs, seed=seed, c_orthogonal=True)
    for _ in range(M - 1):
        arnoldi.step(fact, op.apply, recycle=rs)
    torch.cuda.synchronize()
    return (n, nnz), op, rs, fact, t_gen


def _one_step(fact, op, rs):
    from paper_1604_01713_b200 import arnoldi

    fact.m = fact.m_max - 1
    arnoldi.step(fact, op.apply, recycle=rs)


def _max_over_ranks(x, world, dev):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_step(args, rank, world):
    import torch

    from paper_1604_01713_b200 import device as D

    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    fam = FAMILIES[args.family]
    grid = args.grid or fam["grid"]
    (n, nnz), op, rs, fact, t_gen = _setup_step(grid, dev, seed=rank, world=world, rank=rank, family=args.family)
    model_bytes, parts = step_model_bytes(n, nnz, fam["p"], fam["k"], fam["m"] - 1, fam["esz"])

    for _ in range(args.warmup):
        _one_step(fact, op, rs)
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    # the timed region runs the production path; librgb200 brackets each of
    # its kernel-launching calls with events on the same stream (rg_prof.cu)
    D.LaunchLog.reset(timing=True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        # the ncu launch list (tools/evidence_step.sh) captures exactly this region
        torch.cuda.cudart().cudaProfilerStart()
        ev0.record()
        for _ in range(args.steps):
            _one_step(fact, op, rs)
        ev1.record()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
    ms = ev0.elapsed_time(ev1) / args.steps
    launches = D.LaunchLog.launches()
    per_kernel = D.LaunchLog.summary()
    D.LaunchLog.reset(timing=False)
    ms = _max_over_ranks(ms, world, dev)
    value = model_bytes * world / (ms * 1e-3) / 1e9

    peak, peak_kind = _peaks()
    kernels = sorted(((lbl, *rec) for lbl, rec in per_kernel.items()), key=lambda r: -r[2])
    total_ms = sum(k[2] for k in kernels)
    executed = sum(k[3] for k in kernels) / args.steps
    # dominant kernel: largest share of device time among kernels that move bytes
    top = next(k for k in kernels if k[3] > 0)
    lbl, calls, t_ms, nbytes, flops, nl = top
    per_launch_s = t_ms * 1e-3 / calls
    top_gbs = nbytes / calls / per_launch_s / 1e9
    traffic, traffic_src = _ncu_traffic(lbl, args.family)
    tensor = None
    if flops:
        tensor = {"flops_per_launch": flops, "achieved_tflops": flops / per_launch_s / 1e12,
                  "peak_tflops": DMMA_PEAK_TFLOPS, "frac": flops / per_launch_s / 1e12 / DMMA_PEAK_TFLOPS,
                  "peak_source": "FP64 DMMA m8n8k4, tools/microbench.cu (profiles/microbench_r01.txt)"}
    roofline = {"bound": "hbm", "achieved": top_gbs, "peak": peak, "unit": "GB/s", "frac": top_gbs / peak,
                "traffic": traffic, "traffic_source": traffic_src, "kernel": lbl,
                "kernel_share": t_ms / max(total_ms, 1e-9), "bytes_per_launch": nbytes // calls,
                "peak_source": peak_kind,
                "executed_bytes_per_step": executed,
                "step_achieved": executed / (ms * 1e-3) / 1e9,
                "step_frac": executed / (ms * 1e-3) / 1e9 / peak,
                "fp64_tensor": tensor}

    e2e = None
    if not args.no_e2e:
        e2e = _e2e(fact, op, rs, model_bytes, args)
        e2e["ms_per_step"] = _max_over_ranks(e2e["ms_per_step"], world, dev)
        e2e["value"] = model_bytes * world / (e2e["ms_per_step"] * 1e-3) / 1e9
        e2e["h2d_bytes_per_step"] *= world
        e2e["d2h_bytes_per_step"] *= world

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and args.family == "cfg4" and grid == 256:
        rate, t, info = cpu_step_rate(CPU_WINDOWS, 1)
        cpu = dict(info, value=rate, unit="GB/s")

    del fact, rs, op
    torch.cuda.empty_cache()
    tts = None
    if world == 1 and args.family == "cfg4" and grid == 256 and not args.no_tts:
        try:
            tts = solve_sequence_timed(256, args.tts_systems, 1, 0, dev)
        except Exception as exc:  # reported, never silently dropped
            tts = {"error": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        line = {"metric": STEP_METRIC[args.family],
                "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64" if args.family == "cfg4" else "c128", "data": "synthetic",
                "config": step_config(args.family, grid, world),
                "model_bytes_per_step": model_bytes * world, "model_parts": parts,
                "executed_bytes_per_step": executed * world,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk.summary(),
                "kernels": [{"kernel": k[0], "calls": k[1], "ms": k[2], "bytes": k[3],
                             "GB/s": k[3] / (k[2] * 1e-3) / 1e9 if k[2] > 0 else None} for k in kernels],
                "time_to_solution": tts,
                "setup_s": {"matrix_generation": t_gen}}
        print(json.dumps(line), flush=True)


def _e2e(fact, op, rs, model_bytes, args):
    """Same step, inputs in pinned HOST memory: H2D of V_m's basis (n x 80,
    includes V_10) and C (n x 20) inside the timed region, the step, D2H of
    the new block V_11 (n x 8); the small H/F/R coefficients come back
    inside the step itself."""
    import torch

    n, L, K = fact.n, fact.L, fact.k
    dt = fact.dtype
    esz = 16 if dt == torch.complex128 else 8
    wcols = fact.m_max * L
    hW = torch.empty((wcols, n), dtype=dt).pin_memory()
    hC = torch.empty((K, n), dtype=dt).pin_memory()
    hQ = torch.empty((L, n), dtype=dt).pin_memory()
    hW.copy_(fact._W[:, :wcols].t())
    hC.copy_(rs.c.t())
    W_dev = fact._W[:, :wcols]
    steps = max(1, args.steps)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        W_dev.t().copy_(hW, non_blocking=True)
        rs.c.t().copy_(hC, non_blocking=True)
        _one_step(fact, op, rs)
        hQ.copy_(fact.v_block(fact.m_max).t(), non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    h2d = (wcols + K) * n * esz
    d2h = L * n * esz + (2 * K + 2 * (wcols + L)) * L * esz + 5 * L * L * esz
    return {"value": model_bytes / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms, "steps": steps,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "path": "arnoldi.step with basis/C uploaded from pinned host memory and V_11 downloaded each step"}


# ---------------------------------------------------------------------------
# time to solution (BASELINE configs[3]: "GCRO-DR solve s/system")
# ---------------------------------------------------------------------------


def solve_sequence_timed(grid, nsys, world, rank, dev):
    """Full block GCRO-DR sequence of the config-4 family (3-D conv-diff
    grid^3, beta=20, p=8, m=10, k=20, tol 1e-8, ``nsys`` systems with the
    0.5 %*i*u*diag(A) perturbations).  Strong scaling over ``world`` GPUs:
    the same global problem is row-partitioned on whole z-planes.  Each
    system is timed from the host-resident B to the host-resident X (the
    public API call), max over ranks."""
    import torch

    from paper_1604_01713_b200 import SolverConfig, problems, solve_block_gcrodr
    from paper_1604_01713_b200 import device as D

    t0 = time.perf_counter()
    n_glob = grid ** 3
    if world == 1:
        A, B, system, kw = problems.cfg4_sequence(N=grid, n_systems=nsys)
        ops = [system(i) for i in range(nsys)]
    else:
        from paper_1604_01713_b200 import distributed as DI

        B = np.asfortranarray(np.random.default_rng(0).standard_normal((n_glob, P_BLOCK)))
        u = np.random.default_rng(1).uniform(0.0, 1.0, n_glob)
        comm = DI.CommContext()
        part = DI.RowPartition.even(n_glob, world, rank, align=grid * grid)
        z0, z1 = part.r0 // (grid * grid), part.r1 // (grid * grid)
        rp, ci, v, _ = problems.conv_diff_3d_slab(grid, grid, 20.0, z0, z1)
        rows = np.repeat(np.arange(part.n_local), np.diff(rp))
        on_diag = ci == rows + part.r0
        ops = []
        for i in range(nsys):
            vi = v.copy()
            if i:
                dA = v[on_diag]
                vi[on_diag] = dA + 0.005 * i * u[part.r0:part.r1] * dA
            plan = DI.HaloPlan.from_local_rows(part, rp, ci, vi)
            ops.append(DI.DistCsr(plan, comm, dev))
        D.set_comm(comm, part)
        kw = dict(m=10, k=20, tol=1e-8, max_cycles=200)
    t_setup = time.perf_counter() - t0
    cfg = SolverConfig(**kw)
    rs = None
    per = []
    for i, Ai in enumerate(ops):
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        X, rep, rs_out = solve_block_gcrodr(Ai, B, None, cfg, rs_in=rs)
        torch.cuda.synchronize()
        dt = _max_over_ranks(time.perf_counter() - t1, world, dev)
        rs = rs_out if rs_out is not None else rs
        # reference-model bytes of every block step the solve ran (step j of a
        # cycle: basis width 8(j+1); no recycle space in system 0's first cycle)
        nnz_i = getattr(Ai, "nnz", None) or int(getattr(getattr(Ai, "plan", None), "values", np.zeros(0)).size)
        mb = 0
        for c, h in enumerate(rep.residual_history):
            kk = 0 if (i == 0 and c == 0) else kw["k"]
            mb += sum(step_model_bytes(n_glob // world, nnz_i, P_BLOCK, kk, j)[0] for j in range(len(h)))
        per.append({"system": i, "s": dt, "cycles": rep.cycles,
                    "block_steps": int(sum(len(h) for h in rep.residual_history)),
                    "matvecs": rep.matvec_count, "converged": bool(rep.converged),
                    "rel_residual": float(rep.final_residual_norm / np.linalg.norm(rep.rhs_norms)),
                    "step_model_bytes": mb * world})
    if world > 1:
        D.set_comm(None, None)
        comm.close()
    total_s = sum(r["s"] for r in per)
    total_steps = sum(r["block_steps"] for r in per)
    bsz = n_glob * P_BLOCK * 8
    return {"s_per_system": statistics.mean(r["s"] for r in per), "systems": per, "setup_s": t_setup,
            "workload": f"cfg4 sequence {grid}^3 conv-diff beta=20, p=8, m=10, k=20, tol 1e-8, {nsys} systems",
            "n_gpus": world,
            # the step metric end to end through the public solve API: host B in,
            # host X out, every cycle operation inside the time (numerator: the
            # block steps' reference-model bytes only)
            "e2e_solve": {"value": sum(r["step_model_bytes"] for r in per) / total_s / 1e9, "unit": "GB/s",
                          "path": "solve_block_gcrodr(CsrMatrix, host B) -> host X per system",
                          "h2d_bytes_per_step": nsys * bsz / max(total_steps, 1),
                          "d2h_bytes_per_step": nsys * bsz / max(total_steps, 1)}}


def run_solve(args, rank, world):
    import torch

    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.family == "cfg5":
        return _run_solve_cfg5(args, rank, world)
    grid = args.grid or 256
    rec = solve_sequence_timed(grid, args.systems, world, rank, dev)
    if rank == 0:
        mean = rec["s_per_system"]
        print(json.dumps({"metric": "GCRO-DR solve s/system (cfg4 family)", "value": mean, "unit": "s/system",
                          "n_gpus": world, "steps": args.systems, "warmup": 0, "ms_per_step": mean * 1e3,
                          "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                          "data": "synthetic",
                          "config": {"workload": rec["workload"], "setup_s": rec["setup_s"],
                                     "parallelism": f"row-partition x{world}"},
                          "e2e_solve": rec["e2e_solve"], "systems": rec["systems"]}), flush=True)


def _run_solve_cfg5(args, rank, world):
    """Config-5 sequence (complex 27-point stencil grid^3, p=16, m=8, k=16,
    4 shifts) on one GPU: time per system."""
    import torch

    from paper_1604_01713_b200 import SolverConfig, problems, solve_block_gcrodr

    if world != 1:
        raise SystemExit("the cfg5 solve workload is single-GPU")
    grid = args.grid or 160
    nsys = min(args.systems, 4)
    t0 = time.perf_counter()
    system, B, kw = problems.cfg5_sequence(N=grid)
    ops = [system(i) for i in range(nsys)]
    t_setup = time.perf_counter() - t0
    cfg = SolverConfig(**kw)
    rs, per = None, []
    for i, Ai in enumerate(ops):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        X, rep, rs_out = solve_block_gcrodr(Ai, B, None, cfg, rs_in=rs)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t1
        rs = rs_out if rs_out is not None else rs
        per.append({"system": i, "s": dt, "cycles": rep.cycles,
                    "block_steps": int(sum(len(h) for h in rep.residual_history)),
                    "matvecs": rep.matvec_count, "converged": bool(rep.converged),
                    "rel_residual": float(rep.final_residual_norm / np.linalg.norm(rep.rhs_norms))})
    mean = statistics.mean(r["s"] for r in per)
    print(json.dumps({"metric": "GCRO-DR solve s/system (cfg5 complex family)", "value": mean, "unit": "s/system",
                      "n_gpus": 1, "steps": nsys, "warmup": 0, "ms_per_step": mean * 1e3,
                      "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
                      "data": "synthetic",
                      "config": {"workload": f"cfg5 sequence {grid}^3 complex 27-point stencil, p=16, m=8, k=16, "
                                             f"tol 1e-8, {nsys} shifts", "setup_s": t_setup,
                                 "parallelism": "1 GPU"},
                      "systems": per}), flush=True)


# ---------------------------------------------------------------------------
# kernel microbenches: configs[2] (ortho) and configs[1] (spmm)
# ---------------------------------------------------------------------------


def _timed(fn, steps, warmup):
    import torch

    from paper_1604_01713_b200 import device as D

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    D.LaunchLog.reset(timing=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    launches = D.LaunchLog.launches()
    recs = D.LaunchLog.summary()
    D.LaunchLog.reset(timing=False)
    return e0.elapsed_time(e1) / steps, launches, recs


def run_ortho(args, rank, world):
    """BASELINE configs[2] at n = 2^24: W = C^T V; V - C W; CGS2 of V against
    the 10-block basis Q (2 passes); thin QR of the n x 8 result -- each timed
    separately, GB/s of SURVEY §8d's algorithmic bytes."""
    import torch

    from paper_1604_01713_b200 import device as D
    from paper_1604_01713_b200 import problems
    from paper_1604_01713_b200.dense_kernels import QrScratch, cholqr2_launch
    from paper_1604_01713_b200.ortho import project_chain

    torch.cuda.set_device(0)
    n = 2 ** (args.log2n or 24)
    C, V, Q = problems.cfg3_inputs(n)
    k, p, w = C.shape[1], V.shape[1], Q.shape[1]
    Wc = D.small(k, p)
    Z = D.empty_block(n, p)
    Z2 = D.empty_block(n, p)
    c1, c2 = D.small(w, p), D.small(w, p)
    scr = QrScratch(p, V.device, torch.float64)
    Qo = D.empty_block(n, p)
    D.tall(V, None, gram=("basis", C, Wc))
    ops = {
        "CtV": (lambda: D.tall(V, None, gram=("basis", C, Wc)), 8 * n * (k + p)),
        "V-CW": (lambda: D.tall(V, Z, [(C, Wc, -1.0)]), 8 * n * (k + 2 * p)),
        "CGS2 vs Q (2 passes)": (lambda: project_chain(V, Z2, [Q, Q], [c1, c2]),
                                 2 * (8 * n * (w + p) + 8 * n * (w + 2 * p))),
        "QR n x 8 (CholQR2)": (lambda: cholqr2_launch(Z2, Qo, scr), 24 * n * p),
    }
    peak, peak_kind = _peaks()
    out, total_b, total_ms = [], 0, 0.0
    for name, (fn, nb) in ops.items():
        ms, launches, recs = _timed(fn, args.steps, args.warmup)
        executed = sum(r[2] for r in recs.values()) / args.steps
        out.append({"op": name, "ms": ms, "algorithmic_bytes": nb, "GB/s": nb / (ms * 1e-3) / 1e9,
                    "frac": nb / (ms * 1e-3) / 1e9 / peak, "executed_bytes": executed,
                    "launches_per_op": launches / args.steps})
        total_b += nb
        total_ms += ms
    print(json.dumps({"metric": "block-orthogonalization GB/s (configs[2], algorithmic bytes)",
                      "value": total_b / (total_ms * 1e-3) / 1e9, "unit": "GB/s", "n_gpus": 1,
                      "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms,
                      "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                      "data": "synthetic", "config": {"workload": f"cfg3 ortho microbench n=2^{int(np.log2(n))}, "
                                                                  f"C n x 20, V n x 8, Q n x 80"},
                      "peak": peak, "peak_source": peak_kind, "ops": out}), flush=True)


def run_spmm(args, rank, world):
    """BASELINE configs[1]: SpMM with the 128^3 7-point Laplacian, p in
    {1, 2, 4, 8, 16}; GB/s of the reference's own bytes model."""
    import torch

    from paper_1604_01713_b200 import device as D
    from paper_1604_01713_b200 import problems
    from paper_1604_01713_b200.sparse_core import spmm_device

    torch.cuda.set_device(0)
    grid = args.grid or 128
    A = problems.laplacian_3d(grid)
    n = A.n_rows
    peak, peak_kind = _peaks()
    out = []
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    dA = A.device(torch.device("cuda", 0))
    for p in (1, 2, 4, 8, 16):
        V = D.empty_block(n, p)
        V.copy_(torch.randn(n, p, generator=g, device="cuda", dtype=torch.float64))
        Y = D.empty_block(n, p)
        # kernel time: events around each library call on its stream (these
        # products take 30-160 us, the same order as a Python call)
        _, launches, recs = _timed(lambda: spmm_device(dA, V, Y), args.steps, args.warmup)
        ms = sum(r[1] for r in recs.values()) / args.steps
        # back-to-back calls through the Python entry point, no per-call events
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            spmm_device(dA, V, Y)
        e1.record()
        torch.cuda.synchronize()
        nb = A.nnz * 12 + (n + 1) * 4 + 16 * p * n
        out.append({"p": p, "ms": ms, "GB/s": nb / (ms * 1e-3) / 1e9, "frac": nb / (ms * 1e-3) / 1e9 / peak,
                    "launches_per_call": launches / args.steps, "call_ms": e0.elapsed_time(e1) / args.steps})
    best = max(o["GB/s"] for o in out)
    print(json.dumps({"metric": "SpMM GB/s (configs[1], reference bytes model bench.py:44-47)", "value": best,
                      "unit": "GB/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                      "ms_per_step": min(o["ms"] for o in out), "higher_is_better": True, "scaling": "weak",
                      "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                      "config": {"workload": f"cfg2 SpMM {grid}^3 7-point Laplacian, n={n}, nnz={A.nnz}",
                                 "timing": "ms = device time of the library call (events on its stream); call_ms = "
                                           "back-to-back spmm_device calls from Python",
                                 "l2": "operands (A 175 MB + blocks) exceed the 126 MB L2 from p = 2; p = 1 "
                                       "re-reads part of A from L2"},
                      "peak": peak, "peak_source": peak_kind, "per_p": out}), flush=True)


# ---------------------------------------------------------------------------


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _spawn(args_list, n):
    """`bench.py --gpus N` without a launcher: re-exec under torchrun, one
    rank per GPU on this node (NCCL's init log stays visible on stderr)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(ROOT / "bench.py"), *args_list]
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"))
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--grid", type=int, default=None)
    ap.add_argument("--log2n", type=int, default=None)
    ap.add_argument("--family", choices=sorted(FAMILIES), default="cfg4")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tts", action="store_true", help="skip the time-to-solution record of the step line")
    ap.add_argument("--tts-systems", type=int, default=5)
    ap.add_argument("--workload", choices=["step", "solve", "ortho", "spmm"], default="step")
    ap.add_argument("--systems", type=int, default=5)
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_spawn(sys.argv[1:], args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        # the CPU arm: rank 0 alone runs and prints it, the other ranks exit 0 without
        # work (no process group: nothing is exchanged)
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1))
        # RG_BENCH_BACKEND=gloo runs the N>1 code path on a single GPU (test only)
        dist.init_process_group(os.environ.get("RG_BENCH_BACKEND", "nccl"))
    if args.workload == "solve":
        run_solve(args, rank, world)
    elif args.workload == "ortho":
        run_ortho(args, rank, world)
    elif args.workload == "spmm":
        run_spmm(args, rank, world)
    else:
        run_step(args, rank, world)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
