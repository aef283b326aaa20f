#!/usr/bin/env python
"""Benchmark of the block GCRO-DR hot path on B200 (driver contract).

Default workload ("step", BASELINE configs[3]/[2] shapes): one block Arnoldi
step of the 256^3 3-D convection-diffusion operator (n = 16,777,216 = 2^24,
nnz = 117,047,296, beta = 20) at its widest point of a cycle (m = 10, step 10):

    Ahat = A V_10                    CSR SpMM, p = 8            (configs[1] kernel)
    CGS2 of Ahat vs C (n x 20) and the 10-block basis (n x 80), 2 passes
    thin QR of the n x 8 result                                  (configs[2] shapes)

one "step" = that whole arnoldi.step call.  metric = algorithmic HBM bytes of
the step (SURVEY.md §8d model: SpMM nnz*12 + (n+1)*4 + 16*p*n; CGS2
8n(4k + 4w + 12p); QR 24np) / device time per step, in GB/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload step|spmm|ortho|solve] [--grid N]

--impl reference times the oracle (CPU restatement of the reference path:
C SpMM with the reference's arithmetic + numpy/OpenBLAS CGS2 + LAPACK QR) on
the host cores, on a bounded sample (a 64^3 grid of the same operator family
with the same k, p, basis width).
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

P_BLOCK, K_RECYCLE, M_STEPS = 8, 20, 10
SAMPLE_GRID = 64  # CPU sample: 64^3 rows of the same operator family
DMMA_PEAK_TFLOPS = 36.7  # measured FP64 tensor (DMMA) throughput, profiles/microbench_r01.txt

# operator families of the step workload: cfg4 (real conv-diff, BASELINE
# configs[3]) and cfg5 (complex 27-point stencil, BASELINE configs[4])
FAMILIES = {
    "cfg4": dict(p=8, k=20, m=10, grid=256, esz=8),
    "cfg5": dict(p=16, k=16, m=8, grid=160, esz=16),
}


def step_model_bytes(n, nnz, p=P_BLOCK, k=K_RECYCLE, j=M_STEPS - 1, esz=8):
    w = (j + 1) * p
    spmm = nnz * (esz + 4) + (n + 1) * 4 + 2 * p * n * esz
    cgs2 = esz * n * (4 * k + 4 * w + 12 * p)
    qr = 3 * esz * n * p
    return spmm + cgs2 + qr, dict(spmm=spmm, cgs2=cgs2, qr=qr)


def _ncu_traffic(label, family):
    """DRAM bytes (read + write) per launch of the kernel with this launch
    label, from the committed ncu --set full capture of the same step
    (profiles/ncu_traffic_r01*.json, written by tools/ncu_traffic.py)."""
    name = "ncu_traffic_r01.json" if family == "cfg4" else f"ncu_traffic_r01_{family}.json"
    f = ROOT / "profiles" / name
    if not f.exists():
        return None, None
    for rec in json.loads(f.read_text())["launches"]:
        if rec["label"] == label:
            return rec["traffic_bytes"], f"profiles/{name}"
    return None, None


def _peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


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
# CPU arm (oracle)
# ---------------------------------------------------------------------------


def _cpu_sample_inputs(grid=SAMPLE_GRID, seed=0):
    from paper_1604_01713_b200 import problems

    A = problems.conv_diff_3d(grid, 20.0)
    n = A.n_rows
    rng = np.random.default_rng(seed)
    C = np.linalg.qr(rng.standard_normal((n, K_RECYCLE)))[0]
    W = np.linalg.qr(rng.standard_normal((n, M_STEPS * P_BLOCK)))[0]
    W = np.asfortranarray(W - C @ (C.T @ W))
    Vm = np.asfortranarray(W[:, -P_BLOCK:])
    return A, np.asfortranarray(C), W, Vm


def cpu_step_rate(steps=3, warmup=1, grid=SAMPLE_GRID):
    """Oracle block Arnoldi step on the CPU sample; returns (GB/s, s/step, info)."""
    import oracle

    A, C, W, Vm = _cpu_sample_inputs(grid)
    nthreads = oracle.host_threads()
    for _ in range(warmup):
        oracle.arnoldi_step(A.row_ptr, A.col_idx, A.values, Vm, C, W, nthreads=nthreads)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle.arnoldi_step(A.row_ptr, A.col_idx, A.values, Vm, C, W, nthreads=nthreads)
        ts.append(time.perf_counter() - t0)
    b, _ = step_model_bytes(A.n_rows, A.nnz)
    t = statistics.mean(ts)
    info = {"kind": "port", "cores": nthreads,
            "sample": f"oracle arnoldi_step (C SpMM, reference arithmetic, {nthreads} threads + numpy/OpenBLAS "
                      f"CGS2 + LAPACK QR) on the {grid}^3 conv-diff operator, n={A.n_rows}, p=8, k=20, "
                      f"basis 80 cols; mean of {steps} after {warmup} warm-up"}
    return b / t / 1e9, t, info


def run_reference(args, rank, world):
    if rank != 0:
        return
    rate, t, info = cpu_step_rate(steps=max(1, args.steps), warmup=max(1, min(args.warmup, 2)))
    line = {"metric": "SpMM+block-orthog HBM GB/s (block Arnoldi step, cfg4 256^3 p=8 k=20 m=10)",
            "value": rate, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": "cfg4-step sample (64^3 of the same operator family) on host cores",
                       "grid": SAMPLE_GRID, "p": P_BLOCK, "k": K_RECYCLE, "basis_cols": M_STEPS * P_BLOCK},
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


def run_ours(args, rank, world):
    import torch

    from paper_1604_01713_b200 import device as D

    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

    fam = FAMILIES[args.family]
    grid = args.grid or fam["grid"]
    (n, nnz), op, rs, fact, t_gen = _setup_step(grid, dev, seed=rank, world=world, rank=rank, family=args.family)
    model_bytes, parts = step_model_bytes(n, nnz, fam["p"], fam["k"], fam["m"] - 1, fam["esz"])

    for _ in range(args.warmup):
        _one_step(fact, op, rs)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    D.LaunchLog.reset(timing=True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            _one_step(fact, op, rs)
        ev1.record()
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    launches = D.LaunchLog.count
    per_kernel = D.LaunchLog.summary()
    D.LaunchLog.reset(timing=False)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = model_bytes * world / (ms * 1e-3) / 1e9

    # dominant kernel (largest share of device time inside the timed region)
    peak, peak_kind = _peaks()
    kernels = sorted(((lbl, c, t_ms, b) for lbl, (c, t_ms, b) in per_kernel.items()), key=lambda r: -r[2])
    top = kernels[0]
    top_gbs = top[3] / (top[2] * 1e-3) / 1e9
    total_ms = sum(k[2] for k in kernels)
    traffic, traffic_src = _ncu_traffic(top[0], args.family)
    top_flops = D.LaunchLog.flops.get(top[0], 0) if hasattr(D.LaunchLog, "flops") else 0
    tensor = None
    if top_flops:
        per_launch_s = top[2] * 1e-3 / max(top[1], 1)
        tensor = {"flops_per_launch": top_flops, "achieved_tflops": top_flops / per_launch_s / 1e12,
                  "peak_tflops": DMMA_PEAK_TFLOPS, "frac": top_flops / per_launch_s / 1e12 / DMMA_PEAK_TFLOPS,
                  "peak_source": "FP64 DMMA m8n8k4, tools/microbench.cu (profiles/microbench_r01.txt)"}
    roofline = {"bound": "hbm", "achieved": top_gbs, "peak": peak, "unit": "GB/s", "frac": top_gbs / peak,
                "traffic": traffic, "traffic_source": traffic_src, "kernel": top[0],
                "kernel_share": top[2] / max(total_ms, 1e-9),
                "bytes_per_launch": top[3] // max(top[1], 1), "peak_source": peak_kind,
                "fp64_tensor": tensor}

    # end to end through the reference-facing call with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = _e2e(fact, op, rs, model_bytes, args, dev)
        if world > 1:
            import torch.distributed as dist

            t = torch.tensor([e2e["ms_per_step"]], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["ms_per_step"] = float(t.item())
            e2e["value"] = model_bytes * world / (e2e["ms_per_step"] * 1e-3) / 1e9
            e2e["h2d_bytes_per_step"] *= world
            e2e["d2h_bytes_per_step"] *= world

    cpu = None
    if rank == 0 and not args.no_cpu and args.family == "cfg4":
        rate, t, info = cpu_step_rate(steps=3, warmup=1)
        cpu = dict(info, value=rate, unit="GB/s")

    if rank == 0:
        if args.family == "cfg4":
            metric = "SpMM+block-orthog HBM GB/s (block Arnoldi step, cfg4 256^3 p=8 k=20 m=10)"
            workload = (f"cfg4-step: arnoldi.step #10 of a cycle, {grid}^3 conv-diff beta=20 "
                        f"per GPU, n={n}, nnz={nnz} per GPU, p=8, k=20, basis 80 cols (cfg3 shapes)")
        else:
            metric = "SpMM+block-orthog HBM GB/s (complex block Arnoldi step, cfg5 160^3 p=16 k=16 m=8)"
            workload = (f"cfg5-step: arnoldi.step #8 of a cycle, {grid}^3 complex 27-point stencil, "
                        f"n={n}, nnz={nnz}, p=16, k=16, basis 128 cols, complex128")
        line = {"metric": metric,
                "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64" if args.family == "cfg4" else "c128", "data": "synthetic",
                "config": {"workload": workload,
                           "model_bytes_per_step": model_bytes, "model_parts": parts,
                           "l2": "inputs (>14 GB) far larger than the 126 MB L2; no flush needed",
                           "parallelism": f"row-partition x{world}" if world > 1 else "1 GPU"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk.summary(),
                "kernels": [{"kernel": k[0], "calls": k[1], "ms": k[2], "GB/s": k[3] / (k[2] * 1e-3) / 1e9
                             if k[2] > 0 else None} for k in kernels],
                "setup_s": {"matrix_generation": t_gen}}
        print(json.dumps(line), flush=True)


def _e2e(fact, op, rs, model_bytes, args, dev):
    """Same step, inputs in pinned HOST memory: H2D of V_m's basis (n x 80,
    includes V_10) and C (n x 20) inside the timed region, the step, D2H of
    the new block V_11 (n x 8); the small H/F/R coefficients come back
    inside the step itself."""
    import torch

    from paper_1604_01713_b200 import device as D

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
    steps = max(1, min(args.steps, 3))
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
    return {"value": model_bytes / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "path": "arnoldi.step with basis/C uploaded from pinned host memory and V_11 downloaded each step"}


# ---------------------------------------------------------------------------
# time-to-solution workload (BASELINE configs[3]: "GCRO-DR solve s/system")
# ---------------------------------------------------------------------------


def run_solve(args, rank, world):
    """Full block GCRO-DR sequence of the config-4 family (3-D conv-diff
    grid^3, beta=20, p=8, m=10, k=20, tol 1e-8, `--systems` systems with the
    0.5 %*i*u*diag(A) perturbations).  Strong scaling over `world` GPUs: the
    same global problem is row-partitioned on whole z-planes."""
    import torch

    from paper_1604_01713_b200 import SolverConfig, problems, solve_block_gcrodr
    from paper_1604_01713_b200 import device as D

    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.family == "cfg5":
        return _run_solve_cfg5(args, rank, world)
    grid, nsys = args.grid or 256, args.systems
    t0 = time.perf_counter()
    n_glob = grid ** 3
    B = np.asfortranarray(np.random.default_rng(0).standard_normal((n_glob, P_BLOCK)))
    u = np.random.default_rng(1).uniform(0.0, 1.0, n_glob)
    if world == 1:
        A, _, system, kw = problems.cfg4_sequence(N=grid, n_systems=nsys)
        ops = [system(i) for i in range(nsys)]
        part = None
    else:
        from paper_1604_01713_b200 import distributed as DI
        from paper_1604_01713_b200.problems import add_diagonal  # noqa: F401

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
        dt = time.perf_counter() - t1
        if world > 1:
            t = torch.tensor([dt], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        rs = rs_out if rs_out is not None else rs
        per.append({"system": i, "s": dt, "cycles": rep.cycles, "block_steps": int(sum(len(h) for h in rep.residual_history)),
                    "matvecs": rep.matvec_count, "converged": bool(rep.converged),
                    "rel_residual": float(rep.final_residual_norm / np.linalg.norm(rep.rhs_norms))})
    if rank == 0:
        mean = statistics.mean(r["s"] for r in per)
        line = {"metric": "GCRO-DR solve s/system (cfg4 family)", "value": mean, "unit": "s/system",
                "n_gpus": world, "steps": nsys, "warmup": 0, "ms_per_step": mean * 1e3,
                "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": {"workload": f"cfg4 sequence {grid}^3 conv-diff beta=20, p=8, m=10, "
                                                            f"k=20, tol 1e-8, {nsys} systems",
                                                "setup_s": t_setup, "parallelism": f"row-partition x{world}"},
                "systems": per}
        print(json.dumps(line), flush=True)


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--grid", type=int, default=None)
    ap.add_argument("--family", choices=sorted(FAMILIES), default="cfg4")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", choices=["step", "solve"], default="step")
    ap.add_argument("--systems", type=int, default=5)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        if args.impl == "reference":
            dist.init_process_group("gloo")
        else:
            import torch

            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1))
            # RG_BENCH_BACKEND=gloo runs the N>1 code path on a single GPU (test only)
            dist.init_process_group(os.environ.get("RG_BENCH_BACKEND", "nccl"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.workload == "solve":
        run_solve(args, rank, world)
    else:
        run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
