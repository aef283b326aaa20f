"""Block vs one-at-a-time sweeps of A and of (I - CC^T)A on the B200.

Drop-in for ``recgmres.bench`` (/root/reference/pkg/src/recgmres/bench.py):
same names, bytes model, CSV schema and ratio helpers; the timed operations
run on the device kernels (rg_spmm_csr_f64 and the fused projection chain)
and are timed with CUDA events on the launch stream (mean / min / std over
``reps`` after one warm-up, as ``_time_reps`` does at bench.py:58-67).
This reproduces the paper's §6.2 experiments on B200.
"""

from __future__ import annotations

import csv
import pathlib
from dataclasses import dataclass

import numpy as np
import torch

from . import device as _dev
from .dense_kernels import reduced_qr_device
from .ortho import project_chain
from .sparse_core import CsrMatrix, spmm_device

DEFAULT_BLOCK_SIZES = (1, 2, 4, 6, 8, 10, 12, 14, 16, 18, 20)

_VAL_BYTES = 8
_IDX_BYTES = 4


@dataclass
class BenchResult:
    matrix_id: str
    n: int
    nnz: int
    L: int
    mode: str  # "all-at-once" | "one-at-a-time"
    projector: str  # "none" | "mgs" | "cgs2"
    dim_c: int
    reps: int
    mean_seconds: float
    min_seconds: float
    stddev_seconds: float
    bytes_model: int


def matvec_bytes(n_rows: int, nnz: int, L: int) -> int:
    """Matrix values/indices read once, block read and result written
    (bench.py:44-47)."""
    return nnz * (_VAL_BYTES + _IDX_BYTES) + (n_rows + 1) * _IDX_BYTES + 2 * L * n_rows * _VAL_BYTES


def projector_bytes(n: int, dim_c: int, L: int, ortho: str) -> int:
    """Extra bytes of (I - CC^T) per the reference's model (bench.py:50-55)."""
    passes = 2 if ortho == "cgs2" else 1
    return passes * (2 * dim_c * n * _VAL_BYTES + 2 * L * n * _VAL_BYTES)


def _time_reps(fn, reps: int, warmup: bool):
    if warmup:
        fn()
    times = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
    t = np.array(times)
    return float(t.mean()), float(t.min()), float(t.std())


def _random_block(n: int, L: int, seed: int) -> torch.Tensor:
    """Same seeded uniform(0,1) block as bench.py:70-72, uploaded."""
    rng = np.random.default_rng(seed)
    return _dev.to_device_block(np.asfortranarray(rng.uniform(0.0, 1.0, size=(n, L))))


def bench_matvec(A: CsrMatrix, L_values=None, reps: int = 100, warmup: bool = True, *, matrix_id: str = "matrix",
                 seed: int = 0):
    """spmm(A, n x L) against L single-column products, per block size
    (bench.py:75-107)."""
    L_values = list(L_values) if L_values else list(DEFAULT_BLOCK_SIZES)
    results = []
    for L in L_values:
        X = _random_block(A.n_cols, L, seed)
        Y = _dev.empty_block(A.n_rows, L, X.device)
        cols = [X[:, j:j + 1] for j in range(L)]
        outs = [Y[:, j:j + 1] for j in range(L)]

        def block_once():
            spmm_device(A, X, Y)

        def one_at_a_time():
            for c, o in zip(cols, outs):
                spmm_device(A, c, o)

        mean_b, min_b, std_b = _time_reps(block_once, reps, warmup)
        if L == 1:
            mean_s, min_s, std_s = mean_b, min_b, std_b
        else:
            mean_s, min_s, std_s = _time_reps(one_at_a_time, reps, warmup)
        results.append(BenchResult(matrix_id, A.n_rows, A.nnz, L, "all-at-once", "none", 0, reps,
                                   mean_b, min_b, std_b, matvec_bytes(A.n_rows, A.nnz, L)))
        results.append(BenchResult(matrix_id, A.n_rows, A.nnz, L, "one-at-a-time", "none", 0, reps,
                                   mean_s, min_s, std_s, L * matvec_bytes(A.n_rows, A.nnz, 1)))
    return results


def make_projector_basis(n: int, dim_c: int, seed: int) -> torch.Tensor:
    """Orthonormalised seeded N(0,1) n x dim_c basis (bench.py:110-113), on
    the device."""
    rng = np.random.default_rng(seed)
    G = _dev.to_device_block(rng.standard_normal((n, dim_c)))
    return reduced_qr_device(G, 1e-12).q


def _project(Y: torch.Tensor, C: torch.Tensor, ortho: str) -> torch.Tensor:
    """(I - CC^T) Y in place: one vector of C at a time ("mgs") or two dense
    block passes ("cgs2") (bench.py:116-126), as fused device passes."""
    if C.shape[1] == 0:
        return Y
    L = Y.shape[1]
    if ortho == "mgs":
        bases = [C[:, i:i + 1] for i in range(C.shape[1])]
    else:
        bases = [C, C]
    coefs = [_dev.small(b.shape[1], L, Y.device) for b in bases]
    project_chain(Y, Y, bases, coefs)
    return Y


def bench_projected(A: CsrMatrix, C_dims, L_values=None, ortho: str = "cgs2", reps: int = 100, *,
                    warmup: bool = True, matrix_id: str = "matrix", seed: int = 0):
    """(I - CC^T)A applied all-at-once vs one column at a time, per
    projector dimension (bench.py:129-166)."""
    if ortho not in ("mgs", "cgs2"):
        raise ValueError(f"unknown ortho '{ortho}'")
    L_values = list(L_values) if L_values else list(DEFAULT_BLOCK_SIZES)
    results = []
    for dim_c in C_dims:
        C = make_projector_basis(A.n_rows, dim_c, seed + dim_c) if dim_c else _dev.empty_block(A.n_rows, 0)
        tag = "none" if dim_c == 0 else ortho
        for L in L_values:
            X = _random_block(A.n_cols, L, seed)
            Y = _dev.empty_block(A.n_rows, L, X.device)
            cols = [X[:, j:j + 1] for j in range(L)]
            outs = [Y[:, j:j + 1] for j in range(L)]

            def block_once():
                _project(spmm_device(A, X, Y), C, ortho)

            def one_at_a_time():
                for c, o in zip(cols, outs):
                    _project(spmm_device(A, c, o), C, ortho)

            mean_b, min_b, std_b = _time_reps(block_once, reps, warmup)
            if L == 1:
                mean_s, min_s, std_s = mean_b, min_b, std_b
            else:
                mean_s, min_s, std_s = _time_reps(one_at_a_time, reps, warmup)
            base = matvec_bytes(A.n_rows, A.nnz, L)
            proj = projector_bytes(A.n_rows, dim_c, L, ortho)
            single = matvec_bytes(A.n_rows, A.nnz, 1) + projector_bytes(A.n_rows, dim_c, 1, ortho)
            results.append(BenchResult(matrix_id, A.n_rows, A.nnz, L, "all-at-once", tag, dim_c, reps,
                                       mean_b, min_b, std_b, base + proj))
            results.append(BenchResult(matrix_id, A.n_rows, A.nnz, L, "one-at-a-time", tag, dim_c, reps,
                                       mean_s, min_s, std_s, L * single))
    return results


CSV_HEADER = ["matrix_id", "n", "nnz", "L", "mode", "projector", "dim_c", "ortho", "reps", "mean_s", "min_s",
              "stddev_s", "bytes_model"]


def emit_csv(results, path) -> None:
    """Header row, '.' decimal, %.6e floats, LF endings (bench.py:169-186)."""
    with open(path, "wt", newline="\n") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(CSV_HEADER)
        for r in results:
            ortho = r.projector if r.projector in ("mgs", "cgs2") else ""
            w.writerow([r.matrix_id, r.n, r.nnz, r.L, r.mode, r.projector, r.dim_c, ortho, r.reps,
                        f"{r.mean_seconds:.6e}", f"{r.min_seconds:.6e}", f"{r.stddev_seconds:.6e}", r.bytes_model])


def block_single_ratios(results):
    """{(matrix_id, projector, dim_c): [(L, mean(block L) / (mean(L singles)/L))]}."""
    index = {(r.matrix_id, r.projector, r.dim_c, r.L, r.mode): r for r in results}
    groups = sorted({(r.matrix_id, r.projector, r.dim_c) for r in results})
    out = {}
    for g in groups:
        pts = []
        for L in sorted({r.L for r in results if (r.matrix_id, r.projector, r.dim_c) == g}):
            blk = index.get((*g, L, "all-at-once"))
            one = index.get((*g, L, "one-at-a-time"))
            if blk is not None and one is not None:
                pts.append((L, blk.mean_seconds / (one.mean_seconds / L)))
        out[g] = pts
    return out


_SERIES_COLORS = ("#1f3a93", "#b03a2e", "#1e8449", "#7d3c98", "#ca6f1e", "#5d6d7e")


def emit_plot(results, path) -> None:
    """SVG of the block / single-product time ratio against the block size L,
    one polyline per (matrix, projector, dim_c) group (the figure the
    reference's ``emit_plot`` draws, bench.py:212-251; drawn here with tick
    labels on both axes and a dashed ratio-1 reference line)."""
    series = {g: pts for g, pts in sorted(block_single_ratios(results).items()) if pts}
    W, H, M = 640, 420, 56
    xs = [L for pts in series.values() for L, _ in pts] or [1]
    ys = [v for pts in series.values() for _, v in pts] or [1.0]
    x_hi, y_hi = max(max(xs), 1), max(max(ys), 1.0)

    def px(L):
        return M + (W - 2 * M) * L / x_hi

    def py(v):
        return H - M - (H - 2 * M) * v / y_hi

    el = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{H}" font-family="sans-serif">',
          f'<rect x="0" y="0" width="{W}" height="{H}" fill="#ffffff"/>',
          f'<path d="M{M},{M} V{H - M} H{W - M}" fill="none" stroke="#000000"/>',
          f'<line x1="{M}" y1="{py(1.0):.1f}" x2="{W - M}" y2="{py(1.0):.1f}" stroke="#999999" '
          f'stroke-dasharray="4,3"/>']
    for L in sorted(set(xs)):
        el.append(f'<text x="{px(L):.1f}" y="{H - M + 16}" font-size="10" text-anchor="middle">{L}</text>')
    for k in range(5):
        v = y_hi * k / 4
        el.append(f'<text x="{M - 6}" y="{py(v) + 3:.1f}" font-size="10" text-anchor="end">{v:.2f}</text>')
    el.append(f'<text x="{W / 2:.0f}" y="{H - 14}" font-size="12" text-anchor="middle">block size L</text>')
    el.append(f'<text x="{M}" y="{M - 18}" font-size="12">time(one block of L) / time(one single product)</text>')
    for i, (g, pts) in enumerate(series.items()):
        col = _SERIES_COLORS[i % len(_SERIES_COLORS)]
        xy = " ".join(f"{px(L):.1f},{py(v):.1f}" for L, v in pts)
        el.append(f'<polyline points="{xy}" fill="none" stroke="{col}" stroke-width="1.5"/>')
        el.append(f'<text x="{W - M - 230}" y="{M + 14 * (i + 1)}" font-size="11" fill="{col}">'
                  f'{g[0]} projector={g[1]} dim_c={g[2]}</text>')
    el.append("</svg>")
    pathlib.Path(path).write_text("\n".join(el) + "\n")


def read_results_csv(path):
    out = []
    with open(path, "rt", newline="") as fh:
        for row in csv.DictReader(fh):
            out.append(BenchResult(matrix_id=row["matrix_id"], n=int(row["n"]), nnz=int(row["nnz"]), L=int(row["L"]),
                                   mode=row["mode"], projector=row["projector"], dim_c=int(row["dim_c"]),
                                   reps=int(row["reps"]), mean_seconds=float(row["mean_s"]),
                                   min_seconds=float(row["min_s"]), stddev_seconds=float(row["stddev_s"]),
                                   bytes_model=int(row["bytes_model"])))
    return out
