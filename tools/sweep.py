"""The paper's section 6.2 sweeps on B200 through the package's bench module
(reference bench.py:75-166 protocol): block SpMM vs L single products, and the
projected operator (I - C C^T) A with CGS2 and MGS projectors of growing
dimension, on the config-2 operator.  Writes the reference CSV schema and
the SVG ratio plot.

    python tools/sweep.py --grid 128 --out gpurun_out/sweep
"""
import argparse
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=128)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="gpurun_out/sweep")
    args = ap.parse_args()
    from paper_1604_01713_b200 import bench, problems

    A = problems.laplacian_3d(args.grid)
    mid = f"lap3d_{args.grid}"
    Ls = [1, 2, 4, 8, 16]
    res = bench.bench_matvec(A, Ls, reps=args.reps, matrix_id=mid)
    for ortho in ("cgs2", "mgs"):
        res += [r for r in bench.bench_projected(A, [0, 10, 20, 40], Ls, ortho=ortho, reps=args.reps, matrix_id=mid)
                if not (ortho == "mgs" and r.dim_c == 0)]
    out = pathlib.Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    bench.emit_csv(res, out.with_suffix(".csv"))
    bench.emit_plot(res, out.with_suffix(".svg"))
    for g, pts in sorted(bench.block_single_ratios(res).items()):
        print(g, " ".join(f"L={L}:{v:.3f}" for L, v in pts))


if __name__ == "__main__":
    main()
