"""Cold vs warm time to solution: bench.solve_sequence_timed twice in one
process on the cfg4 family (the second run has the modules loaded, the
allocator warm and the kernels' attributes set).

    python tools/prof_tts.py [--grid 256] [--systems 2]
"""
import argparse
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--systems", type=int, default=2)
    ap.add_argument("--no-dia", action="store_true", help="keep every SpMM on the CSR kernel")
    args = ap.parse_args()
    from paper_1604_01713_b200 import device as D

    D.SPMM_DIA = not args.no_dia
    dev = torch.device("cuda", 0)
    out = {}
    for run in ("cold", "warm"):
        t0 = time.perf_counter()
        rec = bench.solve_sequence_timed(args.grid, args.systems, 1, 0, dev)
        out[run] = {"wall_s": time.perf_counter() - t0, "setup_s": rec["setup_s"],
                    "systems": [(r["s"], r["cycles"], r["block_steps"]) for r in rec["systems"]]}
        print(run, json.dumps(out[run]), flush=True)


if __name__ == "__main__":
    main()
