"""cProfile of the host side of a cfg4 solve (system 0, --cycles cycles at
grid^3): where the Python thread spends its time (blocking syncs show up as
time in .item() / synchronize / numpy() calls)."""
import argparse
import cProfile
import pathlib
import pstats
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=256)
ap.add_argument("--cycles", type=int, default=20)
args = ap.parse_args()
from paper_1604_01713_b200 import SolverConfig, problems, solver  # noqa: E402

A, B, system, kw = problems.cfg4_sequence(N=args.grid, n_systems=1)
solver.solve_block_gcrodr(system(0), B, None, SolverConfig(m=2, k=4, max_cycles=1))
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
solver.solve_block_gcrodr(system(0), B, None, SolverConfig(**dict(kw, max_cycles=args.cycles)))
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
st.sort_stats("cumulative").print_stats(40)
