"""Golden run of the REAL reference on the config-4 family at a reduced grid
(3-D conv-diff 64^3, beta=20, p=8, m=10, k=20, tol 1e-8, 5 systems with the
0.5 %*i*u*diag(A) perturbations of problems.cfg4_sequence).  Stores the
iteration record of every system plus the reference's wall time on this
container's CPU (the CPU time-to-solution baseline quoted in DESIGN.md).

    python tests/golden/make_golden_cfg4_64.py      (~6 min, 8 cores)
"""

import os
import pathlib
import sys
import time

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parents[1]))

from make_golden import _import_reference, _report_arrays  # noqa: E402


def main(grid=64, n_systems=5):
    _import_reference()
    from recgmres.solver import SolverConfig, solve_sequence
    from recgmres.sparse_core import CsrMatrix
    from paper_1604_01713_b200 import problems

    A, B, system, kw = problems.cfg4_sequence(N=grid, n_systems=n_systems)
    mats = [system(i) for i in range(n_systems)]
    ref_systems = [(CsrMatrix(M.n_rows, M.n_cols, M.row_ptr, M.col_idx, M.values), B) for M in mats]
    t0 = time.perf_counter()
    reps = solve_sequence(ref_systems, SolverConfig(**kw))
    wall = time.perf_counter() - t0
    out = {"grid": np.array(grid), "n_systems": np.array(n_systems), "wall_s": np.array(wall),
           "cpu_count": np.array(os.cpu_count())}
    for i, rep in enumerate(reps):
        _report_arrays(f"sys{i}/", rep, out, with_solution=False)
        out[f"sys{i}/Xnorms"] = np.linalg.norm(rep.solution, axis=0)
    np.savez_compressed(HERE / f"cfg4_{grid}_cases.npz", **out)
    print(f"reference cfg4 family at {grid}^3: {wall:.1f} s for {n_systems} systems "
          f"({[int(r.cycles) for r in reps]} cycles, {[int(r.matvec_count) for r in reps]} matvecs)")


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
