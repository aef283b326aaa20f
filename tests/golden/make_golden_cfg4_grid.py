"""Golden run of the REAL reference on the config-4 operator family at a
chosen grid, system 0 only, optionally truncated to the first cycles:

    python tests/golden/make_golden_cfg4_grid.py 256 2     # first 2 cycles at 256^3 (~20 min, 8 cores)
    python tests/golden/make_golden_cfg4_grid.py 128 200   # system 0 to convergence at 128^3 (~40 min)

Same recipe as make_golden_cfg4_64.py (problems.cfg4_sequence: 3-D conv-diff
beta=20, p=8 N(0,1) RHS from default_rng(0), m=10, k=20, tol 1e-8); only
`max_cycles` differs.  Writes tests/golden/cfg4_<grid>_c<max_cycles>.npz
with the iteration record of system 0 (per-step residual histories,
per-cycle true residuals, matvecs, cycles), X column norms, and the
reference's wall time per block step on this container (8 cores) -- the
full-size CPU step time that BASELINE.md §2 asks for.

The 256^3 record pins the full-size solve ("first cycles at
full size"); the 128^3 record pins the cycle-count growth between the 64^3
golden and the 256^3 device runs.
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


def main(grid=256, max_cycles=2):
    _import_reference()
    import recgmres.arnoldi as ra
    from recgmres.solver import SolverConfig, solve_block_gcrodr
    from recgmres.sparse_core import CsrMatrix
    from paper_1604_01713_b200 import problems

    A, B, _system, kw = problems.cfg4_sequence(N=grid, n_systems=1)
    kw = dict(kw, max_cycles=max_cycles)
    t0 = time.perf_counter()
    Aref = CsrMatrix(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, A.values)
    t_csr = time.perf_counter() - t0

    step_times = []
    orig_step = ra.step

    def timed_step(*a, **k):
        t = time.perf_counter()
        r = orig_step(*a, **k)
        step_times.append(time.perf_counter() - t)
        return r

    ra.step = timed_step
    import recgmres.solver as rsol
    if getattr(rsol, "arnoldi", None) is ra:
        pass  # the solver calls arnoldi.step through the module attribute
    t0 = time.perf_counter()
    X, rep, _rs = solve_block_gcrodr(Aref, B, None, SolverConfig(**kw))
    wall = time.perf_counter() - t0
    ra.step = orig_step
    out = {"grid": np.array(grid), "max_cycles": np.array(max_cycles), "wall_s": np.array(wall),
           "csr_validation_s": np.array(t_csr), "cpu_count": np.array(os.cpu_count()),
           "step_s": np.array(step_times)}
    _report_arrays("sys0/", rep, out, with_solution=False)
    out["sys0/Xnorms"] = np.linalg.norm(X, axis=0)
    out["sys0/Bnorm"] = np.array(np.linalg.norm(B))
    np.savez_compressed(HERE / f"cfg4_{grid}_c{max_cycles}.npz", **out)
    print(f"reference cfg4 system 0 at {grid}^3, max_cycles={max_cycles}: {wall:.1f} s, "
          f"{rep.cycles} cycles, {sum(len(h) for h in rep.residual_history)} block steps, "
          f"{rep.matvec_count} matvecs, converged={rep.converged}, "
          f"median step {np.median(step_times) if step_times else float('nan'):.2f} s")


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
