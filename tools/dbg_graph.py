import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1604_01713_b200 import SolverConfig, arnoldi, problems, solve_block_gcrodr
systems, kw = problems.cfg1_sequence()
A, B = systems[1]
A0 = systems[0][0]
cfg = SolverConfig(**kw)
# system 0 to get a recycle space
_, r0, rs = solve_block_gcrodr(A0, B, None, cfg)
log = {}
orig = arnoldi.step
def rec(tag):
    def f(fact, opA, recycle=None, ortho="cgs2"):
        out = orig(fact, opA, recycle, ortho)
        log.setdefault(tag, []).append((fact.m, fact._H[: (fact.m + 1) * fact.L, (fact.m - 1) * fact.L: fact.m * fact.L].copy(), fact.k, fact.c_orthogonal))
        return out
    return f
for tag, rows in (("eager", 0), ("graph", 1 << 18)):
    arnoldi.GRAPH_MAX_ROWS = rows
    arnoldi.step = rec(tag)
    _, rep, _ = solve_block_gcrodr(A, B, None, SolverConfig(**dict(kw, max_cycles=4)), rs_in=rs)
    print(tag, rep.cycles, [len(h) for h in rep.residual_history])
arnoldi.step = orig
for i, (a, b) in enumerate(zip(log["eager"], log["graph"])):
    d = np.abs(a[1] - b[1]).max()
    if d > 1e-12:
        print("first divergence at call", i, "m", a[0], "k", a[2], a[3], "diff", d)
        print(a[1][:6, :2]); print(b[1][:6, :2])
        break
else:
    print("no divergence in", len(log["eager"]), "steps")
