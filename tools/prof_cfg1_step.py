"""Per-step host+device time of the config-1 solve (n = 4096, p = 4, m = 20,
k = 10; latency-bound) with and without the captured step graphs
(arnoldi.StepWorkspace), and the sequence wall time.  Writes one JSON line.

    python tools/prof_cfg1_step.py
"""
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1604_01713_b200 import SolverConfig, arnoldi, problems, solve_sequence  # noqa: E402


def run(graphs: bool, reps: int = 3, after: int = 2):
    orig_ws = arnoldi.StepWorkspace.__init__

    def ws_init(self, graphs_=None, capture_after=after):
        orig_ws(self, graphs, capture_after)

    arnoldi.StepWorkspace.__init__ = ws_init
    systems, kw = problems.cfg1_sequence()
    step_t = []
    orig = arnoldi.step

    def timed(*a, **k):
        t = time.perf_counter()
        r = orig(*a, **k)
        step_t.append(time.perf_counter() - t)
        return r

    arnoldi.step = timed
    walls = []
    try:
        for _ in range(reps):
            step_t.clear()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            reps_ = solve_sequence(systems, SolverConfig(**kw))
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
    finally:
        arnoldi.step = orig
        arnoldi.StepWorkspace.__init__ = orig_ws
    steps = [int(sum(len(h) for h in r.residual_history)) for r in reps_]
    return {"graphs": graphs, "capture_after": after, "sequence_s": min(walls), "steps": steps,
            "step_ms_median": 1e3 * float(np.median(step_t)), "step_ms_mean": 1e3 * float(np.mean(step_t)),
            "hist": [np.concatenate(r.residual_history).tolist() for r in reps_]}


if __name__ == "__main__":
    torch.cuda.set_device(0)
    off = run(False)
    ons = [run(True, after=a) for a in (1, 2, 3, 5)]
    same = all(off["hist"] == on["hist"] for on in ons)
    for r in [off] + ons:
        r.pop("hist")
    print(json.dumps({"cfg1_step_eager": off, "cfg1_step_graphs": ons, "identical_histories": same}))
