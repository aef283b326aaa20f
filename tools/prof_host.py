"""Host-side profile (cProfile) of the config-1 sequence on the GPU: where
the per-step Python / launch / sync overhead goes at small n."""
import cProfile, pathlib, pstats, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1604_01713_b200 import SolverConfig, problems, solve_sequence

systems, kw = problems.cfg1_sequence()
solve_sequence(systems[:1], SolverConfig(**kw))  # warm-up
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
reps = solve_sequence(systems, SolverConfig(**kw))
torch.cuda.synchronize()
pr.disable()
print(f"cfg1 sequence wall {time.perf_counter() - t0:.3f} s; steps", [sum(len(h) for h in r.residual_history) for r in reps])
st = pstats.Stats(pr).sort_stats("tottime")
st.print_stats(25)
