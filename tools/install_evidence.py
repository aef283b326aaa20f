"""Copy the outputs of tools/evidence_step.sh (gpurun_out/) into profiles/ under
the round's names: the bench line, the ncu launch list of the timed region, the
per-launch DRAM traffic, the full-set summary / details and the cycle profile.

    python tools/install_evidence.py r02
"""
import csv
import pathlib
import shutil
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
G, P = ROOT / "gpurun_out", ROOT / "profiles"
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"

shutil.copy(G / "bench_step.json", P / f"bench_{tag}_step.json")
shutil.copy(G / "launches.csv", P / f"ncu_launches_bench_{tag}.csv")
shutil.copy(G / "ncu_traffic.json", P / f"ncu_traffic_{tag}.json")
if (G / "cycle_256.json").exists():
    shutil.copy(G / "cycle_256.json", P / f"cycle_{tag}_256.json")

rows = list(csv.reader(open(G / "step_raw.csv")))
h, units = rows[0], rows[1]
keep = [i for i, c in enumerate(h) if c == "Kernel Name" or "." in c]
with open(P / f"ncu_step_{tag}_summary.txt", "w") as f:
    f.write("# ncu --set full --clock-control none, one cfg4 block Arnoldi step (tools/prof_step.py via "
            "tools/evidence_step.sh):\n# SpMM on the diagonal layout (spmm_dia_kernel), TMA-fed ws CGS2 passes "
            "(tall_ws_kernel: P1 <9,1,13,0,1,32>, P2 <8,1,13,26,1,32>, P3 <8,1,2,0,1,28>), CholQR2 solves on the "
            "256-row TMA ring (tall_nr_kernel)\n")
    f.write("# " + " | ".join(f"{h[i]}" + (f" ({units[i]})" if units[i] else "") for i in keep) + "\n")
    for r in rows[2:]:
        f.write(" | ".join(r[i].split("(")[0].replace("void ", "") if h[i] == "Kernel Name" else r[i] for i in keep)
                + "\n")
out = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_details.py"), str(G / "step_details.csv")],
                     capture_output=True, text=True, check=True).stdout
(P / f"ncu_step_{tag}_details.txt").write_text(out)
print("installed", tag)
