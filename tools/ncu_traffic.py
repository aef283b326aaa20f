"""Pair an ncu capture of tools/prof_step.py with the step's launch labels
and write the per-launch DRAM traffic table bench.py reports as
roofline.traffic.

    ncu --set full --clock-control none --profile-from-start off -o step \\
        python tools/prof_step.py --steps 1 --labels labels.json
    python tools/ncu_traffic.py step.ncu-rep labels.json profiles/ncu_traffic_r01.json
"""
import csv
import io
import json
import subprocess
import sys


OURS = ("spmm", "tall", "chol", "tsqr", "ilu0", "sptrsv", "permute_rows", "gather_kernel")


def main():
    rep, labels_path, out = sys.argv[1:4]
    if rep.endswith(".csv"):  # an exported `ncu -i ... --page raw --csv`
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    col = {k: h.index(k) for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum",
                                   "dram__bytes_write.sum")}
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    launches = []
    for r in rows[2:]:
        rd = float(r[col["dram__bytes_read.sum"]]) * scale[units[col["dram__bytes_read.sum"]]]
        wr = float(r[col["dram__bytes_write.sum"]]) * scale[units[col["dram__bytes_write.sum"]]]
        ms = float(r[col["gpu__time_duration.sum"]]) * (1e-3 if units[col["gpu__time_duration.sum"]] == "us" else 1.0)
        name = r[col["Kernel Name"]]
        if not any(k in name for k in OURS):
            continue  # torch plumbing (fills, copies) between our launches
        launches.append((name, ms, rd, wr))
    labels = json.load(open(labels_path))
    if len(labels) != len(launches):
        raise SystemExit(f"{len(labels)} labels vs {len(launches)} ncu launches")
    table = []
    for lab, (kname, ms, rd, wr) in zip(labels, launches):
        kind = lab["label"].split()[0]
        if not (("spmm" in kind and "spmm" in kname) or ("tall" in kind and "tall" in kname)
                or ("chol" in kind and "chol" in kname)):
            raise SystemExit(f"label {lab['label']!r} does not match kernel {kname!r}")
        table.append({"label": lab["label"], "kernel": kname.split("(")[0], "ncu_ms": ms,
                      "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
                      "algorithmic_bytes": lab["bytes"]})
    json.dump({"source": rep, "launches": table}, open(out, "w"), indent=1)
    print(json.dumps(table, indent=1))


if __name__ == "__main__":
    main()
