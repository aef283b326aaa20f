"""Summarise bench.py step lines: step time, per-kernel time and GB/s."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as exc:  # noqa: BLE001
        print(f, "unreadable", exc)
        continue
    print(f"{f}: {d['ms_per_step']:.3f} ms/step  value {d['value']:.0f}  step_frac {d['roofline']['step_frac']:.3f}"
          f"  sm {d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')}")
    for k in d["kernels"]:
        print(f"   {k['ms'] / k['calls']:.3f} ms  {k['GB/s'] or 0:6.0f} GB/s  {k['kernel']}")
