"""Host-side checks of the driver bench (bench.py): the CPU arm's row-window
sample of the step and the config both arms print."""

import json
import sys

import numpy as np

import bench


def test_cpu_window_sample_covers_the_operator():
    s = bench.CpuStepSample(grid=16, windows=4)
    rows = [w[3] for w in s.win]
    nnz = [w[4] for w in s.win]
    assert sum(rows) == s.n and sum(nnz) == s.nnz
    t, b = s.run(5)  # window 1
    assert t > 0 and b == bench.step_model_bytes(rows[1], nnz[1])[0]


def test_reference_arm_prints_the_step_config(capsys, monkeypatch):
    class Small(bench.CpuStepSample):
        def __init__(self):
            super().__init__(grid=16, windows=4)

    monkeypatch.setattr(bench, "CpuStepSample", Small)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--steps", "3", "--warmup", "3"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    bench.main()
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["steps"] == 3 and line["warmup"] == 3
    assert line["config"] == bench.step_config("cfg4", 256, 1)
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert np.isfinite(line["value"]) and line["value"] > 0
