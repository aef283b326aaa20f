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


def _fake_results():
    from paper_1604_01713_b200.bench import BenchResult

    out = []
    for proj, dim_c in (("none", 0), ("cgs2", 4)):
        for L in (1, 2, 4, 8):
            blk = 1e-3 * (1 + 0.3 * L) * (1 + dim_c / 10)
            one = 1e-3 * L * (1 + dim_c / 10)
            out.append(BenchResult("cfg2", 100, 700, L, "all-at-once", proj, dim_c, 3, blk, blk, 0.0, 10 * L))
            out.append(BenchResult("cfg2", 100, 700, L, "one-at-a-time", proj, dim_c, 3, one, one, 0.0, 10 * L))
    return out


def test_emit_plot_one_polyline_per_group(tmp_path):
    """The reference's SVG contract (tests/test_bench_cli.py:97-103): an <svg>
    document with one polyline per (matrix, projector, dim_c) group."""
    from paper_1604_01713_b200.bench import block_single_ratios, emit_plot

    res = _fake_results()
    path = tmp_path / "ratios.svg"
    emit_plot(res, path)
    text = path.read_text()
    assert text.startswith("<svg") and text.rstrip().endswith("</svg>")
    assert text.count("<polyline") == len(block_single_ratios(res)) == 2
    emit_plot(res, tmp_path / "again.svg")
    assert (tmp_path / "again.svg").read_bytes() == path.read_bytes()


def test_emit_csv_round_trip(tmp_path):
    from paper_1604_01713_b200.bench import CSV_HEADER, emit_csv, read_results_csv

    res = _fake_results()
    emit_csv(res, tmp_path / "r.csv")
    assert (tmp_path / "r.csv").read_text().splitlines()[0] == ",".join(CSV_HEADER)
    back = read_results_csv(tmp_path / "r.csv")
    assert [(r.L, r.mode, r.projector, r.dim_c, r.bytes_model) for r in back] == \
        [(r.L, r.mode, r.projector, r.dim_c, r.bytes_model) for r in res]
