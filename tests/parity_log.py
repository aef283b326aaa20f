"""Observed parity errors of the GPU tests, appended as JSON lines to
$RG_PARITY_LOG (default gpurun_out/parity.jsonl) so that the tolerances in
the tests can be checked against what the device actually achieves."""

import json
import os
import pathlib


def record(test: str, **errors) -> None:
    path = pathlib.Path(os.environ.get("RG_PARITY_LOG", "gpurun_out/parity.jsonl"))
    try:
        path.parent.mkdir(parents=True, exist_ok=True)
        with open(path, "a") as fh:
            fh.write(json.dumps({"test": test, **{k: float(v) for k, v in errors.items()}}) + "\n")
    except OSError:
        pass
