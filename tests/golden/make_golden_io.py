"""Golden fixtures for the host-side utilities, produced by the REAL
reference (recgmres.sparse_core: Matrix Market reader/writer, CsrMatrix
validation, gen_banded).  Run in the build container:

    python tests/golden/make_golden_io.py

Writes tests/golden/io_cases.npz: for every Matrix Market text below, either
the parsed CSR arrays or the reference's error class and message.
"""

from __future__ import annotations

import json
import pathlib
import tempfile

import numpy as np

from make_golden import OUT, _import_reference

MM_CASES = {
    "general": "%%MatrixMarket matrix coordinate real general\n% c\n3 3 4\n1 1 2.5\n2 3 -1\n3 1 4e-3\n3 3 7\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n1 1 1\n2 1 2\n3 2 3\n",
    "integer": "%%MatrixMarket matrix coordinate integer general\n2 2 2\n1 2 5\n2 1 -6\n",
    "empty": "",
    "bad_header": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "complex_field": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "size_line": "%%MatrixMarket matrix coordinate real general\n3 3\n1 1 1\n",
    "size_nonint": "%%MatrixMarket matrix coordinate real general\n3 x 1\n1 1 1\n",
    "missing_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "entry_fields": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "entry_malformed": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 a 3\n",
    "out_of_range": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",
    "count_mismatch": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 1\n",
    "duplicates": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 1 2\n",
}
ARRAY_CASES = {
    "array_ok": "%%MatrixMarket matrix array real general\n3 2\n1\n2\n3\n4\n5\n6\n",
    "array_short": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n",
    "array_bad": "%%MatrixMarket matrix coordinate real general\n2 2\n",
}


def main():
    _import_reference()
    from recgmres.sparse_core import CsrMatrix, gen_banded, read_matrix_market, read_matrix_market_array

    out = {}
    tmp = pathlib.Path(tempfile.mkdtemp())
    for name, text in MM_CASES.items():
        f = tmp / f"{name}.mtx"
        f.write_text(text)
        try:
            A = read_matrix_market(f)
            out[f"mm/{name}/row_ptr"] = np.asarray(A.row_ptr)
            out[f"mm/{name}/col_idx"] = np.asarray(A.col_idx)
            out[f"mm/{name}/values"] = np.asarray(A.values)
            out[f"mm/{name}/shape"] = np.array([A.n_rows, A.n_cols])
        except Exception as e:  # noqa: BLE001 - the class and message are the fixture
            out[f"mm/{name}/error"] = np.array(json.dumps([type(e).__name__, str(e)]))
    for name, text in ARRAY_CASES.items():
        f = tmp / f"{name}.mtx"
        f.write_text(text)
        try:
            out[f"arr/{name}/value"] = read_matrix_market_array(f)
        except Exception as e:  # noqa: BLE001
            out[f"arr/{name}/error"] = np.array(json.dumps([type(e).__name__, str(e)]))
    for n, band, seed in ((50, 2, 3), (200, 5, 11)):
        B = gen_banded(n, band, seed)
        out[f"banded/{n}_{band}_{seed}/row_ptr"] = np.asarray(B.row_ptr)
        out[f"banded/{n}_{band}_{seed}/col_idx"] = np.asarray(B.col_idx)
        out[f"banded/{n}_{band}_{seed}/values"] = np.asarray(B.values)
    bad = {
        "rp_len": (2, 2, [0, 1], [0], [1.0]),
        "rp_start": (2, 2, [1, 1, 2], [0], [1.0]),
        "len_mismatch": (2, 2, [0, 1, 2], [0, 1], [1.0]),
        "col_range": (2, 2, [0, 1, 2], [0, 2], [1.0, 2.0]),
        "unsorted": (2, 3, [0, 2, 2], [1, 0], [1.0, 2.0]),
        "duplicate": (2, 3, [0, 2, 2], [1, 1], [1.0, 2.0]),
    }
    for name, args in bad.items():
        try:
            CsrMatrix(*[np.asarray(a) if isinstance(a, list) else a for a in args])
            out[f"csr/{name}/error"] = np.array(json.dumps(["none", ""]))
        except Exception as e:  # noqa: BLE001
            out[f"csr/{name}/error"] = np.array(json.dumps([type(e).__name__, str(e)]))
    np.savez_compressed(OUT / "io_cases.npz", **out)
    print("wrote", OUT / "io_cases.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
