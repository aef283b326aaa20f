"""A/B of SpMM builds: time rg_spmm_csr_f64 on the config-2 and config-4
operators for each library given (default build first; variants from
tools/ab_build.py) in fresh subprocesses, and check that every variant's
output is bitwise the default's.

    python tools/ab_spmm.py [variant.so ...]
"""
import hashlib
import json
import os
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]


def child():
    sys.path.insert(0, str(ROOT))
    import torch

    from paper_1604_01713_b200 import device as D, problems
    from paper_1604_01713_b200.sparse_core import spmm_device

    out = {}
    for name, A in (("cfg2_lap128", problems.laplacian_3d(128)), ("cfg4_cd256", problems.conv_diff_3d(256, 20.0))):
        g = torch.Generator(device="cuda")
        g.manual_seed(1)
        for p in (1, 4, 8, 16):
            X = D.empty_block(A.n_rows, p)
            X.copy_(torch.randn(A.n_rows, p, generator=g, device="cuda", dtype=torch.float64))
            Y = D.empty_block(A.n_rows, p)
            for _ in range(3):
                spmm_device(A, X, Y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                spmm_device(A, X, Y)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            b = A.nnz * 12 + (A.n_rows + 1) * 4 + 16 * p * A.n_rows
            h = hashlib.sha1(D.to_numpy_block(Y).tobytes()).hexdigest()[:16]
            out[f"{name}/p{p}"] = {"us": round(ms * 1e3, 1), "GB/s": round(b / ms / 1e6), "sha": h}
    print(json.dumps(out))


if __name__ == "__main__":
    if "--child" in sys.argv:
        child()
        sys.exit(0)

    libs = [None] + sys.argv[1:]
    res = {}
    for lib in libs:
        env = dict(os.environ)
        if lib:
            env["RG_LIB_PATH"] = str(pathlib.Path(lib).resolve())
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        res[lib or "default"] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-2000:]
    base = res["default"]
    for lib, r in res.items():
        if isinstance(r, str):
            print(lib, "FAILED", r)
            continue
        same = all(r[k]["sha"] == base[k]["sha"] for k in r)
        print(f"{lib}: bitwise={'yes' if same else 'NO'}  " + "  ".join(f"{k} {v['us']}us {v['GB/s']}GB/s" for k, v in r.items()))
    print(json.dumps(res))
