"""CSR kernel vs diagonal-layout kernel (rg_spmm_dia_f64) on the config-2 and
config-4 operators: time per call (20 calls after 3 warm-up) and bitwise
agreement; GB/s of the reference's byte model (bench.py:44-47)."""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1604_01713_b200 import device as D, problems  # noqa: E402

out = {}
for name, A in (("cfg2_lap128", problems.laplacian_3d(128)), ("cfg4_cd256", problems.conv_diff_3d(256, 20.0))):
    dA = A.device(torch.device("cuda", 0))
    plan = dA.dia()
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    for p in (1, 4, 8, 16):
        X = D.empty_block(A.n_rows, p)
        X.copy_(torch.randn(A.n_rows, p, generator=g, device="cuda", dtype=torch.float64))
        Y = D.empty_block(A.n_rows, p)
        res = {}
        for mode in (False, True):
            D.SPMM_DIA = mode
            for _ in range(3):
                D.spmm(dA, X, Y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                D.spmm(dA, X, Y)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            res[mode] = (ms, Y.clone())
        b = A.nnz * 12 + (A.n_rows + 1) * 4 + 16 * p * A.n_rows
        same = torch.equal(res[False][1], res[True][1])
        out[f"{name}/p{p}"] = {"csr_us": round(res[False][0] * 1e3, 1), "dia_us": round(res[True][0] * 1e3, 1),
                               "csr_GB/s": round(b / res[False][0] / 1e6), "dia_GB/s": round(b / res[True][0] / 1e6),
                               "bitwise": same}
        print(name, p, out[f"{name}/p{p}"], flush=True)
print(json.dumps(out))
