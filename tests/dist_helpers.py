"""Test-only helpers for the multi-process tests: a host restatement of
rg_tall's semantics (driving ortho.project_chain without a GPU) and a local
SpMM for DistCsr built on the oracle."""

import numpy as np
import torch

import oracle


def host_tall_factory(comm=None):
    """rg_tall semantics on CPU torch tensors (float64, any layout)."""

    def tall(Zin, Zout, terms=(), r1=None, r2=None, gram=None, n=None, p=None):
        z = (Zin.numpy().copy() if Zin is not None else np.zeros((n, p)))
        for X, S, alpha in terms:
            z = z + alpha * (X.numpy() @ S.numpy())
        for R in (r1, r2):
            if R is not None:
                z = np.linalg.solve(R.numpy().T, z.T).T
        if Zout is not None:
            Zout.copy_(torch.from_numpy(z))
        if gram is not None:
            kind = gram[0]
            if kind == "basis":
                out = gram[2]
                out.copy_(torch.from_numpy(gram[1].numpy().T @ z))
            elif kind == "self":
                out = gram[1]
                out.copy_(torch.from_numpy(z.T @ z))
            else:
                out = gram[1]
                out.copy_(torch.from_numpy((z * z).sum(axis=0)))
            if comm is not None:
                comm.allreduce_(out)

    return tall


def oracle_local_spmm(plan, Z, out, rb, re, Xg):
    """DistCsr local product on the host with the reference arithmetic."""
    Xext = Z.numpy()
    if Xg is not None and plan.n_ghost:
        Xext = np.vstack([Xext, Xg.numpy()])
    rp = plan.row_ptr.astype(np.int64)
    sub_rp = rp[rb:re + 1] - rp[rb]
    ci = plan.col_idx[rp[rb]:rp[re]]
    v = plan.values[rp[rb]:rp[re]]
    Y = oracle.spmm(sub_rp, ci, v, Xext, nthreads=1)
    out[rb:re].copy_(torch.from_numpy(Y))
