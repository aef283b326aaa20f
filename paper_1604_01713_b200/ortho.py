"""Block orthogonalisation schedules on the device (K4 of the hot path).

``project_chain`` performs the sequential classical Gram-Schmidt projections
the reference writes as numpy products,

    for B in bases:  coef = B^T z;  z -= B @ coef        (arnoldi.py:172-180,
                                                         solver.py:154-155)

but schedules them as fused rg_tall passes: pass i applies the updates that
are still pending and computes the Gram of the next basis in the same sweep,
so every basis is streamed once per dependency level.  An intermediate z is
written back only when that is cheaper than carrying its pending updates
into the next pass (or when more than two updates would be pending).  The
arithmetic per element is the reference's: products formed first, then
subtracted, updates applied in the reference's order.
"""

from __future__ import annotations

import torch

from . import device as _dev


def project_chain(zin: torch.Tensor, zbuf: torch.Tensor, bases, coefs, tail_gram=None, tall=None):
    """z = zin projected sequentially against ``bases``; the final z lands in
    ``zbuf`` (which may alias zin); coefs[i] (device, a_i x p, column-major)
    receives B_i^T z_{i}.  ``tail_gram`` (e.g. ("self", G)) is fused into the
    final pass.  ``tall`` defaults to the rg_tall wrapper (tests substitute a
    host restatement to exercise the schedule without a GPU).  Returns the
    number of passes launched."""
    tall = _dev.tall if tall is None else tall
    p = zin.shape[1]
    pending = []  # (B, coef) updates not yet folded into the stored z
    cur = zin
    nb = len(bases)
    launches = 0
    for i, B in enumerate(bases):
        if B.shape[1] == 0:
            coefs[i].zero_()
            continue
        nxt = [bases[i + 1]] if i + 1 < nb else []
        next_reads = {B.data_ptr()} | {b.data_ptr() for b in nxt}
        carry_cols = sum(b.shape[1] for b, _ in pending if b.data_ptr() not in next_reads)
        store = len(pending) + 1 > 2 or carry_cols > p
        terms = [(b, c, -1.0) for b, c in pending]
        if store:
            tall(cur, zbuf, terms, gram=("basis", B, coefs[i]))
            cur = zbuf
            pending = []
        else:
            tall(cur, None, terms, gram=("basis", B, coefs[i]))
        pending.append((B, coefs[i]))
        launches += 1
    terms = [(b, c, -1.0) for b, c in pending]
    if terms or tail_gram is not None or cur.data_ptr() != zbuf.data_ptr():
        tall(cur, zbuf, terms, gram=tail_gram)
        launches += 1
    return launches
