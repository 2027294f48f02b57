"""Oracle: renormalization pieces — TEST INFRASTRUCTURE ONLY.

Restates dmrg.py:204-251 (global top-D selection, reduced density matrix per
sector) and the per-block rotation of dmrg.py:298-312 (W^T O W, no sum over
positions), on plain dicts:

  psi blocks   {(ql, q1, q2, qr): (dl x dr) array}
  layout       {(qa, qb): row offset inside fused sector qa+qb}  (FusedBasis)
  fused dims   {q: dim}
  op blocks    {(rq, cq): array};  W blocks {q: (dim(q) x kept(q)) array}
"""

import numpy as np


def select_states(sector_scores, d_max):
    """dmrg.py:204-218: ties break by (score, qn lexicographic, index)."""
    ranked = []
    for q in sorted(sector_scores):
        for idx, s in enumerate(sector_scores[q]):
            ranked.append((-s, q, idx))
    ranked.sort()
    kept = {}
    for _negs, q, idx in ranked[:d_max]:
        kept.setdefault(q, []).append(idx)
    return kept


def rdm_slabs(psi_blocks, side, layout, fused_dims):
    """dmrg.py:226-242: gather ψ blocks into per-(sector, spectator) slabs."""
    slabs = {}
    if side == "L":
        for (ql, q1, q2, qr), blk in psi_blocks.items():
            qe = tuple(a + b for a, b in zip(ql, q1))
            off = layout[(ql, q1)]
            key = (qe, q2, qr)
            if key not in slabs:
                slabs[key] = np.zeros((fused_dims[qe], blk.shape[1]))
            slabs[key][off:off + blk.shape[0], :] = blk
    else:
        for (ql, q1, q2, qr), blk in psi_blocks.items():
            qf = tuple(a + b for a, b in zip(q2, qr))
            off = layout[(q2, qr)]
            key = (qf, ql, q1)
            if key not in slabs:
                slabs[key] = np.zeros((fused_dims[qf], blk.shape[0]))
            slabs[key][off:off + blk.shape[1], :] = blk.T
    return slabs


def rdm_blocks(slabs):
    """dmrg.py:243-246: rho[qe] = sum over spectators of slab @ slab.T."""
    rho = {}
    for (qe, _a, _b), slab in slabs.items():
        acc = rho.get(qe)
        rho[qe] = slab @ slab.T if acc is None else acc + slab @ slab.T
    return rho


def rdm_eigensystem(rho):
    """dmrg.py:247-251: descending eigenpairs per sector."""
    out = {}
    for qe, mat in rho.items():
        evals, evecs = np.linalg.eigh(mat)
        out[qe] = (evals[::-1].copy(), evecs[:, ::-1].copy())
    return out


def truncate(eig, d_max):
    """dmrg.py:342-352: kept states, truncation error, W blocks."""
    scores = {q: vals for q, (vals, _) in eig.items()}
    kept = select_states(scores, d_max)
    total = sum(float(np.sum(v)) for v in scores.values())
    kept_weight = sum(float(np.sum(scores[q][idx])) for q, idx in kept.items())
    trunc = min(1.0, max(0.0, 1.0 - kept_weight / max(total, 1e-300)))
    w = {q: eig[q][1][:, idx] for q, idx in kept.items()}
    return kept, trunc, w


def rotate_op(op_blocks, w):
    """dmrg.py:303-312: every block (rq, cq) -> W[rq]^T @ blk @ W[cq]."""
    res = {}
    for (rq, cq), blk in op_blocks.items():
        wl = w.get(rq)
        wr = w.get(cq)
        if wl is None or wr is None:
            continue
        tmp = wl.T @ blk
        res[(rq, cq)] = tmp @ wr
    return res
