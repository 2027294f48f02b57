"""Device renormalization — drop-in for dmrg.py:204-357 (the block update that
follows each two-site diagonalization).

Pipeline (all arithmetic on the GPU except the global top-D selection, a
sort of <= D eigenvalues that the reference also does on the host):

  1. slabs      ψ blocks gathered into per-(sector, spectator) slabs
                (dmrg.py:226-242) — one device gather;
  2. ρ          ρ_q = Σ_spectators S S^T on the grouped FP64 engine
                (sdmrg_rdm_accumulate: one problem per sector, one segment
                per slab, fixed order);
  3. eigh       per sector, descending (dmrg.py:247-251) — cuSOLVER through
                torch.linalg.eigh;
  4. selection  global top-D with the reference's tie-breaking
                (dmrg.py:204-218), truncation error (dmrg.py:345-347);
  5. rotation   W^T O W for every block of every maintained operator, no sum
                over positions (dmrg.py:254-320, paper §IV.D) — two grouped
                engine launches for all blocks of all operators
                (sdmrg_rotate).

Inputs use plain containers so the module is usable both from the
reference's objects (``renormalize_store`` takes a BlockStore-like object:
``.basis.entries``, ``.ops`` of SectorMatrix-like objects with ``.delta`` and
``.blocks``, ``.fused.layout``) and from fixtures.
"""

from typing import NamedTuple

import numpy as np
import torch

from . import _lib


class RenormError(Exception):
    pass


class Eigensystem(NamedTuple):
    values: dict     # q -> descending eigenvalues (host float64)
    vectors: dict    # q -> matching eigenvector columns (device, fused dim x dim)


class TruncationResult(NamedTuple):
    kept: dict           # q -> kept eigen-indices (reference order)
    truncation_error: float
    w: dict              # q -> W block (device, fused dim(q) x kept(q))
    n_kept: int


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _i64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64))


def _i32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


# ------------------------------------------------------------ density matrix

def reduced_density_matrix(psi_blocks, side, layout, fused_dims, device=None):
    """ρ of the enlarged block, per sector (dmrg.py:221-246).

    ``psi_blocks``: {(ql, q1, q2, qr): (dl x dr) block} (numpy or CUDA
    tensors); ``layout``: {(qa, qb): row offset inside fused sector qa+qb}
    (FusedBasis.layout); ``fused_dims``: {q: dim}.  Returns {q: CUDA tensor}.
    """
    device = torch.device(device or "cuda")
    slabs = {}           # (qe, spectator...) -> [(offset, block key)]
    for key in sorted(psi_blocks):
        ql, q1, q2, qr = key
        if side == "L":
            qe = tuple(a + b for a, b in zip(ql, q1))
            off = layout[(ql, q1)]
            skey = (qe, q2, qr)
        elif side == "R":
            qe = tuple(a + b for a, b in zip(q2, qr))
            off = layout[(q2, qr)]
            skey = (qe, ql, q1)
        else:
            raise RenormError(f"side must be 'L' or 'R', got {side!r}")
        slabs.setdefault(skey, []).append((off, key))
    # slab buffer: each slab fused_dim(qe) x spectator dim, row-major, zeroed
    order = sorted(slabs)
    s_off, rho_q, rows, cols = [], [], [], []
    pos = 0
    for skey in order:
        qe = skey[0]
        first = psi_blocks[slabs[skey][0][1]]
        spec = first.shape[1] if side == "L" else first.shape[0]
        s_off.append(pos)
        rows.append(fused_dims[qe])
        cols.append(spec)
        rho_q.append(qe)
        pos += fused_dims[qe] * spec
    sbuf = torch.zeros(max(pos, 1), dtype=torch.float64, device=device)
    for skey, base, nrow, ncol in zip(order, s_off, rows, cols):
        slab = sbuf[base:base + nrow * ncol].view(nrow, ncol)
        for off, key in slabs[skey]:
            blk = psi_blocks[key]
            blk = blk if isinstance(blk, torch.Tensor) else torch.from_numpy(np.asarray(blk))
            blk = blk.to(device=device, dtype=torch.float64)
            if side == "L":
                slab[off:off + blk.shape[0], :] = blk
            else:
                slab[off:off + blk.shape[1], :] = blk.T
    # ρ sectors in sorted order, one contiguous buffer
    sectors = sorted(set(rho_q))
    r_off, rpos = {}, 0
    for q in sectors:
        r_off[q] = rpos
        rpos += fused_dims[q] ** 2
    rbuf = torch.zeros(max(rpos, 1), dtype=torch.float64, device=device)
    n = len(order)
    if n:
        _lib.check(_lib.load().sdmrg_rdm_accumulate(
            n, _lib.as_p(_i64(s_off), _lib.ctypes.c_int64),
            _lib.as_p(_i64([r_off[q] for q in rho_q]), _lib.ctypes.c_int64),
            _lib.as_p(_i32(rows), _lib.ctypes.c_int32), _lib.as_p(_i32(cols), _lib.ctypes.c_int32),
            sbuf.data_ptr(), rbuf.data_ptr(), _stream()))
    return {q: rbuf[r_off[q]:r_off[q] + fused_dims[q] ** 2].view(fused_dims[q], fused_dims[q])
            for q in sectors}


def rdm_eigensystem(rho):
    """Descending eigenpairs per sector (dmrg.py:247-251)."""
    values, vectors = {}, {}
    for q, mat in rho.items():
        evals, evecs = torch.linalg.eigh(mat)
        values[q] = evals.flip(0).cpu().numpy()
        vectors[q] = evecs.flip(1).contiguous()
    return Eigensystem(values, vectors)


def select_states(sector_scores, d_max):
    """Global top-D, ties by (score, qn lexicographic, index) — dmrg.py:204."""
    ranked = []
    for q in sorted(sector_scores):
        for idx, s in enumerate(np.asarray(sector_scores[q]).tolist()):
            ranked.append((-s, q, idx))
    ranked.sort()
    kept = {}
    for _negs, q, idx in ranked[:d_max]:
        kept.setdefault(q, []).append(idx)
    return kept


def truncate(eig, d_max):
    """Kept states, truncation error and W blocks (dmrg.py:342-352)."""
    scores = eig.values
    kept = select_states(scores, d_max)
    total = sum(float(np.sum(v)) for v in scores.values())
    kept_weight = sum(float(np.sum(scores[q][idx])) for q, idx in kept.items())
    trunc = min(1.0, max(0.0, 1.0 - kept_weight / max(total, 1e-300)))
    w = {}
    for q, idx in kept.items():
        sel = torch.as_tensor(idx, dtype=torch.int64, device=eig.vectors[q].device)
        w[q] = eig.vectors[q].index_select(1, sel).contiguous()
    return TruncationResult(kept, trunc, w, sum(len(v) for v in kept.values()))


# ----------------------------------------------------------------- rotation

def rotate_operators(ops, w, workspace_doubles=None):
    """W^T O W for every block of every operator (dmrg.py:298-312).

    ``ops``: {key: {(rq, cq): block}} (numpy or CUDA); ``w``: {q: CUDA W}.
    Blocks whose row or column sector was truncated away are dropped, like
    the reference.  Returns {key: {(rq, cq): CUDA tensor}} from ONE pair of
    grouped engine launches over all blocks of all operators.
    """
    device = next(iter(w.values())).device if w else torch.device("cuda")
    wq = sorted(w)
    w_off, pos = {}, 0
    for q in wq:
        w_off[q] = pos
        pos += w[q].numel()
    wbuf = torch.empty(max(pos, 1), dtype=torch.float64, device=device)
    for q in wq:
        wbuf[w_off[q]:w_off[q] + w[q].numel()] = w[q].reshape(-1)
    tasks = []       # (key, (rq, cq), block)
    for key in sorted(ops, key=repr):
        for (rq, cq), blk in sorted(ops[key].items()):
            if rq in w and cq in w:
                tasks.append((key, (rq, cq), blk))
    obuf_parts, o_off, d_off = [], [], []
    opos = dpos = 0
    wl, wr, rows, cols, kl, kr = [], [], [], [], [], []
    tmp_need = 0
    for key, (rq, cq), blk in tasks:
        b = blk if isinstance(blk, torch.Tensor) else torch.from_numpy(np.asarray(blk))
        b = b.to(device=device, dtype=torch.float64).contiguous()
        obuf_parts.append(b.reshape(-1))
        o_off.append(opos)
        opos += b.numel()
        r, c = b.shape
        a, z = w[rq].shape[1], w[cq].shape[1]
        wl.append(w_off[rq])
        wr.append(w_off[cq])
        rows.append(r)
        cols.append(c)
        kl.append(a)
        kr.append(z)
        d_off.append(dpos)
        dpos += a * z
        tmp_need = max(tmp_need, a * c)
    out = {key: {} for key in ops}
    if not tasks:
        return out
    obuf = torch.cat(obuf_parts)
    dbuf = torch.empty(max(dpos, 1), dtype=torch.float64, device=device)
    ws = int(workspace_doubles or sum(a * c for a, c in zip(kl, cols)))
    ws = max(ws, tmp_need)
    wsp = torch.empty(max(ws, 1), dtype=torch.float64, device=device)
    P = _lib.as_p
    _lib.check(_lib.load().sdmrg_rotate(
        len(tasks), P(_i64(wl), _lib.ctypes.c_int64), P(_i64(wr), _lib.ctypes.c_int64),
        P(_i64(o_off), _lib.ctypes.c_int64), P(_i64(d_off), _lib.ctypes.c_int64),
        P(_i32(rows), _lib.ctypes.c_int32), P(_i32(cols), _lib.ctypes.c_int32),
        P(_i32(kl), _lib.ctypes.c_int32), P(_i32(kr), _lib.ctypes.c_int32),
        wbuf.data_ptr(), obuf.data_ptr(), dbuf.data_ptr(), wsp.data_ptr(), ws, _stream()))
    for (key, bkey, _blk), off, a, z in zip(tasks, d_off, kl, kr):
        out[key][bkey] = dbuf[off:off + a * z].view(a, z)
    return out


# ------------------------------------------------------------- whole update

class RenormResult(NamedTuple):
    ops: dict                 # key -> {(rq, cq): CUDA block} in the new basis
    basis: list               # [(q, kept dim)] sorted — the new SectorBasis entries
    w: dict                   # q -> W block
    truncation_error: float
    kept: int


def renormalize_blocks(psi_blocks, side, layout, fused_dims, ops, d_max):
    """ρ -> eigh -> top-D -> W^T O W on plain containers (dmrg.py:335-357
    after the enlargement)."""
    rho = reduced_density_matrix(psi_blocks, side, layout, fused_dims)
    eig = rdm_eigensystem(rho)
    tr = truncate(eig, d_max)
    new_ops = rotate_operators(ops, tr.w)
    basis = [(q, len(idx)) for q, idx in sorted(tr.kept.items())]
    return RenormResult(new_ops, basis, tr.w, tr.truncation_error, tr.n_kept)


def renormalize_store(enlarged, psi, side, d_max):
    """Drop-in for the arithmetic of dmrg.py:335 renormalize on the
    reference's objects: ``enlarged`` is the enlarged BlockStore
    (blocks.py:190 enlarge_block output — the caller keeps building it), ``psi``
    the SuperblockWavefunction.  Returns a RenormResult whose ``ops`` maps
    every maintained operator key to its rotated blocks (CUDA tensors); the
    identity is rebuilt by the caller as in dmrg.py:318."""
    fused = enlarged.fused
    fused_dims = {q: d for q, d in fused.basis.entries}
    ops = {key: dict(mat.blocks) for key, mat in enlarged.ops.items() if key != ("I",)}
    return renormalize_blocks(psi.blocks, side, fused.layout, fused_dims, ops, d_max)
