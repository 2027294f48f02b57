"""Oracle: task generation + H_eff·ψ on the compact plan form (numpy).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates
  * blocks.py:503-579  build_plan   — row x ψ-key matching, scale folding,
    grouping by (ψ key, out key), members in table-row order;
  * dmrg.py:107-176    apply_plan   — per group: stage L/R stacks (R scaled,
    dmrg.py:136-140), then sbmm4s's two kernels (sbmm4s.py:127-157).
"""

import numpy as np

from .sbmm4s import batched_gemm_interleaved, concat_gemm_accumulate


def psi_layout(pi):
    """(keys, offsets) of the ψ vector — blocks.py:416-429 and :448."""
    keys = pi.psi_keys()
    return keys, pi.psi_offsets(keys)


def build_groups(pi):
    """Reference grouping restated on the compact form (blocks.py:521-567).

    Returns a list of (psi index, out index, [(row, scale), ...]) in sorted
    (ψ key, out key) order; members in row order.
    """
    keys, _ = psi_layout(pi)
    index = {k[:3]: i for i, k in enumerate(keys)}
    qn_l = [tuple(q) for q in pi.qn_l.tolist()]
    qn_r = [tuple(q) for q in pi.qn_r.tolist()]
    lidx = {q: j for j, q in enumerate(qn_l)}
    ridx = {q: j for j, q in enumerate(qn_r)}

    def shifted(idx, qns, j, delta):
        return idx.get(tuple(a + b for a, b in zip(qns[j], delta)), -1)

    groups = {}
    for t in range(pi.nrows):                                   # blocks.py:521
        lo, ro = int(pi.lop[t]), int(pi.rop[t])
        dl, dr = pi.delta_l[lo].tolist(), pi.delta_r[ro].tolist()
        for i, (jl, s1, s2, jr) in enumerate(keys):               # blocks.py:535
            d1 = int(pi.site1_dst[t, s1])
            d2 = int(pi.site2_dst[t, s2])
            if d1 < 0 or d2 < 0:                                  # blocks.py:539
                continue
            jlp = shifted(lidx, qn_l, jl, dl)                     # blocks.py:543
            if jlp < 0 or pi.blk_off_l[lo, jl] < 0:
                continue
            jrp = shifted(ridx, qn_r, jr, dr)                     # blocks.py:547
            if jrp < 0 or pi.blk_off_r[ro, jr] < 0:
                continue
            o = index.get((jlp, d1, d2), -1)                      # blocks.py:551
            if o < 0 or keys[o][3] != jrp:
                continue
            scale = float(pi.alpha[t]) * float(pi.site1_val[t, s1]) * float(pi.site2_val[t, s2])
            if pi.e_l[t]:                                         # blocks.py:555
                scale *= float(pi.left_sign[jl])
            if scale == 0.0:                                      # blocks.py:561
                continue
            groups.setdefault((i, o), []).append((t, scale))
    return [(i, o, groups[(i, o)]) for (i, o) in sorted(groups)]


def _block(arena, off, rows, cols):
    return arena[off:off + rows * cols].reshape(rows, cols)


def _group_product(pi, keys, offs, grp, psi):
    """One group's SBMM4S contribution (q x r) — dmrg.py:120-163 body."""
    i, o, members = grp
    jl, _s1, _s2, jr = keys[i]
    m, n = int(pi.dim_l[jl]), int(pi.dim_r[jr])
    ojl, ojr = keys[o][0], keys[o][3]
    q, r = int(pi.dim_l[ojl]), int(pi.dim_r[ojr])
    a = psi[offs[i]:offs[i] + m * n].reshape(m, n)
    b = np.zeros((q, r))
    p = len(members)
    l_stack = np.empty((q, m, p), order="F")                      # dmrg.py:130
    r_stack = np.empty((r, n, p), order="F")                      # dmrg.py:136
    for k, (t, s) in enumerate(members):
        lo, ro = int(pi.lop[t]), int(pi.rop[t])
        l_stack[:, :, k] = _block(pi.arena_l, int(pi.blk_off_l[lo, jl]), q, m)
        np.multiply(_block(pi.arena_r, int(pi.blk_off_r[ro, jr]), r, n), s,
                    out=r_stack[:, :, k])
    ws = np.zeros(m * p * r)
    temp = batched_gemm_interleaved(a, r_stack, ws)               # dmrg.py:152
    concat_gemm_accumulate(l_stack, temp, 1.0, b)                 # dmrg.py:156
    return b


def apply_groups(pi, groups, psi, out=None):
    """out += H_eff psi, group by group, sbmm4s two-step (dmrg.py:120-163)."""
    keys, offs = psi_layout(pi)
    out = np.zeros_like(psi) if out is None else out
    for grp in groups:
        o = grp[1]
        out[offs[o]:offs[o + 1]] += _group_product(pi, keys, offs, grp, psi).ravel()
    return out


def apply_groups_threaded(pi, groups, psi, out=None, workers=None):
    """dmrg.py:107 apply_plan with a worker pool: the reference's maze-runner
    runs one task per group on ``pool.workers`` threads and locks the output
    block (dmrg.py:158-163).  Same per-group SBMM4S; BLAS single-threaded per
    call, groups spread over ``workers`` host threads (numpy releases the GIL
    inside the products).  Accumulation order per output block follows
    completion order, as in the reference's pool."""
    import os
    import threading
    from concurrent.futures import ThreadPoolExecutor
    keys, offs = psi_layout(pi)
    out = np.zeros_like(psi) if out is None else out
    workers = workers or os.cpu_count()
    locks = {grp[1]: threading.Lock() for grp in groups}

    def run(grp):
        o = grp[1]
        b = _group_product(pi, keys, offs, grp, psi).ravel()
        with locks[o]:
            out[offs[o]:offs[o + 1]] += b

    try:
        from threadpoolctl import threadpool_limits
        ctx = threadpool_limits(limits=1)
    except ImportError:  # pragma: no cover - threadpoolctl ships in the image
        ctx = None
    try:
        with ThreadPoolExecutor(max_workers=workers) as ex:
            list(ex.map(run, groups))
    finally:
        if ctx is not None:
            ctx.restore_original_limits()
    return out


def apply_heff(pi, psi, groups=None):
    """H_eff psi from scratch (zeroed output), the Lanczos apply_op."""
    groups = build_groups(pi) if groups is None else groups
    return apply_groups(pi, groups, psi)


def ref_flops(pi, groups):
    """plan.flops — sbmm4s.py:205 flops_fused summed over groups (blocks.py:571)."""
    keys, _ = psi_layout(pi)
    total = 0
    for i, o, members in groups:
        m, n = int(pi.dim_l[keys[i][0]]), int(pi.dim_r[keys[i][3]])
        q, r = int(pi.dim_l[keys[o][0]]), int(pi.dim_r[keys[o][3]])
        p = len(members)
        total += 2 * m * r * n * p + 2 * q * r * m * p
    return total


def build_groups_fast(pi, key_subset=None):
    """``build_groups`` vectorised over table rows (same grouping, same member
    order, same folded scales, blocks.py:521-567): one numpy pass per ψ key.
    ``key_subset``: iterable of ψ key indices to generate groups for (None =
    all).  Used by the bench's CPU arm and the bench-scale parity tests, which
    must not touch the product library."""
    keys, _ = psi_layout(pi)
    nk = len(keys)
    nl, nr = len(pi.dim_l), len(pi.dim_r)
    ns = pi.nsite
    qn_l = [tuple(q) for q in pi.qn_l.tolist()]
    qn_r = [tuple(q) for q in pi.qn_r.tolist()]
    lidx = {q: j for j, q in enumerate(qn_l)}
    ridx = {q: j for j, q in enumerate(qn_r)}

    def shift_table(deltas, qns, idx):
        tab = np.full((len(deltas), len(qns)), -1, np.int64)
        for o, d in enumerate(deltas.tolist()):
            for j, q in enumerate(qns):
                tab[o, j] = idx.get(tuple(a + b for a, b in zip(q, d)), -1)
        return tab

    lsh = shift_table(pi.delta_l, qn_l, lidx)
    rsh = shift_table(pi.delta_r, qn_r, ridx)
    key3 = np.full((nl, ns, ns), -1, np.int64)
    keyr = np.array([k[3] for k in keys], np.int64)
    for i, (jl, s1, s2, _jr) in enumerate(keys):
        key3[jl, s1, s2] = i
    lop = pi.lop.astype(np.int64)
    rop = pi.rop.astype(np.int64)
    alpha = pi.alpha
    e_l = pi.e_l != 0
    out = []
    subset = range(nk) if key_subset is None else sorted(int(i) for i in key_subset)
    for i in subset:
        jl, s1, s2, jr = keys[i]
        d1 = pi.site1_dst[:, s1].astype(np.int64)
        d2 = pi.site2_dst[:, s2].astype(np.int64)
        jlp = lsh[lop, jl]
        jrp = rsh[rop, jr]
        ok = (d1 >= 0) & (d2 >= 0) & (jlp >= 0) & (pi.blk_off_l[lop, jl] >= 0) \
            & (jrp >= 0) & (pi.blk_off_r[rop, jr] >= 0)
        o = np.full(len(lop), -1, np.int64)
        o[ok] = key3[jlp[ok], d1[ok], d2[ok]]
        ok &= o >= 0
        ok[ok] &= keyr[o[ok]] == jrp[ok]
        scale = alpha * pi.site1_val[:, s1] * pi.site2_val[:, s2]
        scale = np.where(e_l, scale * pi.left_sign[jl], scale)
        ok &= scale != 0.0
        rows = np.nonzero(ok)[0]
        if rows.size == 0:
            continue
        oo = o[rows]
        order = np.argsort(oo, kind="stable")
        rows, oo = rows[order], oo[order]
        cuts = np.nonzero(np.diff(oo))[0] + 1
        for seg_rows, seg_o in zip(np.split(rows, cuts), np.split(oo, cuts)):
            out.append((i, int(seg_o[0]),
                        list(zip(seg_rows.tolist(), scale[seg_rows].tolist()))))
    return out
