"""Synthetic two-site partitions at bench scale (CAS(L, L), U(1) x U(1)).

The operator table is the reference's own factorization of an L-orbital
random-integral Hamiltonian at the middle partition (committed fixture, see
tools/make_table_fixture.py).  What is synthetic is the renormalized block
data: each block's D states are spread over (N, 2Sz) sectors with Gaussian
weights calibrated on reference DMRG runs (a CAS(8,8) D=128 run's middle
block: sigma_N ~ 1.6, sigma_S ~ 1.5 for 4 orbitals; widths scaled with the
block's orbital count) and capped by the sector's true Fock-space dimension,
and every operator block allowed by the selection rule is filled with seeded
normal deviates (identities stay identities).  Data: synthetic.
"""

import math
import os

import numpy as np

from .plan_input import PlanInput

DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")


def load_table(n_orb):
    path = os.path.join(DATA, f"table_L{n_orb}.npz")
    if not os.path.exists(path):
        raise FileNotFoundError(f"no operator-table fixture for L={n_orb}: {path}")
    return dict(np.load(path))


def sector_dims(norb, d, n_mean=None, sig_n=None, sig_s=None):
    """(N, 2Sz) -> dim for a block of ``norb`` spatial orbitals, total <= d."""
    n_mean = norb if n_mean is None else n_mean
    sig_n = 0.14 * norb if sig_n is None else sig_n
    sig_s = 0.13 * norb if sig_s is None else sig_s
    ents = []
    for n in range(0, 2 * norb + 1):
        for nup in range(0, norb + 1):
            ndn = n - nup
            if not 0 <= ndn <= norb:
                continue
            sz = nup - ndn
            true = math.comb(norb, nup) * math.comb(norb, ndn)
            w = math.exp(-((n - n_mean) ** 2) / (2 * sig_n ** 2) - sz ** 2 / (2 * sig_s ** 2))
            ents.append(((n, sz), w, true))
    tot = sum(w for _, w, _ in ents)
    dims = {}
    for q, w, true in ents:
        k = min(true, int(round(d * w / tot)))
        if k >= 1:
            dims[q] = k
    return dict(sorted(dims.items()))


def synthetic_plan_input(n_orb=30, d=2048, seed=0, n_elec=None, sig_scale=1.0):
    """PlanInput (without arenas) for the middle partition of CAS(n_orb, n_orb)."""
    tab = load_table(n_orb)
    nl, nr = int(tab["n_left_orb"]), int(tab["n_right_orb"])
    target = tab["target"].astype(np.int32)
    if n_elec is not None:
        target = np.array([n_elec, n_elec % 2], np.int32)
    tot_n = int(target[0])
    # expected electrons on each block: proportional to its orbital count
    nbar_l = tot_n * nl / n_orb
    nbar_r = tot_n * nr / n_orb
    left = sector_dims(nl, d, nbar_l, 0.14 * nl * sig_scale, 0.13 * nl * sig_scale)
    right = sector_dims(nr, d, nbar_r, 0.14 * nr * sig_scale, 0.13 * nr * sig_scale)
    qn_l = np.array(list(left), np.int32)
    dim_l = np.array(list(left.values()), np.int32)
    qn_r = np.array(list(right), np.int32)
    dim_r = np.array(list(right.values()), np.int32)

    def offsets(deltas, kinds, qn, dim):
        index = {tuple(q): j for j, q in enumerate(qn.tolist())}
        offs = np.full((len(deltas), len(dim)), -1, np.int64)
        pos = 0
        for o, dq in enumerate(deltas.tolist()):
            for j, q in enumerate(qn.tolist()):
                jr = index.get(tuple(a + b for a, b in zip(q, dq)))
                if jr is None:
                    continue
                offs[o, j] = pos
                pos += int(dim[jr]) * int(dim[j])
        return offs, pos

    ol, size_l = offsets(tab["delta_l"], tab["kind_l"], qn_l, dim_l)
    orr, size_r = offsets(tab["delta_r"], tab["kind_r"], qn_r, dim_r)
    pi = PlanInput(
        site_qn=tab["site_qn"], target=target, qn_l=qn_l, dim_l=dim_l,
        left_sign=np.array([(-1.0) ** (int(q[0]) % 2) for q in qn_l]),
        qn_r=qn_r, dim_r=dim_r,
        delta_l=tab["delta_l"], blk_off_l=ol, kind_l=(tab["kind_l"] == 1).astype(np.int32),
        delta_r=tab["delta_r"], blk_off_r=orr, kind_r=(tab["kind_r"] == 1).astype(np.int32),
        lop=tab["lop"], rop=tab["rop"], alpha=tab["alpha"], e_l=tab["e_l"],
        site1_dst=tab["site1_dst"], site1_val=tab["site1_val"],
        site2_dst=tab["site2_dst"], site2_val=tab["site2_val"],
        row_map=np.arange(len(tab["lop"]), dtype=np.int64))
    pi.meta.update(dict(arena_size_l=size_l, arena_size_r=size_r, n_orb=n_orb, d=d,
                        seed=seed, kind_l_tag=tab["kind_l"], kind_r_tag=tab["kind_r"]))
    return pi.normalized()


def fill_arenas_host(pi, seed=0):
    """Host arenas: seeded normal blocks, identity ops exact (oracle sizes)."""
    rng = np.random.default_rng(seed)
    out = []
    for side in ("l", "r"):
        size = pi.meta[f"arena_size_{side}"]
        arena = rng.standard_normal(max(size, 1)) / 8.0
        _identities(pi, side, arena)
        out.append(arena)
    pi.arena_l, pi.arena_r = out
    return pi


def fill_arenas_device(pi, seed=0, device="cuda"):
    """Device arenas generated in place (bench scale: GBs, no host staging)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = []
    for side in ("l", "r"):
        size = pi.meta[f"arena_size_{side}"]
        arena = torch.randn(max(size, 1), generator=g, dtype=torch.float64, device=device)
        arena.mul_(0.125)
        _identities(pi, side, arena)
        out.append(arena)
    return out


def _identities(pi, side, arena):
    kind = pi.kind_l if side == "l" else pi.kind_r
    offs = pi.blk_off_l if side == "l" else pi.blk_off_r
    dim = pi.dim_l if side == "l" else pi.dim_r
    for o in np.nonzero(kind == 1)[0]:
        for j, off in enumerate(offs[o]):
            if off < 0:
                continue
            n = int(dim[j])
            if isinstance(arena, np.ndarray):
                blk = arena[off:off + n * n].reshape(n, n)
                blk[...] = 0.0
                blk[np.diag_indices(n)] = 1.0
            else:
                blk = arena[off:off + n * n].view(n, n)
                blk.zero_()
                blk.fill_diagonal_(1.0)


def fill_plan_arenas(plan, pi, seed=0):
    """Fill a plan built with ``empty_arenas=True`` in place: seeded normal
    blocks (scale 1/8), identity ops exact, pad columns zero.  The padded
    arenas are column-sector-major (sdmrg_plan_arena), so each column sector's
    blocks form one (rows x even stride) run filled by two tensor ops — no
    dense copy of the operators ever exists beside the padded one."""
    import torch
    g = torch.Generator(device=plan.device)
    g.manual_seed(seed)
    for side in ("l", "r"):
        view, offs = plan.padded_arena(side)
        dim = pi.dim_l if side == "l" else pi.dim_r
        kind = pi.kind_l if side == "l" else pi.kind_r
        for j in range(offs.shape[1]):
            col = offs[:, j]
            present = col >= 0
            if not present.any():
                continue
            ld = int(dim[j]) + (int(dim[j]) & 1)
            lo = int(col[present].min())
            # run end: last block's offset + its rows * ld
            hi_op = int(np.argmax(np.where(present, col, -1)))
            rows_last = _rows_of(pi, side, hi_op, j)
            hi = int(col[hi_op]) + rows_last * ld
            run = view[lo:hi].view(-1, ld)
            run.normal_(generator=g).mul_(0.125)
            if int(dim[j]) & 1:
                run[:, -1].zero_()
            for o in np.nonzero((kind == 1) & present)[0]:
                n = int(dim[j])
                blk = view[int(col[o]):int(col[o]) + n * ld].view(n, ld)
                blk.zero_()
                blk[:, :n].fill_diagonal_(1.0)
    torch.cuda.synchronize()
    plan.invalidate()  # operator pre-sums (if any) follow the new arenas


def _rows_of(pi, side, op, j):
    """Row count of block (op, column sector j): dim of sector j + delta(op)."""
    qn = pi.qn_l if side == "l" else pi.qn_r
    dim = pi.dim_l if side == "l" else pi.dim_r
    delta = (pi.delta_l if side == "l" else pi.delta_r)[op]
    target = tuple(int(a) + int(b) for a, b in zip(qn[j], delta))
    for k, q in enumerate(qn.tolist()):
        if tuple(q) == target:
            return int(dim[k])
    raise ValueError("block without a row sector")
