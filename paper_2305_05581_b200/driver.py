"""Closed-loop two-site DMRG on the device — drop-in for the reference's
driver.py (``SweepSchedule``, ``warmup``, ``run_sweeps``, ``solve``) and
the block updates of dmrg.py / blocks.py.

Every iteration (driver.py:131 ``_iterate``): the operator table at the
partition (native ``model.factorize``, cached per position like
``DmrgState.table_at``), the complementary operators of both blocks
(blocks.py:331 ``materialize_aux`` — ``blockops.composites`` on the device
stores), the H_eff·ψ plan on the persistent engine (``DevicePlan`` from the
device arenas), device Lanczos (dmrg.py:43), the renormalization of the
grown block (dmrg.py:335: ψ-slab ρ, cuSOLVER eigh per sector, the
reference's global top-D selection, enlargement + W^T O W fused on the
engine) and White's prediction of the next ψ (driver.py:200/:228), all with
the operators resident in HBM.  Nothing of the reference's per-block numpy
work is on this path; host work is task/work-list construction and the
top-D selection over eigenvalues.

The ``Engine`` hooks (plan factory, Lanczos, grouped-GEMM runner) default to
the sm_100a library; tests may substitute checkers, the product never does.
"""

import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import blockops as bo
from .blockops import Basis, ClassArena, DeviceStore, Fused, KronTerm
from .model import KEY_H, KEY_I, OperatorTable, compact, decode, factorize
from .plan_input import PlanInput


class DmrgError(Exception):
    pass


# ----------------------------------------------------------------- schedule

@dataclass
class SweepSchedule:
    """driver.py:31 SweepSchedule."""

    n_sweeps: int
    d: object = 64
    lanczos_tol: float = 1e-12
    lanczos_max_iter: int = 300
    # "lanczos": the reference's eigensolver (dmrg.py:43), iteration for
    # iteration; "davidson": diagonal-preconditioned Davidson on the device
    # (lanczos.davidson_ground) — same acceptance test, fewer H_eff·ψ
    eigensolver: str = "lanczos"

    def __post_init__(self):
        if self.n_sweeps < 0:
            raise DmrgError("sweep count must be non-negative")
        if self.lanczos_tol <= 0 or self.lanczos_max_iter < 1:
            raise DmrgError("tolerances must be positive")
        if self.eigensolver not in ("lanczos", "davidson"):
            raise DmrgError(f"unknown eigensolver {self.eigensolver!r}")
        ds = self.d if isinstance(self.d, (list, tuple)) else [self.d]
        if any(int(x) < 1 for x in ds):
            raise DmrgError("bond dimension must be >= 1")

    def d_for(self, sweep_index):
        if isinstance(self.d, (list, tuple)):
            i = min(max(sweep_index - 1, 0), len(self.d) - 1)
            return int(self.d[i])
        return int(self.d)


@dataclass
class SweepRecord:
    """driver.py:55 SweepRecord (+ the device time breakdown)."""

    sweep: int
    position: int
    direction: str
    energy: float
    truncation_error: float
    lanczos_iterations: int
    wall_seconds: float
    flops: int
    converged: bool = True
    timing: dict = field(default_factory=dict)

    CSV_HEADER = "sweep,position,direction,energy,truncation_error," \
                 "lanczos_iterations,wall_seconds,flops,converged"

    def csv_line(self):
        return (f"{self.sweep},{self.position},{self.direction},"
                f"{self.energy:.17g},{self.truncation_error:.17g},"
                f"{self.lanczos_iterations},{self.wall_seconds:.17g},"
                f"{self.flops},{int(self.converged)}")


class Engine:
    """Device hooks: plan factory, eigensolver, device."""

    def __init__(self, device=None):
        self.device = torch.device(device or "cuda")
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())

    def plan(self, pi, arena_l, arena_r):
        from .plan import DevicePlan
        return DevicePlan(pi, device=self.device, arena_l=arena_l, arena_r=arena_r)

    def lanczos(self, apply_op, guess, tol, max_iter):
        from .lanczos import lanczos_ground
        return lanczos_ground(apply_op, guess, tol=tol, max_iter=max_iter)

    def davidson(self, apply_op, guess, diag, tol, max_iter):
        from .lanczos import davidson_ground
        return davidson_ground(apply_op, guess, diag, tol=tol, max_iter=max_iter)

    def eigh(self, mat):
        return torch.linalg.eigh(mat)


# --------------------------------------------------------------- ψ structure

class PsiStruct:
    """blocks.py:408 SuperblockWavefunction layout: keys (qL,q1,q2,qR)
    fusing to the target, sorted; blocks dim(qL) x dim(qR), concatenated."""

    def __init__(self, left_basis, site_qns, right_basis, target):
        self.left_basis, self.right_basis = left_basis, right_basis
        self.site_qns = [tuple(q) for q in site_qns]
        self.target = tuple(target)
        keys = []
        for ql in left_basis.qns:
            for q1 in self.site_qns:
                for q2 in self.site_qns:
                    rest = tuple(t - x - y - z for t, x, y, z in zip(self.target, ql, q1, q2))
                    if rest in right_basis.index:
                        keys.append((ql, q1, q2, rest))
        keys.sort()
        self.keys = keys
        self.index = {k: i for i, k in enumerate(keys)}
        self.shapes = [(left_basis.dim(k[0]), right_basis.dim(k[3])) for k in keys]
        sizes = [a * b for a, b in self.shapes]
        self.offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.size = int(self.offsets[-1])

    def same_bases(self, other):
        return (other is not None and self.left_basis == other.left_basis
                and self.right_basis == other.right_basis and self.target == other.target)

    def blocks(self, vec):
        return {k: vec[self.offsets[i]:self.offsets[i + 1]].view(*self.shapes[i])
                for i, k in enumerate(self.keys)}


@dataclass
class PsiState:
    struct: PsiStruct
    vec: torch.Tensor


# -------------------------------------------------------------- block stores

def mode_range(model, store):
    mps = model.local.modes_per_site
    return store.sites[0] * mps, store.sites[1] * mps


def required_keys(model, lo, hi):
    """blocks.py:135 _required_keys with their QN shifts."""
    zero = model.local.zero_qn()
    keys = [(KEY_I, zero), (KEY_H, zero)]
    for m in range(lo, hi):
        keys.append((("C", (m, 1)), model.factor_delta(((m, 1),))))
        keys.append((("C", (m, 0)), model.factor_delta(((m, 0),))))
    for c1, c2 in model.pair_codes.tolist():
        f = decode([c1, c2])
        if all(lo <= x[0] < hi for x in f):
            keys.append((("P",) + f, model.factor_delta(f)))
    return keys


def empty_store(model, side, site_index, device):
    """blocks.py:147 empty_store: width-zero block (I = [[1]], H = [[0]])."""
    basis = Basis([(model.local.zero_qn(), 1)])
    zero = model.local.zero_qn()
    ops = ClassArena(basis, [(KEY_I, zero), (KEY_H, zero)], device)
    bo._write_identity(ops, KEY_I)
    return DeviceStore(side, (site_index, site_index), ops)


def _site_terms_dense(model, site_index, lo, hi, codes_mask=None):
    """Σ coef · string_matrix over the terms whose modes all lie in [lo, hi)."""
    local = model.local
    m0, _ = model.site_mode_range(site_index)
    codes = model.codes
    valid = codes >= 0
    modes = np.where(valid, codes >> 1, lo)
    inside = np.all((modes >= lo) & (modes < hi), axis=1)
    h = np.zeros((local.dim, local.dim))
    for t in np.nonzero(inside)[0].tolist():
        h += model.coef[t] * local.string_matrix(decode(codes[t]), m0)
    return h


def site_store(model, site_index, side, device):
    """blocks.py:156 site_store: exact width-one block, exactified (dmrg.py:364)."""
    local = model.local
    m0, m1 = model.site_mode_range(site_index)
    basis = Basis(local.basis_entries)
    keys = required_keys(model, m0, m1)
    ops = ClassArena(basis, keys, device)
    host = np.zeros(ops.size)
    qidx = {q: i for i, q in enumerate(local.state_qns)}
    for key, _delta in keys:
        if key == KEY_I:
            dense = np.eye(local.dim)
        elif key == KEY_H:
            dense = _site_terms_dense(model, site_index, m0, m1)
        else:
            dense = local.string_matrix(key[1:], m0)
        cl, r = ops.ops[key]
        for j, jr, o in zip(cl.col, cl.row, cl.off):
            # basis sector order == local.state_qns order (QN-sorted, 1-dim)
            host[cl.base + r * cl.size + o] = dense[qidx[basis.qns[jr]], qidx[basis.qns[j]]]
    ops.arena.copy_(torch.from_numpy(host))
    store = DeviceStore(side, (site_index, site_index + 1), ops)
    store.transform = bo.identity_w(basis, device)          # exactify_store
    return store


def _identity_map(ns):
    return (np.arange(ns, dtype=np.int64), np.ones(ns))


def enlarge_spec(model, store, site_index, comp_device):
    """The enlarged operators of blocks.py:190 enlarge_block as Kronecker
    terms (nothing is materialised): returns (fused layout, new keys,
    kron terms, composite definitions for the Hamiltonian cross sums)."""
    local = model.local
    left = store.side == "L"
    if left and site_index != store.sites[1]:
        raise DmrgError("left block must grow onto the next site")
    if not left and site_index != store.sites[0] - 1:
        raise DmrgError("right block must grow onto the previous site")
    m0, m1 = model.site_mode_range(site_index)
    blk_lo, blk_hi = mode_range(model, store)
    new_lo, new_hi = (blk_lo, m1) if left else (m0, blk_hi)
    site_basis = Basis(local.basis_entries)
    fused = Fused(store.basis, site_basis) if left else Fused(site_basis, store.basis)
    keys = required_keys(model, new_lo, new_hi)
    ns = local.dim
    eye = _identity_map(ns)

    def smap(factors, dress=False):
        return bo.site_map(local, local.string_matrix(factors, m0), dress)

    terms = []
    for key, _d in keys:
        if key == KEY_I:
            continue
        if key == KEY_H:
            continue
        if key[0] == "C":
            (m, dag), = key[1:]
            if m0 <= m < m1:
                # left: parity of the block dragged by the later site factor
                terms.append(KronTerm(key, ("op", KEY_I), smap(((m, dag),)), 1.0, left))
            else:
                terms.append(KronTerm(key, ("op", key), eye))
        else:
            f1, f2 = key[1], key[2]
            on1, on2 = m0 <= f1[0] < m1, m0 <= f2[0] < m1
            if on1 and on2:
                terms.append(KronTerm(key, ("op", KEY_I), smap((f1, f2))))
            elif not on1 and not on2:
                terms.append(KronTerm(key, ("op", key), eye))
            elif left:      # (c_f1 P_blk) x c_f2
                terms.append(KronTerm(key, ("op", ("C", f1)), smap((f2,)), 1.0, True))
            else:           # (c_f1 P_site) x c_f2
                terms.append(KronTerm(key, ("op", ("C", f2)), smap((f1,), dress=True)))
    # the enlarged Hamiltonian (blocks.py:262): H_old x 1, cross sums, site terms
    h_terms = [KronTerm(KEY_H, ("op", KEY_H), eye)]
    codes = model.codes
    valid = codes >= 0
    modes = np.where(valid, codes >> 1, -1)
    in_new = np.all(~valid | ((modes >= new_lo) & (modes < new_hi)), axis=1)
    on_site = valid & (modes >= m0) & (modes < m1)
    in_old = valid & (modes >= blk_lo) & (modes < blk_hi)
    n_site = on_site.sum(axis=1)
    n_old = in_old.sum(axis=1)
    cross = np.nonzero(in_new & (n_site > 0) & (n_old > 0))[0]
    defs_keys, aux, coef, inside = [], [], [], []
    kidx = {}
    for t in cross.tolist():
        row = codes[t]
        s_codes = tuple(int(c) for c, f in zip(row, on_site[t]) if f)
        o_codes = [int(c) for c, f in zip(row, in_old[t]) if f]
        dress = (len(s_codes) % 2 == 1) if left else (len(o_codes) % 2 == 1)
        if not model.fermionic:
            dress = False
        gk = ("HX", s_codes, dress)
        if gk not in kidx:
            kidx[gk] = len(defs_keys)
            defs_keys.append((gk, model.factor_delta(decode(o_codes))))
        aux.append(kidx[gk])
        coef.append(model.coef[t])
        inside.append((o_codes + [-1, -1, -1])[:3])
    comp_defs = {"keys": defs_keys, "aux": np.array(aux, np.int64),
                 "coef": np.array(coef, float), "inside": np.array(inside, np.int64).reshape(-1, 3)}
    for gk, _delta in defs_keys:
        _, s_codes, dress = gk
        sf = decode(s_codes)
        if left:
            h_terms.append(KronTerm(KEY_H, ("comp", gk), smap(sf), 1.0, dress))
        else:
            h_terms.append(KronTerm(KEY_H, ("comp", gk), smap(sf, dress=dress)))
    site_h = _site_terms_dense(model, site_index, m0, m1)
    if np.any(site_h):
        h_terms.append(KronTerm(KEY_H, ("op", KEY_I), bo.site_map(local, site_h)))
    return fused, keys, h_terms + terms, comp_defs


def _grow(model, store, site_index, w, new_basis, fused, keys, terms, comp_defs, device,
          only=None):
    comp = bo.composites(store, comp_defs, model, device) if comp_defs["keys"] else None
    if only is not None:
        keys = [(k, d) for k, d in keys if k in only]
        terms = [t for t in terms if t.key in only]
    ops = bo.enlarge_rotate(store, comp, model.local, terms, keys, fused, w, new_basis, device)
    left = store.side == "L"
    sites = (store.sites[0], site_index + 1) if left else (site_index, store.sites[1])
    return DeviceStore(store.side, sites, ops, fused=fused)


TIE_RTOL = 1e-11


def select_states(sector_scores, d_max, info=None):
    """dmrg.py:204 _select_states: global top-D, ties broken by (score, qn
    lexicographic, intra-sector index) — on the raw floats, exactly as the
    reference orders them.

    The Hamiltonians are spin-summed, so ±Sz sectors share spectra: members
    of an exactly degenerate multiplet are then ordered by rounding noise
    (the reference's LAPACK noise there, cuSOLVER's here).  ``info`` (dict)
    receives ``tie_at_cut``: whether the D-th state splits a class of scores
    equal within TIE_RTOL of the largest — the only case where the kept set
    can legitimately differ from the reference's."""
    ranked = []
    for q in sorted(sector_scores):
        for idx, s in enumerate(np.asarray(sector_scores[q]).tolist()):
            ranked.append((-s, q, idx))
    ranked.sort()
    if info is not None:
        scale = max((abs(r[0]) for r in ranked), default=0.0)
        tol = TIE_RTOL * max(scale, 1e-300)
        info["tie_at_cut"] = bool(0 < d_max < len(ranked)
                                  and ranked[d_max][0] - ranked[d_max - 1][0] <= tol)
    kept = {}
    for _negs, q, idx in ranked[:d_max]:
        kept.setdefault(q, []).append(idx)
    return kept


def spectral_truncate(model, store, site_index, d_max, engine):
    """Warm-up growth (driver.py:297 enlarge_block + dmrg.py:369
    spectral_truncate): exact when the enlarged basis fits D, else keep the
    D lowest eigenstates of the enlarged block Hamiltonian."""
    dev = engine.device
    fused, keys, terms, comp_defs = enlarge_spec(model, store, site_index, dev)
    fb = fused.basis
    if fb.total_dim <= d_max:                                  # exactify_store
        w = bo.identity_w(fb, dev)
        new = _grow(model, store, site_index, w, fb, fused, keys, terms, comp_defs, dev)
        new.transform = w
        return new
    # the enlarged H on the fused basis (identity W), its sector spectra
    hs = _grow(model, store, site_index, bo.identity_w(fb, dev), fb, fused, keys, terms,
               comp_defs, dev, only={KEY_H})
    hb = hs.ops.blocks(KEY_H)
    scores, vecs = {}, {}
    for q, d in fb.entries:
        mat = hb.get((q, q))
        if mat is None:
            mat = torch.zeros((d, d), dtype=torch.float64, device=dev)
        evals, evecs = engine.eigh(mat)
        scores[q] = -evals.cpu().numpy()          # lowest energy first
        vecs[q] = evecs
    del hs
    info = {}
    kept = select_states(scores, d_max, info)
    w = {q: vecs[q][:, torch.as_tensor(idx, device=dev)].contiguous() for q, idx in kept.items()}
    nb = Basis([(q, len(idx)) for q, idx in kept.items()])
    new = _grow(model, store, site_index, w, nb, fused, keys, terms, comp_defs, dev)
    new.transform = w
    new.tie_at_cut = info["tie_at_cut"]
    return new


def density_matrix(psi, side, fused, device):
    """ρ of the enlarged block per fused sector (dmrg.py:221 rdm_eigensystem)
    without forming the slabs: ρ_qe[a, b] = Σ_spectators B_a B_b^T (side L,
    a/b the (ql, q1) combinations of qe) or Σ B_a^T B_b (side R, a/b the
    (q2, qr) combinations) — one grouped engine launch, one problem per
    sub-block, the spectator sectors its segments (in ψ key order)."""
    ps = psi.struct
    groups = {}          # qe -> {spectator: [(fused offset, rows, block index)]}
    for i, (ql, q1, q2, qr) in enumerate(ps.keys):
        if side == "L":
            qe, comb, spec = qn_add(ql, q1), (ql, q1), (q2, qr)
        else:
            qe, comb, spec = qn_add(q2, qr), (q2, qr), (ql, q1)
        groups.setdefault(qe, {}).setdefault(spec, []).append((fused.layout[comb], i))
    fdims = {q: d for q, d in fused.basis.entries}
    sectors = sorted(groups)
    roff, pos = {}, 0
    for q in sectors:
        roff[q] = pos
        pos += fdims[q] ** 2
    rbuf = torch.zeros(max(pos, 1), dtype=torch.float64, device=device)
    ln = bo.Launch(0, 1) if side == "L" else bo.Launch(1, 0)
    for qe in sectors:
        dq = fdims[qe]
        pairs = {}
        for spec, members in groups[qe].items():
            for oa, ia in members:
                for ob, ib in members:
                    pairs.setdefault((oa, ob), []).append((ia, ib))
        for (oa, ob), segs in sorted(pairs.items()):
            ia0, ib0 = segs[0]
            if side == "L":
                m, n = ps.shapes[ia0][0], ps.shapes[ib0][0]
                ks = [ps.shapes[a][1] for a, _ in segs]
                lda = ks
                ldb = ks
            else:
                m, n = ps.shapes[ia0][1], ps.shapes[ib0][1]
                ks = [ps.shapes[a][0] for a, _ in segs]
                lda = [m] * len(segs)
                ldb = [n] * len(segs)
            ln.add(bo.handle(0, roff[qe] + oa * dq + ob), dq, m, n, 0, len(segs),
                   bo.handle(1, [ps.offsets[a] for a, _ in segs]), lda,
                   bo.handle(1, [ps.offsets[b] for _, b in segs]), ldb, ks, np.ones(len(segs)))
    ln.run([rbuf, psi.vec])
    return {q: rbuf[roff[q]:roff[q] + fdims[q] ** 2].view(fdims[q], fdims[q]) for q in sectors}


def _sector_eigh(mats, engine):
    """Eigenpairs of every ρ sector, descending, with ONE device-to-host
    transfer of all eigenvalues (per-sector eigh calls: a batched call per
    sector size ran slower — torch's batched path, r2ac: renormalization
    164 vs 90 s per L=30 D=1024 sweep)."""
    vals, vecs = {}, {}
    for q, mat in mats.items():
        ev, vc = engine.eigh(mat)
        vals[q], vecs[q] = ev.flip(0), vc.flip(1)
    order = list(mats)
    flat = torch.cat([vals[q] for q in order]).cpu().numpy() if order else np.zeros(0)
    scores, pos = {}, 0
    for q in order:
        n = int(vals[q].shape[0])
        scores[q] = flat[pos:pos + n]
        pos += n
    return scores, vecs


def renormalize(model, psi, side, old_store, site_index, d_max, engine):
    """dmrg.py:335 renormalize: enlarge, ρ eigensystem (dmrg.py:221), top-D
    (dmrg.py:204), W^T O W of every maintained operator (dmrg.py:254)."""
    dev = engine.device
    fused, keys, terms, comp_defs = enlarge_spec(model, old_store, site_index, dev)
    rho = density_matrix(psi, side, fused, dev)
    scores, vecs = _sector_eigh(rho, engine)
    info = {}
    kept = select_states(scores, d_max, info)
    total = sum(float(np.sum(v)) for v in scores.values())
    kept_weight = sum(float(np.sum(scores[q][idx])) for q, idx in kept.items())
    trunc = min(1.0, max(0.0, 1.0 - kept_weight / max(total, 1e-300)))
    w = {q: vecs[q][:, torch.as_tensor(idx, device=dev)].contiguous() for q, idx in kept.items()}
    nb = Basis([(q, len(idx)) for q, idx in kept.items()])
    new = _grow(model, old_store, site_index, w, nb, fused, keys, terms, comp_defs, dev)
    new.transform = w
    new.tie_at_cut = info["tie_at_cut"]
    return new, trunc


# --------------------------------------------------------------- prediction

def _w_pack(w, device):
    qs = sorted(w)
    off, pos = {}, 0
    for q in qs:
        off[q] = pos
        pos += w[q].numel()
    buf = torch.empty(max(pos, 1), dtype=torch.float64, device=device)
    for q in qs:
        buf[off[q]:off[q] + w[q].numel()] = w[q].reshape(-1)
    return buf, off


def predict_right(psi, new_left, old_right, struct, device):
    """driver.py:200 _predict_right on the engine: part = W_l^T ψ, then
    σ(qe, q2, q2n, qrn) += part · W_r[rows of (q2n, qrn)]^T."""
    wl, fl = new_left.transform, new_left.fused
    wr, fr = old_right.transform, old_right.fused
    if wl is None or fl is None or wr is None or fr is None:
        return None
    out = torch.zeros(struct.size, dtype=torch.float64, device=device)
    lbuf, loff = _w_pack(wl, device)
    rbuf, roff = _w_pack(wr, device)
    ps = psi.struct
    parts, ppos = [], 0
    l1 = bo.Launch(1, 0)
    for i, (ql, q1, q2, qr) in enumerate(ps.keys):
        qe = qn_add(ql, q1)
        if qe not in wl or qr not in wr:
            continue
        rows, cols = ps.shapes[i]
        ke = int(wl[qe].shape[1])
        off = fl.layout[(ql, q1)]
        l1.add(bo.handle(2, ppos), cols, ke, cols, 0, 1,
               bo.handle(0, loff[qe] + off * ke), ke, bo.handle(1, ps.offsets[i]), cols, rows, 1.0)
        parts.append((i, qe, q2, qr, ppos, ke, cols))
        ppos += ke * cols
    pbuf = torch.empty(max(ppos, 1), dtype=torch.float64, device=device)
    l1.run([lbuf, psi.vec, pbuf])
    probs = {}
    for i, qe, q2, qr, pp, ke, cols in parts:
        for (q2n, qrn), off2 in fr.layout.items():
            if qn_add(q2n, qrn) != qr:
                continue
            key = (qe, q2, q2n, qrn)
            o = struct.index.get(key)
            if o is None:
                continue
            d_r = fr.basis_b.dim(qrn)
            kr = int(wr[qr].shape[1])
            probs.setdefault(o, []).append((pp, cols, roff[qr] + off2 * kr, kr, ke, d_r))
    l2 = bo.Launch(0, 1)
    for o, segs in sorted(probs.items()):
        ke, d_r = segs[0][4], segs[0][5]
        l2.add(bo.handle(0, struct.offsets[o]), d_r, ke, d_r, 0, len(segs),
               bo.handle(1, [s[0] for s in segs]), [s[1] for s in segs],
               bo.handle(2, [s[2] for s in segs]), [s[3] for s in segs],
               [s[1] for s in segs], np.ones(len(segs)))
    l2.run([out, pbuf, rbuf])
    return _normalized_or_none(out)


def predict_left(psi, new_right, old_left, struct, device):
    """driver.py:228 _predict_left on the engine: proj = ψ · W_r, then
    σ(qln, q1n, q1, qf) += W_l[rows of (qln, q1n)] · proj."""
    wr, fr = new_right.transform, new_right.fused
    wl, fl = old_left.transform, old_left.fused
    if wr is None or fr is None or wl is None or fl is None:
        return None
    out = torch.zeros(struct.size, dtype=torch.float64, device=device)
    rbuf, roff = _w_pack(wr, device)
    lbuf, loff = _w_pack(wl, device)
    ps = psi.struct
    parts, ppos = [], 0
    l1 = bo.Launch(0, 0)
    for i, (ql, q1, q2, qr) in enumerate(ps.keys):
        qf = qn_add(q2, qr)
        if qf not in wr or ql not in wl:
            continue
        rows, cols = ps.shapes[i]
        kf = int(wr[qf].shape[1])
        off = fr.layout[(q2, qr)]
        l1.add(bo.handle(2, ppos), kf, rows, kf, 0, 1,
               bo.handle(1, ps.offsets[i]), cols, bo.handle(0, roff[qf] + off * kf), kf, cols, 1.0)
        parts.append((i, ql, q1, qf, ppos, rows, kf))
        ppos += rows * kf
    pbuf = torch.empty(max(ppos, 1), dtype=torch.float64, device=device)
    l1.run([rbuf, psi.vec, pbuf])
    probs = {}
    for i, ql, q1, qf, pp, rows, kf in parts:
        kl = int(wl[ql].shape[1])
        for (qln, q1n), off2 in fl.layout.items():
            if qn_add(qln, q1n) != ql:
                continue
            key = (qln, q1n, q1, qf)
            o = struct.index.get(key)
            if o is None:
                continue
            d_l = fl.basis_a.dim(qln)
            probs.setdefault(o, []).append((loff[ql] + off2 * kl, kl, pp, kf, rows, d_l))
    l2 = bo.Launch(0, 0)
    for o, segs in sorted(probs.items()):
        kf, d_l = segs[0][3], segs[0][5]
        l2.add(bo.handle(0, struct.offsets[o]), kf, d_l, kf, 0, len(segs),
               bo.handle(1, [s[0] for s in segs]), [s[1] for s in segs],
               bo.handle(2, [s[2] for s in segs]), [s[3] for s in segs],
               [s[4] for s in segs], np.ones(len(segs)))
    l2.run([out, lbuf, pbuf])
    return _normalized_or_none(out)


def qn_add(a, b):
    return tuple(x + y for x, y in zip(a, b))


def _normalized_or_none(vec):
    n = float(torch.linalg.vector_norm(vec).item())
    if n < 1e-12:
        return None
    return vec / n


# -------------------------------------------------------------------- plan

def plan_input(model, table, comp_tab, left, right, comp_l, comp_r, target, device):
    """PlanInput of one partition from the device stores (the drop-in of
    blocks.py:503 build_plan's operator resolution): each referenced
    operator is one contiguous slice of its class arena; the plan arena of a
    side is their concatenation with per-(op, column sector) offsets."""
    local = model.local
    sides = {}
    for side, store, comp, keys in (("l", left, comp_l, comp_tab["keys_l"]),
                                    ("r", right, comp_r, comp_tab["keys_r"])):
        basis = store.basis
        slices, offs, deltas, kinds = [], [], [], []
        pos = 0
        for key in keys:
            if key[0] == "AUX":
                src, k2 = comp, key
            else:
                src, k2 = store.ops, key
            if src is None or not src.has(k2):
                raise DmrgError(f"operator {key} not available on block {store.sites}")
            cl, r = src.ops[k2]
            base = cl.base + r * cl.size
            slices.append(src.arena[base:base + cl.size])
            row = np.full(len(basis), -1, np.int64)
            row[cl.col] = pos + cl.off
            offs.append(row)
            deltas.append(cl.delta)
            kinds.append(1 if key == KEY_I else 0)
            pos += cl.size
        arena = torch.cat(slices) if slices else torch.zeros(1, dtype=torch.float64,
                                                             device=device)
        sides[side] = (arena, np.stack(offs) if offs else np.zeros((0, len(basis)), np.int64),
                       np.array(deltas, np.int32).reshape(-1, local.qn_ncomp),
                       np.array(kinds, np.int32))
    lb, rb = left.basis, right.basis
    pi = PlanInput(
        site_qn=np.array(local.state_qns, np.int32), target=np.array(target, np.int32),
        qn_l=np.array(lb.qns, np.int32), dim_l=lb.dims.astype(np.int32),
        left_sign=np.array([local.parity_sign(q) for q in lb.qns]),
        qn_r=np.array(rb.qns, np.int32), dim_r=rb.dims.astype(np.int32),
        delta_l=sides["l"][2], blk_off_l=sides["l"][1], kind_l=sides["l"][3],
        delta_r=sides["r"][2], blk_off_r=sides["r"][1], kind_r=sides["r"][3],
        lop=comp_tab["lop"], rop=comp_tab["rop"], alpha=comp_tab["alpha"], e_l=comp_tab["e_l"],
        site1_dst=comp_tab["site1_dst"], site1_val=comp_tab["site1_val"],
        site2_dst=comp_tab["site2_dst"], site2_val=comp_tab["site2_val"],
        row_map=np.arange(len(comp_tab["lop"]), dtype=np.int64))
    pi.normalized()
    return pi, sides["l"][0], sides["r"][0]


_AUX_DEFS = {}


def aux_defs(model, aux):
    """AuxDefs of one side as composite definitions keyed like the table's
    ("AUX", side, factors) operator keys (memoized per AuxDefs object: the
    tables are cached per position, so one defs object serves every visit
    and carries its term preprocessing, blockops._defs_prep)."""
    hit = _AUX_DEFS.get(id(aux))
    if hit is not None and hit[0] is aux:
        return hit[1]
    keys = []
    for a in range(len(aux.keys)):
        first = np.nonzero(aux.aux == a)[0][0]
        keys.append((("AUX", aux.side, aux.key_tuple(a)),
                     model.factor_delta(decode(aux.inside[first]))))
    defs = {"keys": keys, "aux": aux.aux.astype(np.int64), "coef": aux.coef,
            "inside": aux.inside.astype(np.int64)}
    if len(_AUX_DEFS) > 256:
        _AUX_DEFS.clear()
    _AUX_DEFS[id(aux)] = (aux, defs)
    return defs


# ------------------------------------------------------------------ driver

def _store_tensors(store):
    ts = [store.ops.arena]
    if store.transform:
        ts += list(store.transform.values())
    return ts


def store_bytes(store):
    return sum(t.numel() * t.element_size() for t in _store_tensors(store))


def _move_store(store, device):
    store.ops.arena = store.ops.arena.to(device)
    if store.transform:
        store.transform = {k: v.to(device) for k, v in store.transform.items()}


class StoreDict(dict):
    """Block stores of one side by site count, resident in HBM up to a byte
    budget (default 35% of the device's memory): the least recently used
    stores beyond it wait in host memory and come back on access.  A sweep
    touches one store per side and step, so at L=30 D=2048 (2.5 GB per
    store, 2 x 28 of them) only the stores around the sweep position stay on
    the device."""

    def __init__(self, device=None, budget=None):
        super().__init__()
        self.device = device
        if budget is None and os.environ.get("SDMRG_STORE_BUDGET"):
            budget = int(float(os.environ["SDMRG_STORE_BUDGET"]))
        if budget is None and device is not None and device.type == "cuda":
            budget = int(0.35 * torch.cuda.get_device_properties(device).total_memory)
        self.budget = budget
        self.order = []          # keys, least recently used first
        self.offloads = 0

    def _touch(self, key):
        if key in self.order:
            self.order.remove(key)
        self.order.append(key)

    def _trim(self):
        if self.budget is None:
            return
        resident = [k for k in self.order
                    if dict.__getitem__(self, k).ops.arena.device.type == "cuda"]
        total = sum(store_bytes(dict.__getitem__(self, k)) for k in resident)
        for k in resident[:-2]:            # the two most recent always stay
            if total <= self.budget:
                break
            st = dict.__getitem__(self, k)
            total -= store_bytes(st)
            _move_store(st, "cpu")
            self.offloads += 1

    def __getitem__(self, key):
        st = dict.__getitem__(self, key)
        if self.device is not None and st.ops.arena.device != self.device:
            _move_store(st, self.device)
        self._touch(key)
        self._trim()
        return st

    def __setitem__(self, key, st):
        dict.__setitem__(self, key, st)
        self._touch(key)
        self._trim()


@dataclass
class DmrgState:
    """driver.py:78 DmrgState with device stores."""

    model: object
    target: tuple
    seed: int
    rng: object
    engine: object
    left: dict = field(default_factory=StoreDict)
    right: dict = field(default_factory=StoreDict)
    psi: object = None
    position: int = 0
    sweeps_done: int = 0
    records: list = field(default_factory=list)
    tables: dict = field(default_factory=dict)
    warmup_ties: int = 0       # spectral truncations that split a degenerate multiplet

    def table_at(self, position):
        if position not in self.tables:
            tab = factorize(self.model, position)
            self.tables[position] = (tab, compact(self.model, tab))
        return self.tables[position]


def sweep_positions(model):
    n = model.n_sites
    if n >= 4:
        return 1, n - 3
    return 0, n - 2


def _psi_struct(state, position):
    model = state.model
    n = model.n_sites
    left = state.left[position]
    right = state.right[n - position - 2]
    struct = PsiStruct(left.basis, model.local.state_qns, right.basis, state.target)
    if not struct.keys:
        raise DmrgError(f"target sector {state.target} unreachable at position {position}")
    return struct, left, right


def _psi_struct_safe(state, position):
    try:
        return _psi_struct(state, position)
    except (KeyError, DmrgError):
        return None, None, None


def _guess_vector(state, struct):
    """driver.py:118 _guess_vector: the predicted ψ when its bases match,
    else a seeded normal vector (same generator draws as the reference)."""
    psi = state.psi
    dev = state.engine.device
    if psi is not None and struct.same_bases(psi.struct):
        n = float(torch.linalg.vector_norm(psi.vec).item())
        if n > 0:
            return psi.vec / n
    host = state.rng.standard_normal(struct.size)
    return torch.from_numpy(host).to(dev)


def _sync(dev):
    if dev.type == "cuda":
        torch.cuda.synchronize(dev)


def _iterate(state, position, d_max, schedule, sweep_index, direction):
    model = state.model
    eng = state.engine
    dev = eng.device
    t0 = time.perf_counter()
    tim = {}
    struct, left, right = _psi_struct(state, position)
    table, ctab = state.table_at(position)
    t1 = time.perf_counter()
    tim["table_s"] = t1 - t0
    comp_l = bo.composites(left, aux_defs(model, table.left_aux), model, dev) \
        if len(table.left_aux.keys) else None
    comp_r = bo.composites(right, aux_defs(model, table.right_aux), model, dev) \
        if len(table.right_aux.keys) else None
    pi, al, ar = plan_input(model, table, ctab, left, right, comp_l, comp_r, state.target, dev)
    pi.arena_l, pi.arena_r = None, None
    _sync(dev)
    t2 = time.perf_counter()
    tim["aux_s"] = t2 - t1
    if dev.type == "cuda":
        # the plan sizes its T workspace from the driver's free HBM: hand
        # torch's cached-but-unused blocks back when they are a large share
        # (L=30 D=2048 ran out of memory with 55 GB held in torch's cache);
        # releasing them every step made the next step's allocations slow
        idle = torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
        if idle > 0.15 * torch.cuda.get_device_properties(dev).total_memory:
            torch.cuda.empty_cache()
    plan = eng.plan(pi, al, ar)
    del al, ar, comp_l, comp_r
    if plan.psi_size != struct.size:
        raise DmrgError("plan ψ layout disagrees with the superblock structure")
    _sync(dev)
    t3 = time.perf_counter()
    tim["plan_s"] = t3 - t2
    buf = torch.empty(struct.size, dtype=torch.float64, device=dev)

    def apply_op(vec):
        return plan.apply(vec, buf)

    if schedule.eigensolver == "davidson":
        res = eng.davidson(apply_op, _guess_vector(state, struct), plan.diagonal(),
                           schedule.lanczos_tol, schedule.lanczos_max_iter)
    else:
        res = eng.lanczos(apply_op, _guess_vector(state, struct), schedule.lanczos_tol,
                          schedule.lanczos_max_iter)
    flops = int(plan.flops) * (res.iterations + 1)
    plan.close()
    del plan, buf
    psi = PsiState(struct, res.vector.contiguous())
    state.psi = psi
    state.position = position
    _sync(dev)
    t4 = time.perf_counter()
    tim["lanczos_s"] = t4 - t3

    lo, hi = sweep_positions(model)
    n = model.n_sites
    if direction == "R":
        new, trunc = renormalize(model, psi, "L", left, position, d_max, eng)
        state.left[position + 1] = new
        _sync(dev)
        t5 = time.perf_counter()
        if position < hi:
            nxt, _l, _r = _psi_struct_safe(state, position + 1)
            if nxt is not None:
                vec = predict_right(psi, new, right, nxt, dev)
                state.psi = PsiState(nxt, vec) if vec is not None else psi
    else:
        new, trunc = renormalize(model, psi, "R", right, position + 1, d_max, eng)
        state.right[n - position - 1] = new
        _sync(dev)
        t5 = time.perf_counter()
        if position > lo:
            nxt, _l, _r = _psi_struct_safe(state, position - 1)
            if nxt is not None:
                vec = predict_left(psi, new, left, nxt, dev)
                state.psi = PsiState(nxt, vec) if vec is not None else psi
    _sync(dev)
    t6 = time.perf_counter()
    tim["renorm_s"] = t5 - t4
    tim["predict_s"] = t6 - t5
    tim["tie_at_cut"] = bool(getattr(new, "tie_at_cut", False))
    rec = SweepRecord(sweep_index, position, direction, float(res.energy), float(trunc),
                      int(res.iterations), t6 - t0, flops, bool(res.converged), tim)
    state.records.append(rec)
    return rec


def warmup(model, schedule, target=None, seed=42, engine=None):
    """driver.py:262 warmup: exact growth truncated spectrally to the first
    bond dimension, then the bootstrap half-pass from the middle."""
    engine = engine or Engine()
    dev = engine.device
    target = tuple(target) if target is not None else model.default_target()
    state = DmrgState(model, target, seed, np.random.default_rng(seed), engine,
                      left=StoreDict(dev), right=StoreDict(dev))
    d = schedule.d_for(1)
    lo, hi = sweep_positions(model)
    n = model.n_sites
    m0 = min(max((n - 2) // 2, lo), hi)
    state.left[0] = empty_store(model, "L", 0, dev)
    state.right[0] = empty_store(model, "R", n, dev)
    state.left[1] = site_store(model, 0, "L", dev)
    state.right[1] = site_store(model, n - 1, "R", dev)
    for w in range(2, m0 + 1):
        state.left[w] = spectral_truncate(model, state.left[w - 1], w - 1, d, engine)
        state.warmup_ties += int(getattr(state.left[w], "tie_at_cut", False))
    for w in range(2, n - m0 - 1):
        state.right[w] = spectral_truncate(model, state.right[w - 1], n - w, d, engine)
        state.warmup_ties += int(getattr(state.right[w], "tie_at_cut", False))
    for p in range(m0, lo - 1, -1):
        _iterate(state, p, d, schedule, 0, "W")
    return state


def run_sweeps(state, schedule, start_sweep=None):
    """driver.py:307 run_sweeps: full left-to-right then right-to-left passes."""
    lo, hi = sweep_positions(state.model)
    first = state.sweeps_done + 1 if start_sweep is None else start_sweep
    new_records = []
    for s in range(first, schedule.n_sweeps + 1):
        d = schedule.d_for(s)
        for p in range(lo, hi + 1):
            new_records.append(_iterate(state, p, d, schedule, s, "R"))
        for p in range(hi, lo - 1, -1):
            new_records.append(_iterate(state, p, d, schedule, s, "L"))
        state.sweeps_done = s
    return new_records


sweep = run_sweeps


@dataclass
class SolveResult:
    energy: float
    records: list
    state: DmrgState

    def sweep_final_energies(self):
        out = {}
        for r in self.records:
            if r.sweep > 0:
                out[r.sweep] = r.energy
        return [out[k] for k in sorted(out)]


def solve(model, schedule, target=None, seed=42, engine=None):
    """driver.py:356 solve: warm-up plus the scheduled sweeps."""
    state = warmup(model, schedule, target=target, seed=seed, engine=engine)
    run_sweeps(state, schedule)
    energy = state.records[-1].energy if state.records else float("nan")
    return SolveResult(energy, list(state.records), state)
