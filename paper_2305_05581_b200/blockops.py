"""Device block stores and the block algebra of a DMRG step.

The reference keeps every maintained operator of a block (identity, block
Hamiltonian, single-mode creators/annihilators, two-factor strings) as a
``SectorMatrix`` dict of numpy blocks (blocks.py:45 ``BlockStore``) and
grows, truncates and partially sums them with per-block numpy calls
(blocks.py:190 ``enlarge_block``, :262 ``_enlarged_hamiltonian``, :331
``materialize_aux``; dmrg.py:254 ``_transform_tree``, :335 ``renormalize``,
:376 ``spectral_truncate``; driver.py:200/:228 White's prediction).  Here:

* **Layout.**  A ``DeviceStore`` owns ONE fp64 device arena.  Operators are
  grouped into *delta classes* (all operators with the same quantum-number
  shift share one block structure over the store basis); a class is a
  row-major ``[n_ops, class_size]`` matrix whose row is one operator, its
  blocks (q + delta, q) row-major in column-sector order.  Every allowed
  block is stored (absent = zero), so an operator is one contiguous slice
  and a class is a dense operand of the tensor engine.

* **Partial sums** (complementary operators, the enlarged-Hamiltonian cross
  sums): Σ_t c_t · O_t over one- and two-factor strings is a coefficient
  matrix times the class matrix — one engine GEMM per class; three-factor
  strings (blocks.py:104 ``resolve`` = C_i · P_jk) are refactored as
  Σ_i C_i · (Σ_jk c · P_jk): a GEMM for the inner sums, then one grouped
  engine launch whose segments are the heads i.

* **Enlargement fused with truncation.**  The enlarged operators are never
  materialised: every new operator is a sum of Kronecker pieces s · X(q_r, q_c)
  placed at (row, column) offsets of the fused sectors (sectors.py:176
  FusedBasis layout), so its rotated block is
  Σ_pieces s · W_r[rows]^T · (X · W_c[cols]) — one grouped launch for the
  distinct X · W_c products and one whose segments sum the pieces.  With an
  identity W (un-truncated growth, exactify_store) the same two launches
  reproduce the enlarged operators exactly.

* **Prediction** and the ψ-slab reduced density matrix are grouped launches
  on the same engine; eigendecompositions are cuSOLVER (torch.linalg.eigh).

All device work goes through ``sdmrg_grouped_gemm`` (include/sdmrg_b200.h) —
the engine of the H_eff·ψ plan.  Host work is the per-step work-list
construction (numpy) and the global top-D selection over eigenvalues.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .model import KEY_H, KEY_I, decode

SHIFT = 60


# ------------------------------------------------------------------ bases

class Basis:
    """sectors.py:44 SectorBasis: sorted (qn, dim) entries."""

    def __init__(self, entries):
        ents = sorted((tuple(int(x) for x in q), int(d)) for q, d in entries)
        self.entries = tuple(ents)
        self.qns = [q for q, _ in ents]
        self.dims = np.array([d for _, d in ents], dtype=np.int64)
        self.index = {q: i for i, q in enumerate(self.qns)}
        self.offsets = np.concatenate([[0], np.cumsum(self.dims)]).astype(np.int64)
        self.total_dim = int(self.offsets[-1])

    def __eq__(self, other):
        return isinstance(other, Basis) and self.entries == other.entries

    def __hash__(self):
        return hash(self.entries)

    def __len__(self):
        return len(self.qns)

    def dim(self, q):
        return int(self.dims[self.index[tuple(q)]])


def qn_add(a, b):
    return tuple(x + y for x, y in zip(a, b))


class Fused:
    """sectors.py:176 FusedBasis: (qa, qb) -> row offset inside sector qa+qb;
    combinations in (basis_a, basis_b) order."""

    def __init__(self, basis_a, basis_b):
        self.basis_a, self.basis_b = basis_a, basis_b
        sizes, layout = {}, {}
        for qa, da in basis_a.entries:
            for qb, db in basis_b.entries:
                q = qn_add(qa, qb)
                layout[(qa, qb)] = sizes.get(q, 0)
                sizes[q] = sizes.get(q, 0) + da * db
        self.layout = layout
        self.basis = Basis(sizes.items())


class OpClass:
    """All operators of one store with one QN shift: a [n_ops, size] matrix."""

    def __init__(self, basis, delta):
        self.delta = tuple(delta)
        cols, rows, offs = [], [], []
        pos = 0
        for j, q in enumerate(basis.qns):
            jr = basis.index.get(qn_add(q, self.delta))
            if jr is None:
                continue
            cols.append(j)
            rows.append(jr)
            offs.append(pos)
            pos += int(basis.dims[jr]) * int(basis.dims[j])
        self.col = np.array(cols, np.int64)
        self.row = np.array(rows, np.int64)
        self.off = np.array(offs, np.int64)
        self.size = pos
        self.col_pos = {int(j): i for i, j in enumerate(cols)}   # column sector -> slot
        self.keys = []
        self.base = 0

    @property
    def nops(self):
        return len(self.keys)


class ClassArena:
    """Operators on one basis, grouped in delta classes, in one device arena."""

    def __init__(self, basis, key_deltas, device, zero=True):
        self.basis = basis
        self.classes = {}
        self.ops = {}
        for key, delta in key_deltas:
            cl = self.classes.get(tuple(delta))
            if cl is None:
                cl = self.classes[tuple(delta)] = OpClass(basis, delta)
            if key in self.ops:
                raise ValueError(f"duplicate operator {key}")
            self.ops[key] = (cl, len(cl.keys))
            cl.keys.append(key)
        pos = 0
        for cl in self.classes.values():
            cl.base = pos
            pos += cl.nops * cl.size
        self.size = pos
        alloc = torch.zeros if zero else torch.empty
        self.arena = alloc(max(pos, 1), dtype=torch.float64, device=device)

    def op_offset(self, key):
        cl, r = self.ops[key]
        return cl.base + r * cl.size

    def block_offsets(self, key):
        """{column sector j: element offset of block (j + delta, j)}."""
        cl, r = self.ops[key]
        base = cl.base + r * cl.size
        return {int(j): base + int(o) for j, o in zip(cl.col, cl.off)}

    def has(self, key):
        return key in self.ops

    def delta(self, key):
        return self.ops[key][0].delta

    def dense(self, key):
        """Dense host matrix of one operator (tests / small bases)."""
        cl, r = self.ops[key]
        b = self.basis
        out = np.zeros((b.total_dim, b.total_dim))
        data = self.arena[cl.base + r * cl.size: cl.base + (r + 1) * cl.size].cpu().numpy()
        for j, jr, o in zip(cl.col, cl.row, cl.off):
            dr, dc = int(b.dims[jr]), int(b.dims[j])
            out[b.offsets[jr]:b.offsets[jr] + dr, b.offsets[j]:b.offsets[j] + dc] = \
                data[o:o + dr * dc].reshape(dr, dc)
        return out

    def blocks(self, key):
        """{(row qn, col qn): device view} of one operator."""
        cl, r = self.ops[key]
        b = self.basis
        base = cl.base + r * cl.size
        out = {}
        for j, jr, o in zip(cl.col, cl.row, cl.off):
            dr, dc = int(b.dims[jr]), int(b.dims[j])
            out[(b.qns[jr], b.qns[j])] = self.arena[base + o: base + o + dr * dc].view(dr, dc)
        return out


@dataclass
class DeviceStore:
    """blocks.py:45 BlockStore on the device."""

    side: str                 # "L" grows rightward, "R" leftward
    sites: tuple              # (lo, hi) site range, hi exclusive
    ops: ClassArena
    fused: Fused = None       # fusion layout that built this basis
    transform: dict = None    # fused qn -> W (device, dimF x kept)

    @property
    def basis(self):
        return self.ops.basis

    @property
    def n_sites(self):
        return self.sites[1] - self.sites[0]


# --------------------------------------------------------- grouped launches

def handle(base, off):
    return (np.int64(base) << np.int64(SHIFT)) | np.asarray(off, dtype=np.int64)


class Launch:
    """Host staging of one sdmrg_grouped_gemm call (numpy chunks)."""

    def __init__(self, ta, tb):
        self.ta, self.tb = int(ta), int(tb)
        self.p = {k: [] for k in ("c", "ldc", "m", "n", "beta", "nseg")}
        self.s = {k: [] for k in ("a", "lda", "b", "ldb", "k", "scale")}

    def add(self, c, ldc, m, n, beta, nseg, a, lda, b, ldb, k, scale):
        for name, v in (("c", c), ("ldc", ldc), ("m", m), ("n", n), ("beta", beta),
                        ("nseg", nseg)):
            self.p[name].append(np.atleast_1d(np.asarray(v)))
        for name, v in (("a", a), ("lda", lda), ("b", b), ("ldb", ldb), ("k", k),
                        ("scale", scale)):
            self.s[name].append(np.atleast_1d(np.asarray(v)))

    def run(self, bases, stream=None):
        if not self.p["c"]:
            return
        P = {k: np.concatenate(v) for k, v in self.p.items()}
        S = {k: np.concatenate(v) for k, v in self.s.items()}
        i64 = lambda x: np.ascontiguousarray(x, dtype=np.int64)   # noqa: E731
        i32 = lambda x: np.ascontiguousarray(x, dtype=np.int32)   # noqa: E731
        nprob = len(P["c"])
        seg_begin = np.concatenate([[0], np.cumsum(P["nseg"])]).astype(np.int64)
        if seg_begin[-1] != len(S["a"]):
            raise ValueError("segment count mismatch")
        arrs = dict(c=i64(P["c"]), ldc=i32(P["ldc"]), m=i32(P["m"]), n=i32(P["n"]),
                    beta=i32(P["beta"]), sb=i64(seg_begin), a=i64(S["a"]), lda=i32(S["lda"]),
                    b=i64(S["b"]), ldb=i32(S["ldb"]), k=i32(S["k"]),
                    scale=np.ascontiguousarray(S["scale"], dtype=np.float64))
        ptrs = (_lib.c_vp * 8)(*([t.data_ptr() for t in bases] + [0] * (8 - len(bases))))
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        P_ = _lib.as_p
        c64, c32, cd = _lib.c_i64, _lib.ctypes.c_int32, _lib.c_dbl
        _lib.check(_lib.load().sdmrg_grouped_gemm(
            self.ta, self.tb, nprob, P_(arrs["c"], c64), P_(arrs["ldc"], c32),
            P_(arrs["m"], c32), P_(arrs["n"], c32), P_(arrs["beta"], c32),
            P_(arrs["sb"], c64), P_(arrs["a"], c64), P_(arrs["lda"], c32),
            P_(arrs["b"], c64), P_(arrs["ldb"], c32), P_(arrs["k"], c32),
            P_(arrs["scale"], cd), ptrs, len(bases), st))


# ---------------------------------------------------------- partial sums

def _defs_prep(defs):
    """Store-independent preprocessing of a definition set (the term keys,
    the three-factor head/tail split), cached in ``defs`` — the driver
    reuses one defs object per partition for the whole run."""
    prep = defs.get("_prep")
    if prep is not None:
        return prep
    aux, inside = defs["aux"], defs["inside"]
    nf = (inside >= 0).sum(axis=1)

    def op_key(codes):
        f = decode(codes)
        return ("C",) + f if len(f) == 1 else ("P",) + f

    direct = np.nonzero(nf <= 2)[0]
    three = np.nonzero(nf == 3)[0]
    prep = {"direct": direct, "direct_keys": [op_key(inside[t]) for t in direct.tolist()],
            "three": three}
    if len(three):
        heads = [("C",) + decode(inside[t][:1]) for t in three.tolist()]
        tails = [("P",) + decode(inside[t][1:3]) for t in three.tolist()]
        mkeys, mindex = [], {}
        m_of = np.empty(len(three), np.int64)
        for i, (t, h) in enumerate(zip(three.tolist(), heads)):
            mk = (int(aux[t]), h)
            if mk not in mindex:
                mindex[mk] = len(mkeys)
                mkeys.append(mk)
            m_of[i] = mindex[mk]
        prep.update(tails=tails, mkeys=mkeys, m_of=m_of)
    defs["_prep"] = prep
    return prep


def composites(store, defs, model, device):
    """Σ_t coef_t · resolve(factors_t) for each definition (blocks.py:331
    materialize_aux / the cross sums of blocks.py:262).

    ``defs``: list of (key, delta, aux_ids, coefs, inside codes) where the
    three arrays list the terms of all definitions (aux_ids index ``defs``),
    inside strings of 1-3 factors (-1 padded codes).  Returns a ClassArena
    on the store basis holding the composites under their keys."""
    ops = store.ops
    out = ClassArena(ops.basis, [(d[0], d[1]) for d in defs["keys"]], device, zero=True)
    aux, coef = defs["aux"], defs["coef"]
    if len(aux) == 0:
        return out
    prep = _defs_prep(defs)
    keys = [k for k, _ in defs["keys"]]
    # one- and two-factor strings: out_class = K @ store_class
    direct = prep["direct"]
    for tk in prep["direct_keys"]:
        if not ops.has(tk):
            raise KeyError(f"operator {tk} not maintained on block {store.sites}")
    _class_gemm(out, keys, ops, aux, coef, direct, prep["direct_keys"],
                cache=prep.setdefault("_k_direct", {}))
    # three-factor strings: M_(c, head) = Σ c · P (GEMM), out += Σ_head C · M
    three = prep["three"]
    if len(three):
        mkeys = prep["mkeys"]
        mdeltas = []
        for (c, h) in mkeys:
            hd = ops.delta(h)
            cd = out.delta(keys[c])
            mdeltas.append(tuple(a - b for a, b in zip(cd, hd)))
        marena = ClassArena(ops.basis, [(mk, dl) for mk, dl in zip(mkeys, mdeltas)], device)
        _class_gemm(marena, mkeys, ops, prep["m_of"], coef[three], np.arange(len(three)),
                    prep["tails"], cache=prep.setdefault("_k_three", {}))
        _head_products(out, keys, ops, marena, mkeys)
    return out


def _class_gemm(out, out_keys, ops, aux, coef, terms, term_keys, cache=None):
    """out[key] (=) Σ coef · ops[term key] for each output key: one engine
    GEMM per (output class, source class): C = K · S.

    ``cache`` (a dict kept with the definition set): the coefficient
    matrices K depend only on the key layouts of ``out`` and ``ops`` — fixed
    for a partition — so they are built once per layout (and uploaded once
    per device) and every later visit only launches the GEMMs."""
    if len(terms) == 0:
        return
    dev = out.arena.device
    sig = None
    if cache is not None:
        sig = (hash(tuple(ops.ops)), hash(tuple(out.ops)), len(ops.ops), len(out.ops))
        plan = cache.get(sig)
        if plan is not None:
            ocl, scl = list(out.classes.values()), list(ops.classes.values())
            for oi, si, k, kdev in plan:
                cl_o, cl_s = ocl[oi], scl[si]
                if cl_o.size == 0:
                    continue
                kd = kdev.get(dev)
                if kd is None:
                    kd = kdev[dev] = torch.from_numpy(k).to(dev)
                ln = Launch(0, 0)
                ln.add(handle(0, cl_o.base), cl_o.size, cl_o.nops, cl_o.size, 0, 1,
                       handle(1, 0), cl_s.nops, handle(2, cl_s.base), cl_s.size, cl_s.nops, 1.0)
                ln.run([out.arena, kd, ops.arena])
            return
    terms = np.asarray(terms)
    outs = [out.ops[out_keys[a]] for a in np.asarray(aux)[terms].tolist()]
    srcs = [ops.ops[tk] for tk in term_keys]
    oidx = {id(c): i for i, c in enumerate(out.classes.values())}
    sidx = {id(c): i for i, c in enumerate(ops.classes.values())}
    co = np.array([oidx[id(c)] for c, _ in outs], np.int64)
    ro = np.array([r for _, r in outs], np.int64)
    cs = np.array([sidx[id(c)] for c, _ in srcs], np.int64)
    rs = np.array([r for _, r in srcs], np.int64)
    cf = np.asarray(coef, np.float64)[terms]
    ocl, scl = list(out.classes.values()), list(ops.classes.values())
    pair = co * max(len(scl), 1) + cs
    order = np.argsort(pair, kind="stable")
    bounds = np.nonzero(np.diff(pair[order]))[0] + 1
    plan = []
    for grp in np.split(order, bounds):
        oi, si = int(co[grp[0]]), int(cs[grp[0]])
        cl_o, cl_s = ocl[oi], scl[si]
        if cl_o.delta != cl_s.delta:
            raise ValueError(f"term shift {cl_s.delta} != composite shift {cl_o.delta}")
        k = np.zeros((cl_o.nops, cl_s.nops))
        np.add.at(k, (ro[grp], rs[grp]), cf[grp])
        kd = torch.from_numpy(k).to(dev)
        plan.append((oi, si, k, {dev: kd}))
        if cl_o.size == 0:
            continue
        ln = Launch(0, 0)
        ln.add(handle(0, cl_o.base), cl_o.size, cl_o.nops, cl_o.size, 0, 1,
               handle(1, 0), cl_s.nops, handle(2, cl_s.base), cl_s.size, cl_s.nops, 1.0)
        ln.run([out.arena, kd, ops.arena])
    if cache is not None:
        if len(cache) > 8:
            cache.clear()
        cache[sig] = plan


def _slot_table(cl, nsec):
    t = getattr(cl, "_slots", None)
    if t is None or len(t) != nsec:
        t = np.full(nsec, -1, np.int64)
        t[cl.col] = np.arange(len(cl.col))
        cl._slots = t
    return t


def _head_products(out, keys, ops, marena, mkeys):
    """out[c] += Σ_head C_head · M_(c, head): per output block one problem,
    the heads its segments (blocks.py:104 resolve of 3-factor strings)."""
    basis = ops.basis
    dims = basis.dims
    nsec = len(basis)
    parts = []
    for mk in mkeys:
        c, h = mk
        cl_o, r_o = out.ops[keys[c]]
        cl_m, r_m = marena.ops[mk]
        cl_h, r_h = ops.ops[h]
        j = cl_o.col
        if len(j) == 0 or len(cl_m.row) == 0 or len(cl_h.row) == 0:
            continue
        ms = _slot_table(cl_m, nsec)[j]
        ok = ms >= 0
        jm = np.where(ok, cl_m.row[np.maximum(ms, 0)], 0)
        hs = np.where(ok, _slot_table(cl_h, nsec)[jm], -1)
        ok &= hs >= 0
        if not ok.any():
            continue
        slot = np.nonzero(ok)[0]
        ms, hs, jm = ms[slot], hs[slot], jm[slot]
        jr = cl_h.row[hs]
        if np.any(jr != cl_o.row[slot]):
            raise ValueError("selection rule mismatch in a three-factor product")
        parts.append((cl_o.base + r_o * cl_o.size + cl_o.off[slot], dims[jr], dims[j[slot]],
                      cl_h.base + r_h * cl_h.size + cl_h.off[hs],
                      cl_m.base + r_m * cl_m.size + cl_m.off[ms], dims[jm]))
    if not parts:
        return
    dst, m, n, a, b, k = (np.concatenate([p[x] for p in parts]) for x in range(6))
    order = np.argsort(dst, kind="stable")       # segments of a block in head order
    dst, m, n, a, b, k = dst[order], m[order], n[order], a[order], b[order], k[order]
    first = np.concatenate([[True], dst[1:] != dst[:-1]])
    starts = np.nonzero(first)[0]
    nseg = np.diff(np.concatenate([starts, [len(dst)]]))
    ln = Launch(0, 0)
    ln.add(handle(0, dst[starts]), n[starts], m[starts], n[starts],
           np.ones(len(starts), np.int64), nseg,
           handle(1, a), k, handle(2, b), n, k, np.ones(len(a)))
    ln.run([out.arena, ops.arena, marena.arena])


# ------------------------------------------------------ site operators

def site_map(local, dense, dress_sign=False):
    """Column map (dst state, value) of a site operator (1-dim sectors:
    <= one nonzero per column); ``dress_sign``: times the parity of the
    input state (op @ par_site)."""
    ns = dense.shape[0]
    dst = np.full(ns, -1, np.int64)
    val = np.zeros(ns)
    for s in range(ns):
        nz = np.nonzero(np.abs(dense[:, s]) > 0)[0]
        if nz.size == 0:
            continue
        if nz.size > 1:
            raise ValueError("site operator mixes quantum-number shifts")
        dst[s] = int(nz[0])
        val[s] = float(dense[nz[0], s]) * (local.parity_sign(local.state_qns[s])
                                          if dress_sign else 1.0)
    return dst, val


# --------------------------------------------- enlargement + rotation

@dataclass
class KronTerm:
    """new op += coef · kron_lr(X (@ par_block), s (@ par_site))."""

    key: tuple               # new operator key
    src: tuple               # ("op", key) in the old store, ("comp", key)
    site: tuple              # (dst, val) column map of the site operator
    coef: float = 1.0
    dress_block: bool = False


def enlarge_rotate(old, comp, local, terms, new_keys, fused, w, new_basis, device,
                   t_budget=None):
    """New operators W^T (Σ kron pieces) W on ``new_basis`` (blocks.py:190
    enlarge_block + dmrg.py:254 _transform_tree, fused).

    ``w``: {fused qn: device W (dimF x kept)} for the kept sectors;
    ``new_keys``: [(key, delta)] of the new store (identity written exactly,
    dmrg.py:318).  Returns the new ClassArena."""
    left = old.side == "L"
    ob = old.basis
    sq = local.state_qns
    out = ClassArena(new_basis, new_keys, device, zero=True)
    # W packed in one buffer
    wq = sorted(w)
    woff, pos = {}, 0
    for q in wq:
        woff[q] = pos
        pos += w[q].numel()
    wbuf = torch.empty(max(pos, 1), dtype=torch.float64, device=device)
    for q in wq:
        wbuf[woff[q]:woff[q] + w[q].numel()] = w[q].reshape(-1)
    kept = {q: int(w[q].shape[1]) for q in wq}
    psign = np.array([local.parity_sign(q) for q in ob.qns])
    # pieces: (out block offset, m, n) <- scale * W_r[rowoff:+dr]^T (X W_c[coloff:+dc])
    pieces = []          # (dst, m_out, n_out, wr_off, x_src(base, off), dr, dc, wc_off, scale)
    for term in terms:
        if term.src[0] == "op":
            arena, base_id = old.ops, 0
        else:
            arena, base_id = comp, 1
        cl, r = arena.ops[term.src[1]]
        cl_n, r_n = out.ops[term.key]
        dst_s, val_s = term.site
        for slot in range(len(cl.col)):
            j, jr = int(cl.col[slot]), int(cl.row[slot])
            xoff = cl.base + r * cl.size + int(cl.off[slot])
            dr, dc = int(ob.dims[jr]), int(ob.dims[j])
            for sc in range(len(sq)):
                sr = int(dst_s[sc])
                if sr < 0:
                    continue
                if left:
                    cpair, rpair = (ob.qns[j], sq[sc]), (ob.qns[jr], sq[sr])
                else:
                    cpair, rpair = (sq[sc], ob.qns[j]), (sq[sr], ob.qns[jr])
                fc = qn_add(*cpair)
                fr = qn_add(*rpair)
                if fc not in kept or fr not in kept:
                    continue
                scale = term.coef * float(val_s[sc])
                if term.dress_block:
                    scale *= psign[j]
                if scale == 0.0:
                    continue
                jn_c = new_basis.index[fc]
                slot_n = cl_n.col_pos.get(jn_c)
                if slot_n is None or new_basis.qns[int(cl_n.row[slot_n])] != fr:
                    raise ValueError("kron piece outside the new operator's block structure")
                dst = cl_n.base + r_n * cl_n.size + int(cl_n.off[slot_n])
                pieces.append((dst, kept[fr], kept[fc], woff[fr] + fused.layout[rpair] * kept[fr],
                               base_id, xoff, dr, dc, woff[fc] + fused.layout[cpair] * kept[fc],
                               scale))
    # identity: exact (dmrg.py:318 SectorMatrix.identity)
    if out.has(KEY_I):
        _write_identity(out, KEY_I)
    if not pieces:
        return out
    # stage A: distinct X·W_c products (dedup on (source, block, W_c slice))
    tkey = {}
    t_list = []
    for pc in pieces:
        k = (pc[4], pc[5], pc[8])
        if k not in tkey:
            tkey[k] = len(t_list)
            t_list.append((pc[4], pc[5], pc[6], pc[7], pc[8], pc[2]))   # base, xoff, dr, dc, wc, n
    t_off = np.zeros(len(t_list) + 1, np.int64)
    t_off[1:] = np.cumsum([t[2] * t[5] for t in t_list])
    if t_budget is None:
        free = torch.cuda.mem_get_info(device)[0] if device.type == "cuda" else 1 << 33
        t_budget = max(1 << 24, int(0.25 * free / 8))
    budget = t_budget
    # chunk the pieces by output so each chunk's T fits the budget
    order = sorted(range(len(pieces)), key=lambda i: pieces[i][0])
    chunks, cur, cur_t, seen = [], [], 0, set()
    for i in order:
        ti = tkey[(pieces[i][4], pieces[i][5], pieces[i][8])]
        need = 0 if ti in seen else t_list[ti][2] * t_list[ti][5]
        if cur and cur_t + need > budget and pieces[i][0] != pieces[cur[-1]][0]:
            chunks.append(cur)
            cur, cur_t, seen = [], 0, set()
            need = t_list[ti][2] * t_list[ti][5]
        cur.append(i)
        if ti not in seen:
            seen.add(ti)
            cur_t += need
    if cur:
        chunks.append(cur)
    for ch in chunks:
        tis = sorted({tkey[(pieces[i][4], pieces[i][5], pieces[i][8])] for i in ch})
        loc = {}
        p = 0
        for ti in tis:
            loc[ti] = p
            p += t_list[ti][2] * t_list[ti][5]
        tbuf = torch.empty(max(p, 1), dtype=torch.float64, device=device)
        la = Launch(0, 0)
        ar = np.array([[loc[ti], t_list[ti][2], t_list[ti][5], t_list[ti][0], t_list[ti][1],
                        t_list[ti][3], t_list[ti][4]] for ti in tis], np.int64)
        # T (dr x n) = X (dr x dc, ld dc) · W_c[coloff:+dc] (dc x n, ld n)
        a_h = np.where(ar[:, 3] == 0, handle(0, ar[:, 4]), handle(1, ar[:, 4]))
        la.add(handle(3, ar[:, 0]), ar[:, 2], ar[:, 1], ar[:, 2], np.zeros(len(ar), np.int64),
               np.ones(len(ar), np.int64), a_h, ar[:, 5], handle(2, ar[:, 6]), ar[:, 2],
               ar[:, 5], np.ones(len(ar)))
        la.run([old.ops.arena, comp.arena if comp is not None else old.ops.arena, wbuf, tbuf])
        # stage B: out block += Σ s · W_r^T T  (segments in piece order)
        lb = Launch(1, 0)
        groups = {}
        for i in ch:
            groups.setdefault(pieces[i][0], []).append(i)
        cs, ms_, ns, nseg, a, b, lda, ldb, kk, sc = [], [], [], [], [], [], [], [], [], []
        for dst, idx in groups.items():
            pc0 = pieces[idx[0]]
            cs.append(dst)
            ms_.append(pc0[1])
            ns.append(pc0[2])
            nseg.append(len(idx))
            for i in idx:
                pc = pieces[i]
                ti = tkey[(pc[4], pc[5], pc[8])]
                a.append(pc[3])
                lda.append(pc[1])
                b.append(loc[ti])
                ldb.append(pc[2])
                kk.append(pc[6])
                sc.append(pc[9])
        lb.add(handle(0, cs), ns, ms_, ns, np.zeros(len(cs), np.int64), nseg,
               handle(1, a), lda, handle(2, b), ldb, kk, sc)
        lb.run([out.arena, wbuf, tbuf])
        del tbuf
    return out


def _write_identity(arena, key):
    cl, r = arena.ops[key]
    b = arena.basis
    host = np.zeros(cl.size)
    for j, jr, o in zip(cl.col, cl.row, cl.off):
        d = int(b.dims[j])
        host[o:o + d * d] = np.eye(d).ravel()
    base = cl.base + r * cl.size
    arena.arena[base:base + cl.size].copy_(torch.from_numpy(host))


def identity_w(basis, device):
    return {q: torch.eye(int(d), dtype=torch.float64, device=device)
            for q, d in basis.entries}
