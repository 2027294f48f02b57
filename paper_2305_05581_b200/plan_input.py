"""Compact operator-table form of an H_eff·ψ plan (host side, numpy).

``PlanInput`` is the wire format of ``sdmrg_plan_desc``: sector bases,
per-operator block offset tables into two packed arenas, and the resolved
operator-table rows.  It is produced three ways:

* ``compile_reference_plan`` — from the reference's own objects (Model,
  OperatorTable, BlockStore, SuperblockWavefunction), resolving every row the
  way blocks.py:503-565 build_plan does (drop-in path);
* ``paper_2305_05581_b200.workload`` — synthetic partitions at bench scale;
* ``PlanInput.load`` — committed fixtures (tests/golden).
"""

from dataclasses import dataclass, field

import numpy as np

KEY_I = ("I",)
KEY_H = ("H",)

_ARRAYS = ("site_qn", "target", "qn_l", "dim_l", "left_sign", "qn_r", "dim_r",
           "delta_l", "blk_off_l", "kind_l", "delta_r", "blk_off_r", "kind_r",
           "lop", "rop", "alpha", "e_l", "site1_dst", "site1_val", "site2_dst",
           "site2_val", "row_map")


@dataclass
class PlanInput:
    site_qn: np.ndarray          # (nsite, ncomp) int32
    target: np.ndarray           # (ncomp,) int32
    qn_l: np.ndarray             # (nL, ncomp) int32, sorted
    dim_l: np.ndarray            # (nL,) int32
    left_sign: np.ndarray        # (nL,) float64
    qn_r: np.ndarray
    dim_r: np.ndarray
    delta_l: np.ndarray          # (nops_l, ncomp) int32
    blk_off_l: np.ndarray        # (nops_l, nL) int64, -1 = absent
    kind_l: np.ndarray           # (nops_l,) int32, 1 = identity
    delta_r: np.ndarray
    blk_off_r: np.ndarray
    kind_r: np.ndarray
    lop: np.ndarray              # (nrows,) int32
    rop: np.ndarray
    alpha: np.ndarray            # (nrows,) float64
    e_l: np.ndarray              # (nrows,) int32
    site1_dst: np.ndarray        # (nrows, nsite) int32
    site1_val: np.ndarray        # (nrows, nsite) float64
    site2_dst: np.ndarray
    site2_val: np.ndarray
    row_map: np.ndarray          # (nrows,) int64: index of the source table row
    arena_l: np.ndarray = None   # host copies of the packed arenas (float64)
    arena_r: np.ndarray = None
    meta: dict = field(default_factory=dict)

    @property
    def ncomp(self):
        return int(self.target.shape[0])

    @property
    def nsite(self):
        return int(self.site_qn.shape[0])

    @property
    def nrows(self):
        return int(self.lop.shape[0])

    def normalized(self):
        """Contiguous arrays of the exact dtypes the C ABI reads."""
        i32 = ("site_qn", "target", "qn_l", "dim_l", "qn_r", "dim_r", "delta_l",
               "kind_l", "delta_r", "kind_r", "lop", "rop", "e_l", "site1_dst", "site2_dst")
        i64 = ("blk_off_l", "blk_off_r", "row_map")
        f64 = ("left_sign", "alpha", "site1_val", "site2_val")
        for name in i32:
            setattr(self, name, np.ascontiguousarray(getattr(self, name), dtype=np.int32))
        for name in i64:
            setattr(self, name, np.ascontiguousarray(getattr(self, name), dtype=np.int64))
        for name in f64:
            setattr(self, name, np.ascontiguousarray(getattr(self, name), dtype=np.float64))
        for name in ("arena_l", "arena_r"):
            arr = getattr(self, name)
            if arr is not None:
                setattr(self, name, np.ascontiguousarray(arr, dtype=np.float64))
        return self

    # ---------------------------------------------------------------- ψ layout
    def psi_keys(self):
        """Sorted (jl, s1, s2, jr) index keys — blocks.py:416-429 order."""
        rindex = {tuple(q): j for j, q in enumerate(self.qn_r.tolist())}
        keys = []
        for jl, ql in enumerate(self.qn_l.tolist()):
            for s1, q1 in enumerate(self.site_qn.tolist()):
                for s2, q2 in enumerate(self.site_qn.tolist()):
                    qr = tuple(t - a - b - c for t, a, b, c in
                               zip(self.target.tolist(), ql, q1, q2))
                    jr = rindex.get(qr)
                    if jr is not None:
                        keys.append((jl, s1, s2, jr))

        def qkey(k):
            return (tuple(self.qn_l[k[0]]), tuple(self.site_qn[k[1]]),
                    tuple(self.site_qn[k[2]]), tuple(self.qn_r[k[3]]))

        keys.sort(key=qkey)
        return keys

    def psi_offsets(self, keys=None):
        keys = self.psi_keys() if keys is None else keys
        sizes = [int(self.dim_l[k[0]]) * int(self.dim_r[k[3]]) for k in keys]
        return np.concatenate([[0], np.cumsum(sizes, dtype=np.int64)]).astype(np.int64)

    # ----------------------------------------------------------- persistence
    def save(self, path, **extra):
        blobs = {name: getattr(self, name) for name in _ARRAYS}
        if self.arena_l is not None:
            blobs["arena_l"] = self.arena_l
            blobs["arena_r"] = self.arena_r
        blobs.update(extra)
        np.savez_compressed(path, **blobs)

    @classmethod
    def load(cls, path):
        z = np.load(path, allow_pickle=False)
        kw = {name: z[name] for name in _ARRAYS}
        pi = cls(**kw, arena_l=z["arena_l"] if "arena_l" in z else None,
                 arena_r=z["arena_r"] if "arena_r" in z else None)
        extra = {k: z[k] for k in z.files if k not in _ARRAYS and k not in ("arena_l", "arena_r")}
        pi.meta.update(extra)
        return pi.normalized()


# ------------------------------------------------------------ reference compile

def _site_map(local, dense, dress):
    """Column map of a site operator: input state -> (output state, value).

    Mirrors blocks.py:526-534 (``_site_sector_op`` then ``site1_map``), with
    the row's parity dressing on the input site state folded into the value
    (blocks.py:557-560; signs are +-1 so folding is exact).
    """
    qns = [tuple(q) for q, _ in local.basis.entries]
    pos = {tuple(q): i for i, q in enumerate(local.state_qns)}
    ns = len(qns)
    dst = np.full(ns, -1, dtype=np.int32)
    val = np.zeros(ns, dtype=np.float64)
    for s, qc in enumerate(qns):
        c = pos[qc]
        nz = np.nonzero(np.abs(dense[:, c]) > 0)[0]
        if nz.size == 0:
            continue
        r = int(nz[0])
        qr = tuple(local.state_qns[r])
        dst[s] = qns.index(qr)
        v = float(dense[r, c])
        if dress:
            v *= local.parity_sign(qc)
        val[s] = v
    return dst, val


class _OpPacker:
    """Packs the operators of one block side into an arena + offset table."""

    def __init__(self, basis):
        self.basis = basis
        self.qns = [tuple(q) for q, _ in basis.entries]
        self.index = {}
        self.deltas = []
        self.kinds = []
        self.offsets = []
        self.chunks = []
        self.size = 0
        self.by_id = {}      # id(block array) -> arena offset (fixture tooling)

    def add(self, key, mat, identity=False):
        if key in self.index:
            return self.index[key]
        if mat.row_basis != self.basis or mat.col_basis != self.basis:
            raise ValueError(f"operator {key} not on the block basis")
        row = np.full(len(self.qns), -1, dtype=np.int64)
        for j, cq in enumerate(self.qns):
            rq = tuple(a + b for a, b in zip(cq, mat.delta))
            blk = mat.blocks.get((rq, cq))
            if blk is None:
                continue
            arr = np.ascontiguousarray(blk, dtype=np.float64)
            row[j] = self.size
            self.by_id[id(blk)] = self.size
            self.chunks.append(arr.ravel())
            self.size += arr.size
        self.index[key] = len(self.deltas)
        self.deltas.append(tuple(mat.delta))
        self.kinds.append(1 if identity else 0)
        self.offsets.append(row)
        return self.index[key]

    def arena(self):
        if not self.chunks:
            return np.zeros(1)
        return np.concatenate(self.chunks)


def materialize_aux(table, left_store, right_store):
    """Partially summed composite operators (blocks.py:331-345), evaluated on
    the host from the stores' own ``resolve`` and the rows' coefficients."""
    out = {"L": {}, "R": {}}
    for side, defs, store in (("L", table.left_aux, left_store),
                              ("R", table.right_aux, right_store)):
        cache = {}
        for key, aux in defs.items():
            acc = None
            for coef, factors in aux.terms:
                mat = store.resolve(factors, cache)
                if acc is None:
                    acc = mat.scaled(0.0)
                    acc.blocks = {}
                for bkey, blk in mat.blocks.items():
                    acc.add_to_block(*bkey, coef * blk)
            out[side][key] = acc
    return out["L"], out["R"]


def _resolve_ref(key, store, aux_mats):
    if key == KEY_I:
        return store.ops[KEY_I]
    if key == KEY_H:
        return store.ops[KEY_H]
    if key[0] == "AUX":
        return aux_mats[key[2]]
    return store.op(key)


def compile_reference_plan(model, table, left_store, right_store, psi_struct,
                           aux_mats=None):
    """Resolve the reference's operator table into a ``PlanInput``.

    Same resolution as blocks.py:503-565: row coefficient, site-operator
    column maps (``_site_sector_op`` of ``local.string_matrix``), left parity
    dressing by input left sector, and operator blocks looked up by column
    sector.  Rows whose operators do not resolve are dropped (blocks.py:524).
    """
    local = model.local
    a, b, _c = table.bounds
    if aux_mats is None:
        laux, raux = materialize_aux(table, left_store, right_store)
    else:
        laux, raux = aux_mats
    packers = (_OpPacker(left_store.basis), _OpPacker(right_store.basis))
    lop, rop, alpha, e_l, rmap = [], [], [], [], []
    s1d, s1v, s2d, s2v = [], [], [], []
    site_cache = {}
    for t, row in enumerate(table.rows):
        lmat = _resolve_ref(row.left, left_store, laux)
        rmat = _resolve_ref(row.right, right_store, raux)
        if lmat is None or rmat is None:
            continue
        e_left, e_1, e_2 = row.dress
        k1 = (row.site1, e_1, a)
        if k1 not in site_cache:
            site_cache[k1] = _site_map(local, local.string_matrix(row.site1, a), e_1)
        k2 = (row.site2, e_2, b)
        if k2 not in site_cache:
            site_cache[k2] = _site_map(local, local.string_matrix(row.site2, b), e_2)
        lop.append(packers[0].add(row.left, lmat, row.left == KEY_I))
        rop.append(packers[1].add(row.right, rmat, row.right == KEY_I))
        alpha.append(float(row.alpha))
        e_l.append(int(bool(e_left)))
        d1, v1 = site_cache[k1]
        d2, v2 = site_cache[k2]
        s1d.append(d1)
        s1v.append(v1)
        s2d.append(d2)
        s2v.append(v2)
        rmap.append(t)

    def basis_arrays(basis):
        qn = np.array([q for q, _ in basis.entries], dtype=np.int32)
        dim = np.array([d for _, d in basis.entries], dtype=np.int32)
        return qn, dim

    qn_l, dim_l = basis_arrays(left_store.basis)
    qn_r, dim_r = basis_arrays(right_store.basis)
    ns = len(local.basis.entries)
    nrow = len(lop)
    pl, pr = packers
    ncomp = len(psi_struct.target)

    def ops_arrays(p, nsec):
        if not p.deltas:
            return (np.zeros((0, ncomp), np.int32), np.zeros((0, nsec), np.int64),
                    np.zeros(0, np.int32))
        return (np.array(p.deltas, dtype=np.int32), np.stack(p.offsets).astype(np.int64),
                np.array(p.kinds, dtype=np.int32))

    dl, ol, kl = ops_arrays(pl, len(dim_l))
    dr, orr, kr = ops_arrays(pr, len(dim_r))
    pi = PlanInput(
        site_qn=np.array([q for q, _ in local.basis.entries], dtype=np.int32),
        target=np.array(psi_struct.target, dtype=np.int32),
        qn_l=qn_l, dim_l=dim_l,
        left_sign=np.array([local.parity_sign(tuple(q)) for q in qn_l.tolist()]),
        qn_r=qn_r, dim_r=dim_r,
        delta_l=dl, blk_off_l=ol, kind_l=kl,
        delta_r=dr, blk_off_r=orr, kind_r=kr,
        lop=np.array(lop, dtype=np.int32), rop=np.array(rop, dtype=np.int32),
        alpha=np.array(alpha, dtype=np.float64), e_l=np.array(e_l, dtype=np.int32),
        site1_dst=np.array(s1d, dtype=np.int32).reshape(nrow, ns),
        site1_val=np.array(s1v, dtype=np.float64).reshape(nrow, ns),
        site2_dst=np.array(s2d, dtype=np.int32).reshape(nrow, ns),
        site2_val=np.array(s2v, dtype=np.float64).reshape(nrow, ns),
        row_map=np.array(rmap, dtype=np.int64),
        arena_l=pl.arena(), arena_r=pr.arena())
    pi.meta["packers"] = packers
    return pi.normalized()
