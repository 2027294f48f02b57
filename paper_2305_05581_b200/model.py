"""Hamiltonian terms and the operator-table factorization, vectorised.

Host-side input preparation for the device sweep (the reference's own
counterpart is pure Python, model.py).  Same definitions, bit for bit:

* ``LocalSpace``        model.py:51   single-site space (fermion / spin-1/2);
* ``Model.from_integrals``  model.py:383 model_from_integrals — the raw term
  list of model.py:400 ``_spin_terms`` / :412 ``_fermion_terms`` merged by
  :257 ``_merge_terms`` (mode-sorted with Jordan-Wigner sign, :238
  ``mode_sorted``; equal strings summed in raw-term order; sorted);
* ``factorize``         model.py:482  distribution of every term over
  (left | site | site | right) with the N^4 -> N^2 partial sums folded into
  auxiliary (complementary) operators, ties to the left; rows summed in term
  order and sorted exactly as Python sorts the reference's row keys.

Terms are arrays, not Python tuples: a factor (mode m, dagger d) is the code
``2*m + d``; strings are padded with -1.  At CAS(113,76) the reference's
Python loop over 1.3e8 raw terms did not finish in 4 h (round 1); here the
same arithmetic is a handful of numpy passes.  Parity with the reference is
pinned by tests/test_model_factorize.py against the reference's own tables
(tests/golden/factorize_*.npz, paper_2305_05581_b200/data/table_L*.npz).
"""

from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

SPIN_HALF = "spinhalf"
FERMION = "fermion"
KEY_I = ("I",)
KEY_H = ("H",)
COEF_TOL = 1e-15                                              # model.py:36


class ModelError(Exception):
    pass


class LocalSpace:
    """model.py:51 LocalSpace: QN-labeled single-site basis + mode operators."""

    def __init__(self, statistics):
        self.statistics = statistics
        if statistics == SPIN_HALF:
            self.modes_per_site = 1
            self.dim = 2
            self.state_qns = [(-1,), (1,)]
            self._creators = [np.array([[0.0, 0.0], [1.0, 0.0]])]
            self.charges = [(2,)]
        elif statistics == FERMION:
            self.modes_per_site = 2
            self.dim = 4
            self.state_qns = [(0, 0), (1, -1), (1, 1), (2, 0)]
            adag = np.array([[0.0, 0.0], [1.0, 0.0]])
            z = np.diag([1.0, -1.0])
            self._creators = [np.kron(adag, np.eye(2)), np.kron(z, adag)]
            self.charges = [(1, 1), (1, -1)]
        else:
            raise ModelError(f"unknown statistics {statistics!r}")
        self.basis_entries = [(q, 1) for q in self.state_qns]
        self.qn_ncomp = len(self.state_qns[0])

    def factor_matrix(self, k, dag):
        return self._creators[k] if dag else self._creators[k].T

    def parity_sign(self, qn):
        if self.statistics == SPIN_HALF:
            return 1.0
        return -1.0 if qn[0] % 2 else 1.0

    def parity_dense(self):
        if self.statistics == SPIN_HALF:
            return np.eye(self.dim)
        return np.diag([(-1.0) ** q[0] for q in self.state_qns])

    def string_matrix(self, factors, site_mode0):
        """model.py:94: dense site operator of a factor string (global modes)."""
        op = np.eye(self.dim)
        for m, dag in factors:
            op = op @ self.factor_matrix(m - site_mode0, dag)
        return op

    def zero_qn(self):
        return tuple(0 for _ in range(self.qn_ncomp))


# ------------------------------------------------------------------ factors

def decode(codes):
    """Padded code row -> tuple of (mode, dagger) factors (reference form)."""
    return tuple((int(c) >> 1, int(c) & 1) for c in codes if c >= 0)


def encode(factors, width=4):
    out = [-1] * width
    for i, (m, d) in enumerate(factors):
        out[i] = 2 * int(m) + int(d)
    return out


def _sort_key(codes):
    """int64 key whose integer order is Python's tuple order of the factor
    strings (shorter prefix first): 9 bits per factor, code+1, pad 0."""
    w = codes.shape[1]
    key = np.zeros(codes.shape[0], dtype=np.int64)
    for i in range(w):
        key = (key << 9) | (codes[:, i].astype(np.int64) + 1)
    return key


def mode_sorted(codes, fermionic):
    """model.py:238 mode_sorted, vectorised over rows of padded codes.

    Stable sort by mode; the sign counts strict mode inversions (the
    reference's insertion-sort swaps); sign 0 when two adjacent factors are
    the same mode with the same dagger."""
    n, w = codes.shape
    valid = codes >= 0
    mode = np.where(valid, codes >> 1, np.iinfo(np.int32).max).astype(np.int64)
    inv = np.zeros(n, dtype=np.int64)
    for i in range(w):
        for j in range(i + 1, w):
            inv += (valid[:, i] & valid[:, j] & (mode[:, i] > mode[:, j]))
    order = np.argsort(mode, axis=1, kind="stable")
    out = np.take_along_axis(codes, order, axis=1)
    sign = np.where(inv % 2 == 1, -1, 1) if fermionic else np.ones(n, dtype=np.int64)
    for i in range(w - 1):
        bad = (out[:, i] >= 0) & (out[:, i] == out[:, i + 1])
        sign = np.where(bad, 0, sign)
    return sign.astype(np.int64), out


@dataclass
class Integrals:
    """model.py:110 Integrals: one-body matrix + ordered two-body entries."""

    n_modes: int
    one_body: np.ndarray
    two_idx: np.ndarray          # (n, 4) int, dict (insertion) order
    two_val: np.ndarray
    core: float = 0.0


def random_integrals(n, seed, scale=0.2, core=0.3):
    """The random-integral models of tests/golden/make_golden.py:57 (the
    configs[0] / sweep fixtures): t symmetric normal, V = scale * normal
    symmetrised V_ijkl = V_lkji, core energy; two-body entries in (i,j,k,l)
    lexicographic order like the reference's dict."""
    rng = np.random.default_rng(seed)
    t = rng.standard_normal((n, n))
    t = (t + t.T) / 2
    v = scale * rng.standard_normal((n, n, n, n))
    v = 0.5 * (v + v.transpose(3, 2, 1, 0))
    idx = np.indices((n, n, n, n)).reshape(4, -1).T
    return Integrals(n, t, idx.astype(np.int32), v.reshape(-1).copy(), core)


class Model:
    """model.py:269 Model: local space, mode-level terms (arrays), core."""

    def __init__(self, integrals, statistics=FERMION):
        self.integrals = integrals
        self.local = LocalSpace(statistics)
        self.n_sites = integrals.n_modes
        self.n_modes = self.n_sites * self.local.modes_per_site
        self.core = float(integrals.core)
        self.fermionic = statistics == FERMION
        self.coef, self.codes = self._terms(integrals)
        self.nf = (self.codes >= 0).sum(axis=1)
        self.pair_codes = self._pair_codes()

    # -- model.py:400 / :412 raw terms, :257 merge
    def _terms(self, ig):
        t = np.asarray(ig.one_body, dtype=float)
        n = ig.n_modes
        ii, jj = np.nonzero(t != 0.0)            # row-major = the reference's i, j loops
        tv = t[ii, jj]
        vals = [np.zeros(0)]
        rows = [np.zeros((0, 4), np.int32)]
        if self.fermionic:
            spins = (0, 1)
            one = np.empty((len(ii), 2, 4), np.int32)
            for s in spins:
                one[:, s] = np.stack([2 * (2 * ii + s) + 1, 2 * (2 * jj + s) + 0,
                                      -np.ones_like(ii), -np.ones_like(ii)], axis=1)
            rows.append(one.reshape(-1, 4))
            vals.append(np.repeat(tv, 2))
            keep = ig.two_val != 0.0
            idx = ig.two_idx[keep].astype(np.int64)
            v = ig.two_val[keep]
            i, j, k, l = idx.T
            two = np.empty((len(v), 2, 2, 4), np.int32)
            for s in (0, 1):
                for tt in (0, 1):
                    two[:, s, tt] = np.stack([2 * (2 * i + s) + 1, 2 * (2 * j + tt) + 1,
                                              2 * (2 * k + tt) + 0, 2 * (2 * l + s) + 0], axis=1)
            rows.append(two.reshape(-1, 4))
            vals.append(np.repeat(v, 4))
        else:
            rows.append(np.stack([2 * ii + 1, 2 * jj + 0, -np.ones_like(ii),
                                  -np.ones_like(ii)], axis=1).astype(np.int32))
            vals.append(tv)
            idx = ig.two_idx.astype(np.int64)
            i, j, k, l = idx.T
            rows.append(np.stack([2 * i + 1, 2 * j + 1, 2 * k, 2 * l], axis=1).astype(np.int32))
            vals.append(np.asarray(ig.two_val, dtype=float))
        raw = np.concatenate(rows)
        coef = np.concatenate(vals)
        keep = coef != 0.0                                     # model.py:260
        raw, coef = raw[keep], coef[keep]
        sign, srt = mode_sorted(raw, self.fermionic)
        ok = sign != 0                                         # model.py:263
        srt, val = srt[ok], (sign[ok] * coef[ok])
        key = _sort_key(srt)
        uniq, first, inv = np.unique(key, return_index=True, return_inverse=True)
        acc = np.zeros(len(uniq))
        np.add.at(acc, inv, val)                 # sequential, raw-term order (model.py:265)
        keep = np.abs(acc) > COEF_TOL                          # model.py:266
        return acc[keep], srt[first[keep]]

    def _pair_codes(self):
        """model.py:306 pair_keys restricted to two-factor keys (codes)."""
        pairs = []
        for i in range(4):
            for j in range(i + 1, 4):
                m = (self.codes[:, i] >= 0) & (self.codes[:, j] >= 0)
                pairs.append(np.stack([self.codes[m, i], self.codes[m, j]], axis=1))
        allp = np.concatenate(pairs) if pairs else np.zeros((0, 2), np.int32)
        return np.unique(allp, axis=0)

    # -- geometry (model.py:284-324)
    def site_mode_range(self, s):
        mps = self.local.modes_per_site
        return s * mps, (s + 1) * mps

    def mode_charge(self, m):
        return self.local.charges[m % self.local.modes_per_site]

    def factor_delta(self, factors):
        delta = [0] * self.local.qn_ncomp
        for m, dag in factors:
            ch = self.mode_charge(m)
            for c in range(len(delta)):
                delta[c] += ch[c] if dag else -ch[c]
        return tuple(delta)

    def default_target(self):
        if self.local.statistics == SPIN_HALF:
            return (self.n_sites % 2,)
        return (self.n_sites, self.n_sites % 2)

    def bounds_at(self, position):
        mps = self.local.modes_per_site
        a = position * mps
        return a, a + mps, a + 2 * mps

    def terms(self):
        """The reference's ``model.terms`` list form (small models / tests)."""
        return [(float(c), decode(r)) for c, r in zip(self.coef, self.codes)]


# ------------------------------------------------------------ factorization

class TableRow(NamedTuple):                                    # model.py:436
    left: tuple
    site1: tuple
    site2: tuple
    right: tuple
    alpha: float
    dress: tuple


@dataclass
class AuxDefs:
    """The auxiliary (complementary) operators of one side (model.py:446
    AuxDef): ``keys[a]`` is the outside factor string (codes, -1 padded);
    terms ``(aux[t], coef[t], inside[t])`` in the reference's append order."""

    side: str
    keys: np.ndarray            # (nkeys, 2)
    aux: np.ndarray             # (nterms,) int
    coef: np.ndarray
    inside: np.ndarray          # (nterms, 3) codes

    def key_tuple(self, a):
        return decode(self.keys[a])

    def as_dict(self):
        """{outside key tuple: [(coef, inside factors)]} (reference form)."""
        out = {}
        for a in range(len(self.keys)):
            out[self.key_tuple(a)] = []
        for a, c, ins in zip(self.aux.tolist(), self.coef.tolist(), self.inside):
            out[self.key_tuple(a)].append((c, decode(ins)))
        return out


_TYPE_RANK = {"AUX": 0, "C": 1, "H": 2, "I": 3, "P": 4}        # Python str order


@dataclass
class OperatorTable:
    """model.py:453 OperatorTable in array form.

    Row t: left op (ltype: 0 AUX / 1 C / 2 H / 3 I / 4 P; lf: its factor
    codes, for AUX the outside key), site strings s1/s2 (codes), right op
    (rtype, rf), alpha, dress (3)."""

    position: int
    bounds: tuple
    ltype: np.ndarray
    lf: np.ndarray
    s1: np.ndarray
    s2: np.ndarray
    rtype: np.ndarray
    rf: np.ndarray
    alpha: np.ndarray
    dress: np.ndarray
    left_aux: AuxDefs
    right_aux: AuxDefs
    meta: dict = field(default_factory=dict)

    @property
    def nrows(self):
        return int(self.alpha.shape[0])

    @staticmethod
    def op_key(typ, codes, side):
        name = {0: "AUX", 1: "C", 2: "H", 3: "I", 4: "P"}[int(typ)]
        if name in ("H", "I"):
            return (name,)
        if name == "AUX":
            return ("AUX", side, decode(codes))
        return (name,) + decode(codes)

    def left_key(self, t):
        return self.op_key(self.ltype[t], self.lf[t], "L")

    def right_key(self, t):
        return self.op_key(self.rtype[t], self.rf[t], "R")

    def row(self, t):
        return TableRow(self.left_key(t), decode(self.s1[t]), decode(self.s2[t]),
                        self.right_key(t), float(self.alpha[t]),
                        tuple(int(x) for x in self.dress[t]))

    @property
    def rows(self):
        return [self.row(t) for t in range(self.nrows)]


def _pad(codes, width):
    n = codes.shape[0]
    out = -np.ones((n, width), np.int32)
    w = min(width, codes.shape[1])
    out[:, :w] = codes[:, :w]
    return out


def _segment(codes, start, length, width):
    """Per row: codes[start : start + length] left-aligned into ``width``."""
    n = codes.shape[0]
    out = -np.ones((n, width), np.int32)
    for i in range(width):
        src = start + i
        ok = (i < length) & (src < codes.shape[1])
        srcc = np.clip(src, 0, codes.shape[1] - 1)
        vals = np.take_along_axis(codes, srcc[:, None], axis=1)[:, 0]
        out[:, i] = np.where(ok, vals, -1)
    return out


def factorize(model, position):
    """model.py:482 factorize(model, model.partition_at(position))."""
    a, b, c = model.bounds_at(position)
    codes = model.codes
    coef = model.coef
    n = codes.shape[0]
    valid = codes >= 0
    mode = np.where(valid, codes >> 1, -1)
    part = np.where(~valid, -1, np.where(mode < a, 0, np.where(mode < b, 1, np.where(mode < c, 2, 3))))
    cnt = [((part == p)).sum(axis=1) for p in range(4)]
    nl, n1, n2, nr = cnt
    k = model.nf
    has_hl = bool(np.any(nl == k))
    has_hr = bool(np.any(nr == k))
    inner = (nl != k) & (nr != k)
    outside_l = n1 + n2 + nr
    outside_r = nl + n1 + n2
    is_l = inner & (nl >= np.maximum(1, nr)) & (outside_l <= 2)
    is_r = inner & ~is_l & (nr >= 1) & (outside_r <= 2)
    plain = inner & ~is_l & ~is_r
    # terms are mode-sorted: the parts are contiguous runs in order
    lam = _segment(codes, np.zeros(n, np.int64), nl, 4)
    s1 = _segment(codes, nl, n1, 4)
    s2 = _segment(codes, nl + n1, n2, 4)
    rho = _segment(codes, nl + n1 + n2, nr, 4)
    if model.fermionic:
        dress = np.stack([(n1 + n2 + nr) % 2, (n2 + nr) % 2, nr % 2], axis=1)
    else:
        dress = np.zeros((n, 3), np.int64)

    def plain_type(cnt_):
        return np.where(cnt_ == 0, 3, np.where(cnt_ == 1, 1, 4))

    ltype = np.where(is_l, 0, plain_type(nl))
    rtype = np.where(is_r, 0, plain_type(nr))
    lkey_l = _segment(codes, nl, outside_l, 4)                # left aux key = s1+s2+rho
    lkey_r = _segment(codes, np.zeros(n, np.int64), outside_r, 4)   # right aux key = lam+s1+s2
    lf = np.where(is_l[:, None], lkey_l, lam)
    rf = np.where(is_r[:, None], lkey_r, rho)
    if np.any(lf[inner, 2:] >= 0) or np.any(rf[inner, 2:] >= 0):
        raise ModelError("operator key longer than two factors")
    lf, rf = lf[:, :2], rf[:, :2]

    # aux buckets: keys in first-occurrence order, terms in term order
    def aux_defs(mask, keys4, inside, side):
        idx = np.nonzero(mask)[0]
        kk = _sort_key(keys4[idx][:, :2])
        uniq, first, inv = np.unique(kk, return_index=True, return_inverse=True)
        order = np.argsort(first, kind="stable")               # first occurrence
        rank = np.empty_like(order)
        rank[order] = np.arange(len(order))
        keys = keys4[idx[first[order]]][:, :2]
        if np.any(inside[idx][:, 3] >= 0):
            raise ModelError("auxiliary inside string longer than three factors")
        return AuxDefs(side, keys.astype(np.int32), rank[inv].astype(np.int64),
                       coef[idx].copy(), inside[idx][:, :3].astype(np.int32)), rank[inv]

    left_aux, _ = aux_defs(is_l, lkey_l, lam, "L")
    right_aux, _ = aux_defs(is_r, lkey_r, rho, "R")

    # rows: aux rows carry alpha 1 (model.py:511), plain rows accumulate coef
    # in term order (model.py:509); keys sorted as Python sorts the tuples
    rmask = inner
    ridx = np.nonzero(rmask)[0]
    comps = [ltype[ridx], lf[ridx, 0], lf[ridx, 1]]
    comps += [s1[ridx, i] for i in range(4)] + [s2[ridx, i] for i in range(4)]
    comps += [rtype[ridx], rf[ridx, 0], rf[ridx, 1]] + [dress[ridx, i] for i in range(3)]
    mat = np.stack([np.asarray(x, np.int64) for x in comps], axis=1)
    uniq, inv = np.unique(mat, axis=0, return_inverse=True)   # lexicographic = tuple order
    inv = inv.reshape(-1)
    alpha = np.zeros(len(uniq))
    is_plain = plain[ridx]
    np.add.at(alpha, inv[is_plain], coef[ridx][is_plain])
    aux_row = np.zeros(len(uniq), bool)
    aux_row[inv[~is_plain]] = True
    alpha[aux_row] = 1.0
    # the Python key order compares the type *names*; AUX < C < H < I < P is
    # already the rank order, and a code -1 pad sorts first like a shorter tuple
    keep = np.abs(alpha) > COEF_TOL                            # model.py:560
    u = uniq[keep]
    alpha = alpha[keep]
    head_t = []
    if has_hl or a > 0:
        head_t.append((2, 3))
    if has_hr or c < model.n_modes:
        head_t.append((3, 2))
    if model.core:
        head_t.append((3, 3))
    nh = len(head_t)
    neg = -np.ones((nh, 4), np.int32)
    ltype_o = np.concatenate([np.array([h[0] for h in head_t], np.int64), u[:, 0]])
    rtype_o = np.concatenate([np.array([h[1] for h in head_t], np.int64), u[:, 11]])
    lf_o = np.concatenate([neg[:, :2], u[:, 1:3]]).astype(np.int32)
    rf_o = np.concatenate([neg[:, :2], u[:, 12:14]]).astype(np.int32)
    s1_o = np.concatenate([neg, u[:, 3:7]]).astype(np.int32)
    s2_o = np.concatenate([neg, u[:, 7:11]]).astype(np.int32)
    alpha_o = np.concatenate([np.array([model.core if h == (3, 3) else 1.0 for h in head_t],
                                       dtype=float), alpha])
    dress_o = np.concatenate([np.zeros((nh, 3), np.int64), u[:, 14:17]]).astype(np.int32)
    return OperatorTable(position, (a, b, c), ltype_o.astype(np.int32), lf_o, s1_o, s2_o,
                         rtype_o.astype(np.int32), rf_o, alpha_o, dress_o, left_aux, right_aux)


# ------------------------------------------------------- compact table form

_KIND = {0: 5, 1: 3, 2: 2, 3: 1, 4: 4}     # AUX, C, H, I, P -> fixture kind tags


def site_map(local, factors, site_mode0, dress):
    """Column map of a site operator: input state -> (output state, value),
    the row's parity dressing of the input state folded in — blocks.py:526-560
    (``_site_sector_op`` of ``local.string_matrix`` + the e_1/e_2 signs)."""
    dense = local.string_matrix(factors, site_mode0)
    qns = [tuple(q) for q, _ in local.basis_entries]
    ns = len(qns)
    dst = np.full(ns, -1, dtype=np.int32)
    val = np.zeros(ns, dtype=np.float64)
    for s in range(ns):
        nz = np.nonzero(np.abs(dense[:, s]) > 0)[0]
        if nz.size == 0:
            continue
        r = int(nz[0])
        dst[s] = r
        v = float(dense[r, s])
        if dress:
            v *= local.parity_sign(qns[s])
        val[s] = v
    return dst, val


def compact(model, table):
    """The operator table as the plan's row arrays (tools/make_table_fixture.py
    format): per side, operator keys numbered by first appearance in row
    order with their QN shift and kind tag; per row lop/rop/alpha/e_l and the
    two site column maps."""
    a, b, _c = table.bounds
    local = model.local
    out = {}
    sides = {}
    for side, typ, fc, aux in (("l", table.ltype, table.lf, table.left_aux),
                               ("r", table.rtype, table.rf, table.right_aux)):
        kk = np.stack([typ.astype(np.int64), fc[:, 0], fc[:, 1]], axis=1)
        uniq, first, inv = np.unique(kk, axis=0, return_index=True, return_inverse=True)
        order = np.argsort(first, kind="stable")
        rank = np.empty_like(order)
        rank[order] = np.arange(len(order))
        ops = uniq[order]
        aux_first = {}
        aux_index = {tuple(k): i for i, k in enumerate(aux.keys.tolist())}
        if len(aux.aux):
            fi = np.unique(aux.aux, return_index=True)
            for ai, ti in zip(*fi):
                aux_first[int(ai)] = int(ti)
        deltas, kinds, keys = [], [], []
        for t, c0, c1 in ops.tolist():
            codes = [x for x in (c0, c1) if x >= 0]
            if t == 0:
                ai = aux_index[tuple([c0, c1])]
                ins = aux.inside[aux_first[ai]]
                deltas.append(model.factor_delta(decode(ins)))
            elif t in (2, 3):
                deltas.append(tuple([0] * local.qn_ncomp))
            else:
                deltas.append(model.factor_delta(decode(codes)))
            kinds.append(_KIND[t])
            keys.append(OperatorTable.op_key(t, np.array([c0, c1]), side.upper()))
        sides[side] = (rank[inv.reshape(-1)].astype(np.int32), np.array(deltas, np.int32),
                       np.array(kinds, np.int32), keys)
    cache = {}
    s1d, s1v, s2d, s2v = [], [], [], []
    for t in range(table.nrows):
        e0, e1, e2 = (int(x) for x in table.dress[t])
        k1 = (tuple(table.s1[t]), e1)
        if k1 not in cache:
            cache[k1] = site_map(local, decode(table.s1[t]), a, e1)
        k2 = (tuple(table.s2[t]), e2, 2)
        if k2 not in cache:
            cache[k2] = site_map(local, decode(table.s2[t]), b, e2)
        s1d.append(cache[k1][0])
        s1v.append(cache[k1][1])
        s2d.append(cache[k2][0])
        s2v.append(cache[k2][1])
    ns = len(local.basis_entries)
    out.update(
        site_qn=np.array(local.state_qns, np.int32),
        target=np.array(model.default_target(), np.int32),
        lop=sides["l"][0], rop=sides["r"][0], delta_l=sides["l"][1], kind_l=sides["l"][2],
        delta_r=sides["r"][1], kind_r=sides["r"][2], alpha=table.alpha.copy(),
        e_l=(table.dress[:, 0] != 0).astype(np.int32),
        site1_dst=np.array(s1d, np.int32).reshape(-1, ns), site1_val=np.array(s1v).reshape(-1, ns),
        site2_dst=np.array(s2d, np.int32).reshape(-1, ns), site2_val=np.array(s2v).reshape(-1, ns))
    out["keys_l"] = sides["l"][3]
    out["keys_r"] = sides["r"][3]
    return out
