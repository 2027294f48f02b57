"""Dump the reference's operator table for a synthetic CAS(L, L) partition.

Runs in the build container only (imports the reference from
/root/reference/pkg/src).  The table of an L-orbital random-integral model at
the middle partition — exactly ``factorize(model, model.partition_at(p))``
(model.py:415) — is stored in compact form (site maps resolved from the
rows' factor strings as blocks.py:526-560 does) together with each operator
key's quantum-number shift.  The bench / workload generator combines it with
synthetic block bases at bond dimension D, so the GPU box needs neither the
reference nor its multi-minute Python factorization.

Usage: python tools/make_table_fixture.py 30 [out.npz]
"""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from sector_dmrg.model import KEY_H, KEY_I, Integrals, ModelSpec, factorize, model_from_integrals  # noqa: E402

from paper_2305_05581_b200.plan_input import _site_map  # noqa: E402


def random_integrals(n, seed=1):
    rng = np.random.default_rng(seed)
    t = rng.standard_normal((n, n))
    t = (t + t.T) / 2
    v = 0.1 * rng.standard_normal((n, n, n, n))
    v = 0.5 * (v + v.transpose(3, 2, 1, 0))
    two = {(i, j, k, l): float(v[i, j, k, l]) for i in range(n) for j in range(n)
           for k in range(n) for l in range(n)}
    return Integrals(n, t, two, 0.0)


def main():
    n = int(sys.argv[1])
    out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(
        ROOT, "paper_2305_05581_b200", "data", f"table_L{n}.npz")
    t0 = time.time()
    model = model_from_integrals(ModelSpec("integral-file", path="synthetic"), random_integrals(n))
    p = (n - 2) // 2
    table = factorize(model, model.partition_at(p))
    a, b, _c = table.bounds
    local = model.local

    def delta_of(factors):
        d = [0] * local.qn_ncomp
        for m, dag in factors:
            ch = model.mode_charge(m)
            for c in range(len(d)):
                d[c] += ch[c] if dag else -ch[c]
        return d

    def key_delta(key, side):
        if key in (KEY_I, KEY_H):
            return [0] * local.qn_ncomp
        if key[0] == "AUX":
            aux = (table.left_aux if side == "L" else table.right_aux)[key[2]]
            return delta_of(aux.terms[0][1])
        return delta_of(key[1:])

    def key_kind(key):
        if key == KEY_I:
            return 1
        if key == KEY_H:
            return 2
        return {"C": 3, "P": 4, "AUX": 5}[key[0]]

    lkeys, rkeys = {}, {}
    lop, rop, alpha, e_l, s1d, s1v, s2d, s2v = [], [], [], [], [], [], [], []
    cache = {}
    for row in table.rows:
        for keys, key in ((lkeys, row.left), (rkeys, row.right)):
            if key not in keys:
                keys[key] = len(keys)
        e0, e1, e2 = row.dress
        k1 = (row.site1, e1)
        if k1 not in cache:
            cache[k1] = _site_map(local, local.string_matrix(row.site1, a), e1)
        k2 = (row.site2, e2, 2)
        if k2 not in cache:
            cache[k2] = _site_map(local, local.string_matrix(row.site2, b), e2)
        lop.append(lkeys[row.left])
        rop.append(rkeys[row.right])
        alpha.append(row.alpha)
        e_l.append(int(bool(e0)))
        s1d.append(cache[k1][0])
        s1v.append(cache[k1][1])
        s2d.append(cache[k2][0])
        s2v.append(cache[k2][1])
    lk = sorted(lkeys, key=lkeys.get)
    rk = sorted(rkeys, key=rkeys.get)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    np.savez_compressed(
        out, n_orb=np.int64(n), position=np.int64(p),
        n_left_orb=np.int64(p), n_right_orb=np.int64(n - p - 2),
        site_qn=np.array([q for q, _ in local.basis.entries], np.int32),
        target=np.array(model.default_target(), np.int32),
        delta_l=np.array([key_delta(k, "L") for k in lk], np.int32),
        kind_l=np.array([key_kind(k) for k in lk], np.int32),
        delta_r=np.array([key_delta(k, "R") for k in rk], np.int32),
        kind_r=np.array([key_kind(k) for k in rk], np.int32),
        lop=np.array(lop, np.int32), rop=np.array(rop, np.int32),
        alpha=np.array(alpha), e_l=np.array(e_l, np.int32),
        site1_dst=np.array(s1d, np.int32), site1_val=np.array(s1v),
        site2_dst=np.array(s2d, np.int32), site2_val=np.array(s2v))
    print(f"L={n} p={p}: {len(lop)} rows, {len(lk)} left ops, {len(rk)} right ops "
          f"in {time.time() - t0:.1f}s -> {out}")


if __name__ == "__main__":
    main()
