"""Operator-table fixture for a synthetic CAS(L, L) partition from the native
(vectorised) factorization — paper_2305_05581_b200.model, bit-exact with the
reference's factorize (tests/test_model_factorize.py: L=12/16/30/50 fixtures
made by the reference itself via tools/make_table_fixture.py).  Same file
format as tools/make_table_fixture.py; runs without the reference, so the
CAS(113,76) table (configs[3]) — which the reference's Python factorize did
not finish in 4 h — can be produced.

Usage: python tools/make_table_native.py 76 [out.npz]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2305_05581_b200 import model as M  # noqa: E402


def main():
    n = int(sys.argv[1])
    out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(
        ROOT, "paper_2305_05581_b200", "data", f"table_L{n}.npz")
    t0 = time.time()
    mm = M.Model(M.random_integrals(n, 1, scale=0.1, core=0.0))
    t1 = time.time()
    p = (n - 2) // 2
    tab = M.factorize(mm, p)
    t2 = time.time()
    c = M.compact(mm, tab)
    keys = ("site_qn", "target", "delta_l", "kind_l", "delta_r", "kind_r", "lop", "rop",
            "alpha", "e_l", "site1_dst", "site1_val", "site2_dst", "site2_val")
    np.savez_compressed(out, n_orb=np.int64(n), position=np.int64(p),
                        n_left_orb=np.int64(p), n_right_orb=np.int64(n - p - 2),
                        **{k: c[k] for k in keys})
    print(f"L={n} p={p}: {len(mm.coef)} terms, {tab.nrows} rows, {len(c['kind_l'])} left ops, "
          f"{len(c['kind_r'])} right ops; model {t1 - t0:.0f}s factorize {t2 - t1:.0f}s -> {out}")


if __name__ == "__main__":
    main()
