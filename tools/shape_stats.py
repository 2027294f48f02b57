"""Engine work shapes of one apply: K-stage efficiency of phase 1 / phase 2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2305_05581_b200.plan import DevicePlan
from paper_2305_05581_b200.workload import synthetic_plan_input
L, D = int(sys.argv[1]), int(sys.argv[2])
pi = synthetic_plan_input(L, D)
p = DevicePlan(pi, dry_run=True, keep_groups=True)
g = p.groups()
keys = np.array(pi.psi_keys())
dl, dr = pi.dim_l.astype(np.int64), pi.dim_r.astype(np.int64)
print("left dims", np.sort(dl)[::-1][:12], "mean", dl.mean())
# phase 2: per group, distinct rops -> products with K = m
k_use = 0; k_st16 = 0; k_st4 = 0; fl = 0
ph1 = {}
for k in range(len(g)):
    i, o = int(g.group_psi[k]), int(g.group_out[k])
    m = dl[keys[i][0]]; n = dr[keys[i][3]]; q = dl[keys[o][0]]; r = dr[keys[o][3]]
    rows = g.member_row[g.group_begin[k]:g.group_begin[k + 1]]
    nprod = len(np.unique(pi.rop[rows]))
    w = q * r  # output area weight
    k_use += nprod * m * w; k_st16 += nprod * (-(-m // 16) * 16) * w; k_st4 += nprod * (-(-m // 4) * 4) * w
    for b in np.unique(pi.rop[rows]):
        if pi.kind_r[b] != 1:
            ph1[(i, b)] = (m, r, n)
print(f"phase2 K efficiency: stage16 {k_use / k_st16:.3f}  k4 {k_use / k_st4:.3f}")
sh = np.array(list(ph1.values()))
m, r, n = sh[:, 0], sh[:, 1], sh[:, 2]
f = 2 * m * r * n
def pad(x, b): return -(-x // b) * b
tiles = np.ceil(m / 64) * np.ceil(r / 64)
print(f"phase1: {len(sh)} problems, mean m {np.average(m, weights=f):.1f} r {np.average(r, weights=f):.1f} n {np.average(n, weights=f):.1f} (flop-weighted)")
print(f"phase1 K efficiency stage16 {np.sum(f) / np.sum(2 * m * r * pad(n, 16)):.3f}, MN 8-pad eff {np.sum(f) / np.sum(2 * pad(m, 8) * pad(r, 8) * n):.3f}")
print(f"phase1 tiles {tiles.sum():.0f}, flops per tile {np.sum(f) / tiles.sum() / 1e6:.2f} MFLOP")
# phase 2 tile costs (per out key: K = sum of m over its products)
kout = {}
for k in range(len(g)):
    i, o = int(g.group_psi[k]), int(g.group_out[k])
    rows = g.member_row[g.group_begin[k]:g.group_begin[k + 1]]
    kout[o] = kout.get(o, 0) + len(np.unique(pi.rop[rows])) * int(dl[keys[i][0]])
costs = []
for o, K in kout.items():
    q, r = int(dl[keys[o][0]]), int(dr[keys[o][3]])
    nt = int(np.ceil(q / 64) * np.ceil(r / 64))
    tq, tr = q / np.ceil(q / 64), r / np.ceil(r / 64)
    costs += [2 * tq * tr * K] * nt
costs = np.sort(np.array(costs))[::-1]
for ctas in (148 * 3, 148 * 4):
    print(f"phase2: {len(costs)} tiles, max tile {costs[0] / 1e9:.2f} GF, total/{ctas} CTAs {costs.sum() / ctas / 1e9:.2f} GF (max/mean-per-CTA {costs[0] / (costs.sum() / ctas):.2f})")
