"""Phase-1 tiling with T = A R^T per (ψ key, rop) vs per run of right
operators whose arena blocks are adjacent (one m x sum(r) x n product)."""
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
need = {}
for k in range(len(g)):
    i = int(g.group_psi[k])
    rows = g.member_row[g.group_begin[k]:g.group_begin[k + 1]]
    need.setdefault(i, set()).update(int(b) for b in np.unique(pi.rop[rows]) if pi.kind_r[b] != 1)
present = pi.blk_off_r >= 0  # [op, sector]
def rows_of(o, j):
    tgt = tuple(int(a) + int(b) for a, b in zip(pi.qn_r[j], pi.delta_r[o]))
    return qmap.get(tgt)
qmap = {tuple(q): int(dr[k]) for k, q in enumerate(pi.qn_r.tolist())}
def p8(x): return -(-x // 8) * 8
def p2(x): return x + (x & 1)
T = 64
base = dict(tiles=0, work=0, flops=0); stk = dict(tiles=0, work=0, flops=0, runs=0)
for i, ops in need.items():
    m, n, j = int(dl[keys[i][0]]), int(dr[keys[i][3]]), int(keys[i][3])
    kp = -(-n // 4) * 4
    pres = [o for o in np.nonzero(present[:, j])[0]]
    pos = {o: x for x, o in enumerate(pres)}
    srt = sorted(ops, key=lambda o: pos[o])
    runs = []; cur = []
    for o in srt:
        if cur and pos[o] != pos[cur[-1]] + 1:
            runs.append(cur); cur = []
        cur.append(o)
    if cur: runs.append(cur)
    for o in srt:
        r = rows_of(o, j)
        base['flops'] += 2 * m * r * n
        for r0 in range(0, m, T):
            for c0 in range(0, r, T):
                base['tiles'] += 1; base['work'] += p8(min(T, m - r0)) * p8(min(T, r - c0)) * kp
    for run in runs:
        R = sum(p2(rows_of(o, j)) for o in run)
        stk['runs'] += 1
        for r0 in range(0, m, T):
            for c0 in range(0, R, T):
                stk['tiles'] += 1; stk['work'] += p8(min(T, m - r0)) * p8(min(T, R - c0)) * kp
f = base['flops']
print(f"L={L} D={D}: per-rop {sum(len(v) for v in need.values())} products, {base['tiles']} tiles, "
      f"eff {f / 2 / base['work']:.3f}; stacked {stk['runs']} runs, {stk['tiles']} tiles, eff {f / 2 / stk['work']:.3f}")
