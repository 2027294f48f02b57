import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sys
from paper_2305_05581_b200.plan import DevicePlan
from paper_2305_05581_b200.workload import synthetic_plan_input
import numpy as np
L, D = int(sys.argv[1]), int(sys.argv[2])
pi = synthetic_plan_input(L, D)
p = DevicePlan(pi, dry_run=True, keep_groups=True)
g = p.groups()
keys = np.array(pi.psi_keys())
dl = pi.dim_l; dr = pi.dim_r
cur1 = {}; cur2 = 0; o1_2 = 0; o2_1 = {}; o2_2 = 0; sum_l = 0; sum_r = 0
ref = p.stats['ref_flops']
for k in range(len(g)):
    i, o = int(g.group_psi[k]), int(g.group_out[k])
    m, n = int(dl[keys[i][0]]), int(dr[keys[i][3]])
    q, r = int(dl[keys[o][0]]), int(dr[keys[o][3]])
    rows = g.member_row[g.group_begin[k]:g.group_begin[k+1]]
    lo = pi.lop[rows]; ro = pi.rop[rows]
    for b in np.unique(ro):
        if pi.kind_r[b] != 1:
            cur1[(i, b)] = 2*m*n*r
    cur2 += len(rows) * 2*q*r*m
    o1_2 += len(np.unique(ro)) * 2*q*r*m
    sum_l += (len(rows) - len(np.unique(ro))) * q*m
    for a in np.unique(lo):
        if pi.kind_l[a] != 1:
            o2_1[(i, a)] = 2*q*m*n
    o2_2 += len(np.unique(lo)) * 2*q*n*r
    sum_r += (len(rows) - len(np.unique(lo))) * r*n
c1 = sum(cur1.values()); x1 = sum(o2_1.values())
print(f"ref {ref/1e12:.3f} TF  current {(c1+cur2)/1e12:.3f} (P1 {c1/1e12:.3f} P2 {cur2/1e12:.3f})")
print(f"opt1 Lsum: {(c1+o1_2)/1e12:.3f} (P2 {o1_2/1e12:.3f}); sum-adds {sum_l/1e9:.2f} G elems")
print(f"opt2 X=LA, Rsum: {(x1+o2_2)/1e12:.3f} (P1 {x1/1e12:.3f}, P2 {o2_2/1e12:.3f}); sum-adds {sum_r/1e9:.2f} G elems")
print("distinct (i,rop)", len(cur1), "distinct (i,lop)", len(o2_1))
