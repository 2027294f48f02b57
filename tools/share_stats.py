"""Sharing structure of H_eff members: how many members of one (group, right
op) / (group, left op) pair exist, split by identity / general operators."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from collections import Counter
import numpy as np
from paper_2305_05581_b200.plan import DevicePlan
from paper_2305_05581_b200.workload import synthetic_plan_input
L, D = int(sys.argv[1]), int(sys.argv[2])
pi = synthetic_plan_input(L, D)
p = DevicePlan(pi, dry_run=True, keep_groups=True)
g = p.groups()
keys = np.array(pi.psi_keys())
dl, dr = pi.dim_l, pi.dim_r
byr = Counter(); byl = Counter(); fl_r = Counter(); fl_l = Counter()
for k in range(len(g)):
    i, o = int(g.group_psi[k]), int(g.group_out[k])
    m = int(dl[keys[i][0]]); q = int(dl[keys[o][0]]); r = int(dr[keys[o][3]]); n = int(dr[keys[i][3]])
    rows = g.member_row[g.group_begin[k]:g.group_begin[k + 1]]
    for b, c in Counter(pi.rop[rows].tolist()).items():
        tag = "Rid" if pi.kind_r[b] == 1 else "Rgen"
        byr[(tag, min(c, 9))] += 1
        fl_r[tag] += c * 2 * q * r * m
    for a, c in Counter(pi.lop[rows].tolist()).items():
        tag = "Lid" if pi.kind_l[a] == 1 else "Lgen"
        byl[(tag, min(c, 9))] += 1
        fl_l[tag] += c * 2 * q * r * n
print("phase-2 member flops by rop kind (TF):", {k: v / 1e12 for k, v in fl_r.items()})
print("(group, rop) multiplicity:", sorted(byr.items()))
print("(group, lop) multiplicity:", sorted(byl.items()))
print("member flops by lop kind (TF):", {k: v / 1e12 for k, v in fl_l.items()})
