"""Phase-2 σ tiles: FLOP-weighted distribution of 8-block tile shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from collections import Counter
from paper_2305_05581_b200.plan import DevicePlan
from paper_2305_05581_b200.workload import synthetic_plan_input
L, D = int(sys.argv[1]), int(sys.argv[2])
pi = synthetic_plan_input(L, D)
p = DevicePlan(pi, dry_run=True, keep_groups=True)
g = p.groups()
keys = np.array(pi.psi_keys())
dl, dr = pi.dim_l.astype(np.int64), pi.dim_r.astype(np.int64)
kout = {}
for k in range(len(g)):
    i, o = int(g.group_psi[k]), int(g.group_out[k])
    rows = g.member_row[g.group_begin[k]:g.group_begin[k + 1]]
    kout[o] = kout.get(o, 0) + len(np.unique(pi.rop[rows])) * int(dl[keys[i][0]])
c = Counter(); tot = 0; work = 0
for o, K in kout.items():
    q, r = int(dl[keys[o][0]]), int(dr[keys[o][3]])
    for r0 in range(0, q, 64):
        for c0 in range(0, r, 64):
            tm, tn = min(64, q - r0), min(64, r - c0)
            f = 2 * tm * tn * K
            c[((tm + 7) // 8, (tn + 7) // 8)] += f; tot += f
            work += 2 * ((tm + 7) // 8 * 8) * ((tn + 7) // 8 * 8) * K
print(f"L={L} D={D}: phase-2 flops {tot/1e12:.3f} T, 8-pad eff {tot/work:.3f}")
acc = 0
for (mb, nb), f in sorted(c.items(), key=lambda x: -x[1])[:20]:
    acc += f
    print(f"  {mb}x{nb} blocks: {f/tot:.3f} (cum {acc/tot:.3f})")
