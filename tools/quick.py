"""Quick per-phase timing of one H_eff·ψ workload (experiments)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2305_05581_b200.plan import DevicePlan
from paper_2305_05581_b200.workload import fill_plan_arenas, synthetic_plan_input
L = int(sys.argv[1]) if len(sys.argv) > 1 else 30
D = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
NE = int(sys.argv[3]) if len(sys.argv) > 3 else None   # electrons (L=76: 113)
pi = synthetic_plan_input(L, D, n_elec=NE)
ws = int(os.environ.get("SDMRG_WS", "0"))
plan = DevicePlan(pi, empty_arenas=True, workspace_doubles=ws)
fill_plan_arenas(plan, pi)
psi = torch.randn(plan.psi_size, dtype=torch.float64, device="cuda")
out = plan.empty_vector()
for _ in range(2):
    plan.apply(psi, out)
plan.set_timing(True)
res = [None] * 3
for _ in range(3):
    plan.apply(psi, out)
    res[_] = plan.last_timing()
ms = [min(r[0][k] for r in res) for k in range(4)]
fl, by = res[0][1], res[0][2]
print(json.dumps({"lib": os.environ.get("SDMRG_LIB", "default"), "L": L, "D": D, "ws": ws,
                  "chunks": plan.stats["chunks"],
                  "ms": [round(x, 2) for x in ms],
                  "tflops": [round(f / max(m, 1e-9) / 1e9, 2) for f, m in zip(fl[1:3], ms[1:3])],
                  "combine_GBs": [round(by[k] / max(ms[k], 1e-9) / 1e6, 1) for k in (0, 3)],
                  "total_ms": round(sum(ms), 2),
                  "ref_tflops": round(plan.stats["ref_flops"] / sum(ms) / 1e9, 2)}))
