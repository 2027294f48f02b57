"""Quick per-phase timing of one H_eff·ψ workload (experiments)."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2305_05581_b200.plan import DevicePlan
from paper_2305_05581_b200.workload import fill_arenas_device, synthetic_plan_input
L = int(sys.argv[1]) if len(sys.argv) > 1 else 30
D = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
pi = synthetic_plan_input(L, D)
al, ar = fill_arenas_device(pi)
plan = DevicePlan(pi, arena_l=al, arena_r=ar)
psi = torch.randn(plan.psi_size, dtype=torch.float64, device="cuda")
out = plan.empty_vector()
for _ in range(2):
    plan.apply(psi, out)
plan.set_timing(True)
res = []
for _ in range(3):
    plan.apply(psi, out)
    res.append(plan.last_timing())
m1 = min(r[0] for r in res); m2 = min(r[1] for r in res)
f1, f2 = res[0][2], res[0][3]
print(json.dumps({"lib": os.environ.get("SDMRG_LIB", "default"), "L": L, "D": D,
                  "ms": [round(m1, 2), round(m2, 2)], "tflops": [round(f1 / m1 / 1e9, 2), round(f2 / m2 / 1e9, 2)],
                  "total_ms": round(m1 + m2, 2), "ref_tflops": round(plan.stats["ref_flops"] / (m1 + m2) / 1e9, 2)}))
