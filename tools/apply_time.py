"""Whole-apply device time (events around plan.apply, no per-phase events)."""
import json, os, sys
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
for _ in range(3):
    plan.apply(psi, out)
ts = []
for _ in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); plan.apply(psi, out); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
best = min(ts)
print(json.dumps({"lib": os.environ.get("SDMRG_LIB", "default"), "L": L, "D": D,
                  "apply_ms": [round(t, 2) for t in ts], "best_ms": round(best, 2),
                  "ref_tflops": round(plan.stats["ref_flops"] / best / 1e9, 2),
                  "exec_tflops": round(plan.stats["exec_flops"] / best / 1e9, 2)}))
