"""Strong-scaling estimate on one GPU: time every rank's shard of the plan
(world = N) one after another; efficiency ~ t_full / (N * max_rank t)."""
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
psi = None


def timed(plan, reps=3):
    global psi
    if psi is None:
        psi = torch.randn(plan.psi_size, dtype=torch.float64, device="cuda")
    out = plan.empty_vector()
    plan.apply(psi, out)
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); plan.apply(psi, out); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


full = DevicePlan(pi, arena_l=al, arena_r=ar)
t_full = timed(full)
full.close()
res = {"L": L, "D": D, "full_ms": round(t_full, 2)}
for world in (2, 4, 8):
    ts = []
    for rank in range(world):
        p = DevicePlan(pi, arena_l=al, arena_r=ar, rank=rank, world=world)
        ts.append(timed(p))
        p.close()
    res[f"N{world}"] = {"max_ms": round(max(ts), 2), "min_ms": round(min(ts), 2),
                        "efficiency": round(t_full / (world * max(ts)), 3)}
print(json.dumps(res))
