"""Where the time of a device Lanczos iteration goes (bench workload)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2305_05581_b200 import lanczos as lz
from paper_2305_05581_b200.plan import DevicePlan
from paper_2305_05581_b200.workload import fill_arenas_device, synthetic_plan_input
L = int(sys.argv[1]) if len(sys.argv) > 1 else 30
D = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
pi = synthetic_plan_input(L, D)
al, ar = fill_arenas_device(pi)
plan = DevicePlan(pi, arena_l=al, arena_r=ar)
psi = torch.randn(plan.psi_size, dtype=torch.float64, device="cuda")
buf = plan.empty_vector()
acc = {"apply": 0.0, "other": 0.0}
def apply_op(v):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = plan.apply(v, buf)
    torch.cuda.synchronize(); acc["apply"] += time.perf_counter() - t0
    return r
for rep in range(2):
    acc["apply"] = 0.0
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = lz.lanczos_ground(apply_op, psi, tol=0.0, max_iter=10)
    torch.cuda.synchronize(); wall = time.perf_counter() - t0
    print(f"rep {rep}: wall {wall*1e3:.1f} ms, applies {acc['apply']*1e3:.1f} ms, "
          f"other {(wall - acc['apply'])*1e3:.1f} ms over {res.iterations} iterations")
# vector algebra alone
basis = lz.KrylovBasis(plan.psi_size, psi.device)
for i in range(10):
    lz._axpby(1.0, psi, 0.0, basis.append_slot(), torch.cuda.current_stream().cuda_stream)
w = psi.clone()
s = torch.cuda.current_stream().cuda_stream
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10):
    basis.project_out(w, s)
torch.cuda.synchronize()
print(f"project_out over 10 vectors: {(time.perf_counter() - t0) * 100:.2f} ms each")

# per-call timing of the loop's pieces (synchronized)
from collections import defaultdict
tm = defaultdict(float)
def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize(); tm[name] += time.perf_counter() - t0
        return r
    return w
lz.KrylovBasis.append_slot = timed("append_slot", lz.KrylovBasis.append_slot)
lz.KrylovBasis.project_out = timed("project_out", lz.KrylovBasis.project_out)
lz.KrylovBasis.combine = timed("combine", lz.KrylovBasis.combine)
lz._nrm2 = timed("nrm2", lz._nrm2)
lz._axpby = timed("axpby", lz._axpby)
acc["apply"] = 0.0
torch.cuda.synchronize(); t0 = time.perf_counter()
res = lz.lanczos_ground(apply_op, psi, tol=0.0, max_iter=10)
torch.cuda.synchronize(); wall = time.perf_counter() - t0
print(f"instrumented: wall {wall*1e3:.1f} ms, applies {acc['apply']*1e3:.1f} ms;",
      ", ".join(f"{k} {v*1e3:.1f} ms" for k, v in tm.items()))
