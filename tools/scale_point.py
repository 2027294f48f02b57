"""One bench scale point (empty plan arenas filled in place): python
tools/scale_point.py L D [n_elec].  Prints the operator sizes first and
refuses workloads whose padded arenas would not leave room in HBM."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2305_05581_b200.workload import synthetic_plan_input

L, D = int(sys.argv[1]), int(sys.argv[2])
n_elec = int(sys.argv[3]) if len(sys.argv) > 3 else None
pi = synthetic_plan_input(L, D, n_elec=n_elec)
gb = (pi.meta["arena_size_l"] + pi.meta["arena_size_r"]) * 8 / 1e9
print(json.dumps({"L": L, "D": D, "rows": pi.nrows, "sectors": [len(pi.dim_l), len(pi.dim_r)],
                  "max_dim": int(max(pi.dim_l.max(), pi.dim_r.max())),
                  "arena_gb_dense": round(gb, 1), "target": pi.target.tolist()}), flush=True)
if gb > 140:
    sys.exit("operators too large for one GPU")
import torch  # noqa: E402
import bench  # noqa: E402
peak = bench.dgemm_peak(torch)
print(json.dumps(bench.scale_point(L, D, 0, peak, n_elec=n_elec)))
