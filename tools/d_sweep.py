"""configs[4] microbench: one H_eff·ψ of the L=30 CAS partition swept over
the bond dimension D (inputs resident, best of 3 after a warm-up), with the
grouped-GEMM work-list statistics (products, tiles, executed FLOPs per tile)
beside the engine's fraction of the live cuBLAS DGEMM peak.

Usage: python tools/d_sweep.py [L] [D,D,...] [out.jsonl]
"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2305_05581_b200.workload import synthetic_plan_input  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 30
ds = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "512,1024,2048,4096,8192").split(",")]
out = open(sys.argv[3], "w") if len(sys.argv) > 3 else None
peak = bench.dgemm_peak(torch)
for d in ds:
    pi = synthetic_plan_input(L, d)
    res = bench.scale_point(L, d, 0, peak)
    res.update({"dgemm_peak_tflops": peak, "max_sector": int(max(pi.dim_l.max(), pi.dim_r.max()))})
    line = json.dumps(res)
    print(line, flush=True)
    if out:
        out.write(line + "\n")
        out.flush()
