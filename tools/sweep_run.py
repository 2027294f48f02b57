"""Closed-loop device DMRG run (paper_2305_05581_b200.driver.solve) with
per-iteration records, seconds per sweep and, when a reference record of
the same run exists (tests/golden/make_sweep_record.py), the per-iteration
energy differences up to the first degenerate-multiplet cut.

  python tools/sweep_run.py L D SWEEPS [--model-seed 16] [--run-seed 42]
         [--tol 1e-10] [--scale 0.2] [--core 0.3] [--ref tests/golden/...jsonl]
         [--out gpurun_out/sweep_L16_D256.jsonl]
"""
import argparse
import json
import os

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("L", type=int)
    ap.add_argument("D", type=int)
    ap.add_argument("sweeps", type=int)
    ap.add_argument("--model-seed", type=int, default=16)
    ap.add_argument("--run-seed", type=int, default=42)
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--max-iter", type=int, default=300)
    ap.add_argument("--scale", type=float, default=0.2)
    ap.add_argument("--core", type=float, default=0.3)
    ap.add_argument("--ref", default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    from paper_2305_05581_b200 import _lib
    from paper_2305_05581_b200 import driver as drv
    from paper_2305_05581_b200 import model as M
    t0 = time.perf_counter()
    mm = M.Model(M.random_integrals(a.L, a.model_seed, scale=a.scale, core=a.core))
    sch = drv.SweepSchedule(n_sweeps=a.sweeps, d=a.D, lanczos_tol=a.tol,
                            lanczos_max_iter=a.max_iter)
    out = open(a.out, "w") if a.out else None
    l0 = _lib.launch_count()
    tw = time.perf_counter()
    st = drv.warmup(mm, sch, seed=a.run_seed)
    torch.cuda.synchronize()
    t_warm = time.perf_counter() - tw
    sweep_t = []
    for s in range(1, a.sweeps + 1):
        ts = time.perf_counter()
        lo, hi = drv.sweep_positions(mm)
        d = sch.d_for(s)
        for p in range(lo, hi + 1):
            drv._iterate(st, p, d, sch, s, "R")
        for p in range(hi, lo - 1, -1):
            drv._iterate(st, p, d, sch, s, "L")
        st.sweeps_done = s
        torch.cuda.synchronize()
        sweep_t.append(time.perf_counter() - ts)
    ref = None
    if a.ref and os.path.exists(a.ref):
        rows = [json.loads(x) for x in open(a.ref)]
        ref = [r for r in rows[1:] if "sweep" in r]
    worst, compared, first_tie = 0.0, 0, None
    for i, r in enumerate(st.records):
        line = {"sweep": r.sweep, "position": r.position, "direction": r.direction,
                "energy": r.energy, "truncation_error": r.truncation_error,
                "lanczos_iterations": r.lanczos_iterations, "converged": r.converged,
                "wall_seconds": r.wall_seconds, **r.timing}
        if ref is not None and i < len(ref):
            line["ref_energy"] = ref[i]["energy"]
            line["dE"] = r.energy - ref[i]["energy"]
            if first_tie is None and st.warmup_ties == 0:
                worst = max(worst, abs(line["dE"]))
                compared += 1
        if first_tie is None and r.timing.get("tie_at_cut"):
            first_tie = i
        if out:
            out.write(json.dumps(line) + "\n")
    summ = {"summary": True, "L": a.L, "D": a.D, "sweeps": a.sweeps,
            "final_energy": st.records[-1].energy, "warmup_s": t_warm,
            "sec_per_sweep": sweep_t, "iterations": len(st.records),
            "warmup_ties": st.warmup_ties, "first_tie_record": first_tie,
            "ref_compared": compared, "ref_worst_dE": worst,
            "kernel_launches": _lib.launch_count() - l0,
            "breakdown_s": {k: sum(r.timing.get(k, 0.0) for r in st.records if r.sweep > 0)
                            for k in ("table_s", "aux_s", "plan_s", "lanczos_s", "renorm_s",
                                      "predict_s")},
            "total_s": time.perf_counter() - t0}
    if out:
        out.write(json.dumps(summ) + "\n")
        out.close()
    print(json.dumps(summ))


if __name__ == "__main__":
    main()
