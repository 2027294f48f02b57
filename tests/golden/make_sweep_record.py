"""Record the reference's configs[0] run: L=16 random-integral CAS, U(1)
two-site DMRG, D=256, 4 sweeps (BASELINE.json configs[0]).

Runs ONLY in the build container (imports the reference from
/root/reference/pkg/src).  The reference's own front door
``driver.py:356 solve`` runs unchanged; ``driver._iterate`` is wrapped only
to stream every SweepRecord (sweep, position, direction, energy, truncation
error, Lanczos iterations, wall seconds, converged) to a JSON-lines file as
it is produced, so a partial run still leaves a usable record.  The device
sweep (paper_2305_05581_b200.sweep) is run closed-loop on the same model
(integrals regenerated from the same seed by ``paper_2305_05581_b200.model``)
and compared record by record (tests/test_gpu_closed_sweep.py).

Usage:  python tests/golden/make_sweep_record.py [L] [D] [sweeps] [out.jsonl]
"""

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import sector_dmrg.driver as drv  # noqa: E402
from sector_dmrg.driver import SweepSchedule, solve  # noqa: E402

from make_golden import random_integral_model  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(
        HERE, f"sweep_record_L{n}_D{d}.jsonl")
    model_seed, run_seed, tol = 16, 42, 1e-10
    model = random_integral_model(n, model_seed)
    real = drv._iterate
    fh = open(out, "w")
    fh.write(json.dumps({"header": True, "L": n, "D": d, "sweeps": sweeps,
                         "model": "random_integral_model", "model_seed": model_seed,
                         "run_seed": run_seed, "lanczos_tol": tol,
                         "lanczos_max_iter": 300, "target": list(model.default_target()),
                         "generator": "tests/golden/make_sweep_record.py"}) + "\n")
    fh.flush()
    t_start = time.time()

    def _iterate(state, position, d_max, *a, **k):
        rec = real(state, position, d_max, *a, **k)
        fh.write(json.dumps({"sweep": rec.sweep, "position": rec.position,
                             "direction": rec.direction, "energy": rec.energy,
                             "truncation_error": rec.truncation_error,
                             "lanczos_iterations": rec.lanczos_iterations,
                             "wall_seconds": rec.wall_seconds, "converged": rec.converged,
                             "left_dim": state.left[position].basis.total_dim,
                             "right_dim": state.right[model.n_sites - position - 2].basis.total_dim,
                             "elapsed": time.time() - t_start}) + "\n")
        fh.flush()
        return rec

    drv._iterate = _iterate
    try:
        res = solve(model, SweepSchedule(n_sweeps=sweeps, d=d, lanczos_tol=tol,
                                         lanczos_max_iter=300), seed=run_seed)
    finally:
        drv._iterate = real
    fh.write(json.dumps({"footer": True, "energy": res.energy,
                         "sweep_final_energies": res.sweep_final_energies(),
                         "total_seconds": time.time() - t_start}) + "\n")
    fh.close()
    print(f"L={n} D={d}: final E {res.energy:.12f} in {time.time() - t_start:.0f}s -> {out}")


if __name__ == "__main__":
    main()
