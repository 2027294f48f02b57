"""Record a whole DMRG sweep of the reference, iteration by iteration.

Runs ONLY in the build container (imports the reference from
/root/reference/pkg/src).  The reference's own driver (driver.py solve ->
_iterate) runs unchanged; build_plan and lanczos_ground are wrapped so that
every two-site iteration is captured: the compact PlanInput of the operators
the reference built at that position, the Lanczos starting vector it used
(White's prediction or the seeded random fallback), and its energy /
convergence.  The GPU test replays every iteration through the device path
(task generation + H_eff·ψ + device Lanczos) and compares the energies
(north star: sweep energies within 1e-8 Eh).

Usage:  python tests/golden/make_sweep_golden.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import sector_dmrg.driver as drv  # noqa: E402
from sector_dmrg.blocks import materialize_aux  # noqa: E402
from sector_dmrg.driver import SweepSchedule, solve  # noqa: E402

from paper_2305_05581_b200.plan_input import compile_reference_plan  # noqa: E402
from make_golden import random_integral_model  # noqa: E402


def main(name="sweep_ints6_d16", n=6, seed=21, d=16, sweeps=2):
    model = random_integral_model(n, seed)
    captured = []
    real_build, real_lanczos = drv.build_plan, drv.lanczos_ground

    def build_plan(model_, table, left, right, struct, aux_mats=None):
        aux = materialize_aux(table, left, right)
        pi = compile_reference_plan(model_, table, left, right, struct, aux)
        captured.append({"pi": pi})
        return real_build(model_, table, left, right, struct, aux)

    def lanczos_ground(apply_op, guess, tol=1e-12, max_iter=200):
        res = real_lanczos(apply_op, guess, tol=tol, max_iter=max_iter)
        captured[-1].update(guess=np.asarray(guess, float).copy(), energy=res.energy,
                            converged=res.converged, iterations=res.iterations,
                            tol=tol, max_iter=max_iter)
        return res

    drv.build_plan, drv.lanczos_ground = build_plan, lanczos_ground
    try:
        res = solve(model, SweepSchedule(n_sweeps=sweeps, d=d, lanczos_tol=1e-10), seed=5)
    finally:
        drv.build_plan, drv.lanczos_ground = real_build, real_lanczos
    out = os.path.join(HERE, name)
    os.makedirs(out, exist_ok=True)
    recs = res.state.records
    assert len(recs) == len(captured), (len(recs), len(captured))
    for k, (cap, rec) in enumerate(zip(captured, recs)):
        cap["pi"].save(os.path.join(out, f"iter_{k:02d}.npz"), guess=cap["guess"],
                       energy=np.float64(cap["energy"]), converged=np.int64(cap["converged"]),
                       iterations=np.int64(cap["iterations"]), tol=np.float64(cap["tol"]),
                       max_iter=np.int64(cap["max_iter"]), sweep=np.int64(rec.sweep),
                       position=np.int64(rec.position),
                       direction=np.array(rec.direction))
    print(f"{name}: {len(captured)} iterations, final E {recs[-1].energy:.12f} -> {out}")


if __name__ == "__main__":
    main()
