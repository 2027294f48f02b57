"""The closed-loop driver's host logic on CPU (no GPU in the build container).

The driver's three device hooks are replaced by checkers (tests/cpu_engine.py:
numpy grouped GEMM, the oracle's H_eff·ψ and Lanczos); everything else —
factorization, store layout, Kronecker placements and parity dressings of
the fused enlargement + rotation, complementary-operator sums, ρ, top-D
selection, White's prediction, the warm-up/sweep schedule — is the product
code.  Compared iteration by iteration with the reference's own run
(tests/golden/make_sweep_golden.py: L=6, D=16, 2 sweeps): energies within
1e-8 Eh (north star), here ~1e-14 — up to and including the first
iteration whose truncation splits an exactly degenerate multiplet (there
the reference's kept state is chosen by its LAPACK rounding noise; see
driver.select_states).
"""

import glob
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def test_closed_loop_cpu_emulation_matches_reference_L6_D16():
    from cpu_engine import emulated
    from paper_2305_05581_b200 import driver as drv
    from paper_2305_05581_b200 import model as M
    files = sorted(glob.glob(os.path.join(HERE, "golden", "sweep_ints6_d16", "iter_*.npz")))
    ref = [np.load(f) for f in files]
    mm = M.Model(M.random_integrals(6, 21))
    sch = drv.SweepSchedule(n_sweeps=2, d=16, lanczos_tol=1e-10)
    with emulated() as eng:
        res = drv.solve(mm, sch, seed=5, engine=eng)
    assert len(res.records) == len(ref) == 14
    assert res.state.warmup_ties == 0
    for a, z in zip(res.records, ref):
        assert (a.sweep, a.position, a.direction) == (int(z["sweep"]), int(z["position"]),
                                                       str(z["direction"]))
        assert abs(a.energy - float(z["energy"])) <= 1e-8
        assert a.lanczos_iterations == int(z["iterations"])
        if a.timing["tie_at_cut"]:
            break


def test_select_states_flags_ties():
    from paper_2305_05581_b200.driver import select_states
    # an exactly degenerate doublet split by the cut: the raw floats decide
    # (as in the reference) and the split is flagged
    scores = {(1, 1): np.array([2.0, 1.0 + 1e-15]), (1, -1): np.array([1.0])}
    info = {}
    kept = select_states(scores, 2, info)
    assert kept == {(1, 1): [0, 1]} and info["tie_at_cut"]
    info = {}
    kept = select_states({(0, 0): np.array([3.0, 2.0]), (1, 1): np.array([1.0])}, 2, info)
    assert kept == {(0, 0): [0, 1]} and not info["tie_at_cut"]
