"""A whole DMRG sweep of the reference, replayed through the device path.

tests/golden/sweep_*/iter_XX.npz (make_sweep_golden.py) hold, for every
two-site iteration of the reference's driver (driver.py _iterate), the
operators it built, the Lanczos starting vector it used and its energy.  Each
iteration is re-run here: native task generation, H_eff·ψ on the engine,
device Lanczos with the reference's tolerance — energies must agree within
1e-8 Eh (north star) and do within 1e-10 relative.
"""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN

ITERS = sorted(glob.glob(os.path.join(GOLDEN, "sweep_*", "iter_*.npz")))


def _load(path):
    from paper_2305_05581_b200.plan_input import PlanInput
    return PlanInput.load(path)


@pytest.mark.parametrize("path", ITERS, ids=[os.path.relpath(p, GOLDEN) for p in ITERS])
def test_sweep_iteration_grouping_cpu(path):
    """CPU: the native task generator and the oracle agree on every iteration."""
    from oracle import heff
    from paper_2305_05581_b200.plan import DevicePlan
    pi = _load(path)
    groups = heff.build_groups(pi)
    st = DevicePlan(pi, dry_run=True).stats
    assert st["groups"] == len(groups)
    assert st["members"] == sum(len(m) for _i, _o, m in groups)
    assert st["ref_flops"] == heff.ref_flops(pi, groups)


@pytest.mark.gpu
def test_sweep_energies_match_reference():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not ITERS:
        pytest.skip("no sweep fixture")
    from paper_2305_05581_b200.lanczos import lanczos_ground
    from paper_2305_05581_b200.plan import DevicePlan
    worst = 0.0
    for path in ITERS:
        pi = _load(path)
        m = pi.meta
        plan = DevicePlan(pi)
        out = plan.empty_vector()
        res = lanczos_ground(lambda v: plan.apply(v, out), m["guess"], tol=float(m["tol"]),
                             max_iter=int(m["max_iter"]))
        e_ref = float(m["energy"])
        err = abs(res.energy - e_ref)
        worst = max(worst, err)
        assert err <= 1e-8, (path, res.energy, e_ref)
        assert err <= 1e-10 * (1 + abs(e_ref)), (path, res.energy, e_ref)
        plan.close()
    print(f"{len(ITERS)} sweep iterations, worst |dE| = {worst:.2e}")
