"""Generate the golden fixtures from the reference itself.

Runs ONLY in the build container (imports the reference package from
/root/reference/pkg/src).  For each case it builds a two-site partition with
the reference's own model / factorize / block stores, then records:

  * the compact PlanInput (compile_reference_plan of the reference objects);
  * the reference plan's grouping: per group (ψ key, out key) and per member
    (L block arena offset, R block arena offset, scale) — resolved by object
    identity from the reference's PlanGroup members (blocks.py:565);
  * plan.flops (blocks.py:575), a seeded ψ and the reference's
    apply_effective_hamiltonian output (dmrg.py:107);
  * the reference's lanczos_ground on that operator (dmrg.py:43);
  * a renormalization step: reference renormalize (dmrg.py:335) outputs —
    kept sector dims, truncation error, W, and the rotated H operator.

Usage:  python tests/golden/make_golden.py [case ...]
"""

import os
import sys
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from sector_dmrg.blocks import (  # noqa: E402
    SuperblockWavefunction, build_plan, enlarge_block, materialize_aux, site_store)
from sector_dmrg.dmrg import apply_effective_hamiltonian, lanczos_ground, renormalize  # noqa: E402
from sector_dmrg.driver import SweepSchedule, solve  # noqa: E402
from sector_dmrg.model import Integrals, ModelSpec, build_model, factorize, model_from_integrals  # noqa: E402
from sector_dmrg.ttcache import Arena  # noqa: E402

from paper_2305_05581_b200.plan_input import compile_reference_plan  # noqa: E402


def exact_stores(model, p):
    """tests/test_dmrg.py:27 exact_stores (reference test helper)."""
    n = model.n_sites
    left = site_store(model, 0, "L")
    for s in range(1, p):
        left = enlarge_block(model, left, s)
    right = site_store(model, n - 1, "R")
    for s in range(n - 2, p + 1, -1):
        right = enlarge_block(model, right, s)
    return left, right


def random_integral_model(n, seed):
    rng = np.random.default_rng(seed)
    t = rng.standard_normal((n, n))
    t = (t + t.T) / 2
    v = 0.2 * rng.standard_normal((n, n, n, n))
    v = 0.5 * (v + v.transpose(3, 2, 1, 0))        # hermitian: V_ijkl = V_lkji
    two = {(i, j, k, l): float(v[i, j, k, l]) for i in range(n) for j in range(n)
           for k in range(n) for l in range(n)}
    return model_from_integrals(ModelSpec("integral-file", path="synthetic"),
                                Integrals(n, t, two, 0.3))


def case_exact(name, model, p, target):
    left, right = exact_stores(model, p)
    return name, model, p, left, right, tuple(target)


def case_truncated(name, model, d, sweeps, p):
    res = solve(model, SweepSchedule(n_sweeps=sweeps, d=d, lanczos_tol=1e-10), seed=42)
    st = res.state
    n = model.n_sites
    return name, model, p, st.left[p], st.right[n - p - 2], st.target


def record(name, model, p, left, right, target, seed=7):
    table = factorize(model, model.partition_at(p))
    struct = SuperblockWavefunction(left.basis, model.local.basis, right.basis, target)
    aux = materialize_aux(table, left, right)
    plan = build_plan(model, table, left, right, struct, aux)
    pi = compile_reference_plan(model, table, left, right, struct, aux)
    pl, pr = pi.meta["packers"]
    key_index = {k: i for i, k in enumerate(struct.keys)}
    g_psi, g_out, g_begin, m_loff, m_roff, m_scale = [], [], [0], [], [], []
    for grp in plan.groups:
        g_psi.append(key_index[grp.psi_key])
        g_out.append(key_index[grp.out_key])
        for lblk, rblk, s in grp.members:
            m_loff.append(pl.by_id[id(lblk)])
            m_roff.append(pr.by_id[id(rblk)])
            m_scale.append(s)
        g_begin.append(len(m_scale))

    rng = np.random.default_rng(seed)
    psi = struct.copy()
    psi.random_fill(rng)
    out = struct.copy()
    out.zero_fill()
    locks = {k: threading.Lock() for k in struct.keys}
    apply_effective_hamiltonian(plan, psi, out, locks=locks,
                                arenas=[Arena(plan.staging_doubles * 8)])

    work = struct.copy().zero_fill()
    res_out = struct.copy().zero_fill()

    def apply_op(vec):
        work.from_vector(vec)
        for k in res_out.keys:
            res_out.blocks[k][...] = 0.0
        apply_effective_hamiltonian(plan, work, res_out, locks=locks,
                                    arenas=[Arena(plan.staging_doubles * 8)])
        return res_out.to_vector()

    lz = lanczos_ground(apply_op, psi.to_vector(), tol=1e-12, max_iter=300)

    extra = dict(
        ref_group_psi=np.array(g_psi, np.int64), ref_group_out=np.array(g_out, np.int64),
        ref_group_begin=np.array(g_begin, np.int64), ref_member_loff=np.array(m_loff, np.int64),
        ref_member_roff=np.array(m_roff, np.int64), ref_member_scale=np.array(m_scale),
        ref_flops=np.int64(plan.flops), psi=psi.to_vector(), sigma=out.to_vector(),
        lanczos_energy=np.float64(lz.energy), lanczos_iterations=np.int64(lz.iterations),
        lanczos_converged=np.int64(lz.converged), lanczos_vector=lz.vector,
        ref_psi_keys=np.array([[list(q) for q in k] for k in struct.keys], np.int64),
    )

    # renormalization of the left block at this partition with the ground state
    gs = struct.copy()
    gs.from_vector(lz.vector)
    d_keep = max(1, (left.basis.total_dim * model.local.dim) // 2)
    rr = renormalize(model, gs, "L", left, p, d_keep)
    fused = enlarge_block(model, left, p).fused
    extra.update(
        renorm_d=np.int64(d_keep),
        renorm_trunc=np.float64(rr.truncation_error),
        renorm_kept_qn=np.array([q for q, _ in rr.store.basis.entries], np.int64),
        renorm_kept_dim=np.array([d for _, d in rr.store.basis.entries], np.int64),
        renorm_fused_layout=np.array([list(qa) + list(qb) + [off]
                                      for (qa, qb), off in sorted(fused.layout.items())],
                                     np.int64),
        renorm_fused_qn=np.array([q for q, _ in fused.basis.entries], np.int64),
        renorm_fused_dim=np.array([d for _, d in fused.basis.entries], np.int64),
    )
    wq = sorted(rr.transform.blocks)
    extra["renorm_w_qn"] = np.array([k[0] for k in wq], np.int64)
    extra["renorm_w_data"] = np.concatenate([rr.transform.blocks[k].ravel() for k in wq])
    # enlarged H and its rotation (the store's H after renormalize)
    enl = enlarge_block(model, left, p)
    hk = sorted(enl.ops[("H",)].blocks)
    extra["renorm_h_qn"] = np.array([k[0] for k in hk], np.int64)
    extra["renorm_h_data"] = np.concatenate([enl.ops[("H",)].blocks[k].ravel() for k in hk])
    hk2 = sorted(rr.store.ops[("H",)].blocks)
    extra["renorm_hrot_qn"] = np.array([k[0] for k in hk2], np.int64)
    extra["renorm_hrot_data"] = np.concatenate(
        [rr.store.ops[("H",)].blocks[k].ravel() for k in hk2])

    path = os.path.join(HERE, f"{name}.npz")
    pi.save(path, **extra)
    print(f"{name}: rows {pi.nrows} psi {psi.size()} groups {len(plan.groups)} "
          f"members {len(m_scale)} flops {plan.flops} E {lz.energy:.12f} "
          f"iters {lz.iterations} trunc {rr.truncation_error:.3e} -> {path}")


CASES = {
    "heis6_p2": lambda: case_exact("heis6_p2", build_model(ModelSpec("heisenberg-chain", n=6)),
                                   2, (0,)),
    "hub4_p1": lambda: case_exact("hub4_p1", build_model(ModelSpec("hubbard-chain", n=4, t=1.0,
                                                                   u=2.0)), 1, (4, 0)),
    "ints4_p1": lambda: case_exact("ints4_p1", random_integral_model(4, 11), 1, (4, 0)),
    "ints6_d24_p2": lambda: case_truncated("ints6_d24_p2", random_integral_model(6, 12), 24, 1, 2),
    # larger truncated case: many sectors, bilinear member blocks, split groups
    "ints7_d32_p2": lambda: case_truncated("ints7_d32_p2", random_integral_model(7, 13), 32, 1, 2),
}


def main():
    names = sys.argv[1:] or list(CASES)
    for name in names:
        record(*CASES[name]())


if __name__ == "__main__":
    main()
