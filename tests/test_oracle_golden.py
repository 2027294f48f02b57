"""Pin the oracle and the native task generator to the reference's outputs.

CPU-only: the golden fixtures were produced by the reference itself
(tests/golden/make_golden.py).  The C++ task generation runs in dry-run mode
(no device) and must reproduce the reference grouping bit for bit.
"""

import numpy as np
import pytest

from oracle import heff, lanczos, renorm


def ref_groups(pi):
    m = pi.meta
    out = []
    gb = m["ref_group_begin"]
    for g in range(len(m["ref_group_psi"])):
        sl = slice(gb[g], gb[g + 1])
        out.append((int(m["ref_group_psi"][g]), int(m["ref_group_out"][g]),
                    list(zip(m["ref_member_loff"][sl].tolist(),
                             m["ref_member_roff"][sl].tolist(),
                             m["ref_member_scale"][sl].tolist()))))
    return out


def oracle_groups_as_offsets(pi, groups):
    keys = pi.psi_keys()
    out = []
    for i, o, members in groups:
        jl, jr = keys[i][0], keys[i][3]
        out.append((i, o, [(int(pi.blk_off_l[pi.lop[t], jl]), int(pi.blk_off_r[pi.rop[t], jr]), s)
                           for t, s in members]))
    return out


def test_psi_layout_matches_reference(golden):
    name, pi = golden
    keys = pi.psi_keys()
    ref = pi.meta["ref_psi_keys"]
    assert len(keys) == ref.shape[0]
    for (jl, s1, s2, jr), rk in zip(keys, ref):
        got = np.concatenate([pi.qn_l[jl], pi.site_qn[s1], pi.site_qn[s2], pi.qn_r[jr]])
        assert np.array_equal(got, rk.ravel())
    assert pi.psi_offsets(keys)[-1] == pi.meta["psi"].size


def test_oracle_grouping_bit_exact(golden):
    name, pi = golden
    mine = oracle_groups_as_offsets(pi, heff.build_groups(pi))
    assert mine == ref_groups(pi)


def test_oracle_flops_match_plan_flops(golden):
    name, pi = golden
    assert heff.ref_flops(pi, heff.build_groups(pi)) == int(pi.meta["ref_flops"])


def test_oracle_apply_matches_reference(golden):
    name, pi = golden
    sigma = heff.apply_heff(pi, pi.meta["psi"])
    ref = pi.meta["sigma"]
    scale = 1.0 + np.max(np.abs(ref))
    assert np.max(np.abs(sigma - ref)) <= 1e-13 * scale


def test_oracle_lanczos_matches_reference(golden):
    name, pi = golden
    if pi.meta["lanczos_iterations"] > 150:
        # the pure-Python oracle would take minutes here; the device Lanczos
        # checks this case against the reference energy directly
        pytest.skip("oracle Lanczos restatement pinned on the smaller cases")
    groups = heff.build_groups(pi)
    res = lanczos.lanczos_ground(lambda v: heff.apply_heff(pi, v, groups), pi.meta["psi"],
                                 tol=1e-12, max_iter=300)
    e_ref = float(pi.meta["lanczos_energy"])
    assert abs(res.energy - e_ref) <= 1e-10 * (1 + abs(e_ref))
    assert res.converged == bool(pi.meta["lanczos_converged"])


def test_native_task_generation_bit_exact(golden):
    """C++ sdmrg_plan_build (dry run) reproduces blocks.py:503 grouping."""
    from paper_2305_05581_b200.plan import DevicePlan
    name, pi = golden
    plan = DevicePlan(pi, keep_groups=True, dry_run=True)
    assert plan.stats["ref_flops"] == int(pi.meta["ref_flops"])
    assert plan.psi_size == pi.meta["psi"].size
    g = plan.groups()
    keys = pi.psi_keys()
    assert np.array_equal(plan.keys, np.array(keys, np.int32).reshape(-1, 4))
    mine = []
    for k in range(len(g)):
        i, o = int(g.group_psi[k]), int(g.group_out[k])
        jl, jr = keys[i][0], keys[i][3]
        sl = slice(g.group_begin[k], g.group_begin[k + 1])
        mine.append((i, o, [(int(pi.blk_off_l[pi.lop[t], jl]), int(pi.blk_off_r[pi.rop[t], jr]),
                             float(s)) for t, s in zip(g.member_row[sl], g.member_scale[sl])]))
    assert mine == ref_groups(pi)


def test_native_sharding_partitions_members(golden):
    from paper_2305_05581_b200.plan import DevicePlan
    name, pi = golden
    total = DevicePlan(pi, dry_run=True).stats["members"]
    for world in (2, 3, 4):
        # dry-run stats count members globally; local counts come from a real
        # build, so here check the global invariants are rank independent
        for rank in range(world):
            st = DevicePlan(pi, dry_run=True, rank=rank, world=world).stats
            assert st["members"] == total


def renorm_inputs(pi):
    m = pi.meta
    nc = pi.ncomp
    layout = {}
    for row in m["renorm_fused_layout"]:
        layout[(tuple(row[:nc]), tuple(row[nc:2 * nc]))] = int(row[2 * nc])
    fdims = {tuple(q): int(d) for q, d in zip(m["renorm_fused_qn"], m["renorm_fused_dim"])}
    keys = pi.psi_keys()
    offs = pi.psi_offsets(keys)
    vec = m["lanczos_vector"]
    blocks = {}
    for i, (jl, s1, s2, jr) in enumerate(keys):
        k = (tuple(pi.qn_l[jl]), tuple(pi.site_qn[s1]), tuple(pi.site_qn[s2]), tuple(pi.qn_r[jr]))
        blocks[k] = vec[offs[i]:offs[i + 1]].reshape(int(pi.dim_l[jl]), int(pi.dim_r[jr]))
    return blocks, layout, fdims


def test_oracle_renorm_truncation_matches_reference(golden):
    name, pi = golden
    blocks, layout, fdims = renorm_inputs(pi)
    rho = renorm.rdm_blocks(renorm.rdm_slabs(blocks, "L", layout, fdims))
    kept, trunc, w = renorm.truncate(renorm.rdm_eigensystem(rho), int(pi.meta["renorm_d"]))
    assert abs(trunc - float(pi.meta["renorm_trunc"])) <= 1e-12
    got = sorted((q, len(idx)) for q, idx in kept.items())
    ref = sorted((tuple(q), int(d)) for q, d in zip(pi.meta["renorm_kept_qn"],
                                                    pi.meta["renorm_kept_dim"]))
    assert got == ref


def test_oracle_rotation_matches_reference(golden):
    """W^T H W with the reference's own W reproduces its rotated H."""
    name, pi = golden
    m = pi.meta
    fdims = {tuple(q): int(d) for q, d in zip(m["renorm_fused_qn"], m["renorm_fused_dim"])}
    kdims = {tuple(q): int(d) for q, d in zip(m["renorm_kept_qn"], m["renorm_kept_dim"])}
    w, pos = {}, 0
    for q in m["renorm_w_qn"]:
        q = tuple(q)
        n = fdims[q] * kdims[q]
        w[q] = m["renorm_w_data"][pos:pos + n].reshape(fdims[q], kdims[q])
        pos += n
    h, pos = {}, 0
    for q in m["renorm_h_qn"]:
        q = tuple(q)
        n = fdims[q] * fdims[q]
        h[(q, q)] = m["renorm_h_data"][pos:pos + n].reshape(fdims[q], fdims[q])
        pos += n
    rot = renorm.rotate_op(h, w)
    pos = 0
    for q in m["renorm_hrot_qn"]:
        q = tuple(q)
        n = kdims[q] * kdims[q]
        ref = m["renorm_hrot_data"][pos:pos + n].reshape(kdims[q], kdims[q])
        pos += n
        assert np.max(np.abs(rot[(q, q)] - ref)) <= 1e-12 * (1 + np.max(np.abs(ref)))


def _rows_subset(pi, sel):
    """The same partition with only table rows ``sel`` (edge cases)."""
    import copy
    q = copy.copy(pi)
    for name in ("lop", "rop", "alpha", "e_l", "site1_dst", "site1_val", "site2_dst",
                 "site2_val", "row_map"):
        setattr(q, name, getattr(pi, name)[sel])
    q.meta = dict(pi.meta)
    return q.normalized()


def test_native_task_generation_edge_cases(golden):
    """No rows -> no members and zero FLOPs; a single row -> the oracle's
    grouping of that row; zero coefficients are dropped (blocks.py:561)."""
    from paper_2305_05581_b200.plan import DevicePlan
    _name, pi = golden
    empty = _rows_subset(pi, np.zeros(pi.nrows, bool))
    st = DevicePlan(empty, dry_run=True).stats
    assert st["members"] == 0 and st["ref_flops"] == 0 and st["groups"] == 0
    assert st["psi_size"] == pi.meta["psi"].size
    one = _rows_subset(pi, np.arange(pi.nrows) == 1)
    plan = DevicePlan(one, dry_run=True, keep_groups=True)
    assert plan.stats["members"] == sum(len(m) for _i, _o, m in heff.build_groups(one))
    zero = _rows_subset(pi, np.ones(pi.nrows, bool))
    zero.alpha = np.zeros_like(zero.alpha)
    assert DevicePlan(zero.normalized(), dry_run=True).stats["members"] == 0


def test_oracle_threaded_apply_matches_serial(golden):
    """The pooled port (bench CPU baseline, the reference's worker-pool
    semantics) computes the same σ as the serial restatement."""
    _name, pi = golden
    groups = heff.build_groups(pi)
    a = heff.apply_groups(pi, groups, pi.meta["psi"])
    b = heff.apply_groups_threaded(pi, groups, pi.meta["psi"], workers=4)
    assert np.max(np.abs(a - b)) <= 1e-13 * (1.0 + np.max(np.abs(a)))
