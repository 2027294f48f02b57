"""Multi-GPU host logic on CPU: world-size-2 gloo ranks.

Each rank takes its ψ-sector shard from the native task generator (dry run,
no device), computes its partial σ with the oracle restricted to that shard,
and the gloo all-reduce of the partials must equal the reference's full σ
(the NCCL all-reduce of bench.py / the multi-GPU apply does the same on the
device).  Also: the shards partition the ψ keys and the members.
"""

import os
import socket

import numpy as np
import pytest

from conftest import GOLDEN, ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, outq):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle import heff
    from paper_2305_05581_b200.plan import DevicePlan
    from paper_2305_05581_b200.plan_input import PlanInput
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pi = PlanInput.load(os.path.join(GOLDEN, case + ".npz"))
    plan = DevicePlan(pi, rank=rank, world=world, dry_run=True)
    mine = plan.shard()
    # the rank holds only the operator blocks its ψ sectors read: zero every
    # other block — the shard's partial σ must not change
    for side, arena, boff in (("l", pi.arena_l, pi.blk_off_l), ("r", pi.arena_r, pi.blk_off_r)):
        held = plan.block_layout(side) >= 0
        dim = pi.dim_l if side == "l" else pi.dim_r
        from paper_2305_05581_b200.workload import _rows_of
        for o, j in zip(*np.nonzero((boff >= 0) & ~held)):
            n = _rows_of(pi, side, o, j) * int(dim[j])
            arena[boff[o, j]:boff[o, j] + n] = 0.0
    groups = [g for g in heff.build_groups(pi) if mine[g[0]]]
    part = heff.apply_groups(pi, groups, pi.meta["psi"])
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    owned = torch.from_numpy(mine.astype(np.int64))
    dist.all_reduce(owned)
    outq.put((rank, t.numpy().copy(), owned.numpy().copy(),
              int(plan.stats["local_members"]), int(plan.stats["members"]),
              int(plan.stats["arena_bytes"]),
              int(DevicePlan(pi, dry_run=True).stats["arena_bytes"])))
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["ints4_p1", "ints6_d24_p2"])
def test_gloo_world2_sharded_sigma_allreduce(case):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2305_05581_b200.plan_input import PlanInput
    pi = PlanInput.load(os.path.join(GOLDEN, case + ".npz"))
    ref = pi.meta["sigma"]
    scale = 1.0 + np.max(np.abs(ref))
    local = 0
    for _rank, sigma, owned, lm, total, held, full in res:
        assert np.max(np.abs(sigma - ref)) <= 1e-12 * scale
        assert np.all(owned == 1)            # every ψ key owned by exactly one rank
        assert held <= full                  # per-rank operator arenas never exceed world 1
        local += lm
    assert sum(r[5] for r in res) < 2 * res[0][6] or res[0][6] == 0
    assert local == res[0][4]                # members partitioned
