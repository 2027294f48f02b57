"""Multi-rank H_eff·ψ on the device: every rank builds its ψ-sector shard of
the plan, applies it, and the all-reduce of the partial σ must equal the
single-plan σ.  Run under torchrun (rank count may exceed the GPU count with
SDMRG_DIST_BACKEND=gloo: ranks then share cuda:0).  Exit code 0 = pass.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
      --master-port 29511 tools/check_multirank.py [L D]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    from paper_2305_05581_b200.plan import DevicePlan
    from paper_2305_05581_b200.workload import fill_arenas_device, synthetic_plan_input
    n_orb = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    backend = os.environ.get("SDMRG_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group(backend)
    pi = synthetic_plan_input(n_orb, d, seed=4)
    al, ar = fill_arenas_device(pi, seed=4)
    shard = DevicePlan(pi, arena_l=al, arena_r=ar, rank=rank, world=world)
    g = torch.Generator(device="cuda").manual_seed(11)
    psi = torch.randn(shard.psi_size, generator=g, dtype=torch.float64, device="cuda")
    sigma = shard.apply(psi)
    dist.all_reduce(sigma)
    mine = torch.from_numpy(shard.shard().astype("int64")).cuda()
    dist.all_reduce(mine)
    members = torch.tensor([shard.stats["local_members"]], dtype=torch.int64, device="cuda")
    dist.all_reduce(members)
    ok = True
    if rank == 0:
        full = DevicePlan(pi, arena_l=al, arena_r=ar).apply(psi)
        err = ((sigma - full).abs().max() / (1 + full.abs().max())).item()
        ok = err <= 1e-12 and bool((mine == 1).all()) and \
            int(members.item()) == shard.stats["members"]
        print(f"multirank world={world} backend={backend}: rel err {err:.2e}, "
              f"keys covered once {bool((mine == 1).all())}, members {int(members.item())}/"
              f"{shard.stats['members']} -> {'PASS' if ok else 'FAIL'}")
    flag = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(flag)
    dist.destroy_process_group()
    sys.exit(int(flag.item() != 0))


if __name__ == "__main__":
    main()
