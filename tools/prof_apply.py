"""Profiling driver: build the bench workload and run a few H_eff·ψ applies.

Meant to run under ncu (one GPU):  python tools/prof_apply.py [L] [D] [applies] [n_elec]
Kernel order per apply: seg_gemm_kernel<0,1> (phase 1, T = A R^T) then
seg_gemm_kernel<0,0> (phase 2, σ += L T), per workspace chunk.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2305_05581_b200.plan import DevicePlan
    from paper_2305_05581_b200.workload import fill_plan_arenas, synthetic_plan_input
    n_orb = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    applies = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    n_elec = int(sys.argv[4]) if len(sys.argv) > 4 else None  # L=76: 113
    pi = synthetic_plan_input(n_orb, d, n_elec=n_elec)
    plan = DevicePlan(pi, empty_arenas=True)
    fill_plan_arenas(plan, pi)
    psi = torch.randn(plan.psi_size, dtype=torch.float64, device="cuda")
    out = plan.empty_vector()
    for _ in range(applies):
        plan.apply(psi, out)
    torch.cuda.synchronize()
    print(plan.stats)


if __name__ == "__main__":
    main()
