"""Diagnostics for the device Lanczos on one B200: (1) a dense symmetric
operator with > 32 Krylov vectors (multi-slab basis) against eigvalsh;
(2) the first two-site iteration of the closed-loop L=16 D=256 run:
H_eff symmetry |x.Hy - y.Hx| on random vectors, device Lanczos vs the
oracle Lanczos on the same operator.   python tools/diag_lanczos.py"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch


def dense_check():
    from paper_2305_05581_b200.lanczos import lanczos_ground
    g = torch.Generator(device="cuda").manual_seed(3)
    n = 6000
    a = torch.randn(n, n, generator=g, dtype=torch.float64, device="cuda")
    h = (a + a.T) / 2
    ev = torch.linalg.eigvalsh(h)
    x0 = torch.randn(n, generator=g, dtype=torch.float64, device="cuda")
    res = lanczos_ground(lambda v: h @ v, x0, tol=1e-10, max_iter=400)
    return {"dense_n": n, "energy": res.energy, "exact": float(ev[0]), "dE": res.energy - float(ev[0]),
            "iters": res.iterations, "converged": res.converged}


def heff_check():
    from paper_2305_05581_b200 import driver as drv, model as M
    from oracle import lanczos as olz
    out = {}

    class Stop(Exception):
        pass

    class DiagEngine(drv.Engine):
        def lanczos(self, apply_op, guess, tol, max_iter):
            n = guess.numel()
            g = torch.Generator(device="cuda").manual_seed(7)
            xs = [torch.randn(n, generator=g, dtype=torch.float64, device="cuda") for _ in range(3)]
            hx = [apply_op(x).clone() for x in xs]
            asym = []
            for i in range(3):
                for j in range(i + 1, 3):
                    a = float(xs[i] @ hx[j]); b = float(xs[j] @ hx[i])
                    asym.append(abs(a - b) / (abs(a) + abs(b)))
            out["n"] = n
            out["asym_rel"] = asym
            # determinism
            h2 = apply_op(xs[0]).clone()
            out["repeat_bitwise"] = bool(torch.equal(h2, hx[0]))
            res = super().lanczos(apply_op, guess, tol, max_iter)
            out["device"] = {"energy": res.energy, "iters": res.iterations, "conv": res.converged}
            hg = guess.detach().cpu().numpy()
            r2 = olz.lanczos_ground(lambda v: apply_op(torch.from_numpy(v).cuda()).cpu().numpy(),
                                    hg, tol=tol, max_iter=max_iter)
            out["oracle_lanczos"] = {"energy": r2.energy, "iters": r2.iterations, "conv": r2.converged}
            raise Stop()

    mm = M.Model(M.random_integrals(16, 16, scale=0.2, core=0.3))
    sch = drv.SweepSchedule(n_sweeps=4, d=256, lanczos_tol=1e-10, lanczos_max_iter=300)
    try:
        drv.warmup(mm, sch, seed=42, engine=DiagEngine())
    except Stop:
        pass
    return out


if __name__ == "__main__":
    print(json.dumps({"dense": dense_check()}), flush=True)
    print(json.dumps({"heff_L16": heff_check()}), flush=True)
