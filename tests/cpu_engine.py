"""TEST INFRASTRUCTURE ONLY: a CPU stand-in for the device engine.

The closed-loop driver (paper_2305_05581_b200/driver.py) routes all of its
arithmetic through three hooks: ``blockops.Launch.run`` (the grouped FP64
GEMM, sdmrg_grouped_gemm), ``Engine.plan`` (the H_eff·ψ plan) and
``Engine.lanczos``.  For the CPU test-suite (no GPU in the build container)
these are replaced here by numpy: the grouped GEMM restated problem by
problem, the oracle's H_eff·ψ (oracle/heff.py, pinned to the reference's
golden vectors) and the oracle's Lanczos (oracle/lanczos.py).  This checks
the driver's host logic — work-list construction, Kronecker placements,
parity dressings, truncation, prediction — against the reference's recorded
sweeps.  The product never imports this module; the GPU tests run the same
driver on the sm_100a library.
"""

import contextlib
from typing import NamedTuple

import numpy as np
import torch
from numpy.lib.stride_tricks import as_strided

from oracle import heff, lanczos as olanczos

MASK = (1 << 60) - 1


def _view(flat, h, rows, cols, ld):
    base, off = int(h) >> 60, int(h) & MASK
    arr = flat[base]
    return as_strided(arr[off:], shape=(rows, cols), strides=(ld * 8, 8), writeable=True)


def emulated_run(self, bases, stream=None):
    """blockops.Launch.run restated in numpy (row-major, see sdmrg_b200.h)."""
    if not self.p["c"]:
        return
    P = {k: np.concatenate(v) for k, v in self.p.items()}
    S = {k: np.concatenate(v) for k, v in self.s.items()}
    flat = [b.detach().view(-1).numpy() for b in bases]
    sb = np.concatenate([[0], np.cumsum(P["nseg"])]).astype(np.int64)
    for p in range(len(P["c"])):
        m, n = int(P["m"][p]), int(P["n"][p])
        if m == 0 or n == 0:
            continue
        c = _view(flat, P["c"][p], m, n, int(P["ldc"][p]))
        acc = np.zeros((m, n))
        for s in range(sb[p], sb[p + 1]):
            k = int(S["k"][s])
            if k == 0:
                continue
            if self.ta:
                a = _view(flat, S["a"][s], k, m, int(S["lda"][s])).T
            else:
                a = _view(flat, S["a"][s], m, k, int(S["lda"][s]))
            if self.tb:
                b = _view(flat, S["b"][s], n, k, int(S["ldb"][s])).T
            else:
                b = _view(flat, S["b"][s], k, n, int(S["ldb"][s]))
            acc += float(S["scale"][s]) * (a @ b)
        if int(P["beta"][p]):
            c += acc
        else:
            c[...] = acc


class _Res(NamedTuple):
    energy: float
    vector: torch.Tensor
    iterations: int
    converged: bool


class OraclePlan:
    def __init__(self, pi, al, ar):
        pi.arena_l = al.detach().numpy().copy()
        pi.arena_r = ar.detach().numpy().copy()
        self.pi = pi
        self.groups = heff.build_groups_fast(pi)
        self.flops = heff.ref_flops(pi, self.groups)
        self.psi_size = int(pi.psi_offsets()[-1])

    def apply(self, v, out):
        res = heff.apply_groups(self.pi, self.groups, v.detach().numpy())
        out.copy_(torch.from_numpy(res))
        return out

    def close(self):
        pass


class CpuEngine:
    device = torch.device("cpu")

    def plan(self, pi, al, ar):
        return OraclePlan(pi, al, ar)

    def lanczos(self, apply_op, guess, tol, max_iter):
        def op(x):
            return apply_op(torch.from_numpy(np.ascontiguousarray(x))).numpy().copy()
        res = olanczos.lanczos_ground(op, guess.detach().numpy(), tol=tol, max_iter=max_iter)
        return _Res(res.energy, torch.from_numpy(np.ascontiguousarray(res.vector)),
                    res.iterations, res.converged)

    def eigh(self, mat):
        return torch.linalg.eigh(mat)


@contextlib.contextmanager
def emulated():
    from paper_2305_05581_b200 import blockops
    real = blockops.Launch.run
    blockops.Launch.run = emulated_run
    try:
        yield CpuEngine()
    finally:
        blockops.Launch.run = real
