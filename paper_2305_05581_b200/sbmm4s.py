"""SBMM4S on the B200 — drop-in for sbmm4s.py:165 ``sbmm4s``.

``B := B + alpha * sum_i L_i A R_i^T`` in two kernels and no reduction pass
(Alg. 2): step 1 is one grouped launch writing the members A R_i^T
interleaved into a column-major workspace of leading dimension m*p; step 2 is
one launch whose K dimension is the member concatenation.  When the
workspace holds fewer than m*p*r doubles the batch splits in halves
recursively (sbmm4s.py:176).

Accepts the reference ``AccumulationProblem`` (numpy, column-major stacks;
operands are copied to the device and B back — the e2e path) or
``DeviceProblem`` (CUDA tensors, nothing copied).
"""

import ctypes

import numpy as np
import torch

from . import _lib


def flops_fused(m, n, q, r, p):
    """sbmm4s.py:201-203."""
    return 2 * m * r * n * p + 2 * q * r * m * p


class DeviceProblem:
    """Column-major device operands of B += alpha * sum_i L_i A R_i^T.

    Storage (all float64 CUDA, column-major == torch shape transposed):
      a        (n, m) tensor   -> A m x n, lda = m
      b        (r, q) tensor   -> B q x r, ldb = q
      l_stack  (p, m, q)       -> L_i q x m, ld q, member stride q*m
      r_stack  (p, n, r)       -> R_i r x n, ld r, member stride r*n
    """

    def __init__(self, alpha, a, b, l_stack, r_stack):
        self.alpha = float(alpha)
        self.a, self.b, self.l_stack, self.r_stack = a, b, l_stack, r_stack
        n, m = a.shape
        r, q = b.shape
        p = l_stack.shape[0]
        if tuple(l_stack.shape) != (p, m, q):
            raise ValueError(f"L members must be {q}x{m}")
        if tuple(r_stack.shape) != (p, n, r):
            raise ValueError(f"R members must be {r}x{n}")
        self.shape = (m, n, q, r, p)

    @classmethod
    def from_host(cls, alpha, a, b, l_stack, r_stack, device="cuda"):
        """From the reference's numpy operands (sbmm4s.py:97 field layout)."""
        def cm(x):
            return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64).T)).to(device)

        ls = np.asarray(l_stack, dtype=np.float64)
        rs = np.asarray(r_stack, dtype=np.float64)
        # F-ordered (q, m, p) stack: member i column-major == transpose (p, m, q)
        lt = torch.from_numpy(np.ascontiguousarray(ls.transpose(2, 1, 0))).to(device)
        rt = torch.from_numpy(np.ascontiguousarray(rs.transpose(2, 1, 0))).to(device)
        return cls(alpha, cm(a), cm(b), lt, rt)

    def workspace_needed(self):
        m, n, q, r, p = self.shape
        return m * p * r

    def b_host(self):
        return self.b.t().cpu().numpy()


def sbmm4s(problem, workspace=None, backend=None, stream=None):
    """Fused accumulation; returns B (numpy for host problems, tensor else).

    ``backend`` is accepted for signature compatibility; kernel accounting
    (multiply kernels, FLOPs) goes to ``backend.counter`` when it has one.
    """
    host = not isinstance(problem, DeviceProblem)
    dp = DeviceProblem.from_host(problem.alpha, problem.a, problem.b, problem.l_stack,
                                 problem.r_stack) if host else problem
    m, n, q, r, p = dp.shape
    if workspace is None:
        ws = torch.empty(m * p * r, dtype=torch.float64, device=dp.a.device)
    elif isinstance(workspace, torch.Tensor):
        ws = workspace
    else:
        ws = torch.empty(int(np.asarray(workspace).size), dtype=torch.float64,
                         device=dp.a.device)
    kernels = ctypes.c_int(0)
    s = (stream or torch.cuda.current_stream(dp.a.device)).cuda_stream
    _lib.check(_lib.load().sdmrg_sbmm4s(
        m, n, q, r, p, dp.alpha, dp.a.data_ptr(), m, dp.l_stack.data_ptr(), q, q * m,
        dp.r_stack.data_ptr(), r, r * n, dp.b.data_ptr(), q, ws.data_ptr(), ws.numel(),
        ctypes.byref(kernels), s))
    counter = getattr(backend, "counter", None)
    if counter is not None:
        counter.count(multiplies=kernels.value, flops=flops_fused(m, n, q, r, p))
    dp.kernels = kernels.value
    if host:
        problem.b[...] = dp.b_host()
        return problem.b
    return dp.b
