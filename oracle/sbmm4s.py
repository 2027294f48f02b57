"""Oracle: SBMM4S (Alg. 2) in numpy — TEST INFRASTRUCTURE ONLY.

Restates sbmm4s.py:127-203 (and the NumpyGemm kernel semantics of
gemm.py:56-85): step 1 writes the members A @ R_i^T interleaved into a
column-major workspace of leading dimension m*p; step 2 multiplies the
horizontally concatenated L stack by that tall matrix, beta = 1.
"""

import numpy as np
from numpy.lib.stride_tricks import as_strided


def _view(buf, rows, cols, ld, start=0):
    item = buf.itemsize
    return as_strided(buf[start:], shape=(rows, cols), strides=(item, ld * item))


def batched_gemm_interleaved(a, r_stack, workspace):
    """sbmm4s.py:127-147: member i at rows [i*m, (i+1)*m) of an (m*p) x r view."""
    m, n = a.shape
    r, n2, p = r_stack.shape
    if n2 != n:
        raise ValueError("A / R inner dimension mismatch")
    if workspace.size < m * p * r:
        raise ValueError("workspace too small")
    for i in range(p):                       # one batched kernel (gemm.py:72)
        _view(workspace, m, r, m * p, i * m)[...] = np.matmul(a, r_stack[:, :, i].T)
    return _view(workspace, m * p, r, m * p)


def concat_gemm_accumulate(l_stack, temp, alpha, b):
    """sbmm4s.py:150-160: B += alpha * [L_1|...|L_p] @ temp."""
    q, m, p = l_stack.shape
    l_concat = l_stack.reshape((q, m * p), order="F")
    prod = np.matmul(l_concat, temp)
    if alpha == 1.0:
        b += prod
    else:
        b += alpha * prod


def sbmm4s(alpha, a, b, l_stack, r_stack, workspace):
    """sbmm4s.py:163-184 incl. the recursive halving fallback."""
    m, n = a.shape
    q, r = b.shape
    p = l_stack.shape[2]
    if workspace.size < m * r:
        raise ValueError("workspace cannot hold a single member")
    if workspace.size < m * p * r and p > 1:
        lo = p // 2
        for sl in (slice(0, lo), slice(lo, p)):
            sbmm4s(alpha, a, b, np.asfortranarray(l_stack[:, :, sl]),
                   np.asfortranarray(r_stack[:, :, sl]), workspace)
        return b
    temp = batched_gemm_interleaved(a, r_stack, workspace)
    concat_gemm_accumulate(l_stack, temp, alpha, b)
    return b


def sbmm4s_naive(alpha, a, b, l_stack, r_stack):
    """sbmm4s.py:187-198: per-member GEMMs plus a standalone accumulation."""
    for i in range(l_stack.shape[2]):
        b += alpha * (l_stack[:, :, i] @ (a @ r_stack[:, :, i].T))
    return b


def flops_fused(m, n, q, r, p):
    """sbmm4s.py:201-203."""
    return 2 * m * r * n * p + 2 * q * r * m * p
