"""Pluggable dense kernels on the B200 — drop-in for gemm.py's backends.

``CudaGemm`` honours the reference backend contract (gemm.py:50-85): ``gemm``
(c := beta*c + alpha*a@b), ``gemm_strided_batched`` (one batched kernel whose
members write into caller-supplied, possibly interleaved strided views) and
``add_inplace`` (the lone standalone reduction kernel), with the same
``KernelCounter`` accounting (one batched call = one multiply kernel,
2*m*n*k FLOPs per GEMM).

Operands may be CUDA tensors (device-resident, no copies) or numpy arrays —
then each call copies its operands to the device and the result back (the
reference-facing e2e path).  Arithmetic always runs in the sm_100a library.
"""

import threading

import numpy as np
import torch

from . import _lib


class KernelCounter:
    """Thread-safe tally of multiply kernels, reduction kernels and FLOPs
    (gemm.py:22-45)."""

    def __init__(self):
        self._lock = threading.Lock()
        self.multiplies = 0
        self.reductions = 0
        self.flops = 0

    def count(self, multiplies=0, reductions=0, flops=0):
        with self._lock:
            self.multiplies += multiplies
            self.reductions += reductions
            self.flops += flops

    def snapshot(self):
        with self._lock:
            return (self.multiplies, self.reductions, self.flops)

    def reset(self):
        with self._lock:
            self.multiplies = self.reductions = self.flops = 0


def _check_dims(a, b, c):
    if a.ndim != 2 or b.ndim != 2 or c.ndim != 2:
        raise ValueError("gemm operands must be 2-d")
    if a.shape[1] != b.shape[0] or tuple(c.shape) != (a.shape[0], b.shape[1]):
        raise ValueError(f"gemm shape mismatch {tuple(a.shape)} x {tuple(b.shape)} -> "
                         f"{tuple(c.shape)}")


def _cm_operand(x):
    """(device tensor, trans flag, ld) describing x as a column-major operand.

    A 2-d strided view with unit row stride is column-major (trans 0); with
    unit column stride it is row-major == transposed column-major (trans 1).
    """
    s0, s1 = x.stride()
    rows, cols = x.shape
    if s0 == 1 and (s1 >= max(rows, 1) or cols == 1):
        return x, 0, max(s1, rows, 1)
    if s1 == 1 and (s0 >= max(cols, 1) or rows == 1):
        return x, 1, max(s0, cols, 1)
    y = x.contiguous()
    return y, 1, max(cols, 1)


def _dev(x, device):
    if isinstance(x, torch.Tensor):
        return x if x.is_cuda else x.to(device)
    return torch.from_numpy(np.asarray(x, dtype=np.float64)).to(device)


class CudaGemm:
    """B200 backend with the reference backend's interface."""

    name = "cuda-sm100a"

    def __init__(self, counter=None, device=None):
        self.counter = counter or KernelCounter()
        self.device = torch.device(device if device is not None else "cuda")
        _lib.load()

    def _stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def _gemm_dev(self, a, b, c, alpha, beta):
        # column-major C(m x n) with ld from its strides
        cs0, cs1 = c.stride()
        if not (cs0 == 1 or c.shape[1] == 1):
            raise ValueError("device gemm output must be column-major (unit row stride)")
        m, n = c.shape
        k = a.shape[1]
        ad, ta, lda = _cm_operand(a)
        bd, tb, ldb = _cm_operand(b)
        ldc = max(cs1, m, 1)
        _lib.check(_lib.load().sdmrg_dgemm(ta, tb, m, n, k, float(alpha), ad.data_ptr(), lda,
                                           bd.data_ptr(), ldb, float(beta), c.data_ptr(), ldc,
                                           self._stream()))

    def gemm(self, a, b, c, alpha=1.0, beta=1.0):
        """c := beta*c + alpha*(a @ b)   (gemm.py:56)."""
        _check_dims(a, b, c)
        m, k = a.shape
        n = b.shape[1]
        if isinstance(c, torch.Tensor) and c.is_cuda and c.stride(0) == 1:
            self._gemm_dev(_dev(a, self.device), _dev(b, self.device), c, alpha, beta)
        elif isinstance(c, torch.Tensor) and c.is_cuda:
            # strided device output (e.g. a column slice of a row-major
            # tensor): compute into a column-major temporary
            cd = c.t().contiguous().t()
            self._gemm_dev(_dev(a, self.device), _dev(b, self.device), cd, alpha, beta)
            c.copy_(cd)
        else:
            ch = c if isinstance(c, np.ndarray) else c.cpu().numpy()
            cd = torch.from_numpy(np.asfortranarray(ch, dtype=np.float64)).to(self.device)
            cd = cd.t().contiguous().t() if cd.stride(0) != 1 else cd
            self._gemm_dev(_dev(a, self.device), _dev(b, self.device), cd, alpha, beta)
            res = cd.cpu().numpy()
            if isinstance(c, np.ndarray):
                c[...] = res
            else:
                c.copy_(torch.from_numpy(res))
        self.counter.count(multiplies=1, flops=2 * m * n * k)

    def gemm_strided_batched(self, a, b_members, c_members, trans_b=True):
        """One batched kernel: c_i := a @ op(b_i)   (gemm.py:72)."""
        flops = 0
        ad = _dev(a, self.device)
        for b_i, c_i in zip(b_members, c_members):
            op_b = b_i.T if trans_b else b_i
            _check_dims(a, op_b, c_i)
            flops += 2 * a.shape[0] * op_b.shape[1] * a.shape[1]
        # members are independent: run them as one grouped launch when they
        # are host views (interleaved workspace), else per-member device gemm
        if b_members and all(isinstance(c, np.ndarray) for c in c_members):
            m, n = c_members[0].shape
            k = a.shape[1]
            bs = [np.asarray(bm, dtype=np.float64) for bm in b_members]
            stack = np.stack([bm.T if trans_b else bm for bm in bs])  # (p, k, n)
            bd = torch.from_numpy(np.ascontiguousarray(stack)).to(self.device)
            ac = torch.from_numpy(np.asfortranarray(np.asarray(a, dtype=np.float64))).to(self.device)
            ac = ac.t().contiguous().t() if ac.stride(0) != 1 else ac
            cd = torch.empty((len(bs), n, m), dtype=torch.float64, device=self.device)
            # column-major: A (m x k, lda = m), B_i = stack[i] row-major (k x n)
            # == column-major transposed (trans 1, ldb = n), C_i col-major ld m
            _lib.check(_lib.load().sdmrg_dgemm_strided_batched(
                0, 1, m, n, k, ac.data_ptr(), max(ac.stride(1), m, 1), 0,
                bd.data_ptr(), max(n, 1), k * n, cd.data_ptr(), max(m, 1), m * n,
                len(bs), self._stream()))
            res = cd.cpu().numpy()
            for i, c_i in enumerate(c_members):
                c_i[...] = res[i].T
        else:
            for b_i, c_i in zip(b_members, c_members):
                op_b = _dev(b_i.T if trans_b else b_i, self.device)
                self._gemm_dev(ad, op_b, c_i, 1.0, 0.0)
        self.counter.count(multiplies=1, flops=flops)

    def add_inplace(self, c, x, alpha=1.0):
        """Standalone summation kernel (gemm.py:82); only fallback paths."""
        if isinstance(c, torch.Tensor) and c.is_cuda and c.is_contiguous():
            xd = _dev(x, self.device).contiguous()
            _lib.check(_lib.load().sdmrg_daxpy(c.numel(), float(alpha), xd.data_ptr(),
                                               c.data_ptr(), self._stream()))
        else:
            cd = torch.from_numpy(np.ascontiguousarray(c, dtype=np.float64)).to(self.device)
            xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(self.device)
            _lib.check(_lib.load().sdmrg_daxpy(cd.numel(), float(alpha), xd.data_ptr(),
                                               cd.data_ptr(), self._stream()))
            c[...] = cd.cpu().numpy().reshape(c.shape)
        self.counter.count(reductions=1)


_default = None


def default_backend():
    global _default
    if _default is None:
        _default = CudaGemm()
    return _default
