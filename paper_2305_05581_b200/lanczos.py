"""Device Lanczos with full reorthogonalisation — drop-in for dmrg.py:43.

Same control flow, convergence tests and restart logic as the reference
``lanczos_ground`` (dmrg.py:43-97); the Krylov basis, the matrix-vector
products and every vector operation stay on the GPU.  Per iteration the host
reads exactly two scalars (alpha, beta) in one transfer, needed for the
tridiagonal Ritz problem the reference also solves on the host
(``np.linalg.eigh`` of a k x k tridiagonal, dmrg.py:76).

Reorthogonalisation: the reference subtracts alpha v_k and beta v_{k-1} and
then runs one modified Gram-Schmidt sweep over the basis (dmrg.py:67-71).
Here the same projector is applied as two classical Gram-Schmidt passes
(CGS2: coef = V^T w; w -= V coef; twice), each pass one fixed set of
launches over all basis slabs (sdmrg_krylov_project: dot partials, their
fixed-order sum, the update — the second pass also yields ||w||); alpha is
the first pass's coefficient on v_k (before any subtraction, exactly the
reference's alpha).
"""

from typing import NamedTuple

import numpy as np
import torch
from scipy.linalg import eigh_tridiagonal

from . import _lib

_CHUNK = 32  # Krylov vectors per contiguous basis slab


class LanczosError(Exception):
    pass


class LanczosResult(NamedTuple):
    energy: float
    vector: torch.Tensor
    iterations: int
    converged: bool


class KrylovBasis:
    """Growable device basis: slabs of _CHUNK contiguous vectors."""

    def __init__(self, n, device):
        self.n = n
        self.device = device
        self.slabs = []
        self.count = 0
        self.coef = torch.zeros(_CHUNK * 64, dtype=torch.float64, device=device)

    def clear(self):
        self.count = 0

    def vec(self, i):
        return self.slabs[i // _CHUNK][i % _CHUNK]

    def append_slot(self):
        if self.count == len(self.slabs) * _CHUNK:
            self.slabs.append(torch.empty((_CHUNK, self.n), dtype=torch.float64,
                                          device=self.device))
        v = self.vec(self.count)
        self.count += 1
        return v

    def project_out(self, w, stream, coef_out=None, norm_out=None):
        """One CGS pass: coef = V^T w ; w -= V coef (sdmrg_krylov_project:
        one launch set over all slabs; ``norm_out`` receives ||w|| after the
        update).  Returns coef (device)."""
        lib = _lib.load()
        if self.count > self.coef.numel():
            self.coef = torch.zeros(2 * self.count, dtype=torch.float64, device=self.device)
        coef = self.coef if coef_out is None else coef_out
        nsl = (self.count + _CHUNK - 1) // _CHUNK
        if nsl <= 16:
            ptrs = (_lib.c_vp * max(nsl, 1))(*[s.data_ptr() for s in self.slabs[:nsl]])
            _lib.check(lib.sdmrg_krylov_project(
                nsl, ptrs, _CHUNK, self.count, self.n, w.data_ptr(), coef.data_ptr(),
                None if norm_out is None else norm_out.data_ptr(), stream))
            return coef
        for s, slab in enumerate(self.slabs):
            k = min(_CHUNK, self.count - s * _CHUNK)
            if k <= 0:
                break
            c = coef[s * _CHUNK:s * _CHUNK + k]
            _lib.check(lib.sdmrg_gemv_t(k, self.n, slab.data_ptr(), self.n, w.data_ptr(),
                                        c.data_ptr(), stream))
        for s, slab in enumerate(self.slabs):
            k = min(_CHUNK, self.count - s * _CHUNK)
            if k <= 0:
                break
            c = coef[s * _CHUNK:s * _CHUNK + k]
            _lib.check(lib.sdmrg_gemv_n(k, self.n, slab.data_ptr(), self.n, c.data_ptr(),
                                        -1.0, w.data_ptr(), stream))
        if norm_out is not None:
            _nrm2(w, norm_out, stream)
        return coef

    def combine(self, coefs, out, stream):
        """out = sum_i coefs[i] V_i (coefs host array)."""
        lib = _lib.load()
        dc = torch.from_numpy(np.ascontiguousarray(coefs, dtype=np.float64)).to(self.device)
        out.zero_()
        for s, slab in enumerate(self.slabs):
            k = min(_CHUNK, len(coefs) - s * _CHUNK)
            if k <= 0:
                break
            _lib.check(lib.sdmrg_gemv_n(k, self.n, slab.data_ptr(), self.n,
                                        dc[s * _CHUNK:].data_ptr(), 1.0, out.data_ptr(), stream))
        return out


def _nrm2(x, out, stream):
    _lib.check(_lib.load().sdmrg_nrm2(x.numel(), x.data_ptr(), out.data_ptr(), stream))


def _axpby(a, x, b, y, stream):
    _lib.check(_lib.load().sdmrg_axpby(x.numel(), float(a), x.data_ptr(), float(b),
                                       y.data_ptr(), stream))


def _lowest_ritz(alphas, betas):
    if len(alphas) == 1:
        return float(alphas[0]), np.ones(1)
    w, v = eigh_tridiagonal(np.asarray(alphas), np.asarray(betas), select="i",
                            select_range=(0, 0))
    return float(w[0]), v[:, 0]


def lanczos_ground(apply_op, guess, tol=1e-12, max_iter=200):
    """Smallest eigenpair of a symmetric operator (dmrg.py:43 semantics).

    ``apply_op(v)`` maps a CUDA float64 vector to H v (a new tensor or a
    reused buffer); ``guess`` is a CUDA tensor or a host array.
    """
    lib = _lib.load()
    if not isinstance(guess, torch.Tensor):
        guess = torch.from_numpy(np.ascontiguousarray(guess, dtype=np.float64)).cuda()
    guess = guess.to(torch.float64).contiguous()
    dim = guess.numel()
    device = guess.device
    stream = torch.cuda.current_stream(device).cuda_stream
    scal = torch.zeros(4, dtype=torch.float64, device=device)
    _nrm2(guess, scal[0:1], stream)
    nrm = float(scal[0].item())
    if nrm == 0.0 or dim == 0:
        raise LanczosError("lanczos needs a nonzero starting vector")
    basis = KrylovBasis(dim, device)
    v0 = torch.empty_like(guess)
    _axpby(1.0 / nrm, guess, 0.0, v0, stream)
    total_iter = 0
    energy, vec = None, None
    for _restart in range(5):                                   # dmrg.py:58
        basis.clear()
        _axpby(1.0, v0, 0.0, basis.append_slot(), stream)
        alphas, betas = [], []
        ritz = None
        exhausted = False
        while total_iter < max_iter and basis.count <= dim:
            w = apply_op(basis.vec(basis.count - 1))            # reused in place
            total_iter += 1
            coef = basis.project_out(w, stream)                 # pass 1 (alpha)
            scal[1:2].copy_(coef[basis.count - 1:basis.count])
            basis.project_out(w, stream, norm_out=scal[2:3])    # pass 2 + ||w||
            host = scal.cpu().numpy()                           # one D2H per step
            alphas.append(float(host[1]))
            beta = float(host[2])
            # dmrg.py:76 eigh of the k x k tridiagonal: only its lowest pair
            # is used, so the O(k^2) tridiagonal solver (LAPACK stebz/stein)
            # replaces the dense O(k^3) eigh — same Ritz pair to rounding, and
            # no k = 300 dense solve per iteration on the host
            energy, ritz = _lowest_ritz(alphas, betas)
            est = abs(beta * ritz[-1])
            if est <= 0.1 * tol * (1.0 + abs(energy)) or beta < 1e-14 \
                    or basis.count == dim:                      # dmrg.py:81
                exhausted = beta < 1e-14 or basis.count == dim
                break
            betas.append(beta)
            _axpby(1.0 / beta, w, 0.0, basis.append_slot(), stream)
        vec = torch.empty_like(v0)
        basis.combine(ritz, vec, stream)                        # dmrg.py:87
        _nrm2(vec, scal[3:4], stream)
        _lib.check(lib.sdmrg_scal_dev(dim, None, scal[3:4].data_ptr(), 1, vec.data_ptr(), stream))
        resid = apply_op(vec)
        _axpby(-energy, vec, 1.0, resid, stream)                # dmrg.py:91
        _nrm2(resid, scal[0:1], stream)
        rn = float(scal[0].item())
        if rn <= tol * (1.0 + abs(energy)):
            return LanczosResult(energy, vec, total_iter, True)
        if total_iter >= max_iter or exhausted:
            return LanczosResult(energy, vec, total_iter, exhausted)
        v0 = vec
    return LanczosResult(energy, vec, total_iter, False)


def davidson_ground(apply_op, guess, diag, tol=1e-12, max_iter=200, max_space=40):
    """Lowest eigenpair by Davidson with the diagonal preconditioner (the
    north star's eigensolver; the reference runs Lanczos, dmrg.py:43).

    ``diag`` is the diagonal of the operator (``DevicePlan.diagonal``).  The
    search space V and H V live on the device in 32-vector slabs; each step:
    Ritz pair of the projected matrix (host, k <= max_space), residual
    r = H u - θ u, correction t = r / (θ - diag) (sdmrg_davidson_precond),
    two CGS passes against V with the norm fused (sdmrg_krylov_project), one
    H_eff·ψ.  A full space collapses to the current Ritz vector.  Converged
    when ||r|| <= tol (1 + |θ|) — the reference's acceptance test
    (dmrg.py:91).  ``iterations`` counts H_eff applications.
    """
    lib = _lib.load()
    if not isinstance(guess, torch.Tensor):
        guess = torch.from_numpy(np.ascontiguousarray(guess, dtype=np.float64)).cuda()
    guess = guess.to(torch.float64).contiguous()
    dim = guess.numel()
    device = guess.device
    stream = torch.cuda.current_stream(device).cuda_stream
    scal = torch.zeros(2, dtype=torch.float64, device=device)
    _nrm2(guess, scal[0:1], stream)
    nrm = float(scal[0].item())
    if nrm == 0.0 or dim == 0:
        raise LanczosError("davidson needs a nonzero starting vector")
    V = KrylovBasis(dim, device)
    W = KrylovBasis(dim, device)
    coef = torch.zeros(max(max_space, 1) + 1, dtype=torch.float64, device=device)
    mat = np.zeros((max_space, max_space))
    u = torch.empty_like(guess)
    hu = torch.empty_like(guess)
    t = torch.empty_like(guess)
    _axpby(1.0 / nrm, guess, 0.0, u, stream)
    iters = 0

    def add(vec):
        """Append vec (normalised) to V, H vec to W, extend the projected matrix."""
        nonlocal iters
        k = V.count
        _axpby(1.0, vec, 0.0, V.append_slot(), stream)
        w = apply_op(V.vec(k))
        iters += 1
        _axpby(1.0, w, 0.0, W.append_slot(), stream)
        # column k of V^T H V (dots only: one gemv_t per slab)
        for s_, slab in enumerate(V.slabs):
            kk = min(_CHUNK, V.count - s_ * _CHUNK)
            if kk <= 0:
                break
            _lib.check(lib.sdmrg_gemv_t(kk, dim, slab.data_ptr(), dim, W.vec(k).data_ptr(),
                                        coef[s_ * _CHUNK:].data_ptr(), stream))
        col = coef[:V.count].cpu().numpy()
        mat[:k + 1, k] = col
        mat[k, :k + 1] = col          # rows from the column (H_eff is near-symmetric)

    add(u)
    theta = None
    while True:
        k = V.count
        m = 0.5 * (mat[:k, :k] + mat[:k, :k].T)
        evals, evecs = np.linalg.eigh(m)
        theta, y = float(evals[0]), evecs[:, 0]
        V.combine(y, u, stream)
        W.combine(y, hu, stream)
        _axpby(-theta, u, 1.0, hu, stream)             # hu := H u - θ u (residual)
        _nrm2(hu, scal[0:1], stream)
        rn = float(scal[0].item())
        if rn <= tol * (1.0 + abs(theta)):
            _nrm2(u, scal[1:2], stream)
            _lib.check(lib.sdmrg_scal_dev(dim, None, scal[1:2].data_ptr(), 1, u.data_ptr(), stream))
            return LanczosResult(theta, u, iters, True)
        if iters >= max_iter:
            return LanczosResult(theta, u, iters, False)
        _lib.check(lib.sdmrg_davidson_precond(dim, hu.data_ptr(), diag.data_ptr(), theta,
                                              t.data_ptr(), stream))
        if V.count >= max_space:
            # collapse: restart from the Ritz vector (its H u is recomputed)
            _nrm2(u, scal[1:2], stream)
            _lib.check(lib.sdmrg_scal_dev(dim, None, scal[1:2].data_ptr(), 1, u.data_ptr(), stream))
            V.clear()
            W.clear()
            mat[:] = 0.0
            add(u)
            continue
        V.project_out(t, stream)
        V.project_out(t, stream, norm_out=scal[1:2])
        tn = float(scal[1].item())
        if tn < 1e-14:
            return LanczosResult(theta, u, iters, False)
        _axpby(1.0 / tn, t, 0.0, t, stream)
        add(t)
