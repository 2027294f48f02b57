"""Oracle: Lanczos with full reorthogonalisation — TEST INFRASTRUCTURE ONLY.

Restates dmrg.py:43-97 lanczos_ground line for line (numpy).
"""

import numpy as np


class LanczosResult(tuple):
    __slots__ = ()

    def __new__(cls, energy, vector, iterations, converged):
        return tuple.__new__(cls, (energy, vector, iterations, converged))

    energy = property(lambda s: s[0])
    vector = property(lambda s: s[1])
    iterations = property(lambda s: s[2])
    converged = property(lambda s: s[3])


def lanczos_ground(apply_op, guess, tol=1e-12, max_iter=200):
    guess = np.asarray(guess, dtype=float)
    nrm = np.linalg.norm(guess)
    if nrm == 0.0 or guess.size == 0:                      # dmrg.py:53
        raise ValueError("lanczos needs a nonzero starting vector")
    dim = guess.size
    v = guess / nrm
    total_iter = 0
    energy, vec = None, None
    for _restart in range(5):                              # dmrg.py:58
        basis = [v]
        alphas, betas = [], []
        ritz = None
        exhausted = False
        while total_iter < max_iter and len(basis) <= dim:
            w = apply_op(basis[-1])
            total_iter += 1
            alphas.append(float(np.dot(basis[-1], w)))
            w = w - alphas[-1] * basis[-1]
            if betas:
                w = w - betas[-1] * basis[-2]
            for b in basis:                                # dmrg.py:70
                w = w - np.dot(b, w) * b
            tri = np.diag(alphas)
            if betas:
                off = np.diag(betas, 1)
                tri = tri + off + off.T
            evals, evecs = np.linalg.eigh(tri)
            energy = float(evals[0])
            ritz = evecs[:, 0]
            beta = float(np.linalg.norm(w))
            est = abs(beta * ritz[-1])
            if est <= 0.1 * tol * (1.0 + abs(energy)) or beta < 1e-14 \
                    or len(basis) == dim:                  # dmrg.py:81
                exhausted = beta < 1e-14 or len(basis) == dim
                break
            betas.append(beta)
            basis.append(w / beta)
        vec = np.zeros(dim)
        for c, b in zip(ritz, basis):
            vec += c * b
        vec /= np.linalg.norm(vec)
        resid = apply_op(vec) - energy * vec               # dmrg.py:91
        if np.linalg.norm(resid) <= tol * (1.0 + abs(energy)):
            return LanczosResult(energy, vec, total_iter, True)
        if total_iter >= max_iter or exhausted:
            return LanczosResult(energy, vec, total_iter, exhausted)
        v = vec
    return LanczosResult(energy, vec, total_iter, False)
