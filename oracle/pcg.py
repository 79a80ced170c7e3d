"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Preconditioned conjugate gradient, textbook form (Hestenes-Stiefel with a
preconditioner; e.g. Saad, "Iterative Methods for Sparse Linear Systems",
Alg. 9.1), for L x = b with b orthogonal to 1 (§1 l.23 "Conjugate
Gradient (CG) method"; Eq. graphL_precsys R L x = R b).

Stopping rule (reading R10): stop after the first iteration whose recursively
updated residual satisfies ||r||_2 <= rtol ||b||_2; x0 = 0; the iteration count
is the number of L-products performed.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class PCGResult:
    x: np.ndarray
    iterations: int
    converged: bool
    resnorms: list = field(default_factory=list)


def pcg(apply_L, b: np.ndarray, apply_R=None, rtol: float = 1e-8, maxit: int = 1000) -> PCGResult:
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    bnorm = float(np.linalg.norm(b))
    hist = [bnorm]
    if bnorm == 0.0:
        return PCGResult(x, 0, True, hist)
    z = apply_R(r) if apply_R is not None else r.copy()
    p = z.copy()
    rho = float(r @ z)
    for it in range(1, maxit + 1):
        q = apply_L(p)
        alpha = rho / float(p @ q)
        x += alpha * p
        r -= alpha * q
        rn = float(np.linalg.norm(r))
        hist.append(rn)
        if rn <= rtol * bnorm:
            return PCGResult(x, it, True, hist)
        z = apply_R(r) if apply_R is not None else r.copy()
        rho_new = float(r @ z)
        beta = rho_new / rho
        p = z + beta * p
        rho = rho_new
    return PCGResult(x, maxit, False, hist)
