"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Dense spectral checks of PAPER.md §3.2: the generalized eigenvalue problem
Eq. general-eigenvalue (l.321) L_G~ v = lambda L_H~ v, the condition number
kappa(L_H~^+ L_G~) = lambda_max / lambda_min(nonzero) (l.364, Tables 1-2),
Lemma dim_G_tilde (l.329), Lemma upper (l.373), Lemma lower-mu (l.396) and
Theorem MSP_cond (l.579).  numpy dense eigensolvers are the library
primitives; sizes are desk scale.
"""
from __future__ import annotations

import numpy as np


def null_dim(A: np.ndarray, rel: float = 1e-10) -> int:
    """Number of singular values <= rel * sigma_max (Lemma dim_G_tilde)."""
    s = np.linalg.svd(A, compute_uv=False)
    return int(np.sum(s <= rel * s[0]))


def _pinv_sqrt(B: np.ndarray, rel: float = 1e-10):
    lam, V = np.linalg.eigh(B)
    keep = lam > rel * lam.max()
    return V[:, keep] @ np.diag(lam[keep] ** -0.5) @ V[:, keep].T


def pencil_eigs(A: np.ndarray, B: np.ndarray, rel: float = 1e-10) -> np.ndarray:
    """Eigenvalues of B^{+1/2} A B^{+1/2} (= those of B^+ A on range(B)),
    i.e. the generalized eigenvalues of A v = lambda B v for v orthogonal to
    Null(B) (case 3 of §3.2 once the zero ones are discarded)."""
    S = _pinv_sqrt(B, rel)
    M = S @ A @ S
    return np.linalg.eigvalsh((M + M.T) / 2)


def kappa(A: np.ndarray, B: np.ndarray, rel: float = 1e-9) -> float:
    """kappa(B^+ A) = lambda_max / smallest nonzero lambda (l.364, l.681)."""
    ev = pencil_eigs(A, B)
    top = ev.max()
    nz = ev[ev > rel * top]
    return float(top / nz.min())


def rho_hat(Lneg: np.ndarray, LH: np.ndarray, LG: np.ndarray, rel: float = 1e-10) -> float:
    """sup_v c_v(mu) = (L^- v, v) / (L_H~ v, v) over v orthogonal to
    Null(L_G~) (Lemma lower-mu, l.401; Theorem MSP_cond restricts to
    v perp Null(L_G~), l.584 -- on Null(L_G~) the ratio is 1, l.403)."""
    lam, V = np.linalg.eigh(LG)
    Q = V[:, lam > rel * lam.max()]
    A = Q.T @ Lneg @ Q
    B = Q.T @ LH @ Q
    Lc = np.linalg.cholesky((B + B.T) / 2)
    Li = np.linalg.inv(Lc)
    M = Li @ A @ Li.T
    return float(np.linalg.eigvalsh((M + M.T) / 2).max())
