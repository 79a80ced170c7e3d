"""ORACLE -- TEST INFRASTRUCTURE ONLY.

PAPER.md §2.1 "Graph": L_G = B^T W B with B^T in R^{n x m} the incidence
matrix and W the diagonal edge-weight matrix.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def incidence(n: int, u: np.ndarray, v: np.ndarray) -> sp.csr_matrix:
    """B in R^{m x n}: row e=(u,v) (u<v) has +1 at u and -1 at v (§2.1)."""
    m = u.shape[0]
    rows = np.concatenate([np.arange(m), np.arange(m)])
    cols = np.concatenate([u, v])
    vals = np.concatenate([np.ones(m), -np.ones(m)])
    return sp.csr_matrix((vals, (rows, cols)), shape=(m, n))


def laplacian(n: int, u: np.ndarray, v: np.ndarray, w: np.ndarray) -> sp.csr_matrix:
    """L_G = B^T W B (§2.1, l.53)."""
    B = incidence(n, u, v)
    L = (B.T @ sp.diags(w) @ B).tocsr()
    L.sum_duplicates()
    L.eliminate_zeros()
    return L


def laplacian_of_graph(g) -> sp.csr_matrix:
    return laplacian(g.n, g.u, g.v, g.w)


def laplacian_from_weights(n: int, W: sp.spmatrix) -> sp.csr_matrix:
    """Laplacian of a graph given by a symmetric nonnegative weight matrix
    (zero diagonal): D - W with D = diag(row sums)."""
    W = sp.csr_matrix(W)
    d = np.asarray(W.sum(axis=1)).ravel()
    return (sp.diags(d) - W).tocsr()


def quadratic_form(u, v, w, x) -> float:
    """x^T L x = sum_e w_e (x_u - x_v)^2 (the identity used in the proof of
    Lemma upper)."""
    return float(np.sum(w * (x[u] - x[v]) ** 2))


def apply_L(g, x: np.ndarray) -> np.ndarray:
    """y = L_G x with L_G = B^T W B (definition, via the incidence matrix)."""
    B = incidence(g.n, g.u, g.v)
    return B.T @ (g.w * (B @ x))
