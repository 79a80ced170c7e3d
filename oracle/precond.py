"""ORACLE -- TEST INFRASTRUCTURE ONLY.

The preconditioner R of Eq. graphL_precsys ("we want to
choose an R that approximates the Moore-Penrose pseudoinverse L^+"), for the
two preconditioners of the paper.

The paper applies PEGP / MSP to the expanded system (§4, l.843: "we solve the
expanded graph Laplacian system ... which is equivalent to the original
system"), preconditioning L_G~ x~ = b~ by L_X^+ with X = H~ (PEGP) or T~ (MSP).
Reading R9: CG on the expanded system with preconditioner L_X^+ is,
iterate by iterate, CG on L_G x = b with

        R_X = P(mu) L_X^+ P(mu)^T            (x = P(mu) x~, Theorem 3.1)

because r~ = P^T r, L_G~ p~ = P^T L_G P p~ and (r~, L_X^+ r~) = (r, R_X r).
This module applies R_X by the definition: b~ = P^T r, the minimum-norm
solution of L_X z~ = b~ (pseudo-inverse: the grounded sparse LU solve of the
compatible part, then the component along 1 removed), and z = P z~.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


class PinvSolver:
    """y -> L^+ y for the Laplacian L of a connected graph (null space span{1}).

    L^+ y = L^+ (y - mean(y) 1); the compatible system L z = y - mean(y) 1 is
    solved by grounding the last node (sparse LU of the leading block, a
    library primitive), and the minimum-norm solution is z - mean(z) 1."""

    def __init__(self, L: sp.spmatrix):
        L = sp.csc_matrix(L)
        self.n = L.shape[0]
        if self.n > 1:
            self.lu = spla.splu(L[:-1, :-1].tocsc())

    def __call__(self, y: np.ndarray) -> np.ndarray:
        y = np.asarray(y, dtype=np.float64)
        if self.n == 1:
            return np.zeros(1)
        yc = y - y.mean()
        z = np.zeros(self.n)
        z[:-1] = self.lu.solve(yc[:-1])
        return z - z.mean()


class Preconditioner:
    """R_X r = P(mu) L_X^+ P(mu)^T r   (Reading R9)."""

    def __init__(self, P: sp.csr_matrix, LX: sp.spmatrix):
        self.P = sp.csr_matrix(P)
        self.PT = self.P.T.tocsr()
        self.inv = PinvSolver(LX)

    def __call__(self, r: np.ndarray) -> np.ndarray:
        return self.P @ self.inv(self.PT @ r)


def msp(sys) -> Preconditioner:
    return Preconditioner(sys.P(), sys.LT)


def pegp(sys) -> Preconditioner:
    return Preconditioner(sys.P(), sys.LH)


def dense_R(P: sp.spmatrix, LX: sp.spmatrix) -> np.ndarray:
    """Dense P L_X^+ P^T with numpy's pinv (tiny graphs; used as a pin)."""
    Pd = P.toarray()
    return Pd @ np.linalg.pinv(LX.toarray()) @ Pd.T
