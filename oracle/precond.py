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


def _ld_matvec(A: sp.csr_matrix, x: np.ndarray) -> np.ndarray:
    """y = A x with every product and row sum in extended precision
    (np.longdouble, 64-bit significand on x86): the residual of iterative
    refinement must be formed more accurately than the solve it corrects."""
    A = sp.csr_matrix(A)
    A.sort_indices()
    xl = np.asarray(x, dtype=np.longdouble)
    prod = A.data.astype(np.longdouble) * xl[A.indices]
    y = np.zeros(A.shape[0], dtype=np.longdouble)
    nz = np.diff(A.indptr) > 0
    y[nz] = np.add.reduceat(prod, A.indptr[:-1][nz])
    return y


def _ld_laplacian_apply(W: sp.csr_matrix, z: np.ndarray) -> np.ndarray:
    """(L_X z)_i = sum_j w_ij (z_i - z_j) from the edge weights themselves, in
    extended precision -- the Laplacian of the fp64 weights with its exact
    diagonal (R7: "diagonal = sum of the kept weights").  An assembled fp64
    L_X rounds that diagonal, and on high-contrast graphs (a heavy matched
    edge beside a light parent edge) the rounding is far larger, relative to
    the light weight, than the weights' own precision."""
    W = sp.csr_matrix(W)
    W.sort_indices()
    zl = np.asarray(z, dtype=np.longdouble)
    rows = np.repeat(np.arange(W.shape[0]), np.diff(W.indptr))
    prod = W.data.astype(np.longdouble) * (zl[rows] - zl[W.indices])
    y = np.zeros(W.shape[0], dtype=np.longdouble)
    nz = np.diff(W.indptr) > 0
    y[nz] = np.add.reduceat(prod, W.indptr[:-1][nz])
    return y


class RefinedPreconditioner:
    """R_X r = P(mu) L_X^+ P(mu)^T r, the same definition as
    :class:`Preconditioner`, evaluated to (nearly) full accuracy for the
    given fp64 edge weights W_X, for use as the parity *reference* (DESIGN.md
    R14): P^T r and P z~ in extended precision, and the grounded LU solve of
    L_X z~ = r~ - mean(r~) followed by iterative refinement -- residual in
    extended precision from the edge weights (exact diagonal), correction by
    the same LU -- until the correction stops shrinking (classical mixed-
    precision refinement, e.g. Higham, "Accuracy and Stability of Numerical
    Algorithms", ch. 12).  The result is R_X r for the given fp64 data,
    rounded once."""

    def __init__(self, P: sp.csr_matrix, WX: sp.spmatrix, max_steps: int = 60):
        from .graph import laplacian_from_weights
        self.P = sp.csr_matrix(P)
        self.PT = self.P.T.tocsr()
        self.WX = sp.csr_matrix(WX)
        # the correction solver only has to approximate L_X^+ (fp64 LU of
        # the assembled Laplacian); the refinement converges while its error
        # contracts, down to the extended-precision residual
        self.inv = PinvSolver(laplacian_from_weights(self.WX.shape[0], self.WX))
        self.max_steps = max_steps
        self.steps = 0

    def __call__(self, r: np.ndarray) -> np.ndarray:
        rt = _ld_matvec(self.PT, r)
        rt = rt - rt.mean()
        z = self.inv(np.asarray(rt, dtype=np.float64)).astype(np.longdouble)
        last = np.inf
        self.steps = 0
        for _ in range(self.max_steps):
            res = rt - _ld_laplacian_apply(self.WX, z)   # z carried in extended precision
            c = self.inv(np.asarray(res, dtype=np.float64))
            z = z + c.astype(np.longdouble)
            self.steps += 1
            cn = float(np.abs(c).max())
            if cn <= 1e-19 * float(np.abs(z).max()) or cn >= 0.9 * last:
                break
            last = cn
        z = z - z.mean()
        return np.asarray(_ld_matvec(self.P, z), dtype=np.float64)


def msp_refined(sys) -> RefinedPreconditioner:
    return RefinedPreconditioner(sys.P(), sys.WT)


def pegp_refined(sys) -> RefinedPreconditioner:
    return RefinedPreconditioner(sys.P(), sys.WH)


def msp(sys) -> Preconditioner:
    return Preconditioner(sys.P(), sys.LT)


def pegp(sys) -> Preconditioner:
    return Preconditioner(sys.P(), sys.LH)


def dense_R(P: sp.spmatrix, LX: sp.spmatrix) -> np.ndarray:
    """Dense P L_X^+ P^T with numpy's pinv (tiny graphs; used as a pin)."""
    Pd = P.toarray()
    return Pd @ np.linalg.pinv(LX.toarray()) @ Pd.T
