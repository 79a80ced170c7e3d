"""Independent check of the refined parity reference (oracle.precond.msp_refined)
at mu = 1/sqrt(n) on the 20x13 log-uniform grid of test_apply_R_other_mu: the
same R r = P L_T~^+ P^T r solved densely in 50-digit mpmath (grounded LU,
exact diagonal from the edge weights).  Takes a few minutes on one core.
Round 2 result: refined vs mpmath 4.1e-16 (max-norm relative)."""
import sys, numpy as np, scipy.sparse as sp, mpmath as mp
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from inputs import graphs as G
from oracle import aggregation as A, expansion as E, precond as PR
mp.mp.dps = 50
g = G.grid2d(20, 13, "loguniform", 7)
mu = 1 / np.sqrt(g.n)
h = A.build_hierarchy(g, 2)
s = E.expand_msp_only(g, h, mu)
r = G.rhs(g.n, 9)
zr = PR.msp_refined(s)(r)
P = s.P().toarray(); W = sp.csr_matrix(s.WT).toarray(); nt = W.shape[0]
print("nt", nt, flush=True)
rt = [mp.fsum(mp.mpf(P[i, j]) * mp.mpf(r[i]) for i in range(P.shape[0]) if P[i, j] != 0) for j in range(nt)]
m = mp.fsum(rt) / nt; rt = [v - m for v in rt]
Lm = mp.zeros(nt - 1, nt - 1)
for i in range(1, nt):
    d = mp.mpf(0)
    for j in range(nt):
        if j != i and W[i, j] != 0:
            d += mp.mpf(W[i, j])
            if j >= 1: Lm[i - 1, j - 1] = -mp.mpf(W[i, j])
    Lm[i - 1, i - 1] = d
z = mp.lu_solve(Lm, mp.matrix(rt[1:]))
z = [mp.mpf(0)] + [z[i] for i in range(nt - 1)]
mz = mp.fsum(z) / nt; z = [v - mz for v in z]
ze = np.array([float(mp.fsum(mp.mpf(P[i, j]) * z[j] for j in range(nt) if P[i, j] != 0)) for i in range(P.shape[0])])
print("refined vs mp:", np.abs(zr - ze).max() / np.abs(ze).max())
np.save('/tmp/mp_ze.npy', ze)
