"""Exact pins of the oracle against the paper's printed tables.

PAPER.md Tables 1-2 (l.726-780) print kappa(L_H~^+ L_G~) to four decimals
and Table 3 (l.859-879) prints PCG/FGMRES step counts.  With the MWM visit
order fixed to the natural vertex order (R1: the paper's tables
are reproduced by that order; ties to the lowest index, R2), the oracle
reproduces these columns *exactly*:

* Table 2, 2D grids, mu = 1/sqrt(n):       1.5680 1.4128 1.1959 1.0926
* Table 1, ring graphs, mu = 0.8:          3.5001 16.9643 83.5291 348.3507
* Table 2, ring graphs, mu = n^(-1/4):     2.6021 3.1655 2.1026 1.6033
* Table 3, PEGP, level = max, 1/sqrt(n):   7 6 5 steps
* Table 3, PEGP, level = 2,   n^(-1/4):    12 10 9 steps

A kappa to four decimals pins the whole chain -- MWM (§2.2), the coarse
graphs, P(mu) (l.86-90), L_G~ (Eq. def:L_ell), the sign split and R7's
Laplacian of H~ (l.301-317) -- and an exact PEGP step count additionally
pins R = P L_H~^+ P^T (R9) and the PCG loop (R10).  A wrong sign, a
dropped level, a transposed P or a diagonal that is not R7's changes these
numbers.

Two readings of printed parameters follow from these matches (DESIGN.md
R12): the Table 2 ring column and the Table 3 level-2 PEGP column were
computed at mu = n^(-1/4) (= 1/sqrt(sqrt n)), not 1/sqrt(n) -- every other
value of mu misses them.  The Table 3 level = max MSP column (58 93 151) is
matched by the MSP of reading R8 at mu = 0.8 (the paper's practical MSP
choice, l.1004) within -6 %, with the same growth per 4x n; R8 at the
header's mu = 1/sqrt(n) is mathematically ruled out (kappa > 1e6 at n = 64,
pinned below), and the literal "every positive inter-level edge" reading at
1/sqrt(n) needs more than 1.5x the printed steps (also pinned below).
"""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import read_tables
from inputs import graphs as G
from oracle import aggregation as A
from oracle import expansion as E
from oracle import graph as GR
from oracle import pcg as PC
from oracle import precond as PR
from oracle import spectral as S

T = read_tables()


def nat(g, levels=0):
    return A.build_hierarchy(g, 0, max_levels=levels, order="natural")


def kappa(g, mu):
    s = E.expand(g, nat(g), mu)
    return S.kappa(s.LG.toarray(), s.LH.toarray())


@pytest.mark.parametrize("n", [16, 64, 256, 1024])
def test_table2_grid_kappa_exact(n):
    side = int(round(np.sqrt(n)))
    g = G.grid2d(side, side, "unit")
    h = nat(g)
    # Table 1/2 "Level" and "Size of L_G~" columns: perfect halving to 2 nodes
    assert h.nlevels == int(np.log2(n)) and h.n_tilde == 2 * n - 2
    k = kappa(g, 1 / np.sqrt(n))
    assert abs(k - T["table2_invsqrtn_grid_kappa"][str(n)]) <= 5e-5, k


@pytest.mark.parametrize("n", [16, 64, 256, 1024])
def test_table1_ring_kappa_exact(n):
    k = kappa(G.ring(n, 4), 0.8)
    assert abs(k - T["table1_mu0.8_ring_kappa"][str(n)]) <= 5e-5, k


@pytest.mark.parametrize("n", [16, 64, 256, 1024])
def test_table2_ring_kappa_exact_at_quarter_power(n):
    k = kappa(G.ring(n, 4), n ** -0.25)
    assert abs(k - T["table2_invsqrtn_ring_kappa"][str(n)]) <= 5e-5, k
    # ... and not at the printed 1/sqrt(n) (n = 16 coincides: 1/sqrt(16) != 16^-1/4)
    k2 = kappa(G.ring(n, 4), 1 / np.sqrt(n))
    assert abs(k2 - T["table2_invsqrtn_ring_kappa"][str(n)]) > 0.05


def _steps(g, h, mu, kind):
    L = GR.laplacian_of_graph(g)
    s = E.expand(g, h, mu) if kind == "pegp" else E.expand_msp_only(g, h, mu)
    R = PR.pegp(s) if kind == "pegp" else PR.msp(s)
    return PC.pcg(lambda x: L @ x, G.rhs_paper(g.n), R, 1e-8, 3000).iterations


@pytest.mark.parametrize("side", [16, 32, 64])
def test_table3_pegp_levelmax_exact(side):
    n = side * side
    g = G.grid2d(side, side, "unit")
    assert _steps(g, nat(g), 1 / np.sqrt(n), "pegp") == T["table3_grid_levelmax_pegp_steps"][str(n)]


@pytest.mark.parametrize("side", [16, 32, 64])
def test_table3_pegp_level2_exact_at_quarter_power(side):
    n = side * side
    g = G.grid2d(side, side, "unit")
    assert _steps(g, nat(g, 2), n ** -0.25, "pegp") == T["table3_grid_level2_pegp_steps"][str(n)]


@pytest.mark.parametrize("side", [16, 32, 64])
def test_table3_msp_levelmax_R8_at_mu08(side):
    """Reading R8 at mu = 0.8 (l.1004): 55 90 146 against the printed
    58 93 151 -- within [-6 %, 0]."""
    n = side * side
    g = G.grid2d(side, side, "unit")
    it = _steps(g, nat(g), 0.8, "msp")
    paper = T["table3_grid_levelmax_msp_steps"][str(n)]
    assert 0.94 * paper <= it <= paper, (n, it, paper)


@pytest.mark.parametrize("side", [16, 32, 64])
def test_table3_msp_level2(side):
    """level = 2, mu = 1/sqrt(n) (every MSP reading coincides at two levels):
    47 48 48 against the printed 48 51 51 -- within [-10 %, 0]."""
    n = side * side
    g = G.grid2d(side, side, "unit")
    it = _steps(g, nat(g, 2), 1 / np.sqrt(n), "msp")
    paper = T["table3_grid_level2_msp_steps"][str(n)]
    assert 0.90 * paper <= it <= paper, (n, it, paper)


def _kappa_RL(g, s, LX):
    L = GR.laplacian_of_graph(g).toarray()
    P = s.P().toarray()
    Rd = P @ np.linalg.pinv(LX.toarray()) @ P.T
    Q = np.linalg.qr(np.c_[np.ones(g.n), np.random.default_rng(0).standard_normal((g.n, g.n - 1))])[0][:, 1:]
    C = np.linalg.cholesky(Q.T @ L @ Q)
    ev = np.linalg.eigvalsh(C.T @ (Q.T @ Rd @ Q) @ C)
    return ev.max() / ev.min()


def test_R8_at_invsqrtn_is_not_table3():
    """R8's T~ is a tree of aggregates whose level-k edges weigh mu^(2k-1):
    at mu = 1/sqrt(n) and level = max, kappa(R L) grows like mu^-(2l-3) --
    4.9e3 at n = 16, 1.9e9 at n = 64 -- so it cannot have produced the
    column's 58 93 151 steps (R8)."""
    g = G.grid2d(8, 8, "unit")
    s = E.expand(g, nat(g), 1 / 8)
    assert _kappa_RL(g, s, s.LT) > 1e6
    assert _kappa_RL(g, s, s.LH) < 2          # PEGP: Table 2's 1.4128


def test_literal_reading_at_invsqrtn_overshoots_table3():
    """The literal alternative to R8 -- every positive inter-level edge of
    H~ (odd-distance ancestors and even-distance neighbour aggregates) --
    converges at 1/sqrt(n) but needs 146 / 296 PCG steps against the
    printed 58 / 93, and eliminating a base pair then fills in among its
    coarse neighbours, against l.830's no-fill statement (R8)."""
    for side in (16, 32):
        n = side * side
        g = G.grid2d(side, side, "unit")
        s = E.expand(g, nat(g), 1 / np.sqrt(n))
        C = s.WH.tocoo()
        lv, par, top = s.level_of, s.parent, s.h.nlevels
        li, lj = lv[C.row], lv[C.col]
        keep = ((li == top) & (lj == top)) | (li != lj) | ((li == lj) & (par[C.row] == par[C.col]))
        W = sp.csr_matrix((C.data[keep], (C.row[keep], C.col[keep])), shape=C.shape)
        L = GR.laplacian_of_graph(g)
        R = PR.Preconditioner(s.P(), GR.laplacian_from_weights(s.n_tilde, W))
        it = PC.pcg(lambda x: L @ x, G.rhs_paper(n), R, 1e-8, 3000).iterations
        assert it > 1.5 * T["table3_grid_levelmax_msp_steps"][str(n)], it
