"""ORACLE -- TEST INFRASTRUCTURE ONLY.

PAPER.md §3 "Building the Positively Weighted Expanded Graph":

* Eq. def:L_ell (l.110-122):  L_G~ = ({P(mu)}^l)^T L_G {P(mu)}^l
* Theorem 3.1 (l.129-179):    x = {P(mu)}^l x~ solves L_G x = b when
                              L_G~ x~ = b~ with b~ = ({P(mu)}^l)^T b
* §3.2 (l.288-291):           PEGP H~ = subgraph of G~ with only the positively
                              weighted edges; L^-_mu = Laplacian of the
                              negative edges (proof of Lemma upper, l.384)
* §3.3 (l.821):               MSP T~ = edges "on the top coarse level, edges
                              between the levels, and edges inside of the
                              aggregations of the original graphs" of H~

L_G~ is formed through the incidence factorisation of §2.1 and of the proof of
Lemma dim_G_tilde (l.339): L_G~ = (B P(mu))^T W (B P(mu)).  Every off-diagonal
entry is then a sum of terms of one sign, so an edge's sign is decided without
cancellation and entries that are zero are structurally zero.

Readings:
  R6  an edge's weight is minus the off-diagonal entry; "positively weighted"
      edges are the negative off-diagonal entries of L_G~ (l.281-285).
  R7  L_H~ is the Laplacian of H~ (diagonal = sum of the kept positive
      weights, as in the displayed matrix l.301-317: (1,1) = 2 + mu).
  R8  MSP edge classes: (a) all edges among top-level nodes; (b) "edges between
      the levels" = edges between consecutive levels k, k+1 (the tree
      structure of Fig. 4; these are exactly node -> own-aggregate edges);
      (c) "edges inside of the aggregations of the original graphs" = at every
      level k < l, same-level edges whose endpoints share their level-(k+1)
      aggregate (the per-level graphs are the "original graphs" of the
      aggregations; keeping only level 1 would disconnect nodes whose cut
      weight is zero).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .aggregation import Hierarchy, P_level, composite_P
from .graph import incidence, laplacian_from_weights


@dataclass
class ExpandedSystem:
    h: Hierarchy
    mu: float
    offsets: np.ndarray        # level-k block = [offsets[k-1], offsets[k])
    level_of: np.ndarray       # 1-based level of each expanded node
    parent: np.ndarray         # expanded index of the level-(k+1) aggregate, -1 on top
    LG: sp.csr_matrix | None   # L_G~ (None when only the MSP blocks were formed)
    WH: sp.csr_matrix | None   # weights of H~ (PEGP), symmetric, zero diagonal
    WN: sp.csr_matrix | None   # weights of the negative edges (|w|)
    WT: sp.csr_matrix          # weights of T~ (MSP)

    @property
    def n_tilde(self) -> int:
        return int(self.offsets[-1])

    @property
    def LH(self) -> sp.csr_matrix:
        return laplacian_from_weights(self.n_tilde, self.WH)

    @property
    def Lneg(self) -> sp.csr_matrix:
        return laplacian_from_weights(self.n_tilde, self.WN)

    @property
    def LT(self) -> sp.csr_matrix:
        return laplacian_from_weights(self.n_tilde, self.WT)

    def P(self) -> sp.csr_matrix:
        return composite_P(self.h, self.mu)


def _structure(h: Hierarchy):
    sizes = h.sizes
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    level_of = np.concatenate([np.full(s, k + 1, dtype=np.int64) for k, s in enumerate(sizes)])
    parent = np.full(offsets[-1], -1, dtype=np.int64)
    for k in range(1, h.nlevels):
        parent[offsets[k - 1]:offsets[k]] = offsets[k] + h.aggs[k - 1]
    return offsets, level_of, parent


def expanded_laplacian(g, h: Hierarchy, mu: float) -> sp.csr_matrix:
    """L_G~ = P(mu)^T L_G P(mu) = (B P(mu))^T W (B P(mu))  (Eq. def:L_ell)."""
    BP = (incidence(g.n, g.u, g.v) @ composite_P(h, mu)).tocsr()
    BP.eliminate_zeros()
    LG = (BP.T @ sp.diags(g.w) @ BP).tocsr()
    LG.sum_duplicates()
    LG.eliminate_zeros()
    return LG


def expanded_block(g, h: Hierarchy, mu: float, k: int, kp: int) -> sp.csr_matrix:
    """Block (k, k') of L_G~: ((-mu)^{k-1} P^k)^T L_G ((-mu)^{k'-1} P^{k'})
    (Eq. def:L_ell written blockwise, cf. Eq. def:LG_ex l.256-259)."""
    B = incidence(g.n, g.u, g.v)
    Bk = (B @ (((-mu) ** (k - 1)) * P_level(h, k))).tocsr(); Bk.eliminate_zeros()
    Bkp = (B @ (((-mu) ** (kp - 1)) * P_level(h, kp))).tocsr(); Bkp.eliminate_zeros()
    blk = (Bk.T @ sp.diags(g.w) @ Bkp).tocsr()
    blk.sum_duplicates(); blk.eliminate_zeros()
    return blk


def split_signs(LG: sp.csr_matrix):
    """(W_H, W_N): weights of the positive edges (negative off-diagonals of
    L_G~) and magnitudes of the negative edges (positive off-diagonals)."""
    off = (LG - sp.diags(LG.diagonal())).tocsr()
    off.eliminate_zeros()
    WH = (-off).multiply(off < 0).tocsr()
    WN = off.multiply(off > 0).tocsr()
    WH.eliminate_zeros(); WN.eliminate_zeros()
    return WH, WN


def _msp_mask(WH: sp.csr_matrix, level_of, parent, top: int) -> sp.csr_matrix:
    C = WH.tocoo()
    li, lj = level_of[C.row], level_of[C.col]
    keep_top = (li == top) & (lj == top)
    keep_between = np.abs(li - lj) == 1
    keep_inside = (li == lj) & (li < top) & (parent[C.row] == parent[C.col])
    keep = keep_top | keep_between | keep_inside
    return sp.csr_matrix((C.data[keep], (C.row[keep], C.col[keep])), shape=WH.shape)


def expand(g, h: Hierarchy, mu: float) -> ExpandedSystem:
    """Full expanded system (small/medium graphs): L_G~, H~, L^-, T~."""
    offsets, level_of, parent = _structure(h)
    LG = expanded_laplacian(g, h, mu)
    WH, WN = split_signs(LG)
    WT = _msp_mask(WH, level_of, parent, h.nlevels)
    return ExpandedSystem(h, mu, offsets, level_of, parent, LG, WH, WN, WT)


def expand_msp_only(g, h: Hierarchy, mu: float) -> ExpandedSystem:
    """T~ from the blocks (k,k) and (k,k+1) of L_G~ only -- the only blocks
    that can hold MSP edges (R8) -- for graphs where the full L_G~ is too
    large for the oracle.  Pinned equal to ``expand(...).WT`` in the tests."""
    offsets, level_of, parent = _structure(h)
    nt = int(offsets[-1])
    rows, cols, vals = [], [], []
    for k in range(1, h.nlevels + 1):
        for kp in (k, k + 1):
            if kp > h.nlevels:
                continue
            blk = expanded_block(g, h, mu, k, kp).tocoo()
            r = blk.row + offsets[k - 1]
            c = blk.col + offsets[kp - 1]
            neg = (blk.data < 0) & (r != c)
            rows.append(r[neg]); cols.append(c[neg]); vals.append(-blk.data[neg])
            if kp != k:   # mirror the (k+1, k) block
                rows.append(c[neg]); cols.append(r[neg]); vals.append(-blk.data[neg])
    WH_part = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                            shape=(nt, nt))
    WT = _msp_mask(WH_part, level_of, parent, h.nlevels)
    return ExpandedSystem(h, mu, offsets, level_of, parent, None, None, None, WT)


def project_rhs(P: sp.csr_matrix, b: np.ndarray) -> np.ndarray:
    """b~ = ({P(mu)}^l)^T b  (Theorem 3.1 proof, l.179)."""
    return P.T @ b


def lift_solution(P: sp.csr_matrix, xt: np.ndarray) -> np.ndarray:
    """x = {P(mu)}^l x~  (Theorem 3.1, l.132)."""
    return P @ xt
