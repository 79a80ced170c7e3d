"""ORACLE -- TEST INFRASTRUCTURE ONLY.

PAPER.md §2.2 "Aggregation": MWM aggregation, the prolongation operators
P^l_{l-1} (0/1 membership, l.75), P^l = P^2_1 P^3_2 ... P^l_{l-1} (Eq. def:P,
l.81) and the composite prolongation
{P(mu)}^l = [I, -mu P^2, (-mu)^2 P^3, ..., (-mu)^{l-1} P^l] (l.86-90).

The sequential MWM itself is plain C (oracle/c/mwm_oracle.c) for speed; this
module marshals arrays and assembles the matrices.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _native


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Level:
    n: int
    rowptr: np.ndarray     # int64
    col: np.ndarray        # int32
    w: np.ndarray          # float64


@dataclass
class Hierarchy:
    levels: list = field(default_factory=list)   # Level objects, k = 1..l (index 0 = level 1)
    aggs: list = field(default_factory=list)     # aggs[k-1][i] = level-(k+1) aggregate of level-k node i
    mates: list = field(default_factory=list)    # mates[k-1][i] = matched partner or -1
    seed: int = 0

    @property
    def nlevels(self) -> int:
        return len(self.levels)

    @property
    def sizes(self):
        return [lv.n for lv in self.levels]

    @property
    def n_tilde(self) -> int:
        return int(sum(self.sizes))

    @property
    def offsets(self):
        return np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int64)


def visit_order(n: int, seed: int, level: int) -> np.ndarray:
    """Reading R1: the 'random order' of PAPER.md l.61 as a counter-based key."""
    out = np.empty(n, dtype=np.int64)
    _native.lib().oracle_visit_order(n, ctypes.c_uint64(seed), level, _p(out))
    return out


def mwm(lv: Level, seed: int, level: int, order: np.ndarray | None = None):
    """MWM aggregation of one level (§2.2 l.61 and l.70).
    Returns (mate, agg, n_aggregates)."""
    if order is None:
        order = visit_order(lv.n, seed, level)
    order = np.ascontiguousarray(order, dtype=np.int64)
    mate = np.empty(lv.n, dtype=np.int32)
    agg = np.empty(lv.n, dtype=np.int32)
    na = _native.lib().oracle_mwm(lv.n, _p(lv.rowptr), _p(lv.col), _p(lv.w), _p(order),
                                  _p(mate), _p(agg))
    if na < 0:
        raise ValueError("MWM: graph has an isolated vertex")
    return mate, agg, int(na)


def coarsen(lv: Level, agg: np.ndarray, nc: int) -> Level:
    """Coarse graph whose Laplacian is (P^l_{l-1})^T L P^l_{l-1} (its
    off-diagonal weights: sums of fine weights between aggregates)."""
    nnz = lv.col.shape[0]
    crowptr = np.empty(nc + 1, dtype=np.int64)
    ccol = np.empty(max(nnz, 1), dtype=np.int32)
    cw = np.empty(max(nnz, 1), dtype=np.float64)
    agg = np.ascontiguousarray(agg, dtype=np.int32)
    cnnz = _native.lib().oracle_coarsen(lv.n, _p(lv.rowptr), _p(lv.col), _p(lv.w), _p(agg), nc,
                                        _p(crowptr), _p(ccol), _p(cw))
    return Level(nc, crowptr, ccol[:cnnz].copy(), cw[:cnnz].copy())


def build_hierarchy(g, seed: int = 0, max_levels: int = 0, orders=None,
                    order: str = "random") -> Hierarchy:
    """Repeated MWM coarsening (§2.2 l.59: "We then continue to
    aggregate nodes until the desired level is achieved").

    max_levels = 0 means "level = max" ("construct the expanded
    graph to the maximum level possible (with only two nodes on the top
    level)").  Reading R5: a level is aggregated only while it has more than
    two nodes, and an aggregation that would leave fewer than two aggregates
    is not taken (the top level keeps >= 2 nodes so H~ stays connected).
    ``orders`` optionally forces the visit order per level (tests).
    ``order="natural"`` visits every level in vertex-index order: the order
    that reproduces PAPER.md Tables 1-3 (R1); the default
    ``"random"`` is reading R1's counter-based key."""
    if order not in ("random", "natural"):
        raise ValueError(order)
    h = Hierarchy(seed=seed)
    h.levels.append(Level(g.n, np.ascontiguousarray(g.rowptr, dtype=np.int64),
                          np.ascontiguousarray(g.col, dtype=np.int32),
                          np.ascontiguousarray(g.val, dtype=np.float64)))
    k = 1
    while True:
        if max_levels and h.nlevels >= max_levels:
            break
        lv = h.levels[-1]
        if lv.n <= 2:
            break
        vo = None if orders is None else orders[k - 1]
        if vo is None and order == "natural":
            vo = np.arange(lv.n, dtype=np.int64)
        mate, agg, nc = mwm(lv, seed, k, vo)
        if nc < 2:
            break
        h.mates.append(mate)
        h.aggs.append(agg)
        h.levels.append(coarsen(lv, agg, nc))
        k += 1
    return h


def P_step(h: Hierarchy, k: int) -> sp.csr_matrix:
    """P^{k+1}_k in R^{n_k x n_{k+1}}: 1 if node i is in aggregation j (l.75)."""
    agg = h.aggs[k - 1]
    nk, nk1 = h.levels[k - 1].n, h.levels[k].n
    return sp.csr_matrix((np.ones(nk), (np.arange(nk), agg)), shape=(nk, nk1))


def P_level(h: Hierarchy, k: int) -> sp.csr_matrix:
    """P^k = P^2_1 P^3_2 ... P^k_{k-1} in R^{n x n_k} (Eq. def:P); P^1 = I."""
    P = sp.identity(h.levels[0].n, format="csr")
    for j in range(1, k):
        P = (P @ P_step(h, j)).tocsr()
    return P


def composite_P(h: Hierarchy, mu: float) -> sp.csr_matrix:
    """{P(mu)}^l = [I, (-mu) P^2, (-mu)^2 P^3, ..., (-mu)^{l-1} P^l] (l.86-90)."""
    blocks = [((-mu) ** (k - 1)) * P_level(h, k) for k in range(1, h.nlevels + 1)]
    return sp.hstack(blocks, format="csr")


def ancestors(h: Hierarchy) -> list:
    """anc[k-1][i] = level-k ancestor of base node i (k = 1..l)."""
    n = h.levels[0].n
    out = [np.arange(n)]
    cur = np.arange(n)
    for k in range(1, h.nlevels):
        cur = h.aggs[k - 1][cur]
        out.append(cur.astype(np.int64))
    return out
