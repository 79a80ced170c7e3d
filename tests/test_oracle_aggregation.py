"""Pins for oracle.graph and oracle.aggregation (§2.1, §2.2).

Each check is fixed by the paper or by mathematics, not by re-running the
oracle's own formula: the paper's worked example (Eq. def:P_12), the Laplacian
identities of §2.1, an independent pure-Python transcription of the MWM rule
on tiny graphs, replay of the greedy rule, maximality, and the Galerkin
identity P^T L P computed by a dense matrix product.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import read_int_matrix
from inputs import graphs as G
from oracle import aggregation as A
from oracle import graph as GR


def dense_laplacian_by_loops(g):
    """D - A assembled entry by entry (independent of the incidence path)."""
    L = np.zeros((g.n, g.n))
    for a, b, w in zip(g.u, g.v, g.w):
        L[a, b] -= w; L[b, a] -= w; L[a, a] += w; L[b, b] += w
    return L


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_laplacian_identities(seed):
    g = G.grid2d(5, 4, "uniform1_10", seed)
    L = GR.laplacian_of_graph(g).toarray()
    np.testing.assert_allclose(L, dense_laplacian_by_loops(g), rtol=0, atol=1e-13)
    np.testing.assert_allclose(L.sum(axis=1), 0.0, atol=1e-12)          # L 1 = 0
    x = np.random.default_rng(seed).standard_normal(g.n)
    assert abs(x @ L @ x - GR.quadratic_form(g.u, g.v, g.w, x)) < 1e-10 * abs(x @ L @ x)
    ev = np.linalg.eigvalsh(L)
    assert ev[0] > -1e-10 and ev[1] > 1e-8                                # connected => one zero


def test_paper_fig2_laplacian_diagonal():
    # upper-left block diag(2,3,3,2,2,3,3,2)
    L = GR.laplacian_of_graph(G.paper_example_8()).toarray()
    assert list(np.diag(L)) == [2, 3, 3, 2, 2, 3, 3, 2]


def python_mwm(n, adj, order):
    """Independent transcription of PAPER.md l.61 / l.70 on adjacency dicts."""
    mate = {}
    for v in order:
        if v in mate:
            continue
        cands = [(w, -u) for u, w in adj[v].items() if u not in mate and u != v]
        if cands:
            w, mu = max(cands)
            u = -mu
            mate[v] = u; mate[u] = v
    pairs = sorted({(min(a, b), max(a, b)) for a, b in mate.items()})
    agg = {}
    for k, (a, b) in enumerate(pairs):
        agg[a] = k; agg[b] = k
    for v in range(n):
        if v not in mate:
            w, mu = max((w, -u) for u, w in adj[v].items())
            agg[v] = agg[-mu]
    return np.array([mate.get(v, -1) for v in range(n)]), np.array([agg[v] for v in range(n)])


def adjacency(g):
    adj = [dict() for _ in range(g.n)]
    for a, b, w in zip(g.u, g.v, g.w):
        adj[a][b] = w; adj[b][a] = w
    return adj


@pytest.mark.parametrize("seed", range(6))
def test_mwm_matches_independent_transcription(seed):
    rng = np.random.default_rng(seed)
    # random connected graph with repeated weights (exercises tie breaking)
    n = 25
    e = set()
    for i in range(1, n):
        e.add((int(rng.integers(0, i)), i))
    while len(e) < 45:
        a, b = sorted(int(x) for x in rng.integers(0, n, 2))
        if a != b:
            e.add((a, b))
    e = sorted(e)
    w = rng.integers(1, 4, size=len(e)).astype(float)
    g = G.from_edges(n, [a for a, _ in e], [b for _, b in e], w)
    lv = A.Level(g.n, g.rowptr, g.col, g.val)
    order = A.visit_order(g.n, seed, 1)
    mate, agg, na = A.mwm(lv, seed, 1, order)
    pm, pa = python_mwm(g.n, adjacency(g), list(order))
    assert np.array_equal(mate, pm)
    assert np.array_equal(agg, pa)
    assert na == agg.max() + 1


@pytest.mark.parametrize("kind,seed", [("unit", 0), ("loguniform", 1), ("uniform1_10", 2)])
def test_mwm_greedy_replay_and_maximality(kind, seed):
    g = G.grid2d(9, 7, kind, seed)
    adj = adjacency(g)
    lv = A.Level(g.n, g.rowptr, g.col, g.val)
    order = A.visit_order(g.n, seed, 1)
    mate, agg, na = A.mwm(lv, seed, 1, order)
    # replay: when v was visited unmatched it took its heaviest unmatched neighbour
    taken = set()
    for v in order:
        v = int(v)
        if v in taken:
            continue
        free = {u: w for u, w in adj[v].items() if u not in taken}
        if free:
            wmax = max(free.values())
            assert mate[v] >= 0 and free[int(mate[v])] == wmax
            assert int(mate[v]) == min(u for u, w in free.items() if w == wmax)
            taken.update({v, int(mate[v])})
        else:
            assert mate[v] == -1
    # maximal matching: no edge joins two leftovers
    left = mate < 0
    assert not np.any(left[g.u] & left[g.v])
    # leftovers join the aggregate of their heaviest neighbour (l.70)
    for v in np.nonzero(left)[0]:
        wmax = max(adj[v].values())
        h = min(u for u, w in adj[v].items() if w == wmax)
        assert agg[v] == agg[h]
    # aggregate numbering: by the smaller endpoint of the matched pair (R3)
    firsts = sorted(v for v in range(g.n) if mate[v] > v)
    assert [agg[v] for v in firsts] == list(range(na))


def test_paper_example_aggregation_and_P12():
    # aggregations {1,2},{3,4},{5,6},{7,8}; Eq. def:P_12
    g = G.paper_example_8()
    lv = A.Level(g.n, g.rowptr, g.col, g.val)
    mate, agg, na = A.mwm(lv, 0, 1, np.array([0, 2, 4, 6, 1, 3, 5, 7]))
    assert na == 4 and list(agg) == [0, 0, 1, 1, 2, 2, 3, 3]
    h = A.build_hierarchy(g, 0, max_levels=2, orders=[np.array([0, 2, 4, 6, 1, 3, 5, 7])])
    assert np.array_equal(A.P_step(h, 1).toarray(), read_int_matrix("paper_example_P12.txt"))


@pytest.mark.parametrize("seed", [0, 3])
def test_galerkin_coarse_graph(seed):
    g = G.grid2d(8, 6, "loguniform", seed)
    h = A.build_hierarchy(g, seed)
    for k in range(1, h.nlevels):
        fine = h.levels[k - 1]
        Lf = GR.laplacian_from_weights(fine.n, sp.csr_matrix((fine.w, fine.col, fine.rowptr),
                                                             shape=(fine.n, fine.n))).toarray()
        P = A.P_step(h, k).toarray()
        Lc = P.T @ Lf @ P                                   # dense Galerkin product
        c = h.levels[k]
        Wc = sp.csr_matrix((c.w, c.col, c.rowptr), shape=(c.n, c.n)).toarray()
        off = ~np.eye(c.n, dtype=bool)
        np.testing.assert_allclose(-Lc[off], Wc[off], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(Wc, Wc.T, rtol=0, atol=0)


def test_hierarchy_level_max_rules():
    for s in (4, 8, 16, 32):
        g = G.grid2d(s, s, "unit")
        h = A.build_hierarchy(g, 0)
        sz = h.sizes
        assert all(a > b for a, b in zip(sz, sz[1:]))       # strictly coarsening
        assert sz[-1] >= 2                                   # top keeps >= 2 nodes (R5)
        # each level at least halves up to leftovers: n_{k+1} <= n_k / 2
        assert all(b <= a // 2 for a, b in zip(sz, sz[1:]))
    # determinism (same seed => same hierarchy, bit for bit)
    g = G.grid2d(16, 16, "loguniform", 5)
    h1, h2 = A.build_hierarchy(g, 9), A.build_hierarchy(g, 9)
    assert all(np.array_equal(a, b) for a, b in zip(h1.aggs, h2.aggs))
    assert all(np.array_equal(a.w, b.w) for a, b in zip(h1.levels, h2.levels))


def test_composite_prolongation_row_sums():
    # {P(mu)}^l 1 = c 1 with c = sum_k (-mu)^{k-1}
    g = G.grid2d(8, 8, "unit")
    h = A.build_hierarchy(g, 1)
    for mu in (0.1, 0.5, 0.8):
        P = A.composite_P(h, mu)
        c = sum((-mu) ** k for k in range(h.nlevels))
        np.testing.assert_allclose(P @ np.ones(h.n_tilde), c, rtol=1e-14)
        # block k equals (-mu)^{k-1} times a 0/1 partition matrix (one 1 per row)
        off = h.offsets
        for k in range(1, h.nlevels + 1):
            blk = P[:, off[k - 1]:off[k]].toarray() / ((-mu) ** (k - 1))
            assert np.all((blk == 0) | (np.abs(blk - 1) < 1e-12))
            np.testing.assert_allclose(blk.sum(axis=1), 1.0, rtol=1e-12)
