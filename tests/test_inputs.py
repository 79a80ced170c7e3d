"""Input generators: shapes, edge counts, determinism, rhs compatibility."""
import numpy as np

from inputs import graphs as G


def test_grid_counts_and_determinism():
    g = G.grid2d(16, 16, "unit")
    assert g.n == 256 and g.m == 2 * 16 * 15
    a, b = G.grid2d(32, 32, "uniform1_10", 0), G.grid2d(32, 32, "uniform1_10", 0)
    assert a.m == 1984 and np.array_equal(a.w, b.w)           # configs[0]: 1,984 edges
    assert a.w.min() >= 1 and a.w.max() <= 10
    c = G.grid2d(64, 64, "loguniform", 0)
    assert c.w.min() >= 1e-3 and c.w.max() <= 1e3
    g3 = G.grid3d(6, 5, 4, seed=1)
    assert g3.m == (5 * 5 * 4) + (6 * 4 * 4) + (6 * 5 * 3)


def test_csr_is_symmetric_sorted():
    g = G.rgg(3000, 12.0, 0)
    for i in range(0, g.n, 97):
        cols = g.col[g.rowptr[i]:g.rowptr[i + 1]]
        assert np.all(np.diff(cols) > 0) and np.all(cols != i)
    import scipy.sparse as sp
    A = sp.csr_matrix((g.val, g.col, g.rowptr), shape=(g.n, g.n))
    assert abs(A - A.T).max() == 0
    deg = np.diff(g.rowptr)
    assert 8 < deg.mean() < 14                                   # mean degree ~12


def test_chung_lu_and_ws_ring():
    g = G.chung_lu(20000, 2.1, 16.0, 0)
    deg = np.diff(g.rowptr)
    assert deg.max() > 20 * np.median(deg)                        # heavy tail
    r = G.ring(10, 4)
    assert r.m == 20 and np.all(np.diff(r.rowptr) == 4)           # PAPER.md Fig. 6
    ws = G.watts_strogatz(16, 4, 0.25, 0)
    assert ws.m == 32                                            # Fig. 7: rewiring keeps m


def test_rhs_orthogonal_to_ones():
    b = G.rhs(1000, 3)
    assert abs(b.sum()) < 1e-10
    assert G.rhs_paper(8).sum() == 0 and G.rhs_paper(8)[-1] == -7


def test_chung_lu_device_recipe_matches_host_on_cpu():
    """inputs.device draws configs[4]'s Chung-Lu graph with torch (on the GPU
    at full size); run here on the CPU it yields the host generator's CSR
    bit for bit (counter-based uniforms, same dedup / weights / LCC)."""
    import torch
    from inputs import device as D
    g = G.chung_lu(20000, 2.1, 16.0, 5)
    n, rp, c, v = D.chung_lu_csr(20000, 2.1, 16.0, 5, "cpu")
    assert n == g.n
    assert np.array_equal(rp.numpy(), g.rowptr) and np.array_equal(c.numpy(), g.col)
    assert np.array_equal(v.numpy(), g.val)
    assert c.dtype == torch.int32 and v.dtype == torch.float64
