"""Seeded synthetic graph / rhs generators (input plumbing, no method arithmetic).

Every generator returns a :class:`Graph` -- an undirected simple graph given as
an edge list ``(u, v, w)`` with ``u < v`` (unique pairs, no self loops) plus the
symmetric CSR view (rows sorted by column) that the C-ABI ``msp_setup`` takes.

Workload recipes:

* ``grid2d``   -- PAPER.md §4.1 (2D regular grids) and BASELINE configs[0..1]
* ``grid3d``   -- BASELINE configs[2] (anisotropic 7-point 3D grid)
* ``rgg``      -- BASELINE configs[3] (random geometric graph, weight 1/dist)
* ``chung_lu`` -- BASELINE configs[4] (power-law expected-degree graph)
* ``ring`` / ``watts_strogatz`` -- PAPER.md §3.2 Tables 1-2 and §4.2
* ``rhs``      -- N(0,1) projected off the ones vector (BASELINE configs)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "Graph", "from_edges", "grid2d", "grid3d", "rgg", "chung_lu", "ring",
    "watts_strogatz", "paper_example_8", "largest_component", "rhs",
    "rhs_paper", "config_graph",
]


@dataclass
class Graph:
    n: int
    u: np.ndarray        # int64 [m], u < v
    v: np.ndarray        # int64 [m]
    w: np.ndarray        # float64 [m], > 0
    rowptr: np.ndarray   # int64 [n+1]   symmetric CSR, columns sorted per row
    col: np.ndarray      # int32 [2m]
    val: np.ndarray      # float64 [2m]
    name: str = ""

    @property
    def m(self) -> int:
        return int(self.u.shape[0])

    @property
    def nnz_laplacian(self) -> int:
        """Nonzeros of the Laplacian L = D - W (off-diagonals + diagonal)."""
        return 2 * self.m + self.n


def from_edges(n: int, u, v, w, name: str = "") -> Graph:
    """Canonicalise an undirected edge list into a Graph (u<v, sorted, CSR)."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    if u.size:
        if np.any(u == v):
            raise ValueError("self loops are not allowed")
        a = np.minimum(u, v)
        b = np.maximum(u, v)
        order = np.lexsort((b, a))
        a, b, w = a[order], b[order], w[order]
        dup = (a[1:] == a[:-1]) & (b[1:] == b[:-1])
        if np.any(dup):
            raise ValueError("duplicate edges are not allowed")
        if np.any(~(w > 0)):
            raise ValueError("edge weights must be positive")
        u, v = a, b
    rows = np.concatenate([u, v])
    cols = np.concatenate([v, u])
    vals = np.concatenate([w, w])
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rowptr, rows + 1, 1)
    rowptr = np.cumsum(rowptr)
    return Graph(n=int(n), u=u, v=v, w=w, rowptr=rowptr,
                 col=cols.astype(np.int32), val=vals, name=name)


def _weights(kind: str, m: int, rng: np.random.Generator) -> np.ndarray:
    if kind == "unit":
        return np.ones(m)
    if kind == "uniform1_10":            # configs[0]: i.i.d. uniform[1,10]
        return rng.uniform(1.0, 10.0, size=m)
    if kind == "loguniform":             # configs[1]: log-uniform over [1e-3,1e3]
        return np.exp(rng.uniform(np.log(1e-3), np.log(1e3), size=m))
    if kind == "uniform0.5_2":           # configs[4]: uniform[0.5,2]
        return rng.uniform(0.5, 2.0, size=m)
    raise ValueError(kind)


def grid2d(nx: int, ny: int | None = None, weights: str = "unit", seed: int = 0) -> Graph:
    """nx x ny 4-neighbour lattice, row-major numbering (node = y*nx + x).

    Edge order for the weight draw: all horizontal edges (row-major), then all
    vertical edges (row-major)."""
    ny = nx if ny is None else ny
    idx = np.arange(nx * ny, dtype=np.int64).reshape(ny, nx)
    hu, hv = idx[:, :-1].ravel(), idx[:, 1:].ravel()
    vu, vv = idx[:-1, :].ravel(), idx[1:, :].ravel()
    u = np.concatenate([hu, vu])
    v = np.concatenate([hv, vv])
    rng = np.random.default_rng(seed)
    w = _weights(weights, u.size, rng)
    return from_edges(nx * ny, u, v, w, name=f"grid2d_{nx}x{ny}_{weights}")


def grid3d(nx: int, ny: int | None = None, nz: int | None = None,
           wxy: float = 1.0, wz: float = 1e-3, jitter: float = 0.1, seed: int = 0) -> Graph:
    """7-point anisotropic 3D grid (configs[2]): weight wxy in x/y and wz in z,
    each times uniform[1-jitter, 1+jitter]; node = (z*ny + y)*nx + x.
    Edge order: x-edges, y-edges, z-edges (each row-major)."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    idx = np.arange(nx * ny * nz, dtype=np.int64).reshape(nz, ny, nx)
    ex = (idx[:, :, :-1].ravel(), idx[:, :, 1:].ravel())
    ey = (idx[:, :-1, :].ravel(), idx[:, 1:, :].ravel())
    ez = (idx[:-1, :, :].ravel(), idx[1:, :, :].ravel())
    u = np.concatenate([ex[0], ey[0], ez[0]])
    v = np.concatenate([ex[1], ey[1], ez[1]])
    base = np.concatenate([np.full(ex[0].size, wxy), np.full(ey[0].size, wxy),
                           np.full(ez[0].size, wz)])
    rng = np.random.default_rng(seed)
    w = base * rng.uniform(1.0 - jitter, 1.0 + jitter, size=u.size)
    return from_edges(nx * ny * nz, u, v, w, name=f"grid3d_{nx}x{ny}x{nz}")


def largest_component(n: int, u: np.ndarray, v: np.ndarray, w: np.ndarray, name: str = "") -> Graph:
    """Restrict an edge list to its largest connected component, relabelled
    contiguously in increasing original-index order (§4.3 preprocessing)."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components
    if u.size == 0:
        return from_edges(1, u, v, w, name)
    a = sp.coo_matrix((np.ones(u.size), (u, v)), shape=(n, n)).tocsr()
    ncomp, lab = connected_components(a, directed=False)
    big = np.argmax(np.bincount(lab))
    keep = lab == big
    newid = np.full(n, -1, dtype=np.int64)
    newid[keep] = np.arange(int(keep.sum()))
    ek = keep[u] & keep[v]
    return from_edges(int(keep.sum()), newid[u[ek]], newid[v[ek]], w[ek], name)


def rgg(npts: int, mean_degree: float = 12.0, seed: int = 0) -> Graph:
    """Random geometric graph (configs[3]): npts uniform points in the unit
    square, edge between points closer than r with n*pi*r^2 = mean_degree,
    weight 1/distance, largest connected component only."""
    rng = np.random.default_rng(seed)
    pts = rng.uniform(0.0, 1.0, size=(npts, 2))
    r = float(np.sqrt(mean_degree / (np.pi * npts)))
    ncell = max(1, int(1.0 / r))
    cx = np.minimum((pts[:, 0] * ncell).astype(np.int64), ncell - 1)
    cy = np.minimum((pts[:, 1] * ncell).astype(np.int64), ncell - 1)
    cell = cy * ncell + cx
    order = np.argsort(cell, kind="stable")
    cell_sorted = cell[order]
    start = np.searchsorted(cell_sorted, np.arange(ncell * ncell), side="left")
    end = np.searchsorted(cell_sorted, np.arange(ncell * ncell), side="right")
    us, vs, ws = [], [], []
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            # pair every point with every point of the neighbouring cell
            ncx = cx + dx
            ncy = cy + dy
            ok = (ncx >= 0) & (ncx < ncell) & (ncy >= 0) & (ncy < ncell)
            src = np.nonzero(ok)[0]
            nb = ncy[src] * ncell + ncx[src]
            cnt = end[nb] - start[nb]
            rep_src = np.repeat(src, cnt)
            offs = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
            dst = order[np.repeat(start[nb], cnt) + offs]
            keep = rep_src < dst
            a, b = rep_src[keep], dst[keep]
            d = np.sqrt(((pts[a] - pts[b]) ** 2).sum(axis=1))
            close = (d < r) & (d > 0)
            us.append(a[close]); vs.append(b[close]); ws.append(1.0 / d[close])
    u = np.concatenate(us); v = np.concatenate(vs); w = np.concatenate(ws)
    return largest_component(npts, u, v, w, name=f"rgg_{npts}")


# ---- counter-based uniforms (splitmix64), shared by the host generator below
# and the device generator in inputs/device.py so both draw the same graph
SM_GAMMA = 0x9E3779B97F4A7C15
SM_M1 = 0xBF58476D1CE4E5B9
SM_M2 = 0x94D049BB133111EB


def splitmix64_np(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser of x + gamma (uint64 in, uint64 out, wraps mod 2^64)."""
    z = np.asarray(x, dtype=np.uint64) + np.uint64(SM_GAMMA)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(SM_M1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(SM_M2)
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, stream: int) -> int:
    """64-bit key of one random stream of one seed."""
    return int(splitmix64_np(np.array([(seed * 0x100000001B3 + stream) & (2**64 - 1)], dtype=np.uint64))[0])


def uniform01_np(key: int, idx: np.ndarray) -> np.ndarray:
    """U[0,1) number idx of the stream `key`: top 53 bits of splitmix64(key ^ idx)."""
    z = splitmix64_np(np.uint64(key) ^ np.asarray(idx, dtype=np.uint64))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def chung_lu_cdf(n: int, exponent: float = 2.1, mean_degree: float = 16.0) -> np.ndarray:
    """Normalised cumulative expected degrees d_i ~ (i+1)^(-1/(exponent-1))
    (the host computes it for both generators)."""
    d = (np.arange(1, n + 1, dtype=np.float64)) ** (-1.0 / (exponent - 1.0))
    d *= mean_degree * n / d.sum()
    cdf = np.cumsum(d)
    cdf /= cdf[-1]
    return cdf


def chung_lu(n: int, exponent: float = 2.1, mean_degree: float = 16.0, seed: int = 0,
             weights: str = "uniform0.5_2") -> Graph:
    """Chung-Lu power-law graph (configs[4]): expected degrees
    d_i proportional to (i+1)^(-1/(exponent-1)) scaled to the requested mean;
    m = n*mean/2 endpoint pairs, endpoint j of pair e drawn by inverting the
    degree cdf at U(stream 1, 2e + j); self loops and duplicate pairs
    dropped; weight of the k-th distinct edge (sorted by (min, max))
    0.5 + 1.5 U(stream 2, k); largest connected component only.  Counter-
    based uniforms, so inputs/device.py draws the identical graph on a GPU."""
    cdf = chung_lu_cdf(n, exponent, mean_degree)
    m = int(n * mean_degree / 2)
    k1 = stream_key(seed, 1)
    e = np.arange(m, dtype=np.uint64)
    a = np.searchsorted(cdf, uniform01_np(k1, 2 * e), side="right").astype(np.int64)
    b = np.searchsorted(cdf, uniform01_np(k1, 2 * e + np.uint64(1)), side="right").astype(np.int64)
    a = np.minimum(a, n - 1); b = np.minimum(b, n - 1)
    keep = a != b
    lo = np.minimum(a[keep], b[keep]); hi = np.maximum(a[keep], b[keep])
    key = np.unique(lo * n + hi)
    lo, hi = key // n, key % n
    if weights != "uniform0.5_2":
        raise ValueError(weights)
    w = 0.5 + 1.5 * uniform01_np(stream_key(seed, 2), np.arange(key.size, dtype=np.uint64))
    return largest_component(n, lo, hi, w, name=f"chunglu_{n}")


def ring(n: int, deg: int = 4) -> Graph:
    """Circulant ring: each node joined to deg/2 nearest neighbours per side,
    unit weights (Fig. 6 / Tables 1-2 'ring graphs')."""
    if deg % 2 or deg >= n:
        raise ValueError("deg must be even and < n")
    us, vs = [], []
    for k in range(1, deg // 2 + 1):
        i = np.arange(n, dtype=np.int64)
        us.append(i); vs.append((i + k) % n)
    u = np.concatenate(us); v = np.concatenate(vs)
    a, b = np.minimum(u, v), np.maximum(u, v)
    key = np.unique(a * n + b)
    return from_edges(n, key // n, key % n, np.ones(key.size), name=f"ring_{n}_{deg}")


def watts_strogatz(n: int, deg: int = 4, beta: float | None = None, seed: int = 0) -> Graph:
    """Watts-Strogatz small world (§4.2): ring(n,deg), then each edge
    (i, i+k) independently with probability beta has its far endpoint rewired to
    a uniform non-neighbour (no self loops / duplicates).  beta defaults to
    1/sqrt(n).  Retries with seed+1 if the result is disconnected."""
    beta = 1.0 / np.sqrt(n) if beta is None else beta
    for attempt in range(100):
        rng = np.random.default_rng(seed + attempt)
        adj = [set() for _ in range(n)]
        edges = []
        for k in range(1, deg // 2 + 1):
            for i in range(n):
                j = (i + k) % n
                edges.append([i, j])
                adj[i].add(j); adj[j].add(i)
        for e in edges:
            if rng.random() < beta:
                i, j = e
                cands = [x for x in range(n) if x != i and x not in adj[i]]
                if not cands:
                    continue
                t = cands[int(rng.integers(len(cands)))]
                adj[i].discard(j); adj[j].discard(i)
                adj[i].add(t); adj[t].add(i)
                e[1] = t
        u = np.array([min(a, b) for a, b in edges], dtype=np.int64)
        v = np.array([max(a, b) for a, b in edges], dtype=np.int64)
        g = from_edges(n, u, v, np.ones(u.size), name=f"ws_{n}_{deg}")
        from scipy.sparse.csgraph import connected_components
        import scipy.sparse as sp
        a = sp.csr_matrix((g.val, g.col, g.rowptr), shape=(n, n))
        if connected_components(a, directed=False)[0] == 1:
            return g
    raise RuntimeError("watts_strogatz: repeatedly disconnected")


def paper_example_8() -> Graph:
    """The unweighted 2x4 lattice of PAPER.md §3.1 Fig. 2 (nodes 1..8 -> 0..7):
    rows {1,2,3,4} and {5,6,7,8}; edges 1-2,2-3,3-4,5-6,6-7,7-8,1-5,2-6,3-7,4-8
    (degrees 2,3,3,2,2,3,3,2 as in the displayed L_G block)."""
    e = [(0, 1), (1, 2), (2, 3), (4, 5), (5, 6), (6, 7), (0, 4), (1, 5), (2, 6), (3, 7)]
    u = np.array([a for a, _ in e]); v = np.array([b for _, b in e])
    return from_edges(8, u, v, np.ones(len(e)), name="paper_fig2")


def rhs(n: int, seed: int = 0) -> np.ndarray:
    """b ~ N(0,1) i.i.d., projected orthogonal to the ones vector."""
    b = np.random.default_rng(seed + 7919).standard_normal(n)
    return b - b.mean()


def rhs_paper(n: int) -> np.ndarray:
    """PAPER.md §4: b = [1, 1, ..., 1, 1-n]^T (sums to zero)."""
    b = np.ones(n)
    b[-1] = 1.0 - n
    return b


def config_graph(idx: int, scale: float = 1.0, seed: int = 0) -> Graph:
    """BASELINE.json configs[idx]; ``scale`` < 1 shrinks the linear size for
    tests (same family and weight distribution)."""
    if idx == 0:
        s = max(4, int(round(32 * scale)))
        return grid2d(s, s, "uniform1_10", seed)
    if idx == 1:
        s = max(4, int(round(1024 * scale)))
        return grid2d(s, s, "loguniform", seed)
    if idx == 2:
        s = max(4, int(round(256 * scale)))
        return grid3d(s, s, s, 1.0, 1e-3, 0.1, seed)
    if idx == 3:
        return rgg(max(64, int(4_000_000 * scale * scale)), 12.0, seed)
    if idx == 4:
        return chung_lu(max(256, int(50_000_000 * scale * scale)), 2.1, 16.0, seed)
    raise ValueError(idx)
