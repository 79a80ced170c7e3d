"""Device-side (torch, CUDA) input generators -- input plumbing only.

The full-size BASELINE configs[4] graph (Chung-Lu, 50M vertices, ~400M
edges) takes tens of minutes and tens of GB through the numpy generator, so
it is drawn on the GPU here with the *same* counter-based recipe as
``inputs.graphs.chung_lu`` (splitmix64 uniforms, the host-computed degree
cdf, the same dedup, weight and largest-component rules): the two produce
identical CSR arrays, which ``tests/test_gpu_inputs.py`` checks at reduced
size.  Like the rest of ``inputs/`` this module holds none of the method's
arithmetic.
"""
from __future__ import annotations

import numpy as np
import torch

from . import graphs as G


def _u64_const(c: int) -> int:
    """A uint64 constant as the int64 with the same bits."""
    return c - (1 << 64) if c >= (1 << 63) else c


_GAMMA = _u64_const(G.SM_GAMMA)
_M1 = _u64_const(G.SM_M1)
_M2 = _u64_const(G.SM_M2)


def _lsr(z: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    z = x + _GAMMA                        # int64 arithmetic wraps mod 2^64
    z = (z ^ _lsr(z, 30)) * _M1
    z = (z ^ _lsr(z, 27)) * _M2
    return z ^ _lsr(z, 31)


def uniform01(key: int, idx: torch.Tensor) -> torch.Tensor:
    z = splitmix64(torch.bitwise_xor(idx, _u64_const(key)))
    return _lsr(z, 11).to(torch.float64) * (1.0 / 9007199254740992.0)


def _largest_component(n: int, lo: torch.Tensor, hi: torch.Tensor):
    """Label of every vertex = smallest vertex id of its component (min-label
    propagation + pointer jumping); returns the keep mask of the largest
    component (ties: smallest label, like np.argmax over the bincount)."""
    dev = lo.device
    lab = torch.arange(n, device=dev, dtype=torch.int64)
    while True:
        m = torch.minimum(lab[lo], lab[hi])
        new = lab.clone()
        new.scatter_reduce_(0, lo, m, reduce="amin")
        new.scatter_reduce_(0, hi, m, reduce="amin")
        while True:  # pointer jumping
            nn = new[new]
            if torch.equal(nn, new):
                break
            new = nn
        if torch.equal(new, lab):
            break
        lab = new
    cnt = torch.bincount(lab, minlength=n)
    big = int(torch.argmax(cnt).item())
    return lab == big


def chung_lu_csr(n: int, exponent: float = 2.1, mean_degree: float = 16.0, seed: int = 0,
                 device="cuda", chunk: int = 1 << 27):
    """inputs.graphs.chung_lu on the device: returns (n_lcc, rowptr int64,
    col int32, val float64) as device tensors, identical to the host
    generator's Graph.rowptr / col / val."""
    dev = torch.device(device)
    cdf = torch.as_tensor(G.chung_lu_cdf(n, exponent, mean_degree), device=dev)
    m = int(n * mean_degree / 2)
    k1 = G.stream_key(seed, 1)
    keys = []
    for e0 in range(0, m, chunk):
        e = torch.arange(e0, min(m, e0 + chunk), device=dev, dtype=torch.int64)
        a = torch.searchsorted(cdf, uniform01(k1, 2 * e), right=True).clamp_(max=n - 1)
        b = torch.searchsorted(cdf, uniform01(k1, 2 * e + 1), right=True).clamp_(max=n - 1)
        keep = a != b
        a, b = a[keep], b[keep]
        keys.append(torch.minimum(a, b) * n + torch.maximum(a, b))
        del e, a, b, keep
    key = torch.unique(torch.cat(keys))
    del keys
    lo, hi = key // n, key % n
    w = 0.5 + 1.5 * uniform01(G.stream_key(seed, 2), torch.arange(key.numel(), device=dev, dtype=torch.int64))
    del key
    keepv = _largest_component(n, lo, hi)
    newid = torch.cumsum(keepv.to(torch.int64), 0) - 1
    ek = keepv[lo] & keepv[hi]
    lo, hi, w = newid[lo[ek]], newid[hi[ek]], w[ek]
    nl = int(keepv.sum().item())
    del newid, ek, keepv
    rows = torch.cat([lo, hi])
    cols = torch.cat([hi, lo])
    vals = torch.cat([w, w])
    del lo, hi, w
    order = torch.argsort(rows * nl + cols)
    rows, cols, vals = rows[order], cols[order], vals[order]
    del order
    rowptr = torch.zeros(nl + 1, device=dev, dtype=torch.int64)
    rowptr[1:] = torch.cumsum(torch.bincount(rows, minlength=nl), 0)
    return nl, rowptr, cols.to(torch.int32), vals


def config_csr(idx: int, scale: float = 1.0, seed: int = 0, device="cuda"):
    """BASELINE configs[idx] as device CSR (n, rowptr, col, val): configs[4]
    drawn on the device, the others drawn on the host and copied."""
    dev = torch.device(device)
    if idx == 4:
        return chung_lu_csr(max(256, int(50_000_000 * scale * scale)), 2.1, 16.0, seed, dev)
    g = G.config_graph(idx, scale, seed)
    return (g.n, torch.as_tensor(g.rowptr, device=dev), torch.as_tensor(g.col, device=dev),
            torch.as_tensor(g.val, device=dev))
