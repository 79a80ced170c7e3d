"""PCG-MSP on assorted graph families and sizes: convergence to rtol 1e-8 and
the true residual ||b - L x|| (a property check across schedule shapes --
tiers, merged coarse, top map, multi-tile CTAs)."""
import os
import sys
import time

import numpy as np
import scipy.sparse as sp
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_07847_b200 as M  # noqa: E402
from inputs import graphs as G  # noqa: E402

dev = torch.device("cuda:0")
cases = [
    ("grid2d 517x389 loguniform", lambda: G.grid2d(517, 389, "loguniform", 3)),
    ("grid2d 1000x37 uniform", lambda: G.grid2d(1000, 37, "uniform1_10", 4)),
    ("grid3d 61x47x53", lambda: G.grid3d(61, 47, 53, seed=5)),
    ("rgg 300k", lambda: G.rgg(300000, 12.0, 6)),
    ("chung_lu 200k", lambda: G.chung_lu(200000, 2.1, 16.0, 7)),
    ("watts_strogatz 150k", lambda: G.watts_strogatz(150000, 6, None, 8)),
    ("ring 100k", lambda: G.ring(100000, 4)),
]
bad = 0
for name, make in cases:
    g = make()
    S = M.setup(g.n, torch.as_tensor(g.rowptr, device=dev), torch.as_tensor(g.col, device=dev),
                torch.as_tensor(g.val, device=dev), mu=0.8)
    info = S.info()
    b = G.rhs(g.n, 1)
    t = time.time()
    out = S.pcg_solve(torch.as_tensor(b, device=dev), rtol=1e-8, maxit=100000)
    x = out["x"].cpu().numpy()
    A = sp.csr_matrix((g.val, g.col, g.rowptr), shape=(g.n, g.n))
    Lx = np.asarray(A.sum(axis=1)).ravel() * x - A @ x
    res = np.linalg.norm(b - Lx) / np.linalg.norm(b)
    ok = out["converged"] == 1 and res <= 2e-8
    bad += not ok
    print(f"{'ok ' if ok else 'BAD'} {name:28s} n={g.n:8d} levels={info['levels']:2d} tiers={info['ntiers']} "
          f"tile_level={info['tile_level']} Kc={info['coarse_level']} merged={info['merged_coarse']} "
          f"iters={out['iterations']:6d} true_res={res:.2e} {time.time() - t:.2f}s", flush=True)
sys.exit(1 if bad else 0)
