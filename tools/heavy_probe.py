"""Setup phase times, aggregate-size structure and per-kernel solve profile of
a (scaled) BASELINE config -- the heavy-vertex behaviour of power-law graphs."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_07847_b200 as M  # noqa: E402
from inputs import graphs as G  # noqa: E402

os.environ.setdefault("MSP_SETUP_TIMING", "1")
dev = torch.device("cuda:0")
cfg, scale = int(sys.argv[1]), float(sys.argv[2])
t0 = time.time()
g = G.config_graph(cfg, scale)
deg = np.diff(g.rowptr)
print(f"config {cfg} scale {scale}: n={g.n} nnz={g.nnz_laplacian} maxdeg={deg.max()} gen {time.time()-t0:.1f}s",
      flush=True)
S = M.setup(g.n, torch.as_tensor(g.rowptr, device=dev), torch.as_tensor(g.col, device=dev),
            torch.as_tensor(g.val, device=dev), mu=0.8)
info = S.info()
print("info", json.dumps(info), flush=True)
sizes = list(S.level_sizes())
print("levels", sizes, flush=True)
b = torch.as_tensor(G.rhs(g.n, 0), device=dev)
x = torch.empty_like(b)
S.pcg_solve(b, x, rtol=0.0, maxit=8)
r = S.pcg_solve(b, x, rtol=0.0, maxit=32)
print(f"us/iter {r['solve_ms'] / r['iterations'] * 1000:.1f}", flush=True)
S.set_profiling(True)
S.pcg_solve(b, x, rtol=0.0, maxit=16)
S.set_profiling(False)
print("profile", {k: (round(v["ms"] / max(v["launches"], 1) * 1000, 1), v["launches"])
                  for k, v in S.get_profile().items() if v["launches"]}, flush=True)
