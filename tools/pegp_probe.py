"""PEGP-preconditioned PCG on a BASELINE config: outer iterations, inner
iterations and time (a bounded number of outer iterations when maxit given)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_07847_b200 as M  # noqa: E402
from inputs import graphs as G  # noqa: E402

dev = torch.device("cuda:0")
cfg = int(sys.argv[1]); maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
g = G.config_graph(cfg)
S = M.setup(g.n, torch.as_tensor(g.rowptr, device=dev), torch.as_tensor(g.col, device=dev),
            torch.as_tensor(g.val, device=dev), mu=0.8)
b = torch.as_tensor(G.rhs(g.n, 0), device=dev)
print("pegp params", S.pegp_params() if hasattr(S, "pegp_params") else None, flush=True)
for pc in ["msp", "pegp"]:
    t = time.time()
    r = S.pcg_solve(b, rtol=1e-8, maxit=maxit, precond=pc)
    torch.cuda.synchronize()
    print(pc, json.dumps({k: v for k, v in r.items() if k != "x"}), f"wall {time.time() - t:.2f}s", flush=True)
