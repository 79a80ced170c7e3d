"""Which operation is not bit-reproducible? One setup; apply_L, apply_R and
short PCG runs twice each (python tools/determinism2.py 4 0.3)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2207_07847_b200 as M  # noqa: E402
from inputs import device as D, graphs as G  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
dev = torch.device("cuda:0")
n, rp, col, val = D.config_csr(cfg, scale, 0, dev)
S = M.setup(n, rp, col, val, mu=0.8)
b = torch.as_tensor(G.rhs(n, 0), device=dev)
for name, f in [("apply_L", lambda: S.apply_L(b)), ("apply_R", lambda: S.apply_R(b))]:
    a1, a2, a3 = f(), f(), f()
    print(name, "bit-identical:", torch.equal(a1, a2), torch.equal(a1, a3),
          "max diff", float((a1 - a2).abs().max()), flush=True)
for it in (1, 2, 3, 5, 10, 65, 130):
    o1 = S.pcg_solve(b, rtol=0.0, maxit=it)
    o2 = S.pcg_solve(b, rtol=0.0, maxit=it)
    print("pcg maxit", it, "bit-identical:", torch.equal(o1["x"], o2["x"]),
          "max diff", float((o1["x"] - o2["x"]).abs().max()), flush=True)
