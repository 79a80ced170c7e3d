"""Run-to-run determinism of setup + PCG-MSP on one config: two setups of
the same graph, two solves each; prints iteration counts and whether the
solutions are bit-identical.   python tools/determinism.py 4 0.3"""
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
outs = []
for rep in range(2):
    n, rp, col, val = D.config_csr(cfg, scale, 0, dev)
    S = M.setup(n, rp, col, val, mu=0.8)
    b = torch.as_tensor(G.rhs(n, 0), device=dev)
    for k in range(2):
        o = S.pcg_solve(b, rtol=1e-8, maxit=100000)
        outs.append((o["iterations"], o["x"].clone()))
        print(rep, k, o["iterations"], flush=True)
    del S
for i in range(1, len(outs)):
    print(f"solve {i}: iterations {outs[i][0]} vs {outs[0][0]}, x bit-identical: {torch.equal(outs[i][1], outs[0][1])}")
