"""One PEGP apply on a BASELINE config with a bounded inner CG (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_07847_b200 as M  # noqa: E402
from inputs import graphs as G  # noqa: E402

dev = torch.device("cuda:0")
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = G.config_graph(cfg, 1.0)
S = M.setup(g.n, torch.as_tensor(g.rowptr, device=dev), torch.as_tensor(g.col, device=dev),
            torch.as_tensor(g.val, device=dev), mu=0.8)
S.pegp_params(1e-13, 64, 0)
b = torch.as_tensor(G.rhs(g.n, 0), device=dev)
S.set_profiling(True)   # no graphs: kernels launched one by one
S.apply_R(b, precond="pegp")
torch.cuda.synchronize()
print("done", S.pegp_info())
