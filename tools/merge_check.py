"""Merged (coarse inside the last tier's down kernel) vs separate coarse
kernel: apply_R and a few PCG iterations must agree bit for bit."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_07847_b200 as M  # noqa: E402
from inputs import graphs as G  # noqa: E402
dev = torch.device("cuda:0")
g = G.grid2d(320, 320, "loguniform", 4)
def mk():
    return M.setup(g.n, torch.as_tensor(g.rowptr, device=dev), torch.as_tensor(g.col, device=dev),
                   torch.as_tensor(g.val, device=dev), mu=0.8, seed=11)
s1 = mk()
os.environ["MSP_NO_MERGE"] = "1"; s2 = mk(); del os.environ["MSP_NO_MERGE"]
print(s1.info()["merged_coarse"], s2.info()["merged_coarse"])
r = torch.as_tensor(G.rhs(g.n, 5), device=dev)
z1 = s1.apply_R(r).cpu().numpy(); z2 = s2.apply_R(r).cpu().numpy()
print("apply_R max abs diff", np.abs(z1 - z2).max(), "rel", np.abs(z1 - z2).max() / np.abs(z2).max())
for it in [1, 2, 5, 20]:
    o1 = s1.pcg_solve(r, rtol=0.0, maxit=it); o2 = s2.pcg_solve(r, rtol=0.0, maxit=it)
    x1 = o1["x"].cpu().numpy(); x2 = o2["x"].cpu().numpy()
    print(it, "x diff", np.abs(x1 - x2).max() / np.abs(x2).max(), o1["relres"], o2["relres"])
