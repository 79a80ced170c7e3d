"""Level sizes n_k of the hierarchy for configs[i] (GPU setup)."""
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_07847_b200 as M  # noqa: E402
from inputs import graphs as G  # noqa: E402

dev = torch.device("cuda:0")
for c in [int(a) for a in sys.argv[1:]] or [1]:
    g = G.config_graph(c)
    S = M.setup(g.n, torch.as_tensor(g.rowptr, device=dev), torch.as_tensor(g.col, device=dev),
                torch.as_tensor(g.val, device=dev), mu=0.8)
    print("config", c, "levels", list(S.level_sizes()), S.info(), flush=True)
