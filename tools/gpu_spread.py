"""Rounding spread of the GPU's own PCG-MSP iteration count on one config:
b = rhs(n, 4) times (1 + 1e-15 N(0,1)) for several seeds (reading R11).

    python tools/gpu_spread.py [--config 1] [--seeds 8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2207_07847_b200 as M  # noqa: E402
from inputs import graphs as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--seeds", type=int, default=8)
    a = ap.parse_args()
    g = G.config_graph(a.config)
    dev = torch.device("cuda:0")
    t = lambda v, d=torch.float64: torch.as_tensor(np.ascontiguousarray(v), dtype=d, device=dev)
    S = M.setup(g.n, t(g.rowptr, torch.int64), t(g.col, torch.int32), t(g.val), mu=0.8, seed=0)
    b0 = G.rhs(g.n, 4)
    res = {}
    for sd in range(0, a.seeds + 1):
        b = b0 if sd == 0 else b0 * (1 + 1e-15 * np.random.default_rng(sd).standard_normal(b0.size))
        out = S.pcg_solve(t(b), rtol=1e-8, maxit=100000)
        res[sd] = out["iterations"]
        print(sd, out["iterations"], flush=True)
    its = np.array(list(res.values()))
    print(json.dumps({"config": a.config, "iterations": res, "min": int(its.min()), "max": int(its.max())}))


if __name__ == "__main__":
    main()
