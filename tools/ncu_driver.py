"""Short PCG-MSP run for ncu captures (not a bench: a few iterations of the
same launch configuration bench.py times).

    python tools/ncu_driver.py [--config 1] [--iters 6] [--precond msp]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2207_07847_b200 as M  # noqa: E402
from inputs import graphs as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--precond", default="msp")
    ap.add_argument("--mu", type=float, default=0.8)
    ap.add_argument("--scale", type=float, default=1.0)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    from inputs import device as D
    n, rp, col, val = D.config_csr(a.config, a.scale, 0, dev)
    S = M.setup(n, rp, col, val, mu=a.mu)
    b = torch.as_tensor(G.rhs(n, 0), device=dev)
    x = torch.empty_like(b)
    rep = S.pcg_solve(b, x, rtol=1e-8, maxit=a.iters, precond=a.precond)
    torch.cuda.synchronize()
    print(S.info(), rep["iterations"], file=sys.stderr)


if __name__ == "__main__":
    main()
