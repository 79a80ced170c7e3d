"""PCG-PEGP against the inner CG's stopping tolerance (reading R13): outer
iterations, total inner iterations and time to rtol 1e-8 on a 256x256
log-uniform grid (to convergence), and the residual reached after a bounded
number of outer iterations on BASELINE configs[1].

    python tools/pegp_inner_rtol.py [OUTER_MAXIT_CFG1]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_07847_b200 as M  # noqa: E402
from inputs import graphs as G  # noqa: E402

dev = torch.device("cuda:0")
maxit1 = int(sys.argv[1]) if len(sys.argv) > 1 else 60


def run(g, tag, maxit, tols):
    S = M.setup(g.n, torch.as_tensor(g.rowptr, device=dev), torch.as_tensor(g.col, device=dev),
                torch.as_tensor(g.val, device=dev), mu=0.8)
    b = torch.as_tensor(G.rhs(g.n, 0), device=dev)
    r = S.pcg_solve(b, rtol=1e-8, maxit=max(maxit, 100000 if maxit > 1000 else maxit), precond="msp")
    print(json.dumps({"case": tag, "precond": "msp", "iterations": r["iterations"], "converged": r["converged"],
                      "relres": r["relres"], "solve_ms": r["solve_ms"]}), flush=True)
    for tol in tols:
        S.pegp_params(tol, 200000, 0)
        S.pcg_solve(b, rtol=1e-8, maxit=2, precond="pegp")  # graph capture
        r = S.pcg_solve(b, rtol=1e-8, maxit=maxit, precond="pegp")
        torch.cuda.synchronize()
        print(json.dumps({"case": tag, "precond": "pegp", "inner_rtol": tol, "iterations": r["iterations"],
                          "converged": r["converged"], "relres": r["relres"], "solve_ms": r["solve_ms"],
                          "inner_total": S.pegp_info()["last_solve_inner_iterations"]}), flush=True)


TOLS = [1e-13, 1e-10, 1e-8, 1e-6, 1e-4, 1e-2]
run(G.grid2d(256, 256, "loguniform", 3), "grid_256x256_loguniform", 5000, TOLS)
run(G.config_graph(1), "configs[1]", maxit1, [1e-13, 1e-8, 1e-4])
