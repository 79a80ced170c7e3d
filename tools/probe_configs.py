"""Setup time, schedule and per-iteration solve time on larger BASELINE
configs (a few hundred iterations, then one full solve if it is short)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2207_07847_b200 as M  # noqa: E402
from inputs import graphs as G  # noqa: E402

dev = torch.device("cuda:0")
for arg in sys.argv[1:]:  # "c" or "c:scale"
    cfg, scale = (int(arg.split(":")[0]), float(arg.split(":")[1])) if ":" in arg else (int(arg), 1.0)
    t0 = time.time()
    g = G.config_graph(cfg, scale)
    tg = time.time() - t0
    print(f"config {cfg} scale {scale}: generated n={g.n} nnz={g.nnz_laplacian} in {tg:.1f}s", flush=True)
    S = M.setup(g.n, torch.as_tensor(g.rowptr, device=dev), torch.as_tensor(g.col, device=dev),
                torch.as_tensor(g.val, device=dev), mu=0.8)
    info = S.info()
    print(f"  setup {info['setup_ms']:.1f} ms, levels {info['levels']}", flush=True)
    b = torch.as_tensor(G.rhs(g.n, 0), device=dev)
    x = torch.empty_like(b)
    S.pcg_solve(b, x, rtol=0.0, maxit=64)
    r = S.pcg_solve(b, x, rtol=0.0, maxit=512)
    us = r["solve_ms"] / r["iterations"] * 1000
    full = S.pcg_solve(b, x, rtol=1e-8, maxit=20000)
    print(json.dumps({"config": cfg, "scale": scale, "n": g.n, "nnz_L": g.nnz_laplacian, "gen_s": round(tg, 1),
                      "setup_ms": round(info["setup_ms"], 1), "levels": info["levels"], "n_tilde": info["n_tilde"],
                      "tile_level": info["tile_level"], "coarse_level": info["coarse_level"], "ntiers": info["ntiers"],
                      "us_per_iter": round(us, 2), "nnz_iters_per_s": g.nnz_laplacian * 1e6 / us,
                      "full_solve": {"iterations": full["iterations"], "converged": full["converged"],
                                     "ms": round(full["solve_ms"], 1), "relres": full["relres"]}}), flush=True)
