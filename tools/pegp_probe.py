"""PEGP on a BASELINE config: H~ size and build time, one apply_R (inner CG
iterations, device time, per-kernel profile), then PCG-PEGP for a bounded
number of outer iterations (argv[2], default 20) next to PCG-MSP.

    python tools/pegp_probe.py CONFIG [OUTER_MAXIT] [MU] [SCALE]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2207_07847_b200 as M  # noqa: E402
from inputs import graphs as G  # noqa: E402

dev = torch.device("cuda:0")
cfg = int(sys.argv[1])
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 20
mu = float(sys.argv[3]) if len(sys.argv) > 3 else 0.8
scale = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
g = G.config_graph(cfg, scale)
S = M.setup(g.n, torch.as_tensor(g.rowptr, device=dev), torch.as_tensor(g.col, device=dev),
            torch.as_tensor(g.val, device=dev), mu=mu)
info = S.info()
t = time.time()
pi = S.pegp_info()
print("n", g.n, "n_tilde", info["n_tilde"], "levels", info["levels"], "pegp", pi, f"wall {time.time() - t:.2f}s",
      flush=True)
b = torch.as_tensor(G.rhs(g.n, 0), device=dev)
S.pegp_params(1e-13, 200000, 0)
z = S.apply_R(b, precond="pegp")  # warm (graph capture)
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
z = S.apply_R(b, precond="pegp")
e1.record(st)
torch.cuda.synchronize()
inner = S.pegp_info()["last_inner_iterations"]
ms = e0.elapsed_time(e1)
print(f"apply_R pegp: inner {inner}, {ms:.1f} ms, {1000 * ms / max(inner, 1):.1f} us per inner iteration", flush=True)
S.set_profiling(True)
S.apply_R(b, precond="pegp")
S.set_profiling(False)
prof = S.get_profile()
hn, nt = pi["hnnz"], info["n_tilde"]
for k in ("pegp_spmv", "pegp_sweeps"):
    v = prof[k]
    if v["launches"]:
        avg = v["ms"] / v["launches"]
        extra = ""
        if k == "pegp_spmv":
            extra = f" {(12 * hn + 44 * nt) / (avg * 1e-3) / 1e9:.0f} GB/s algorithmic"
        print(f"  {k}: {v['launches']} x {1000 * avg:.2f} us{extra}", flush=True)
for pc in ["msp", "pegp"]:
    t = time.time()
    r = S.pcg_solve(b, rtol=1e-8, maxit=maxit, precond=pc)
    torch.cuda.synchronize()
    extra = f" inner total {S.pegp_info()['last_solve_inner_iterations']}" if pc == "pegp" else ""
    print(pc, json.dumps({k: v for k, v in r.items() if k != "x"}), f"wall {time.time() - t:.2f}s{extra}", flush=True)
