"""Full-size probe of one config on the GPU: generation, setup, PCG-MSP to
rtol 1e-8 (time, iterations), true residual.  python tools/probe_cfg.py 4 [scale]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2207_07847_b200 as M  # noqa: E402
from inputs import device as D, graphs as G  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
dev = torch.device("cuda:0")
t = time.time()
n, rp, col, val = D.config_csr(cfg, scale, 0, dev)
torch.cuda.synchronize()
tg = time.time() - t
nnz = int(rp[-1].item())
print(f"generated n={n} nnz_adj={nnz} in {tg:.1f}s; max degree {int((rp[1:] - rp[:-1]).max())}", flush=True)
t = time.time()
S = M.setup(n, rp, col, val, mu=0.8)
info = S.info()
print(f"setup {info['setup_ms']:.0f} ms (wall {time.time() - t:.1f}s): {json.dumps(info)}", flush=True)
print(f"level sizes {list(S.level_sizes())}", flush=True)
print(f"memory: {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB (torch)", flush=True)
b = torch.as_tensor(G.rhs(n, 4), device=dev)
x = torch.empty_like(b)
out = S.pcg_solve(b, x, rtol=1e-8, maxit=int(os.environ.get("MAXIT", "100000")))
print(f"pcg: {out['iterations']} its, converged={out['converged']}, {out['solve_ms']:.1f} ms, "
      f"{out['solve_ms'] / max(out['iterations'], 1) * 1000:.1f} us/it", flush=True)
Lx = S.apply_L(x)
print(f"true relres {float(torch.linalg.norm(b - Lx) / torch.linalg.norm(b)):.3e}", flush=True)
S.set_profiling(True)
S.pcg_solve(b, x, rtol=0.0, maxit=20)
S.set_profiling(False)
print(json.dumps({k: round(v['ms'] / max(v['launches'], 1) * 1000, 1) for k, v in S.get_profile().items() if v['launches']}))
