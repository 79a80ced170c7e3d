"""Per-iteration timing of the PCG-MSP solve under different schedule knobs
(env vars read by libmsp_b200.so at setup), one process per setting.

    python tools/sweep.py --iters 2000 "MSP_TILE_T=512" "MSP_TILE_T=256" ...
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHILD = r"""
import json, sys, torch
sys.path.insert(0, %r)
import paper_2207_07847_b200 as M
from inputs import graphs as G, device as D
dev = torch.device('cuda:0')
n, rp, col, val = D.config_csr(%d, %r, 0, dev)
S = M.setup(n, rp, col, val, mu=0.8)
del rp, col, val
b = torch.as_tensor(G.rhs(n, 0), device=dev); x = torch.empty_like(b)
S.pcg_solve(b, x, rtol=0.0, maxit=200)
rs = [S.pcg_solve(b, x, rtol=0.0, maxit=%d) for _ in range(3)]
ms = min(r['solve_ms'] for r in rs)
S.set_profiling(True); S.pcg_solve(b, x, rtol=0.0, maxit=200); S.set_profiling(False)
prof = {k: round(v['ms'] / max(v['launches'], 1) * 1000, 2) for k, v in S.get_profile().items() if v['launches']}
print(json.dumps({'us_per_iter': round(ms / rs[0]['iterations'] * 1000, 2), 'prof_us': prof, 'info': S.info()}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=2000)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("settings", nargs="*")
    a = ap.parse_args()
    for st in (a.settings or [""]):
        env = dict(os.environ)
        for kv in st.split():
            k, v = kv.split("=", 1)
            if k == "LIB":  # a library variant built with extra nvcc flags, e.g. LIB=-DMSP_TT=128
                from paper_2207_07847_b200 import build as B
                sys.path.insert(0, ROOT)
                path = os.path.join(ROOT, "build_variant_" + v.replace("-D", "").replace("=", "_").replace(",", "+") + ".so")
                B.build(force=True, extra=v.split(","), lib=path)
                env["MSP_LIB_OVERRIDE"] = path
            else:
                env[k] = v
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, a.config, a.scale, a.iters)], env=env,
                           capture_output=True, text=True, timeout=600)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:]
        print(f"[{st}] {line}", flush=True)


if __name__ == "__main__":
    main()
