"""Build a -DMSP_TRACE copy of the library and run apply_R once on config 1
(phase timestamps of CTA 0 printed by the kernels)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2207_07847_b200 import build as B  # noqa: E402

lib = os.path.join(ROOT, "build_trace_libmsp.so")
B.build(force=True, extra=["-DMSP_TRACE"] + [f for f in os.environ.get("TRACE_EXTRA", "").split(",") if f], lib=lib)
code = r"""
import os, sys, torch
sys.path.insert(0, %r)
import paper_2207_07847_b200 as M
from inputs import graphs as G
dev = torch.device('cuda:0')
g = G.config_graph(%d)
S = M.setup(g.n, torch.as_tensor(g.rowptr, device=dev), torch.as_tensor(g.col, device=dev),
            torch.as_tensor(g.val, device=dev), mu=0.8)
r = torch.as_tensor(G.rhs(g.n, 0), device=dev)
import ctypes, numpy as np
L = ctypes.CDLL(%r)
buf = np.zeros((8, 16), dtype=np.uint64)
for _ in range(3):
    z = S.apply_R(r); torch.cuda.synchronize()
x = torch.empty_like(r)
ph = np.zeros((8, 16), dtype=np.uint64)
L.msp_debug_phase(ph.ctypes.data, 1)
S.pcg_solve(r, x, rtol=0.0, maxit=40); torch.cuda.synchronize()
L.msp_debug_phase(ph.ctypes.data, 0)
for kid, nm in {2: 'k_tile_down<FIRST>', 3: 'k_tile_down<tier2>', 4: 'k_tile_up<FIRST>', 5: 'k_tile_up<tier2>'}.items():
    c = int(ph[kid][15])
    if c:
        ghz = float(os.environ.get('SM_GHZ', '1.965'))
        print('PHASE', nm, 'ctas', c, ' '.join(f'{k}:{ph[kid][k] / c / ghz / 1000:.2f}us' for k in range(8) if ph[kid][k]))
L.msp_debug_trace(buf.ctypes.data)
names = {1: 'k_coarse', 2: 'k_tile_down<FIRST>', 3: 'k_tile_down<tier2>', 4: 'k_tile_up<FIRST>', 5: 'k_tile_up<tier2>'}
names[6] = 'k_spmv_pipe'
names[7] = 'k_spmv_up'
T0 = min(int(buf[k][0]) for k in names if buf[k][0])
for kid, nm in sorted(names.items(), key=lambda kv: int(buf[kv[0]][0]) or 1 << 62):
    row = buf[kid].astype(np.int64)
    nz = [i for i in range(16) if row[i]]
    if nz:
        t0 = row[nz[0]]
        end = f' end={(row[15]-T0)/1000:.2f}us' if row[15] else ''
        # tags >= 1 are SM clock cycles (slot 14 = cycles at tag 0), at the bench clock
        ghz = float(os.environ.get('SM_GHZ', '1.965'))
        print('TRACE', nm, f'start={(t0-T0)/1000:.2f}us' + end,
              ' '.join(f'{i}:{(row[i]-row[14])/ghz/1000:.2f}us' for i in nz if 0 < i < 14))
print('INFO', S.info())
""" % (ROOT, int(sys.argv[1]) if len(sys.argv) > 1 else 1, lib)
env = dict(os.environ, MSP_LIB_OVERRIDE=lib)
out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
lines = [l for l in out.stdout.splitlines() if l.startswith("TRACE") or l.startswith("INFO") or l.startswith("PHASE")]
print(out.stderr[-2000:])
# last apply only: group by kernel, print deltas
last = lines[-(len(lines) // 3 + 1):]
prev = {}
for l in lines:
    print(l)
