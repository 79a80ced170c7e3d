#!/usr/bin/env python3
"""Full-size PCG-MSP record of the ORACLE (calls only oracle/ and inputs/).

    python tools/oracle_record.py --config 1 [--perturb SEED] [--out DIR]

Runs the oracle's PCG with the MSP preconditioner (oracle.pcg.pcg with
oracle.precond.msp, mu = 0.8, rtol 1e-8, x0 = 0; R9-R11) on
BASELINE configs[c] at full size with the rhs the GPU parity test uses
(inputs.graphs.rhs(n, 4)), and writes

    <out>/cfg<c>_pcg_msp[_p<seed>].npz : iterations, converged, the residual
        history, and the solution x (fp64)

``--perturb s`` multiplies b by (1 + 1e-15 N(0,1)) from seed s -- the
rounding-level perturbation that defines the R11 iteration band.  Nothing in
this script touches the CUDA path: the stored values come from the oracle
alone (the rule for stored expected values).
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from inputs import graphs as G                                   # noqa: E402
from oracle import aggregation as A, expansion as E, graph as GR  # noqa: E402
from oracle import pcg as PC, precond as PR                      # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--perturb", type=int, default=0)
    ap.add_argument("--mu", type=float, default=0.8)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "full_size"))
    ap.add_argument("--apply-l", default="csr", choices=["csr", "incidence"],
                    help="L p as the assembled CSR Laplacian (default) or as B^T W B p (oracle.graph.apply_L, "
                         "the definition with the exact diagonal)")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    t0 = time.time()
    g = G.config_graph(args.config)
    h = A.build_hierarchy(g, 0)
    R = PR.msp(E.expand_msp_only(g, h, args.mu))
    L = GR.laplacian_of_graph(g)
    b = G.rhs(g.n, 4)
    if args.perturb:
        b = b * (1 + 1e-15 * np.random.default_rng(args.perturb).standard_normal(b.size))
    print(f"setup {time.time() - t0:.1f}s n={g.n} levels={h.nlevels}", flush=True)
    t0 = time.time()
    if args.apply_l == "incidence":
        B = GR.incidence(g.n, g.u, g.v).tocsr()
        BT = B.T.tocsr()
        res = PC.pcg(lambda v: BT @ (g.w * (B @ v)), b, R, 1e-8, 100000)
    else:
        res = PC.pcg(lambda v: L @ v, b, R, 1e-8, 100000)
    print(f"pcg {time.time() - t0:.1f}s iterations={res.iterations} converged={res.converged}", flush=True)
    name = (f"cfg{args.config}_pcg_msp" + (f"_p{args.perturb}" if args.perturb else "")
            + ("_inc" if args.apply_l == "incidence" else "") + ".npz")
    kw = dict(iterations=res.iterations, converged=res.converged, resnorms=np.array(res.resnorms),
              mu=args.mu, rhs_seed=4, hierarchy_seed=0)
    if not args.perturb:
        kw["x"] = res.x
    np.savez_compressed(os.path.join(args.out, name), **kw)


if __name__ == "__main__":
    main()
