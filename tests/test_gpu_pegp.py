"""GPU parity of the PEGP path (§3.2) against the oracle.

* msp_apply_LH: the matrix-free L_H~ x~ equals the oracle's assembled L_H~
  (positive edges of Eq. def:L_ell) within 1e-12 relative (fp64).
* msp_solve_LH: inexact by construction (reading R13): the inner CG's
  residual in the L_H~ system is <= inner_rtol (checked with the oracle's
  L_H~), and the result agrees with the oracle's pseudo-inverse solve within
  the bound that residual implies.
* apply_R PEGP and PCG with PEGP against the oracle's exact PEGP.
"""
import json
import os

import numpy as np
import pytest

from inputs import graphs as G
from oracle import aggregation as A
from oracle import expansion as E
from oracle import graph as GR
from oracle import pcg as PC
from oracle import precond as PR

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2207_07847_b200 as M  # noqa: E402

DEV = torch.device("cuda:0")


def dt(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=DEV)


GRAPHS = {
    "grid_9x7_loguniform": lambda: G.grid2d(9, 7, "loguniform", 1),
    "grid_20x13_u1_10": lambda: G.grid2d(20, 13, "uniform1_10", 2),
    "ws_300": lambda: G.watts_strogatz(300, 4, None, 1),
    "rgg_800": lambda: G.rgg(800, 12.0, 3),
    "chung_lu_600": lambda: G.chung_lu(600, 2.1, 16.0, 4),
    "grid3d_6": lambda: G.grid3d(6, 5, 4, seed=1),
    # >= 10k vertices: several coarse-CTA / large-level splits of the inner CG
    "grid_120x100_loguniform": lambda: G.grid2d(120, 100, "loguniform", 3),
    "rgg_12000": lambda: G.rgg(12000, 12.0, 4),
}

PARITY_LOG = os.environ.get("MSP_PARITY_LOG", os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "parity_log.jsonl"))


def record(case, quantity, err, tol):
    """Append the achieved error and the bar applied to the parity log, then assert."""
    try:
        os.makedirs(os.path.dirname(PARITY_LOG), exist_ok=True)
        with open(PARITY_LOG, "a") as f:
            f.write(json.dumps({"case": case, "quantity": quantity, "err": err, "tol": tol}) + "\n")
    except OSError:
        pass
    assert err <= tol, (case, quantity, err, tol)


@pytest.fixture(scope="module", params=list(GRAPHS))
def case(request):
    g = GRAPHS[request.param]()
    mu, seed = 0.8, 5
    h = A.build_hierarchy(g, seed)
    sysm = E.expand(g, h, mu)
    s = M.setup(g.n, dt(g.rowptr, torch.int64), dt(g.col, torch.int32), dt(g.val), mu=mu, seed=seed)
    return request.param, g, h, sysm, s


def test_apply_LH(case):
    name, g, h, sysm, s = case
    W = sysm.WH.tocsr()
    for seed in (0, 1):
        x = np.random.default_rng(seed).standard_normal(h.n_tilde)
        y = s.apply_LH(dt(x)).cpu().numpy()
        # reference in the difference form from the oracle's H~ edge weights
        # (R7: exact diagonal), extended precision
        ref = np.asarray(PR._ld_laplacian_apply(W, x), dtype=np.float64)
        record(name, "apply_LH", float(np.abs(y - ref).max() / np.abs(ref).max()), 1e-12)


@pytest.mark.parametrize("mu", [0.3, 0.5])
def test_apply_LH_other_mu(mu):
    g = G.grid2d(11, 10, "loguniform", 6)
    h = A.build_hierarchy(g, 2)
    sysm = E.expand(g, h, mu)
    s = M.setup(g.n, dt(g.rowptr, torch.int64), dt(g.col, torch.int32), dt(g.val), mu=mu, seed=2)
    x = np.random.default_rng(3).standard_normal(h.n_tilde)
    ref = sysm.LH @ x
    assert np.abs(s.apply_LH(dt(x)).cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()


def test_solve_LH(case):
    name, g, h, sysm, s = case
    LH = sysm.LH
    r = np.random.default_rng(7).standard_normal(h.n_tilde)
    r -= r.mean()
    # one refinement step (R13): the CG's recursively updated residual drifts
    # from the true one over long runs; the double-double residual restores it
    s.pegp_params(1e-13, 20000, 1)
    z, it = s.solve_LH(dt(r))
    z = z.cpu().numpy()
    assert it > 0
    res = np.linalg.norm(LH @ z - r)
    record(name, "solve_LH_residual", float(res / np.linalg.norm(r)), 2e-13)
    assert abs(z.sum()) <= 1e-10 * np.abs(z).sum()
    zref = PR.PinvSolver(LH)(r)
    # ||z - z*|| <= ||L_H (z - z*)|| / lambda_2(L_H)
    lam2 = np.sort(np.linalg.eigvalsh(LH.toarray()))[1]
    assert np.linalg.norm(z - zref) <= 1.5 * res / lam2 + 1e-12 * np.linalg.norm(zref), name


def test_apply_R_pegp(case):
    """apply_R PEGP at the north star's fixed 1e-12 (relative, max-norm)
    against the oracle's refined R r (R14), with the inner CG followed by two
    double-double refinement steps (R13)."""
    name, g, h, sysm, s = case
    s.pegp_params(1e-13, 20000, 2)
    r = G.rhs(g.n, 8)
    z = s.apply_R(dt(r), precond="pegp").cpu().numpy()
    zr = PR.pegp_refined(sysm)(r)
    record(name, "apply_R_pegp", float(np.abs(z - zr).max() / np.abs(zr).max()), 1e-12)


def test_apply_R_pegp_deterministic(case):
    name, g, h, sysm, s = case
    s.pegp_params(1e-13, 20000, 0)
    r = dt(G.rhs(g.n, 10))
    z1 = s.apply_R(r, precond="pegp").cpu().numpy()
    z2 = s.apply_R(r, precond="pegp").cpu().numpy()
    assert np.array_equal(z1, z2), name


def test_pcg_pegp(case):
    name, g, h, sysm, s = case
    s.pegp_params(1e-13, 20000)
    L = GR.laplacian_of_graph(g)
    b = G.rhs(g.n, 9)
    ref = PC.pcg(lambda v: L @ v, b, PR.pegp(sysm), 1e-8, 2000)
    out = s.pcg_solve(dt(b), rtol=1e-8, maxit=2000, precond="pegp")
    assert out["converged"] == 1 and ref.converged
    assert abs(out["iterations"] - ref.iterations) <= 2, (name, out["iterations"], ref.iterations)
    x = out["x"].cpu().numpy()
    e = x - ref.x
    e -= e.mean()
    xs = ref.x - ref.x.mean()
    assert np.sqrt(abs(e @ (L @ e))) <= 1e-8 * np.sqrt(xs @ (L @ xs)), name


def test_full_size_config1_pegp():
    """configs[1] at full size (1,048,576 vertices, n~ = 1.94M, H~ with 37.9M
    stored entries; the launch configuration `bench.py --precond pegp` times).
    The oracle cannot factor L_H~ at this size in the suite's time, so the
    apply is checked through what it can compute here:
    * apply_LH on every row against the oracle's H~ edge weights in the
      difference form, extended precision (1e-12);
    * solve_LH (inner CG to 1e-13 + one double-double refinement step): its
      true residual, formed with the ORACLE's assembled L_H~, is <= 2e-13
      relative, and the solution has zero mean;
    * apply_R PEGP = P(mu) solve_LH(P(mu)^T r) with the oracle's P on both
      sides of the GPU inner solve (1e-12): the restriction / prolongation
      wiring at this size."""
    g = G.config_graph(1)
    mu, seed = 0.8, 0
    h = A.build_hierarchy(g, seed)
    sysm = E.expand(g, h, mu)
    s = M.setup(g.n, dt(g.rowptr, torch.int64), dt(g.col, torch.int32), dt(g.val), mu=mu, seed=seed)
    assert s.pegp_info()["hnnz"] == sysm.WH.nnz
    name = "config1_full_pegp"
    x = np.random.default_rng(0).standard_normal(h.n_tilde)
    y = s.apply_LH(dt(x)).cpu().numpy()
    ref = np.asarray(PR._ld_laplacian_apply(sysm.WH.tocsr(), x), dtype=np.float64)
    record(name, "apply_LH", float(np.abs(y - ref).max() / np.abs(ref).max()), 1e-12)
    P = sysm.P()
    r = G.rhs(g.n, 8)
    rt = P.T @ r
    s.pegp_params(1e-13, 200000, 1)
    zt, it = s.solve_LH(dt(rt))
    zt = zt.cpu().numpy()
    assert it > 0
    rt0 = rt - rt.mean()
    res = np.linalg.norm(sysm.LH @ zt - rt0)
    record(name, "solve_LH_residual", float(res / np.linalg.norm(rt0)), 2e-13)
    assert abs(zt.sum()) <= 1e-10 * np.abs(zt).sum()
    z = s.apply_R(dt(r), precond="pegp").cpu().numpy()
    zo = P @ zt
    record(name, "apply_R_pegp_vs_P_solve_LH", float(np.abs(z - zo).max() / np.abs(zo).max()), 1e-12)
