"""The partitioned (multi-GPU) solve on one GPU.

* msp_dist_group_solve: the decomposition of W = 2, 3, 4 ranks -- own-rows
  SpMV after the halo exchange, rank-local sweeps of the tiers up to the
  partition level, all-gathered y there, replicated upper tiers and coarse
  levels, all-reduced dots -- driven by one process with loopback
  collectives, against the oracle (iterations within the R11 band, solution
  1e-8 in the L-norm), on a tiled grid, an RGG and a power-law graph whose
  first tier is generic.
* msp_dist_solve with NCCL at world size 1 (the only multi-rank setting one
  GPU may run): the NCCL code path end to end.
"""
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
from paper_2207_07847_b200 import dist as D  # noqa: E402

DEV = torch.device("cuda:0")


def dt(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=DEV)


def setup(g, seed=3):
    return M.setup(g.n, dt(g.rowptr, torch.int64), dt(g.col, torch.int32), dt(g.val), mu=0.8, seed=seed)


def check_against_oracle(name, g, out, seed=3, b=None):
    from test_gpu_parity import iteration_band
    h = A.build_hierarchy(g, seed)
    sysm = E.expand_msp_only(g, h, 0.8)
    L = GR.laplacian_of_graph(g)
    ref = PC.pcg(lambda v: L @ v, b, PR.msp(sysm), 1e-8, 20000)
    assert out["converged"] == 1 and ref.converged
    d = abs(out["iterations"] - ref.iterations)
    if d > 2:
        band = iteration_band(L, b, sysm, ref.iterations)
        assert d <= band, (name, out["iterations"], ref.iterations, band)
    x = out["x"].cpu().numpy() if hasattr(out["x"], "cpu") else out["x"]
    e = x - ref.x
    e -= e.mean()
    xs = ref.x - ref.x.mean()
    assert np.sqrt(abs(e @ (L @ e))) <= 1e-8 * np.sqrt(xs @ (L @ xs)), name


CASES = {
    "grid_90x70": lambda: G.grid2d(90, 70, "loguniform", 8),
    "rgg_12000": lambda: G.rgg(12000, 12.0, 2),
    "chung_lu_30000": lambda: G.chung_lu(30000, 2.1, 16.0, 7),
    "grid3d_24": lambda: G.grid3d(24, 20, 18, seed=1),
}


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("name", list(CASES))
def test_group_solve_matches_oracle(name, world):
    g = CASES[name]()
    ss = [setup(g) for _ in range(world)]
    b = G.rhs(g.n, 6)
    out = D.group_solve(ss, dt(b), rtol=1e-8, maxit=20000)
    check_against_oracle(f"{name}/W{world}", g, out, b=b)


def test_group_solve_partition_and_host_buffers():
    g = G.chung_lu(30000, 2.1, 16.0, 7)
    ss = [setup(g) for _ in range(2)]
    b = G.rhs(g.n, 2)
    out = D.group_solve(ss, b.copy(), rtol=1e-8, maxit=20000)   # host memory
    L = GR.laplacian_of_graph(g)
    assert out["converged"] == 1
    assert np.linalg.norm(L @ out["x"] - b) <= 1.5e-8 * np.linalg.norm(b)
    tiny = G.grid2d(6, 6)
    st = [setup(tiny) for _ in range(4)]
    with pytest.raises(M.MspError) as ei:
        D.group_solve(st, dt(G.rhs(tiny.n, 0)))
    assert ei.value.code == -4


def test_dist_solve_nccl_world1():
    g = G.grid2d(90, 70, "loguniform", 8)
    S = setup(g)
    import ctypes
    idb = ctypes.create_string_buffer(D.unique_id(), 128)
    D._f("msp_dist_init", [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p])(
        S._h, 1, 0, idb, None)
    rng = D.dist_range(S)
    assert rng[0] == 0 and rng[1] == g.n and rng[6] == 1
    b = G.rhs(g.n, 6)
    out = D.dist_solve(S, dt(b), rtol=1e-8, maxit=20000)
    check_against_oracle("nccl_w1", g, out, b=b)
