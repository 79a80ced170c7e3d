"""Multi-GPU host logic on the CPU (no GPU): the partition boundaries
(msp_dist_boundaries) and the halo plan (msp_halo_plan) of the partitioned
solve, and a world-size-2 gloo run in which each process knows only its own
rows, exchanges the planned halo through torch.distributed, and reproduces
the global SpMV on its rows exactly -- the data-path step the NCCL send/recv
of msp_dist_solve performs on GPUs."""
import os
import socket

import numpy as np
import pytest

from inputs import graphs as G

torch = pytest.importorskip("torch")


def _lib_ok():
    try:
        from paper_2207_07847_b200 import build as B
        B.build()
        return True
    except Exception:
        return False


pytestmark = pytest.mark.skipif(not _lib_ok(), reason="libmsp_b200.so does not build here")


def laplacian_apply(g, x, rows):
    y = np.zeros(rows.size)
    for k, i in enumerate(rows):
        c = g.col[g.rowptr[i]:g.rowptr[i + 1]]
        w = g.val[g.rowptr[i]:g.rowptr[i + 1]]
        y[k] = np.sum(w * (x[i] - x[c]))
    return y


def row_bounds(g, world):
    """Rows split by the solve's cost rule (entries + 8 per row), at row level."""
    from paper_2207_07847_b200.dist import boundaries
    cost = g.rowptr.astype(np.int64) + 8 * np.arange(g.n + 1)
    return boundaries(cost, world)


def test_boundaries_balance_and_cover():
    from paper_2207_07847_b200.dist import boundaries
    rng = np.random.default_rng(0)
    cost = np.concatenate([[0], np.cumsum(rng.integers(1, 50, 1000))])
    for W in (1, 2, 3, 8):
        b = boundaries(cost, W)
        assert b[0] == 0 and b[-1] == 1000 and np.all(np.diff(b) > 0)
        share = np.diff(cost[b])
        assert share.max() - share.min() <= 2 * 49 + 1          # within one node of the quantiles
    # a rank that would own nothing: every rank gets MSP_ERR_UNSUPPORTED
    from paper_2207_07847_b200 import _lib as L
    with pytest.raises(L.MspError) as ei:
        boundaries(np.arange(4), 5)
    assert ei.value.code == -4


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_halo_plan_is_symmetric_and_exact(world):
    from paper_2207_07847_b200.dist import halo_plan
    g = G.rgg(700, 12.0, 4)
    rb = row_bounds(g, world)
    plans = [halo_plan(g.n, g.rowptr, g.col, rb, r) for r in range(world)]
    for r, (rc, sc, rr, sr) in enumerate(plans):
        r0, r1 = rb[r], rb[r + 1]
        nb = set()
        for i in range(r0, r1):
            nb.update(int(c) for c in g.col[g.rowptr[i]:g.rowptr[i + 1]] if not (r0 <= c < r1))
        assert sorted(nb) == list(rr)                  # exactly the outside neighbours
        assert rc.sum() == rr.size and sc.sum() == sr.size and rc[r] == 0 and sc[r] == 0
    for r in range(world):                             # what r sends to q is what q receives from r
        soff = np.concatenate([[0], np.cumsum(plans[r][1])])
        for q in range(world):
            roff = np.concatenate([[0], np.cumsum(plans[q][0])])
            assert np.array_equal(plans[r][3][soff[q]:soff[q + 1]], plans[q][2][roff[r]:roff[r + 1]]), (r, q)


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2207_07847_b200.dist import halo_plan
        for g in (G.grid2d(23, 17, "loguniform", 2), G.chung_lu(3000, 2.1, 16.0, 1)):
            rb = row_bounds(g, world)
            rc, sc, rr, sr = halo_plan(g.n, g.rowptr, g.col, rb, rank)
            r0, r1 = int(rb[rank]), int(rb[rank + 1])
            p = np.random.default_rng(5).standard_normal(g.n)  # the reference (same on all ranks)
            mine = np.zeros(g.n)
            mine[r0:r1] = p[r0:r1]                              # a rank only knows its own rows
            send = torch.from_numpy(np.ascontiguousarray(mine[sr]))
            recv = torch.zeros(int(rr.size), dtype=torch.float64)
            dist.all_to_all_single(recv, send, output_split_sizes=[int(c) for c in rc],
                                   input_split_sizes=[int(c) for c in sc])
            mine[rr] = recv.numpy()
            rows = np.arange(r0, r1)
            assert np.array_equal(laplacian_apply(g, mine, rows), laplacian_apply(g, p, rows))
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def test_gloo_world2_halo_exchange_reproduces_global_spmv():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
