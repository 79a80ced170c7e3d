"""Multi-GPU host logic on the CPU (no GPU): the partition / halo plan of
msp_partition_plan and the torch.distributed callbacks of dist.TorchComm,
exercised by world-size-2 gloo processes that emulate the distributed SpMV
(own rows + exchanged halo) and check it against the global product."""
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


def tiles_of(n, T):
    return np.array(sorted(set(list(range(0, n, T)) + [n])), dtype=np.int32)


def laplacian_apply(g, x, rows):
    y = np.zeros(rows.size)
    for k, i in enumerate(rows):
        c = g.col[g.rowptr[i]:g.rowptr[i + 1]]
        w = g.val[g.rowptr[i]:g.rowptr[i + 1]]
        y[k] = np.sum(w * (x[i] - x[c]))
    return y


@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_plan_partitions_rows_and_halos_are_symmetric(world):
    from paper_2207_07847_b200.dist import partition_plan
    g = G.rgg(700, 12.0, 4)
    tr = tiles_of(g.n, 37)
    plans = [partition_plan(g.n, g.rowptr, g.col, tr, world, r) for r in range(world)]
    starts = [int(p[0][0]) for p in plans] + [g.n]
    assert starts[0] == 0 and all(int(plans[r][0][1]) == starts[r + 1] for r in range(world))
    for r, (rng, rc, sc, rr, sr) in enumerate(plans):
        r0, r1, t0, t1 = (int(v) for v in rng)
        assert tr[t0] == r0 and tr[t1] == r1          # whole tiles
        own = np.arange(r0, r1)
        nb = set()
        for i in own:
            nb.update(int(c) for c in g.col[g.rowptr[i]:g.rowptr[i + 1]] if not (r0 <= c < r1))
        assert sorted(nb) == list(rr)                  # exactly the outside neighbours
        assert rc.sum() == rr.size and sc.sum() == sr.size
    # what r sends to q is what q receives from r
    for r in range(world):
        soff = np.concatenate([[0], np.cumsum(plans[r][2])])
        for q in range(world):
            sent = plans[r][4][soff[q]:soff[q + 1]]
            roff = np.concatenate([[0], np.cumsum(plans[q][1])])
            got = plans[q][3][roff[r]:roff[r + 1]]
            assert np.array_equal(sent, got), (r, q)


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2207_07847_b200.dist import TorchComm, partition_plan
        comm = TorchComm(device="cpu")
        g = G.grid2d(23, 17, "loguniform", 2)
        tr = tiles_of(g.n, 29)
        rng, rc, sc, rr, sr = partition_plan(g.n, g.rowptr, g.col, tr, world, rank)
        r0, r1 = int(rng[0]), int(rng[1])
        p = np.random.default_rng(5).standard_normal(g.n)  # same on all ranks (the reference)
        mine = np.zeros(g.n)
        mine[r0:r1] = p[r0:r1]                              # a rank only knows its own rows
        send = np.ascontiguousarray(mine[sr])
        recv = np.zeros(max(rr.size, 1))
        rcc = np.ascontiguousarray(rc, dtype=np.int64)
        scc = np.ascontiguousarray(sc, dtype=np.int64)
        PI = ctypes_ptr = None  # noqa: F841
        import ctypes
        ok = comm._alltoallv(send.ctypes.data, scc.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                             recv.ctypes.data, rcc.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), None)
        assert ok == 0, comm.error
        mine[rr] = recv[:rr.size]
        y_own = laplacian_apply(g, mine, np.arange(r0, r1))
        y_ref = laplacian_apply(g, p, np.arange(r0, r1))
        assert np.array_equal(y_own, y_ref)
        # all-reduce and all-gather callbacks
        v = np.array([float(rank + 1), 2.0])
        assert comm._allreduce(v.ctypes.data, 2, None) == 0
        assert v[0] == world * (world + 1) / 2 and v[1] == 2.0 * world
        s = np.full(3, float(rank))
        out = np.zeros(3 * world)
        assert comm._allgather(s.ctypes.data, out.ctypes.data, 3, None) == 0
        assert np.array_equal(out, np.repeat(np.arange(world, dtype=float), 3))
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


def test_plan_rejects_rank_without_tiles():
    """More ranks than tiles: every rank gets MSP_ERR_UNSUPPORTED from the
    plan (a deterministic check on shared inputs, so all ranks fail together
    before any collective instead of one hanging)."""
    from paper_2207_07847_b200 import _lib as L
    from paper_2207_07847_b200.dist import partition_plan
    g = G.grid2d(6, 5)
    tr = tiles_of(g.n, 16)                       # 2 tiles
    for r in range(3):
        with pytest.raises(L.MspError) as ei:
            partition_plan(g.n, g.rowptr, g.col, tr, 3, r)
        assert ei.value.code == -4
