"""Multi-GPU binding of libmsp_b200.so (marshalling only -- the partition,
the collectives (NCCL, inside the library) and the solve run in the C ABI).

    import torch.distributed as dist
    from paper_2207_07847_b200 import setup
    from paper_2207_07847_b200.dist import dist_init, dist_solve
    S = setup(n, rowptr, col, w)            # every rank, full graph, same seed
    dist_init(S)                            # NCCL communicator from torch.distributed's group
    out = dist_solve(S, b, rtol=1e-8)       # x: own rows, 0 elsewhere

``group_solve`` runs the same decomposition for W ranks in ONE process on one
device (loopback collectives): the single-GPU test of the partitioned
arithmetic.  ``boundaries`` and ``halo_plan`` are the host-only plan steps
(CPU tests).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L

P = ctypes.c_void_p
i32, i64 = ctypes.c_int32, ctypes.c_int64


def _f(name, argtypes):
    f = getattr(L._lib, name)
    f.argtypes = argtypes
    f.restype = ctypes.c_int
    return f


def unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    L._check(_f("msp_dist_unique_id", [P])(buf))
    return buf.raw


def dist_init(solver, group=None, stream=None) -> np.ndarray:
    """msp_dist_init for this rank of torch.distributed's (default) group:
    rank 0's NCCL unique id is broadcast through torch.distributed.  Returns
    msp_dist_range (row0, row1, kp, tp, nsend, nrecv, world, rank)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    obj = [unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    idb = ctypes.create_string_buffer(obj[0], 128)
    L._check(_f("msp_dist_init", [P, i32, i32, P, P])(solver._h, world, rank, idb, L._stream_ptr(stream)))
    return dist_range(solver)


def dist_range(solver) -> np.ndarray:
    out = np.zeros(8, dtype=np.int64)
    L._check(_f("msp_dist_range", [P, P])(solver._h, out.ctypes.data))
    return out


def dist_solve(solver, b, x=None, rtol: float = 1e-8, maxit: int = 100000, stream=None) -> dict:
    """msp_dist_solve on this rank (collective over the ranks)."""
    x = L._like(b) if x is None else x
    pb, mb, _ = L._ptr_mem(b, np.float64)
    px, mx, _ = L._ptr_mem(x, np.float64)
    if mb != mx:
        raise ValueError("b and x must live in the same memory space")
    rep = L._Report()
    f = _f("msp_dist_solve", [P, P, P, ctypes.c_double, i32, ctypes.c_int, P, ctypes.POINTER(L._Report)])
    L._check(f(solver._h, pb, px, float(rtol), int(maxit), mb, L._stream_ptr(stream), ctypes.byref(rep)))
    out = {f_: getattr(rep, f_) for f_, _ in L._Report._fields_}
    out["x"] = x
    return out


def group_solve(solvers, b, x=None, rtol: float = 1e-8, maxit: int = 100000, stream=None) -> dict:
    """msp_dist_group_solve: len(solvers) ranks (each a setup of the same
    graph) driven by this process on one device; x is the assembled
    solution."""
    W = len(solvers)
    x = L._like(b) if x is None else x
    pb, mb, _ = L._ptr_mem(b, np.float64)
    px, mx, _ = L._ptr_mem(x, np.float64)
    if mb != mx:
        raise ValueError("b and x must live in the same memory space")
    hs = (P * W)(*[s._h for s in solvers])
    rep = L._Report()
    f = _f("msp_dist_group_solve", [ctypes.POINTER(P), i32, P, P, ctypes.c_double, i32, ctypes.c_int, P,
                                    ctypes.POINTER(L._Report)])
    L._check(f(hs, W, pb, px, float(rtol), int(maxit), mb, L._stream_ptr(stream), ctypes.byref(rep)))
    out = {f_: getattr(rep, f_) for f_, _ in L._Report._fields_}
    out["x"] = x
    return out


def boundaries(cost, world: int) -> np.ndarray:
    """msp_dist_boundaries (host only): quantile split of the prefix cost."""
    cost = np.ascontiguousarray(cost, dtype=np.int64)
    bnd = np.zeros(world + 1, dtype=np.int64)
    L._check(_f("msp_dist_boundaries", [i64, P, i32, P])(int(cost.size - 1), cost.ctypes.data, int(world),
                                                           bnd.ctypes.data))
    return bnd


def halo_plan(n, rowptr, col, row_bnd, rank: int):
    """msp_halo_plan (host only): (recv_counts, send_counts, recv_rows,
    send_rows) of `rank` given level-1 row boundaries."""
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int32)
    col = np.ascontiguousarray(col, dtype=np.int32)
    row_bnd = np.ascontiguousarray(row_bnd, dtype=np.int64)
    world = row_bnd.size - 1
    rc = np.zeros(world, dtype=np.int64)
    sc = np.zeros(world, dtype=np.int64)
    f = _f("msp_halo_plan", [i64, P, P, i32, P, i32, P, P, P, i64, P, i64])
    args = (int(n), rowptr.ctypes.data, col.ctypes.data, int(world), row_bnd.ctypes.data, int(rank),
            rc.ctypes.data, sc.ctypes.data)
    L._check(f(*args, None, 0, None, 0))
    rr = np.zeros(max(int(rc.sum()), 1), dtype=np.int64)
    sr = np.zeros(max(int(sc.sum()), 1), dtype=np.int64)
    L._check(f(*args, rr.ctypes.data, int(rc.sum()), sr.ctypes.data, int(sc.sum())))
    return rc, sc, rr[:int(rc.sum())], sr[:int(sc.sum())]
