"""Multi-GPU binding: the collectives msp_dist_solve calls back into, over
torch.distributed (NCCL on GPUs, gloo on CPU for tests), and the host-only
partition plan.  Marshalling only -- the solve runs in libmsp_b200.so.

    import torch.distributed as dist
    from paper_2207_07847_b200 import setup
    from paper_2207_07847_b200.dist import TorchComm, dist_solve
    S = setup(n, rowptr, col, w)                     # every rank, full graph
    out = dist_solve(S, TorchComm(), b, rtol=1e-8)   # x: own rows, 0 elsewhere
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L


class msp_comm(ctypes.Structure):
    pass


ALLREDUCE = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)
ALLGATHER = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)
ALLTOALLV = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p,
                             ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p)
msp_comm._fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("allreduce", ALLREDUCE),
                     ("allgather", ALLGATHER), ("alltoallv", ALLTOALLV), ("ctx", ctypes.c_void_p)]


class _CAI:
    """Zero-copy view of n fp64 at a CUDA device pointer (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _view(ptr: int, n: int, device):
    import torch
    if n == 0:
        return torch.empty(0, dtype=torch.float64, device=device)
    if device.type == "cuda":
        return torch.as_tensor(_CAI(ptr, n), device=device)
    buf = (ctypes.c_double * int(n)).from_address(int(ptr))
    return torch.from_numpy(np.frombuffer(buf, dtype=np.float64))


class TorchComm:
    """msp_comm callbacks over a torch.distributed process group.  Buffers
    are device pointers (CUDA) or host pointers when `device` is CPU."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
                else torch.device("cpu")
        self.device = torch.device(device)
        self._cb = (ALLREDUCE(self._allreduce), ALLGATHER(self._allgather), ALLTOALLV(self._alltoallv))
        self.c = msp_comm(self.world, self.rank, self._cb[0], self._cb[1], self._cb[2], None)
        self.error = None

    def _guard(self, f):
        try:
            f()
            return 0
        except Exception as e:  # reported through the C error path
            self.error = e
            return -1

    def _allreduce(self, ptr, n, ctx):
        return self._guard(lambda: self.dist.all_reduce(_view(ptr, n, self.device), group=self.group))

    def _allgather(self, sptr, rptr, n_each, ctx):
        def f():
            s = _view(sptr, n_each, self.device)
            r = _view(rptr, n_each * self.world, self.device)
            self.dist.all_gather_into_tensor(r, s, group=self.group)
        return self._guard(f)

    def _alltoallv(self, sptr, scounts, rptr, rcounts, ctx):
        def f():
            sc = [int(scounts[q]) for q in range(self.world)]
            rc = [int(rcounts[q]) for q in range(self.world)]
            s = _view(sptr, sum(sc), self.device)
            r = _view(rptr, sum(rc), self.device)
            self.dist.all_to_all_single(r, s, output_split_sizes=rc, input_split_sizes=sc, group=self.group)
        return self._guard(f)


def partition_plan(n, rowptr, col, tile_rows, world: int, rank: int):
    """msp_partition_plan (host only): (range, recv_counts, send_counts,
    recv_rows, send_rows) of `rank` for the CSR (rowptr, col) whose first-tier
    tiles start at tile_rows."""
    lib = L._lib
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int32)
    col = np.ascontiguousarray(col, dtype=np.int32)
    tile_rows = np.ascontiguousarray(tile_rows, dtype=np.int32)
    rng = np.zeros(4, dtype=np.int64)
    rc = np.zeros(world, dtype=np.int64)
    sc = np.zeros(world, dtype=np.int64)
    P = ctypes.c_void_p
    f = lib.msp_partition_plan
    f.argtypes = [ctypes.c_int64, P, P, ctypes.c_int64, P, ctypes.c_int32, ctypes.c_int32, P, P, P, P,
                  ctypes.c_int64, P, ctypes.c_int64]
    f.restype = ctypes.c_int
    args = (int(n), rowptr.ctypes.data, col.ctypes.data, int(tile_rows.size - 1), tile_rows.ctypes.data,
            int(world), int(rank), rng.ctypes.data, rc.ctypes.data, sc.ctypes.data)
    L._check(f(*args, None, 0, None, 0))
    rr = np.zeros(max(int(rc.sum()), 1), dtype=np.int64)
    sr = np.zeros(max(int(sc.sum()), 1), dtype=np.int64)
    L._check(f(*args, rr.ctypes.data, int(rc.sum()), sr.ctypes.data, int(sc.sum())))
    return rng, rc, sc, rr[:int(rc.sum())], sr[:int(sc.sum())]


def dist_solve(solver, comm: TorchComm, b, x=None, rtol: float = 1e-8, maxit: int = 100000, stream=None) -> dict:
    """msp_dist_solve on this rank (collective: every rank of comm calls it)."""
    lib = L._lib
    x = L._like(b) if x is None else x
    pb, mb, kb = L._ptr_mem(b, np.float64)
    px, mx, kx = L._ptr_mem(x, np.float64)
    if mb != mx:
        raise ValueError("b and x must live in the same memory space")
    rep = L._Report()
    f = lib.msp_dist_solve
    f.argtypes = [ctypes.c_void_p, ctypes.POINTER(msp_comm), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                  ctypes.c_int32, ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(L._Report)]
    f.restype = ctypes.c_int
    rc = f(solver._h, ctypes.byref(comm.c), pb, px, float(rtol), int(maxit), mb, L._stream_ptr(stream),
           ctypes.byref(rep))
    if comm.error is not None:
        e, comm.error = comm.error, None
        raise RuntimeError(f"communication callback failed: {e}")
    L._check(rc)
    out = {f_: getattr(rep, f_) for f_, _ in L._Report._fields_}
    out["x"] = x
    return out
