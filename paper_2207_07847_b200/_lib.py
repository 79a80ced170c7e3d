"""ctypes binding of libmsp_b200.so -- marshalling only (no arithmetic).

Array arguments may be torch tensors (CUDA -> MSP_MEM_DEVICE, CPU ->
MSP_MEM_HOST) or numpy arrays (MSP_MEM_HOST).  All vectors are fp64 in the
original vertex numbering.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.environ.get("MSP_LIB_OVERRIDE") or os.path.join(HERE, "libmsp_b200.so")

MSP_OK = 0
MSP_MEM_DEVICE = 0
MSP_MEM_HOST = 1
MSP_PRECOND_NONE = 0
MSP_PRECOND_MSP = 1
MSP_PRECOND_PEGP = 2
_PRECOND = {"none": MSP_PRECOND_NONE, "msp": MSP_PRECOND_MSP, "pegp": MSP_PRECOND_PEGP}


class MspError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"msp error {code}: {msg}")
        self.code = code


class _Params(ctypes.Structure):
    _fields_ = [("mu", ctypes.c_double), ("max_levels", ctypes.c_int32),
                ("top_max", ctypes.c_int32), ("seed", ctypes.c_uint64)]


class _Info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("n_tilde", ctypes.c_int64),
                ("levels", ctypes.c_int32), ("mwm_rounds", ctypes.c_int32), ("mu", ctypes.c_double),
                ("setup_ms", ctypes.c_double), ("tile_level", ctypes.c_int32),
                ("coarse_level", ctypes.c_int32), ("ntiles", ctypes.c_int64),
                ("ntiers", ctypes.c_int32), ("spmv_grid", ctypes.c_int32),
                ("merged_coarse", ctypes.c_int32)]


class _Report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("relres", ctypes.c_double), ("solve_ms", ctypes.c_double),
                ("kernel_launches", ctypes.c_int64)]


def library_path() -> str:
    return _LIBPATH


def _load():
    if not os.path.exists(_LIBPATH):
        raise ImportError(f"{_LIBPATH} is not built: run `python -m paper_2207_07847_b200.build` "
                          "(there is no CPU fallback)")
    # libmsp_b200.so needs libnccl.so.2.  torch bundles the NCCL build it was
    # linked against; if the system's (older) copy were loaded first through
    # our dependency, a later `import torch` in the same process would bind to
    # it and fail on missing symbols.  Loading torch first makes both use
    # torch's copy (same soname).
    try:
        import torch  # noqa: F401
    except ImportError:
        pass
    L = ctypes.CDLL(_LIBPATH)
    P, i32, i64, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    L.msp_setup.argtypes = [i64, P, P, P, ctypes.c_int, ctypes.POINTER(_Params), P, ctypes.POINTER(P)]
    L.msp_destroy.argtypes = [P]
    L.msp_info.argtypes = [P, ctypes.POINTER(_Info)]
    L.msp_level_sizes.argtypes = [P, P]
    L.msp_get_aggregates.argtypes = [P, i32, P]
    L.msp_get_msp_edges.argtypes = [P, ctypes.POINTER(i64), P, P, P]
    L.msp_apply_L.argtypes = [P, P, P, ctypes.c_int, P]
    L.msp_apply_R.argtypes = [P, ctypes.c_int, P, P, ctypes.c_int, P]
    L.msp_pcg_solve.argtypes = [P, ctypes.c_int, P, P, d, i32, ctypes.c_int, P, ctypes.POINTER(_Report)]
    L.msp_set_profiling.argtypes = [P, ctypes.c_int]
    L.msp_get_profile.argtypes = [P, P, P]
    L.msp_apply_LH.argtypes = [P, P, P, ctypes.c_int, P]
    L.msp_solve_LH.argtypes = [P, P, P, ctypes.c_int, P, ctypes.POINTER(i32)]
    L.msp_pegp_params.argtypes = [P, d, i32, i32]
    L.msp_pegp_info.argtypes = [P, P, P]
    L.msp_last_error.restype = ctypes.c_char_p
    for f in ("msp_setup", "msp_destroy", "msp_info", "msp_level_sizes", "msp_get_aggregates",
              "msp_get_msp_edges", "msp_apply_L", "msp_apply_R", "msp_pcg_solve", "msp_set_profiling",
              "msp_get_profile", "msp_apply_LH", "msp_solve_LH", "msp_pegp_params",
              "msp_pegp_info"):
        getattr(L, f).restype = ctypes.c_int
    return L


class _LazyLib:
    """Loads libmsp_b200.so on first use and raises ImportError if it is not
    built (no CPU fallback).  Lazy so that ``paper_2207_07847_b200.build`` can
    be imported to build it."""

    _L = None

    def __getattr__(self, name):
        if _LazyLib._L is None:
            _LazyLib._L = _load()
        return getattr(_LazyLib._L, name)


_lib = _LazyLib()


def load():
    """Force-load the native library (raises ImportError if missing)."""
    return _lib.msp_last_error and _LazyLib._L


def _check(rc: int):
    if rc != MSP_OK:
        raise MspError(rc, _lib.msp_last_error().decode())


def _ptr_mem(a, dtype):
    """(pointer, mem kind, keepalive) for a torch tensor or numpy array."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            tdt = {np.float64: torch.float64, np.int64: torch.int64, np.int32: torch.int32}[dtype]
            if a.dtype != tdt or not a.is_contiguous():
                raise TypeError(f"expected contiguous {tdt}, got {a.dtype}")
            return a.data_ptr(), (MSP_MEM_DEVICE if a.is_cuda else MSP_MEM_HOST), a
    except ImportError:
        pass
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data, MSP_MEM_HOST, arr


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    return getattr(stream, "cuda_stream", stream)


class Solver:
    """Handle of one set-up graph (msp_setup ... msp_destroy)."""

    def __init__(self, n, rowptr, col, w, mu: float = 0.8, max_levels: int = 0, seed: int = 0,
                 top_max: int = 0, stream=None):
        prp, m1, k1 = _ptr_mem(rowptr, np.int64)
        pcol, m2, k2 = _ptr_mem(col, np.int32)
        pw, m3, k3 = _ptr_mem(w, np.float64)
        if not (m1 == m2 == m3):
            raise ValueError("rowptr, col, w must live in the same memory space")
        prm = _Params(mu, max_levels, top_max, seed)
        h = ctypes.c_void_p()
        _check(_lib.msp_setup(int(n), prp, pcol, pw, m1, ctypes.byref(prm), _stream_ptr(stream),
                              ctypes.byref(h)))
        self._h = h
        self.n = int(n)

    def close(self):
        if getattr(self, "_h", None):
            _lib.msp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------- queries
    def info(self) -> dict:
        i = _Info()
        _check(_lib.msp_info(self._h, ctypes.byref(i)))
        return {f: getattr(i, f) for f, _ in _Info._fields_}

    def level_sizes(self) -> np.ndarray:
        L = self.info()["levels"]
        out = np.zeros(L, dtype=np.int64)
        _check(_lib.msp_level_sizes(self._h, out.ctypes.data))
        return out

    def get_aggregates(self, level: int) -> np.ndarray:
        sizes = self.level_sizes()
        out = np.zeros(int(sizes[level - 1]), dtype=np.int32)
        _check(_lib.msp_get_aggregates(self._h, level, out.ctypes.data))
        return out

    def get_msp_edges(self):
        cnt = ctypes.c_int64(0)
        _check(_lib.msp_get_msp_edges(self._h, ctypes.byref(cnt), None, None, None))
        i = np.zeros(cnt.value, dtype=np.int64)
        j = np.zeros(cnt.value, dtype=np.int64)
        w = np.zeros(cnt.value, dtype=np.float64)
        _check(_lib.msp_get_msp_edges(self._h, ctypes.byref(cnt), i.ctypes.data, j.ctypes.data,
                                      w.ctypes.data))
        return i, j, w

    PROFILE_CATEGORIES = ("spmv", "tile_up", "mid_up", "coarse", "mid_down", "tile_down",
                          "pegp_spmv", "pegp_sweeps")

    def set_profiling(self, on: bool = True):
        _check(_lib.msp_set_profiling(self._h, 1 if on else 0))

    def get_profile(self) -> dict:
        ms = np.zeros(8, dtype=np.float64)
        cnt = np.zeros(8, dtype=np.int64)
        _check(_lib.msp_get_profile(self._h, ms.ctypes.data, cnt.ctypes.data))
        return {c: {"ms": float(ms[i]), "launches": int(cnt[i])}
                for i, c in enumerate(self.PROFILE_CATEGORIES)}

    # ---------------------------------------------------------- hot path
    def apply_L(self, x, y=None, stream=None):
        y = _like(x) if y is None else y
        px, mx, kx = _ptr_mem(x, np.float64)
        py, my, ky = _ptr_mem(y, np.float64)
        if mx != my:
            raise ValueError("x and y must live in the same memory space")
        _check(_lib.msp_apply_L(self._h, px, py, mx, _stream_ptr(stream)))
        return y

    def apply_R(self, r, z=None, precond="msp", stream=None):
        z = _like(r) if z is None else z
        pr, mr, kr = _ptr_mem(r, np.float64)
        pz, mz, kz = _ptr_mem(z, np.float64)
        if mr != mz:
            raise ValueError("r and z must live in the same memory space")
        _check(_lib.msp_apply_R(self._h, _PRECOND[precond], pr, pz, mr, _stream_ptr(stream)))
        return z

    def n_tilde(self) -> int:
        return int(self.info()["n_tilde"])

    def pegp_params(self, inner_rtol: float = 1e-13, inner_maxit: int = 5000, refine_steps: int = 0):
        _check(_lib.msp_pegp_params(self._h, float(inner_rtol), int(inner_maxit), int(refine_steps)))

    def pegp_info(self, stream=None) -> dict:
        out = np.zeros(5, dtype=np.int64)
        _check(_lib.msp_pegp_info(self._h, _stream_ptr(stream), out.ctypes.data))
        return {"hnnz": int(out[0]), "last_inner_iterations": int(out[1]), "coarse_level": int(out[2]),
                "build_ms": out[3] / 1000.0, "last_solve_inner_iterations": int(out[4])}

    def apply_LH(self, x, y=None, stream=None):
        """y~ = L_H~ x~ on expanded vectors (canonical expanded numbering)."""
        y = _like(x) if y is None else y
        px, mx, kx = _ptr_mem(x, np.float64)
        py, my, ky = _ptr_mem(y, np.float64)
        if mx != my:
            raise ValueError("x and y must live in the same memory space")
        _check(_lib.msp_apply_LH(self._h, px, py, mx, _stream_ptr(stream)))
        return y

    def solve_LH(self, r, z=None, stream=None):
        """z~ = L_H~^+ r~ (inner CG); returns (z~, inner iterations)."""
        z = _like(r) if z is None else z
        pr, mr, kr = _ptr_mem(r, np.float64)
        pz, mz, kz = _ptr_mem(z, np.float64)
        if mr != mz:
            raise ValueError("r and z must live in the same memory space")
        it = ctypes.c_int32(0)
        _check(_lib.msp_solve_LH(self._h, pr, pz, mr, _stream_ptr(stream), ctypes.byref(it)))
        return z, it.value

    def pcg_solve(self, b, x=None, rtol: float = 1e-8, maxit: int = 100000, precond="msp",
                  stream=None) -> dict:
        x = _like(b) if x is None else x
        pb, mb, kb = _ptr_mem(b, np.float64)
        px, mx, kx = _ptr_mem(x, np.float64)
        if mb != mx:
            raise ValueError("b and x must live in the same memory space")
        rep = _Report()
        _check(_lib.msp_pcg_solve(self._h, _PRECOND[precond], pb, px, float(rtol), int(maxit), mb,
                                  _stream_ptr(stream), ctypes.byref(rep)))
        out = {f: getattr(rep, f) for f, _ in _Report._fields_}
        out["x"] = x
        return out


def _like(a):
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return torch.empty_like(a)
    except ImportError:
        pass
    return np.empty_like(np.asarray(a, dtype=np.float64))


def setup(n, rowptr, col, w, **kw) -> Solver:
    """msp_setup: build the hierarchy, expanded graph and MSP on the GPU."""
    return Solver(n, rowptr, col, w, **kw)
