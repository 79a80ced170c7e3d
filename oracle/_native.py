"""ORACLE -- TEST INFRASTRUCTURE ONLY.  ctypes loader for oracle/c/*.c
(built by __graft_entry__.build(); compiled on demand with gcc if missing)."""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "c", "mwm_oracle.c")
_LIB = os.path.join(_HERE, "c", "libmwm_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", _LIB, _SRC])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, i32, u64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
        P = ctypes.c_void_p
        L.oracle_visit_priority.argtypes = [u64, i32, i64]
        L.oracle_visit_priority.restype = u64
        L.oracle_visit_order.argtypes = [i64, u64, i32, P]
        L.oracle_visit_order.restype = None
        L.oracle_mwm.argtypes = [i64, P, P, P, P, P, P]
        L.oracle_mwm.restype = i64
        L.oracle_coarsen.argtypes = [i64, P, P, P, P, i64, P, P, P]
        L.oracle_coarsen.restype = i64
        _lib = L
    return _lib
