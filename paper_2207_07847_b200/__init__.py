"""B200-native PEGP/MSP graph-Laplacian solver (arxiv 2207.07847).

Thin Python binding of the C ABI in ``include/msp_b200.h`` (argument
marshalling only -- every step of the method runs in the CUDA kernels of
``libmsp_b200.so``).  There is no CPU fallback: importing this package on a
box without the built library raises.

    from paper_2207_07847_b200 import setup
    h = setup(n, rowptr, col, w, mu=0.8)       # GPU: hierarchy, expansion, MSP
    y = h.apply_L(x); z = h.apply_R(r)         # L_G x ; R r = P L_T~^+ P^T r
    rep = h.pcg_solve(b, x, rtol=1e-8)         # PCG, reading R10
"""
from ._lib import (  # noqa: F401
    MSP_MEM_DEVICE, MSP_MEM_HOST, MSP_PRECOND_MSP, MSP_PRECOND_NONE, MSP_PRECOND_PEGP,
    MspError, Solver, library_path, load, setup,
)

__all__ = ["setup", "Solver", "MspError", "library_path", "MSP_PRECOND_MSP", "MSP_PRECOND_PEGP",
           "MSP_PRECOND_NONE", "MSP_MEM_DEVICE", "MSP_MEM_HOST"]
