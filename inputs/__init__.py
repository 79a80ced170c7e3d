"""Seeded synthetic input generators shared by the oracle tests, the GPU parity
tests and bench.py.

This package holds NO arithmetic of the paper's method (no Laplacian, no
aggregation, no expansion, no preconditioner): it only draws graphs (edge lists
with fp64 weights, converted to symmetric CSR) and right-hand sides, with the
shapes/weight distributions that BASELINE.json's configs and the paper's §4
workloads name.  Both sides (oracle/ and the CUDA path) consume its output.
"""
from .graphs import *  # noqa: F401,F403
