import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def read_poly_matrix(name: str, mu: float):
    """Parse a golden "c0:c1:c2" matrix (see tests/golden/*.txt) at mu."""
    import numpy as np
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            row = []
            for tok in line.split():
                c0, c1, c2 = (float(t) for t in tok.split(":"))
                row.append(c0 + c1 * mu + c2 * mu * mu)
            rows.append(row)
    return np.array(rows)


def read_int_matrix(name: str):
    import numpy as np
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append([int(t) for t in line.split()])
    return np.array(rows)


def read_tables():
    import json
    with open(os.path.join(GOLDEN, "paper_tables.json")) as f:
        return json.load(f)
