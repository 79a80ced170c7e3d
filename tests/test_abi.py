"""C-ABI surface (CPU, no GPU calls): libmsp_b200.so loads and exports every
function that include/*.h declares; the Python binding names the same calls.
"""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s+\**\s*(msp_[A-Za-z0-9_]+)\s*\(",
                             src, flags=re.M):
            names.append(m.group(1))
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2207_07847_b200 import build as B
    B.build()
    return ctypes.CDLL(B.LIB)


def test_header_declares_the_hot_path():
    names = declared_functions()
    for f in ("msp_setup", "msp_destroy", "msp_apply_L", "msp_apply_R", "msp_pcg_solve",
              "msp_last_error"):
        assert f in names, names


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 10
    missing = [f for f in names if not hasattr(lib, f)]
    assert not missing, missing


def test_binding_uses_only_declared_calls():
    src = open(os.path.join(ROOT, "paper_2207_07847_b200", "_lib.py")).read()
    used = set(re.findall(r"_lib\.(msp_[A-Za-z0-9_]+)", src))
    assert used <= set(declared_functions()), used - set(declared_functions())


def test_last_error_without_gpu(lib):
    lib.msp_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.msp_last_error(), bytes)
    # argument errors are reported before any CUDA call
    lib.msp_setup.restype = ctypes.c_int
    out = ctypes.c_void_p()
    rc = lib.msp_setup(ctypes.c_int64(1), None, None, None, 1, None, None, ctypes.byref(out))
    assert rc == -1 and out.value is None
    assert b"n must be" in lib.msp_last_error()


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2207_07847_b200")
    for f in glob.glob(os.path.join(pkg, "**", "*.*"), recursive=True):
        if f.endswith((".py", ".cu", ".cuh", ".h")):
            s = open(f).read()
            assert "oracle" not in re.sub(r"#.*|//.*", "", s).replace("no oracle", ""), f


def test_library_load_then_torch_import():
    """build() followed by smoke() in one process: loading the native library
    (which depends on libnccl.so.2) before `import torch` must not bind torch
    to an older system NCCL -- the binding loads torch's copy first."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import paper_2207_07847_b200 as M; M.load(); import torch; "
            "import torch.distributed; print('ok')")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
