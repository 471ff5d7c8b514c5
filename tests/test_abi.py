"""CPU-side checks of the C-ABI boundary: the library builds for sm_100a,
loads, exports every symbol include/mcinv.h declares, and the product path
never touches the oracle. No compute calls (no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mcinv.h")
PKG = os.path.join(ROOT, "paper_cs_0412107_b200")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mcinv_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_cs_0412107_b200 import build
    so = build.build()
    return ctypes.CDLL(so)


def test_header_declares_the_boundary():
    names = declared_functions()
    for need in ("mcinv_create", "mcinv_set_trace_q", "mcinv_set_pattern", "mcinv_workspace_size", "mcinv_run",
                 "mcinv_accumulators", "mcinv_result", "mcinv_destroy", "mcinv_status_string",
                 "mcinv_error_detail", "mcinv_debug_philox", "mcinv_debug_gaussian", "mcinv_debug_get_state",
                 "mcinv_debug_set_state", "mcinv_pattern_size"):
        assert need in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_binding_covers_every_symbol():
    import paper_cs_0412107_b200 as M
    assert set(M.SYMBOLS) == set(declared_functions())


def test_library_is_sm100a_native(lib):
    from paper_cs_0412107_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.SO], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", build.SO], capture_output=True,
                          text=True).stdout
    assert "DMMA" in sass, "the X Y^dagger contraction must use FP64 tensor cores"


def test_status_strings(lib):
    lib.mcinv_status_string.restype = ctypes.c_char_p
    assert lib.mcinv_status_string(0) == b"ok"
    assert b"diverged" in lib.mcinv_status_string(4)


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_cs_0412107_b200 as M
    import workloads as W
    with pytest.raises(M.MCInvError) as e:
        M.Inverter(W.random_dense(4, seed=1))
    assert e.value.code == 6


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "oracle.h" not in txt and "liboracle" not in txt, f


def test_v6_gathers_do_not_wait_behind_global_loads(lib):
    """Regression guard for the late-round-2 finding ("K1 v6, late r2"): ptxas put
    the column reads of a gather chunk on the scoreboard of the chunk's first global loads, so
    the fifth address waited a whole round trip. The config-2 kernel (C = 8, 512 threads) must
    have no instruction that waits for a load's result behind a later global load on the same
    scoreboard (tools/sass_sbcheck.py, run on the built library's SASS)."""
    import importlib.util
    import os
    from paper_cs_0412107_b200 import build
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", build.SO], capture_output=True,
                          text=True).stdout
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("sbcheck", os.path.join(root, "tools", "sass_sbcheck.py"))
    sb = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(sb)
    blocks = [b for b in sass.split("Function : ")[1:]
              if b.startswith("_ZN5mcinv13sweep6_kernelILi6ELi512ELi3ELi2ELb0ELb1E")]
    assert len(blocks) == 1
    assert sb.false_waits(blocks[0]) == []
