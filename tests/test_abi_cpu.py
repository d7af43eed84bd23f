"""CPU-only checks of the C ABI: the library loads and exports every symbol
include/pdnn.h declares; host-side argument validation (no GPU needed)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pdnn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pdnn_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2008_08636_b200 import build

    build.build()
    from paper_2008_08636_b200 import load_library

    return load_library()


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    from paper_2008_08636_b200 import EXPORTS

    assert sorted(EXPORTS) == names


def test_library_is_sm100a(lib):
    import subprocess

    so = os.path.join(ROOT, "paper_2008_08636_b200", "libpdnn.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings(lib):
    assert lib.pdnn_status_string(0) == b"PDNN_OK"
    assert lib.pdnn_status_string(-2) == b"PDNN_ECYCLE"
    assert lib.pdnn_status_string(-6) == b"PDNN_EWORKSPACE"


def test_host_argument_validation(lib):
    h = C.c_void_p()
    # negative sizes / null output are rejected before any CUDA call
    assert lib.pdnn_build_csr(-1, 0, None, None, None, None, C.byref(h)) == -1
    assert lib.pdnn_build_csr(3, 2, None, None, None, None, C.byref(h)) == -1
    assert lib.pdnn_build_csr(3, 0, None, None, None, None, None) == -1
    assert lib.pdnn_graph_query(None, None, None, None, None, None) == -1
    assert lib.pdnn_weighted_levels(None, None, None, None, None, None, None, 0, None) == -1
    assert lib.pdnn_memory_potential(None, None, 2, *([None] * 11), 0, None) == -1
    assert lib.pdnn_workspace_bytes(None, 1, 0) == 0
    assert lib.pdnn_workspace_init(None, 0, None) == -6
    assert b"null" in lib.pdnn_last_error()
    assert lib.pdnn_launch_count() == 0


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2008_08636_b200 import Graph

    with pytest.raises(Exception):
        Graph(3, [0, 1], [1, 2])
