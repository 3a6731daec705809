"""CPU-side checks of the boundary: the C-ABI library builds for sm_100a,
loads, exports every symbol include/o3g.h declares, answers status/error
queries, and fails loudly (no CPU fallback) without a GPU. Also checks the
product package never imports the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1801_09847_b200 import _build
    _build.build()
    import paper_1801_09847_b200 as m
    return m.lib()


def _declared():
    src = open(os.path.join(ROOT, "include", "o3g.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(o3g_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert "o3g_icp_point_to_plane" in names and "o3g_icp_step" in names
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (o3g_\w+)", out))
    assert set(names) <= exported
    assert all(e in names for e in exported), exported - set(names)


def test_built_for_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib._name],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_no_cpu_fallback(lib):
    import torch
    assert lib.o3g_status_string(0) == b"ok"
    assert lib.o3g_status_string(1) == b"invalid argument"
    if torch.cuda.is_available():
        pytest.skip("GPU present: the no-device path is not reachable")
    h = ctypes.c_void_p()
    st = lib.o3g_create(ctypes.byref(h), 0, None)
    assert st == 3 and lib.o3g_last_error()          # O3G_ERR_CUDA, with a message
    import numpy as np
    import paper_1801_09847_b200 as m
    with pytest.raises(m.O3GError):
        m.icp_point_to_plane(np.zeros((4, 3)), np.zeros((4, 3)), np.zeros((4, 3)), 0.1)


def test_null_context_is_invalid_argument(lib):
    assert lib.o3g_set_option(None, 1, 0) == 1
    assert lib.o3g_icp_step(None, None, None, None, None, None, None, None) == 1
    assert lib.o3g_destroy(None) == 0


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1801_09847_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "o3g_oracle" not in txt and "liborc" not in txt, f
