"""The C-ABI library: loads on CPU, exports every symbol include/sieveball_cuda.h
declares, the Python binding covers them, and device entry points fail loudly
(SB_ECUDA) when no GPU is present -- there is no CPU fallback."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "sieveball_cuda.h")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sb_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    from paper_2604_08374_b200 import _lib
    L = ctypes.CDLL(_lib.LIB_PATH)
    names = declared()
    assert len(names) > 30
    for n in names:
        assert hasattr(L, n), n
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sb_\w+)", nm))
    assert set(names) <= exported
    assert set(names) == set(_lib.EXPORTED), set(names) ^ set(_lib.EXPORTED)


def test_library_is_sm100a():
    from paper_2604_08374_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _has_gpu():
    from paper_2604_08374_b200 import lib
    n = ctypes.c_int()
    lib().sb_device_count(ctypes.byref(n))
    return n.value > 0


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_device_entry_points_fail_loudly_without_gpu():
    from paper_2604_08374_b200 import CompressedCsr, CudaError, DeviceGraph
    g = CompressedCsr.from_adjacency([[1], [0]])
    with pytest.raises(CudaError, match="no CPU fallback"):
        DeviceGraph(g)


def test_argument_validation_before_device():
    from paper_2604_08374_b200 import DeviceGraph, HllParams
    with pytest.raises(ValueError):
        HllParams(3)
    with pytest.raises(ValueError):
        DeviceGraph.from_raw(2, [0, 1, 2], [1, 1], [1, 0], node_range=(1, 3))
    with pytest.raises(RuntimeError):  # offsets[N] != stream length
        DeviceGraph.from_raw(2, [0, 1, 5], [1, 1], [1, 0])


def test_cpp_facade_tool_builds_and_reports_missing_gpu():
    tool = os.path.join(ROOT, "tools", "sb_hyperball")
    assert os.path.exists(tool), "make builds tools/sb_hyperball (C++ host over the C-ABI)"
    if _has_gpu():
        pytest.skip("covered by the gpu tests")
    r = subprocess.run([tool, "synth", "8", "8", "0", "1", "1", "1", "0", "10", "2"], capture_output=True, text=True)
    assert r.returncode == 1 and "no CUDA device" in r.stderr
    r = subprocess.run([tool, "synth", "8", "8", "0", "1", "1", "1", "0", "3", "2"], capture_output=True, text=True)
    assert r.returncode in (1, 2)


def test_version_and_last_error_strings():
    from paper_2604_08374_b200 import lib
    assert b"sm_100a" in lib().sb_version()
    assert isinstance(lib().sb_last_error(), bytes)


def test_library_then_torch_import_order():
    """Loading libsieveball_cuda before torch must not pin the system NCCL under torch."""
    import subprocess
    import sys
    code = ("import paper_2604_08374_b200 as P; P.lib()\n"
            "import torch, torch.distributed\n"
            "print('ok')\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
