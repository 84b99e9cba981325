"""libphmm.so: builds, loads, and exports exactly the C-ABI of include/phmm.h."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2411_11547_b200 import _native
from paper_2411_11547_b200.build import build_native

HEADER = os.path.join(ROOT, "include", "phmm.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(phmm_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    build_native()
    return _native.load()


def test_header_declares_the_entry_points():
    assert declared_functions() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (phmm_\w+)", out))
    assert set(declared_functions()) <= exported
    for name in declared_functions():
        assert getattr(lib, name) is not None


def test_library_is_built_for_sm_100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_abi_version(lib):
    assert lib.phmm_abi_version() == 1


def test_fast_geometry_is_host_only(lib):
    P, K, Q = _native.fast_geometry(250, 250)
    assert P * K * Q >= 251 and P in (4, 8, 16, 32) and K % 4 == 0
    for m in (1, 7, 100, 255, 511, 512, 1024, 3000):
        P, K, Q = _native.fast_geometry(m, 300)
        assert P * K * Q >= m + 1
    assert lib.phmm_fast_geometry(0, 5, None, None, None) == -1
    # reads of 128-255 bases pad to a 16-row grid: odd-K tilings between the even ones
    assert [_native.fast_geometry(m, 300)[:2] for m in (143, 175, 207, 239, 255)] == [
        (16, 9), (16, 11), (16, 13), (16, 15), (16, 16)]


def test_no_device_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2411_11547_b200.errors import EngineUnavailableError
    with pytest.raises(EngineUnavailableError):
        _native.Context(0)


def test_kernels_use_packed_fp32_and_shuffles(lib):
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _native.LIB_PATH],
                          capture_output=True, text=True, check=True).stdout
    funcs = {c.split("\n", 1)[0].strip(): c for c in sass.split("Function : ")[1:]}
    # the production FP32 kernel k_stream<kFast32, 16, 16, false>: packed FFMA2 recurrence,
    # neighbour exchange by shuffles, emissions from shared memory (LDS.128)
    fast = [body for name, body in funcs.items() if "k_streamILi0ELi16ELi16ELb0E" in name]
    assert len(fast) == 1
    assert "FFMA2" in fast[0] and "SHFL.UP" in fast[0] and "LDS.128" in fast[0]
    # bit-exactness of the k_exact kernels (no contraction in the recurrence) is
    # verified numerically by tests/test_gpu_parity.py; their setup code legitimately
    # uses DFMA inside IEEE double division.
