"""The C-ABI library loads on a CPU host and exports every symbol include/capsim_b200.h declares.
No device compute is attempted here; the product path must refuse to run without a GPU."""

from __future__ import annotations

import ctypes
import re

import pytest

from conftest import ROOT


def header_symbols() -> set[str]:
    text = (ROOT / "include" / "capsim_b200.h").read_text()
    return set(re.findall(r"^\s*(?:const\s+char\s*\*|int|void)\s+(cs_\w+)\s*\(", text, flags=re.M))


def test_header_and_binding_agree():
    from paper_2306_12247_b200 import _native as N

    assert header_symbols() == set(N.EXPORTS)


def test_library_exports_every_declared_symbol():
    from paper_2306_12247_b200 import _native as N

    lib = ctypes.CDLL(str(N.LIB_PATH))
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing
    assert N.lib().cs_abi_version() == 1


def test_library_is_sm100a_only():
    import subprocess

    from paper_2306_12247_b200 import _native as N

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present: the GPU tests cover this host")
    import paper_2306_12247_b200 as cs
    from paper_2306_12247_b200._native import NativeLibraryError

    g = cs.synthesize_grid(cs.SynthParams(mtl_cap=1, bs_cap=4))
    tr = cs.PowerTrace("x", 60, __import__("datetime").datetime(2020, 1, 1), (100.0, 200.0))
    with pytest.raises(NativeLibraryError):
        cs.simulate(g, tr, cs.COMBINATION)
    with pytest.raises(NativeLibraryError):
        cs.select_config(g, cs.COMBINATION, 150.0)


def test_staging_errors_are_validation_errors():
    import numpy as np

    from paper_2306_12247_b200 import _native as N
    from paper_2306_12247_b200.errors import ValidationError

    mtl = np.array([1, 1], np.int32)
    bs = np.array([1, 1], np.int32)
    thr = np.array([1.0, 2.0])
    pw = np.array([10.0, 20.0])
    d = (N.GridDesc * 1)()
    d[0] = N.GridDesc(2, mtl.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                      bs.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                      thr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                      pw.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), float("nan"))
    h = ctypes.c_void_p()
    with pytest.raises(ValidationError, match="duplicate"):
        N.check(N.lib().cs_tables_create(d, 1, 0, 1, 1, ctypes.byref(h)), invalid=ValidationError)


def test_comm_without_gpu_fails_cleanly():
    """cs_comm_init_all on a host without a usable GPU / NCCL reports an error code, never crashes."""
    import ctypes as C

    import torch

    from paper_2306_12247_b200 import _native as N

    if torch.cuda.is_available():
        pytest.skip("GPU host: covered by tests/test_gpu_multi_device.py")
    h = C.c_void_p()
    devs = (C.c_int32 * 1)(0)
    rc = N.lib().cs_comm_init_all(1, devs, C.byref(h))
    assert rc != 0 and not h.value
    assert N.lib().cs_comm_init_all(0, devs, C.byref(h)) != 0
    assert N.lib().cs_comm_destroy(None) == 0
