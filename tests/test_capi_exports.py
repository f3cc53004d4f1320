"""The C-ABI library loads on a CPU-only host and exports exactly what
include/tbgpu.h declares; host-side status mapping without a device."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "tbgpu.h")).read()
    return sorted(set(re.findall(r"^TB_API\s+[\w\s\*]+?\b(tb_\w+)\(", text, flags=re.M)))


def test_header_matches_binding_list():
    from paper_2509_04594_b200 import _lib

    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    from paper_2509_04594_b200 import _lib

    lib = _lib.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = sorted(set(re.findall(r" T (tb_\w+)", out)))
    assert exported == declared_symbols()


def test_library_is_sm100a():
    from paper_2509_04594_b200 import _lib

    _lib.lib()
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_kernels_use_dmma_and_tma():
    """SASS evidence (B200_PROFILING.md): DMMA for the FP64 tensor path, UTMALDG for TMA."""
    from paper_2509_04594_b200 import _lib

    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass
    assert "DFMA" in sass  # comparison variant
    assert "UTMALDG" in sass
    assert "LDGSTS" in sass  # cp.async variant


def test_metadata_calls_without_device():
    from paper_2509_04594_b200 import _lib

    lib = _lib.lib()
    assert lib.tb_version().decode().startswith("tbgpu")
    assert [lib.tb_variant_name(i).decode() for i in range(5)] == ["auto", "paper", "dmma_tma", "dmma_cpasync", "dfma"]
    assert lib.tb_variant_name(99) is None
    assert lib.tb_resolve_variant(ctypes.c_void_p(4096), 10, ctypes.c_void_p(4096), 10, 0) == 2
    assert lib.tb_resolve_variant(ctypes.c_void_p(4096), 11, ctypes.c_void_p(4096), 10, 0) == 3
    assert lib.tb_resolve_variant(ctypes.c_void_p(4104), 10, ctypes.c_void_p(4096), 10, 2) == 3
    assert lib.tb_resolve_variant(None, 10, None, 10, 4) == 4
    assert lib.tb_resolve_variant(None, 10, None, 10, 7) == -1


def test_no_device_is_a_status_not_a_crash():
    """multiply.ts:65 / kernel.test.ts:136-149: missing device -> NO_DEVICE."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("this host has a GPU")
    import paper_2509_04594_b200 as tb
    from paper_2509_04594_b200 import _lib

    assert _lib.device_count() == 0
    a = np.ones((2, 2))
    out_c, out_s = np.zeros(4), np.zeros(1)
    assert tb.gpu_tiled_multiply_flat(0, a, a, 2, 2, 2, 32, out_c, out_s) == tb.STATUS_NO_DEVICE
    assert tb.gpu_tiled_multiply_flat(None, a, a, 2, 2, 2, 32, out_c, out_s) == tb.STATUS_NO_DEVICE
    assert _lib.lib().tb_validate_launch(2, 2, 2, 32, 0, 0) == tb.STATUS_NO_DEVICE
    assert "no CUDA device" in _lib.last_error()
    sec = ctypes.c_double()
    assert _lib.lib().tb_dgemm(None, None, None, 2, 2, 2, 32, 0, 0, None, ctypes.byref(sec)) == tb.STATUS_NO_DEVICE
    with pytest.raises(_lib.TbStatusError):
        _lib.check(_lib.lib().tb_dgemm(None, None, None, 2, 2, 2, 32, 0, 0, None, ctypes.byref(sec)))
