"""ctypes binding of ``libtbgpu.so`` (declared in ``include/tbgpu.h``).

This is the reference-side binding a maintainer would add beside
``gpuTiledMultiplyFlat`` (reference ``pkg/gpu/src/multiply.ts:54-79``): plain
pointers and sizes, integer status codes mapped onto the reference's
exception tree (``pkg/src/tilebench/errors.py``). There is no fallback: if the
library cannot be loaded every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import InvalidConfigError, ShapeError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtbgpu.so")
# Tooling only (tools/kernel_timeline.py, A/B experiments): load another build
# of the same sources, libtbgpu_<variant>.so, instead.
if os.environ.get("TB_LIB_VARIANT"):
    LIB_PATH = os.path.join(HERE, f"libtbgpu_{os.environ['TB_LIB_VARIANT']}.so")

STATUS_OK = 0
STATUS_BAD_DIMS = 1
STATUS_OVER_LIMITS = 2
STATUS_NO_DEVICE = 3
STATUS_RUNTIME = 4

VARIANT_AUTO = 0
VARIANT_PAPER = 1
VARIANT_DMMA_TMA = 2
VARIANT_DMMA_CPASYNC = 3
VARIANT_DFMA = 4
VARIANTS = {"auto": VARIANT_AUTO, "paper": VARIANT_PAPER, "dmma_tma": VARIANT_DMMA_TMA,
            "dmma_cpasync": VARIANT_DMMA_CPASYNC, "dfma": VARIANT_DFMA}

DEFAULT_TILE_EDGE = 32

# Every symbol include/tbgpu.h declares (checked by tests/test_capi_exports.py).
EXPORTS = [
    "tb_gpu_tiled_multiply_flat", "tb_gpu_tiled_multiply_flat_ex", "tb_dgemm", "tb_dgemm_launch",
    "tb_cublas_dgemm", "tb_validate_launch", "tb_device_count", "tb_variant_name",
    "tb_resolve_variant", "tb_last_error", "tb_version", "tb_release", "tb_pipeline_plan",
    "tb_kernel_launches", "tb_dgemm_mgpu", "tb_copy2d_async", "tb_runtime_info", "tb_launch_plan",
]

_D = ctypes.POINTER(ctypes.c_double)
_VP = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64

_lock = threading.Lock()
_lib = None


class TbStatusError(RuntimeError):
    """A CUDA/NCCL runtime failure (TB_STATUS_RUNTIME) or a missing device."""

    def __init__(self, status: int, message: str):
        self.status = status
        super().__init__(message)


def _declare(l):
    l.tb_gpu_tiled_multiply_flat.argtypes = [_I32, _VP, _VP, _I64, _I64, _I64, _I32, _VP, _I64, _D]
    l.tb_gpu_tiled_multiply_flat_ex.argtypes = [_I32, _VP, _VP, _I64, _I64, _I64, _I32, _I32, _VP, _I64, _D, _D]
    l.tb_dgemm.argtypes = [_VP, _VP, _VP, _I64, _I64, _I64, _I32, _I32, _I32, _VP, _D]
    l.tb_cublas_dgemm.argtypes = [_VP, _VP, _VP, _I64, _I64, _I64, _I32, _I32, _I32, _VP, _D]
    l.tb_dgemm_launch.argtypes = [_VP, _I64, _VP, _I64, _VP, _I64, _I64, _I64, _I64, _I32, _I32, _I32, _VP]
    l.tb_validate_launch.argtypes = [_I64, _I64, _I64, _I32, _I32, _I32]
    l.tb_device_count.argtypes = []
    l.tb_variant_name.argtypes = [_I32]
    l.tb_variant_name.restype = ctypes.c_char_p
    l.tb_resolve_variant.argtypes = [_VP, _I64, _VP, _I64, _I32]
    l.tb_last_error.argtypes = []
    l.tb_last_error.restype = ctypes.c_char_p
    l.tb_version.argtypes = []
    l.tb_version.restype = ctypes.c_char_p
    l.tb_release.argtypes = []
    l.tb_release.restype = None
    _P64 = ctypes.POINTER(ctypes.c_int64)
    _P32 = ctypes.POINTER(ctypes.c_int32)
    l.tb_kernel_launches.argtypes = []
    l.tb_kernel_launches.restype = ctypes.c_longlong
    l.tb_pipeline_plan.argtypes = [_I64, _I64, _I64, _I32, _I32, _I32, _P64, _P32, _P64, _I32, _P32, _P64, _I32,
                                   _P32]
    l.tb_dgemm_mgpu.argtypes = [_I32, _P32, _VP, _VP, _VP, _VP, _P64, _I64, _I64, _I32, _D, _D]
    l.tb_copy2d_async.argtypes = [_VP, _I64, _VP, _I64, _I64, _I64, _VP]
    l.tb_runtime_info.argtypes = [_I32, ctypes.c_char_p, _I64]
    l.tb_launch_plan.argtypes = [_I64, _I64, _I64, _I32, _I32, ctypes.c_char_p, _I64]
    for name in ("tb_runtime_info", "tb_launch_plan", "tb_copy2d_async", "tb_dgemm_mgpu", "tb_gpu_tiled_multiply_flat", "tb_gpu_tiled_multiply_flat_ex", "tb_dgemm", "tb_cublas_dgemm",
                 "tb_dgemm_launch", "tb_validate_launch", "tb_device_count", "tb_resolve_variant",
                 "tb_pipeline_plan"):
        getattr(l, name).restype = ctypes.c_int


def lib():
    """Load libtbgpu.so (building it first if it is missing and nvcc exists)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                from . import build as _build
                _build.build()
            l = ctypes.CDLL(LIB_PATH)
            _declare(l)
            _lib = l
    return _lib


def last_error() -> str:
    msg = lib().tb_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    """Map a TB_STATUS_* code onto the reference's exception kinds
    (multiply.ts:49-52 semantics; errors.py)."""
    if status == STATUS_OK:
        return
    msg = last_error()
    if status == STATUS_BAD_DIMS:
        raise ShapeError(msg)
    if status == STATUS_OVER_LIMITS:
        raise InvalidConfigError(msg)
    raise TbStatusError(status, msg or f"status {status}")


def device_count() -> int:
    return int(lib().tb_device_count())


def version() -> str:
    return lib().tb_version().decode()


def kernel_launches() -> int:
    """Kernels this library has launched in this process (tb_kernel_launches)."""
    return int(lib().tb_kernel_launches())


def pipeline_plan(m: int, k: int, n: int, sms: int = 148, fused_ok: bool = True, staged: bool = False,
                  staged_output: bool = False) -> dict:
    """Shape of the host-buffer pipeline tb_gpu_tiled_multiply_flat_ex would
    run for an m x k x n call (pure host computation; no device needed)."""
    mq, fused = ctypes.c_int64(), ctypes.c_int32()
    npan, nblk = ctypes.c_int32(), ctypes.c_int32()
    panels = (ctypes.c_int64 * 256)()
    blocks = (ctypes.c_int64 * 256)()
    check(lib().tb_pipeline_plan(m, k, n, sms, 1 if fused_ok else 0, (1 if staged else 0) | (2 if staged_output else 0),
                                 ctypes.byref(mq), ctypes.byref(fused), panels,
                                 256, ctypes.byref(npan), blocks, 256, ctypes.byref(nblk)))
    return {"mq": mq.value, "fused": bool(fused.value), "panels": list(panels[:npan.value]),
            "blocks": list(blocks[:nblk.value])}


def _json_call(fn, *args) -> object:
    import json

    size = 4096
    while True:
        buf = ctypes.create_string_buffer(size)
        st = fn(*args, buf, size)
        if st == STATUS_OVER_LIMITS and size < (1 << 22):
            size *= 4
            continue
        check(st)
        return json.loads(buf.value.decode())


def runtime_info(device: int | None = 0) -> dict:
    """tb_runtime_info: library / CUDA / cuBLAS versions and paths, the pinned
    cuBLAS math mode and the GPU's facts (run metadata, harness.py:126-142)."""
    return _json_call(lib().tb_runtime_info, -1 if device is None else int(device))


def launch_plan(m: int, k: int, n: int, variant="auto", sms: int = 148) -> list:
    """tb_launch_plan: the launches (kernel, tile, grid, schedule) tb_dgemm
    would enqueue for a packed m x k x n product (no device needed)."""
    return _json_call(lib().tb_launch_plan, int(m), int(k), int(n), variant_id(variant), int(sms))


def variant_id(variant) -> int:
    if isinstance(variant, str):
        try:
            return VARIANTS[variant]
        except KeyError:
            raise InvalidConfigError(f"unknown kernel variant {variant!r}; known: {', '.join(VARIANTS)}") from None
    return int(variant)
