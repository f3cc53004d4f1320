"""B200-native FP64 square GEMM — the hot path of arXiv 2509.04594 (tilebench).

Public surface mirrors the reference package's plug-in API for this path
(/root/reference/pkg/src/tilebench/__init__.py): ``BackendDescriptor``,
``BackendRegistry``, ``register_external``, ``default_registry``,
``TileConfig``, ``GenSpec``/``generate``/``flop_count``/``max_abs_rel_diff``,
``RunConfig``/``TrialRecord``/``run_trials``/``write_records``, plus the GPU
entry points (``gpu_tiled_multiply`` — the "gpu-tiled" MultiplyFn —,
``dgemm`` on torch tensors, the flat host-buffer ABI and the cuBLAS baseline).

The arithmetic is the sm_100a kernels of ``libtbgpu.so`` (C ABI in
``include/tbgpu.h``); there is no CPU fallback.
"""
from ._lib import (STATUS_BAD_DIMS, STATUS_NO_DEVICE, STATUS_OK, STATUS_OVER_LIMITS, STATUS_RUNTIME, VARIANTS,
                   TbStatusError)
from .backends import (CUBLAS_BACKEND_NAME, GPU_BACKEND_NAME, PAPER_BACKEND_NAME, BackendDescriptor,
                       BackendRegistry, TileConfig, cublas_dgemm, cublas_multiply, default_registry, dgemm,
                       dgemm_launch, gpu_tiled_multiply, gpu_tiled_multiply_flat, gpu_tiled_multiply_timed,
                       probe_device, register_external, register_gpu_backend, register_into)
from .errors import (BackendConflictError, InvalidConfigError, ShapeError, TilebenchError, TrialError,
                     UnknownBackendError)
from .harness import RunConfig, RunMetadata, TrialRecord, run_trials, trial_operands, write_records
from .matrices import GenSpec, flop_count, generate, max_abs_rel_diff, normwise_rel, require_operands

__version__ = "0.1.0"

__all__ = [
    "BackendConflictError", "BackendDescriptor", "BackendRegistry", "CUBLAS_BACKEND_NAME", "GPU_BACKEND_NAME",
    "GenSpec", "InvalidConfigError", "PAPER_BACKEND_NAME", "RunConfig", "RunMetadata", "STATUS_BAD_DIMS",
    "STATUS_NO_DEVICE", "STATUS_OK", "STATUS_OVER_LIMITS", "STATUS_RUNTIME", "ShapeError", "TbStatusError",
    "TileConfig", "TilebenchError", "TrialError", "TrialRecord", "UnknownBackendError", "VARIANTS",
    "cublas_dgemm", "cublas_multiply", "default_registry", "dgemm", "dgemm_launch", "flop_count", "generate",
    "gpu_tiled_multiply", "gpu_tiled_multiply_flat", "gpu_tiled_multiply_timed", "max_abs_rel_diff",
    "normwise_rel", "probe_device", "register_external", "register_gpu_backend", "register_into",
    "require_operands", "run_trials", "trial_operands", "write_records",
]
