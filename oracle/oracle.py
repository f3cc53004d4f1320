"""CPU oracle for the FP64 square-GEMM hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and
only as the checker / the timed CPU reference — never as the product path.

It wraps ``oracle/tb_oracle.c`` (a C restatement of the reference's
``tilebench`` CPU kernels; see that file for per-function citations) and adds
the reference's operand generator, which is numpy's PCG64 exactly as
``/root/reference/pkg/src/tilebench/matrices.py:50-58`` calls it.

Parity pin: ``tests/golden/*`` were produced by importing the reference package
itself (``tests/golden/make_golden.py``); ``tests/test_oracle.py`` checks every
function here against them bitwise.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libtb_oracle.so")
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64


def build() -> str:
    """Compile the oracle library in place (make; gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "tb_oracle.c")
        if not os.path.exists(_LIB_PATH) or (
            os.path.exists(src) and os.path.getmtime(src) > os.path.getmtime(_LIB_PATH)
        ):
            build()
        l = ctypes.CDLL(_LIB_PATH)
        l.tbo_naive.argtypes = [_D, _D, _D, _I64, _I64, _I64]
        l.tbo_naive.restype = None
        l.tbo_tile_range.argtypes = [_D, _D, _D, _I64, _I64, _I64, _I64, _I64, _I64]
        l.tbo_tile_range.restype = None
        l.tbo_tiled_parallel.argtypes = [_D, _D, _D, _I64, _I64, _I64, _I64, _I64]
        l.tbo_tiled_parallel.restype = None
        l.tbo_paper_kernel.argtypes = [_D, _D, _D, _I64, _I64, _I64, _I64]
        l.tbo_paper_kernel.restype = None
        l.tbo_plan_partitions.argtypes = [_I64, _I64, ctypes.POINTER(ctypes.c_int64)]
        l.tbo_plan_partitions.restype = _I64
        l.tbo_max_abs_rel_diff.argtypes = [_D, _D, _I64]
        l.tbo_max_abs_rel_diff.restype = ctypes.c_double
        l.tbo_normwise_rel.argtypes = [_D, _D, _I64]
        l.tbo_normwise_rel.restype = ctypes.c_double
        l.tbo_max_threads.argtypes = []
        l.tbo_max_threads.restype = ctypes.c_int
        _lib = l
    return _lib


def _p(x: np.ndarray):
    return x.ctypes.data_as(_D)


def _operands(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ValueError(f"bad operand shapes {a.shape} @ {b.shape}")
    return a, b


def generate(rows: int, cols: int, seed: int, lo: float = 2.0, hi: float = 5.0) -> np.ndarray:
    """reference matrices.py:50-58: PCG64(seed).random((rows, cols)) scaled to [lo, hi]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    u = rng.random((rows, cols))
    return lo + u * (hi - lo)


def flop_count(n: int) -> int:
    """reference matrices.py:61-70: exact 2n^3 - n^2 in Python ints."""
    n = int(n)
    return 2 * n**3 - n**2


def naive(a, b) -> np.ndarray:
    """reference backends.py:92-97 / kernels.py:19-29."""
    a, b = _operands(a, b)
    out = np.zeros((a.shape[0], b.shape[1]))
    lib().tbo_naive(_p(a), _p(b), _p(out), a.shape[0], a.shape[1], b.shape[1])
    return out


def tiled_seq(a, b, tk: int = 32) -> np.ndarray:
    """reference backends.py:106-116 (one call to tile_range_kernel over all tiles)."""
    a, b = _operands(a, b)
    m, k, n = a.shape[0], a.shape[1], b.shape[1]
    out = np.zeros((m, n))
    tiles = ((m + tk - 1) // tk) * ((n + tk - 1) // tk)
    lib().tbo_tile_range(_p(a), _p(b), _p(out), m, k, n, 0, tiles, tk)
    return out


def tiled_parallel(a, b, tk: int = 32, threads: int | None = None) -> np.ndarray:
    """reference backends.py:139-160 (plan_partitions static split, pthreads).

    Bitwise identical to ``tiled_seq`` for any thread count (backends.py:21-24).
    """
    a, b = _operands(a, b)
    threads = threads or max_threads()
    m, k, n = a.shape[0], a.shape[1], b.shape[1]
    out = np.zeros((m, n))
    lib().tbo_tiled_parallel(_p(a), _p(b), _p(out), m, k, n, tk, threads)
    return out


def paper_kernel(a, b, tile_edge: int = 32) -> np.ndarray:
    """reference gpu/src/kernel.ts:50-78 restated on the CPU (running sum over phases)."""
    a, b = _operands(a, b)
    m, k, n = a.shape[0], a.shape[1], b.shape[1]
    out = np.zeros((m, n))
    lib().tbo_paper_kernel(_p(a), _p(b), _p(out), m, k, n, tile_edge)
    return out


def plan_partitions(num_tiles: int, threads: int) -> list[tuple[int, int]]:
    """reference backends.py:119-136."""
    buf = np.zeros(2 * max(1, min(threads, max(num_tiles, 1))), dtype=np.int64)
    w = lib().tbo_plan_partitions(num_tiles, threads, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(w)]


def max_abs_rel_diff(x, y) -> float:
    """reference matrices.py:73-86."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if x.shape != y.shape:
        raise ValueError(f"shape mismatch: {x.shape} vs {y.shape}")
    if x.size == 0:
        return 0.0
    return float(lib().tbo_max_abs_rel_diff(_p(x), _p(y), x.size))


def normwise_rel(x, ref) -> float:
    """||x - ref||_F / ||ref||_F (north-star parity metric, bound 1e-12)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    ref = np.ascontiguousarray(ref, dtype=np.float64)
    if x.shape != ref.shape:
        raise ValueError(f"shape mismatch: {x.shape} vs {ref.shape}")
    return float(lib().tbo_normwise_rel(_p(x), _p(ref), x.size))


def max_threads() -> int:
    return int(lib().tbo_max_threads())
