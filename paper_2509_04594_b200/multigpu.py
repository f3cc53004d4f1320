"""Row-sharded multi-GPU FP64 GEMM: one process per GPU, NCCL broadcast of B.

No reference counterpart (multi-GPU is a SPEC non-goal); the
partition rule is the reference's ``plan_partitions`` (backends.py:119-136)
applied to rows, so each rank owns the contiguous row block
``C[r0:r1, :] = A[r0:r1, :] · B`` — independent units, the same ownership
argument that makes the reference's tiles race-free (backends.py:21-24).

The only exchange step is B, which rank ``src`` broadcasts once over
NVLink/NVSwitch. With ``panels > 1`` the broadcast is split into K-panels
``B[k0:k1, :]`` (contiguous row slices of row-major B) issued back to back on
NCCL's stream, and the compute stream runs
``C_local (+)= A_local[:, k0:k1] · B[k0:k1, :]`` for panel p as soon as panel
p has landed (``work.wait()`` makes the compute stream, not the host, wait),
so the transfer of panel p+1 overlaps the GEMM of panel p.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

__all__ = ["row_partitions", "panel_bounds", "ShardedGemm", "gather_rows"]


def row_partitions(m: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row blocks by the plan_partitions base + extra rule
    (backends.py:119-136); ranks beyond ``m`` get empty blocks."""
    if world < 1:
        raise ValueError("world must be >= 1")
    workers = min(world, m)
    base, extra = divmod(m, workers) if workers > 0 else (0, 0)
    out, start = [], 0
    for w in range(world):
        stop = start + (base + (1 if w < extra else 0) if w < workers else 0)
        out.append((start, stop))
        start = stop
    return out


def panel_bounds(k: int, panels: int) -> list[tuple[int, int]]:
    """Split [0, k) into ``panels`` K-panels with even boundaries (keeps the
    TMA 16-byte base alignment of A[:, k0:] and B[k0:, :] for float64)."""
    panels = max(1, min(int(panels), max(1, k // 2)))
    if panels == 1:
        return [(0, k)]
    step = -(-k // panels)
    step += step % 2
    out, k0 = [], 0
    while k0 < k:
        k1 = min(k, k0 + step)
        out.append((k0, k1))
        k0 = k1
    return out


def _gpu_matmul(a, b, out, accumulate: bool) -> None:
    from .backends import dgemm_launch
    dgemm_launch(a, b, out, accumulate=accumulate)


class ShardedGemm:
    """``C_local = A_local · B`` with B broadcast from ``src``.

    ``local_matmul(a, b, out, accumulate)`` defaults to the sm_100a kernel
    (asynchronous, current stream); CPU tests substitute a torch matmul to
    exercise the exchange logic over gloo."""

    def __init__(self, group=None, panels: int = 1, src: int = 0,
                 local_matmul: Callable | None = None):
        self.group = group
        self.panels = panels
        self.src = src
        self.local_matmul = local_matmul or _gpu_matmul

    def __call__(self, a_local: torch.Tensor, b: torch.Tensor, out_local: torch.Tensor) -> torch.Tensor:
        if a_local.shape[1] != b.shape[0] or out_local.shape != (a_local.shape[0], b.shape[1]):
            raise ValueError(f"shapes {tuple(a_local.shape)} @ {tuple(b.shape)} -> {tuple(out_local.shape)}")
        if not b.is_contiguous():
            raise ValueError("b must be contiguous (row-major)")
        bounds = panel_bounds(b.shape[0], self.panels)
        if len(bounds) == 1:
            dist.broadcast(b, self.src, group=self.group)
            if a_local.shape[0] > 0:
                self.local_matmul(a_local, b, out_local, False)
            return out_local
        works = [dist.broadcast(b[k0:k1], self.src, group=self.group, async_op=True) for k0, k1 in bounds]
        for i, ((k0, k1), w) in enumerate(zip(bounds, works)):
            w.wait()
            if a_local.shape[0] > 0:
                self.local_matmul(a_local[:, k0:k1], b[k0:k1], out_local, i > 0)
        return out_local


def gather_rows(out_local: torch.Tensor, parts: list[tuple[int, int]], dst: int = 0, group=None):
    """Collect the row blocks on ``dst`` (untimed; for parity checks). Returns
    the full matrix on ``dst`` and None elsewhere."""
    rank = dist.get_rank(group)
    n = out_local.shape[1]
    rows_max = max(r1 - r0 for r0, r1 in parts)
    buf = torch.zeros((rows_max, n), dtype=out_local.dtype, device=out_local.device)
    buf[: out_local.shape[0]].copy_(out_local)
    gathered = [torch.empty_like(buf) for _ in parts] if rank == dst else None
    dist.gather(buf, gathered, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([g[: r1 - r0] for g, (r0, r1) in zip(gathered, parts)], dim=0)
