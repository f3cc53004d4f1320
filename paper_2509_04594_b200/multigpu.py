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

__all__ = ["row_partitions", "panel_bounds", "ramp_panel_bounds", "geometric_panel_bounds", "host_panel_bounds", "shrinking_chunks", "gathered_panels", "ShardedGemm", "HostShardedGemm", "gather_rows", "peer_sharded_dgemm"]


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


def ramp_panel_bounds(k: int, panels: int) -> list[tuple[int, int]]:
    """``panel_bounds`` with a short first panel: only panel 0's broadcast is
    exposed before the first GEMM (each later panel's broadcast hides under
    the previous panel's GEMM — NVLink moves a B panel ~4x faster than a
    1250-row shard multiplies it), so it is 1/8 of an even panel."""
    even = panel_bounds(k, panels)
    if len(even) < 2:
        return even
    first = max(2, ((even[0][1] - even[0][0]) // 8) & ~1)
    rest = panel_bounds(k - first, max(1, len(even) - 1))
    return [(0, first)] + [(first + a, first + b) for a, b in rest]


def geometric_panel_bounds(k: int, first: int = 128, growth: int = 3) -> list[tuple[int, int]]:
    """K-panels growing geometrically from ``first`` rows by ``growth``: the
    default for ``ShardedGemm``. Panel p+1's broadcast must land while panel
    p multiplies: per k-row a 1250-row shard of N = 10000 multiplies in
    2·1250·10^4 / 35 TF/s = 0.71 us, and NCCL moves the k-row (80 KB) in
    ~0.2 us at ~400 GB/s, so the next panel may be ~3x larger. Only the
    first (short) broadcast is exposed, and the panel count — each panel
    costs a C re-read and a wave tail — stays logarithmic in k (N = 10000:
    128, 384, 1152, 3456, 4880). Boundaries are even (TMA alignment)."""
    out, k0, step = [], 0, max(2, first + first % 2)
    while k0 < k:
        k1 = k if k0 + step >= k - step // 4 else k0 + step
        out.append((k0, k1))
        k0 = k1
        step *= max(1, int(growth))
    return out


def gathered_panels(k: int, world: int, panels: int) -> list[tuple[int, int]]:
    """K-panels for the host-buffer path: every panel but the last spans a
    multiple of 2*world rows of B, so each rank uploads an equal, even-sized
    share and the panel is rebuilt by one equal-chunk all-gather; the last
    panel's shares run past ``k`` (padding rows that are gathered but never
    multiplied)."""
    unit = 2 * world
    kp = -(-k // unit) * unit                     # padded row count
    panels = max(1, min(int(panels), kp // unit))
    step = -(-kp // panels)
    step = -(-step // unit) * unit
    out, k0 = [], 0
    while k0 < kp:
        k1 = min(kp, k0 + step)
        out.append((k0, k1))
        k0 = k1
    return out


def host_panel_bounds(k: int, world: int, first: int = 128, growth: float = 1.6,
                      last_min: int = 3328) -> list[tuple[int, int]]:
    """K-panels for ``HostShardedGemm`` (default plan). Every bound is a
    multiple of 2*world (equal, even per-rank shares; the last panel padded
    past k like ``gathered_panels``).

    * A ramp from ``first`` rows growing by ``growth``: per k-row a rank
      uploads 8*m_local + 8n/world bytes over PCIe (N = 10000, 8 GPUs:
      20 KB, 0.36 us at 55 GB/s, plus the 80 KB gather over NVLink) and
      multiplies for 2*m_local*n / 35 TF/s = 0.71 us, so each panel may be
      ~1.6x its predecessor and still land while the previous one computes.
    * One last panel of at least ``last_min`` rows, split into row chunks
      whose D2H copies run while later chunks compute: hiding the whole C
      shard's D2H (8*m_local*n bytes) under the last panel needs
      2*kl/F >= 8/H_d2h, i.e. kl >= 4F/H = 4 * 35e12 / 55e9 ~ 2550 (x1.3).
    """
    unit = 2 * world
    kp = -(-k // unit) * unit
    out, k0 = [], 0
    step = -(-max(first, 1) // unit) * unit
    while k0 < kp:
        if kp - k0 <= max(last_min, step + step // 2):
            out.append((k0, kp))
            break
        k1 = min(k0 + step, kp - last_min)
        k1 = max(k0 + unit, k1 // unit * unit)
        out.append((k0, k1))
        k0 = k1
        step = -(-int(step * growth) // unit) * unit
    return out


def shrinking_chunks(m: int, align: int = 128, last: int = 128) -> list[tuple[int, int]]:
    """Row chunks for the last panel: each half of what remains (on
    ``align``-row bounds) until at most ``last`` rows are left, so the D2H
    after the final chunk is small (N = 10000, 1250 rows: 640, 384, 128, 98)."""
    out, r0 = [], 0
    while m - r0 > last:
        step = -(-((m - r0) // 2) // align) * align
        step = min(step, m - r0)
        out.append((r0, r0 + step))
        r0 += step
    if r0 < m:
        out.append((r0, m))
    return out


def _gpu_matmul(a, b, out, accumulate: bool) -> None:
    from .backends import dgemm_launch
    dgemm_launch(a, b, out, accumulate=accumulate)


class ShardedGemm:
    """``C_local = A_local · B`` with B broadcast from ``src``.

    ``panels=None`` (default) broadcasts B in geometrically growing K-panels
    (``geometric_panel_bounds``); an integer gives that many panels after a
    short first one (``ramp_panel_bounds``).
    ``local_matmul(a, b, out, accumulate)`` defaults to the sm_100a kernel
    (asynchronous, current stream); CPU tests substitute a torch matmul to
    exercise the exchange logic over gloo."""

    def __init__(self, group=None, panels: int | None = None, src: int = 0,
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
        k = b.shape[0]
        bounds = geometric_panel_bounds(k) if not self.panels else ramp_panel_bounds(k, self.panels)
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


class HostShardedGemm:
    """End-to-end form over host buffers: ``C_local = A_local · B`` where each
    rank holds its rows of A and C in (pinned) host memory and can read B's
    rows from its own host copy.

    B crosses PCIe once in total rather than once per GPU: for K-panel q each
    rank uploads an equal share of the panel's rows over its own link, and one
    NCCL all-gather over NVLink/NVSwitch rebuilds the panel on every rank; the
    panel's GEMM ``C_local (+)= A_local[:, q] · B[q, :]`` runs as soon as its
    gather completes. The last panel's GEMM is split into row chunks whose
    D2H copies overlap the remaining chunks. Device buffers are cached across
    calls. With ``device='cpu'`` (gloo tests) copies are plain copies.

    Default plan (``panels=None``, ``chunks=None``): ``host_panel_bounds``
    (a ramp of small panels, then one deep last panel) and
    ``shrinking_chunks``; A is uploaded panel by panel (A[:, q] as a 2D copy
    from the pinned rows), so the first GEMM waits for ~1 MB of A and one
    small B share rather than the whole A shard. Integers give the even
    ``gathered_panels`` split and even chunks."""

    def __init__(self, group=None, panels: int | None = None, chunks: int | None = None,
                 local_matmul: Callable | None = None, device=None):
        self.group = group
        self.panels = panels
        self.chunks = chunks
        self.local_matmul = local_matmul or _gpu_matmul
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._bufs = None

    def plan(self, k: int, world: int) -> list[tuple[int, int]]:
        """The K-panel bounds a call with inner dimension ``k`` uses."""
        return host_panel_bounds(k, world) if not self.panels else gathered_panels(k, world, self.panels)

    def share_rows(self, k: int, world: int, rank: int) -> list[tuple[int, int]]:
        """Rows of B this rank uploads, panel by panel: ``[(s0, s1), ...]``
        (clipped to ``k``; the last panel's padding rows are not read). A
        rank that holds only these rows, packed in this order as a
        ``(sum of panel shares) x n`` pinned buffer, passes it with
        ``b_packed=True`` and never needs all of B in host memory."""
        out = []
        for k0, k1 in self.plan(k, world):
            sh = (k1 - k0) // world
            out.append((min(k, k0 + rank * sh), min(k0 + (rank + 1) * sh, k)))
        return out

    def packed_rows(self, k: int, world: int) -> int:
        """Rows of the packed share buffer (``b_packed=True``)."""
        return sum((k1 - k0) // world for k0, k1 in self.plan(k, world))

    def _buffers(self, m, k, kp, n, share_rows):
        key = (m, k, kp, n, share_rows)
        if self._bufs is None or self._bufs[0] != key:
            dev = self.device
            a = torch.empty((m, k), dtype=torch.float64, device=dev)
            b = torch.empty((kp, n), dtype=torch.float64, device=dev)
            c = torch.empty((m, n), dtype=torch.float64, device=dev)
            stage = torch.zeros((share_rows, n), dtype=torch.float64, device=dev)  # this rank's shares; pad rows 0
            self._bufs = (key, a, b, c, stage)
        return self._bufs[1:]

    def __call__(self, a_local_h: torch.Tensor, b_h: torch.Tensor, c_local_h: torch.Tensor,
                 b_packed: bool = False) -> torch.Tensor:
        """``b_h`` is all of B (k x n), or with ``b_packed=True`` only this
        rank's panel shares packed in panel order (``share_rows``)."""
        world = dist.get_world_size(self.group)
        rank = dist.get_rank(self.group)
        m, k = a_local_h.shape
        n = b_h.shape[1]
        if b_packed:
            if b_h.shape[0] != self.packed_rows(k, world):
                raise ValueError(f"packed B shares need {self.packed_rows(k, world)} rows, got {b_h.shape[0]}")
        elif b_h.shape[0] != k:
            raise ValueError(f"shapes {tuple(a_local_h.shape)} @ {tuple(b_h.shape)} -> {tuple(c_local_h.shape)}")
        if tuple(c_local_h.shape) != (m, n):
            raise ValueError(f"shapes {tuple(a_local_h.shape)} @ {tuple(b_h.shape)} -> {tuple(c_local_h.shape)}")
        bounds = self.plan(k, world)
        kp = bounds[-1][1]
        shares = [(k1 - k0) // world for k0, k1 in bounds]
        a_d, b_d, c_d, stage = self._buffers(m, k, kp, n, sum(shares))
        cuda = self.device.type == "cuda"
        comp = torch.cuda.current_stream(self.device) if cuda else None
        copy_s = torch.cuda.Stream(self.device) if cuda else None
        back_s = torch.cuda.Stream(self.device) if cuda else None

        def on(stream):
            return torch.cuda.stream(stream) if stream is not None else _null()

        # Uploads and gathers are issued from the copy stream, panel by panel:
        # NCCL orders gather q after the uploads enqueued before it (this
        # rank's B shares and A column slices of panels <= q).
        works, off = [], 0
        with on(copy_s):
            if cuda:
                copy_s.wait_stream(comp)  # the cached buffers are free once earlier compute is done
            for q, (k0, k1) in enumerate(bounds):
                sh = shares[q]
                s0, s1 = k0 + rank * sh, min(k0 + (rank + 1) * sh, k)
                if s1 > s0:
                    src = b_h[off:off + s1 - s0] if b_packed else b_h[s0:s1]
                    stage[off:off + s1 - s0].copy_(src, non_blocking=cuda)
                kk1 = min(k1, k)
                if m > 0 and kk1 > k0:
                    _copy_cols(a_d, a_local_h, k0, kk1, copy_s)
                works.append(dist.all_gather_into_tensor(b_d[k0:k1], stage[off:off + sh], group=self.group,
                                                         async_op=True))
                off += sh
        if self.chunks:
            step = -(-max(m, 1) // self.chunks)     # ceil(m / chunks) ...
            step = -(-step // 128) * 128            # ... on 128-row tile bounds
            chunks = [(r0, min(m, r0 + step)) for r0 in range(0, m, step)]
        else:
            chunks = shrinking_chunks(m)
        for q, (k0, k1) in enumerate(bounds):
            works[q].wait()  # the compute stream (not the host) waits for the gather
            kk1 = min(k1, k)
            if kk1 <= k0 or m == 0:
                continue
            if q < len(bounds) - 1:
                self.local_matmul(a_d[:, k0:kk1], b_d[k0:kk1], c_d, q > 0)
                continue
            # last panel: row chunks, each copied back as soon as it is final
            for r0, r1 in chunks:
                self.local_matmul(a_d[r0:r1, k0:kk1], b_d[k0:kk1], c_d[r0:r1], q > 0)
                if cuda:
                    back_s.wait_stream(comp)
                with on(back_s):
                    c_local_h[r0:r1].copy_(c_d[r0:r1], non_blocking=cuda)
        if cuda:
            back_s.synchronize()  # synchronous call: C is in host memory on return
            comp.wait_stream(back_s)
        return c_local_h


def _copy_cols(dst: torch.Tensor, src: torch.Tensor, k0: int, k1: int, stream) -> None:
    """dst[:, k0:k1] = src[:, k0:k1] between host and device without a
    host-side gather: one cudaMemcpy2DAsync on ``stream`` (CUDA), or a plain
    slice copy (CPU tensors, the gloo tests)."""
    if stream is None:
        dst[:, k0:k1].copy_(src[:, k0:k1])
        return
    from . import _lib

    es = dst.element_size()
    _lib.check(_lib.lib().tb_copy2d_async(dst.data_ptr() + k0 * es, dst.stride(0) * es, src.data_ptr() + k0 * es,
                                          src.stride(0) * es, (k1 - k0) * es, dst.shape[0], stream.cuda_stream))


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


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


def peer_sharded_dgemm(a_rows: list, b_root: torch.Tensor, c_rows: list, b_replicas: list | None = None,
                       variant="auto") -> tuple[float, float]:
    """EXPERIMENTAL, unmeasured (see include/tbgpu.h): the measured
    multi-GPU paths are ``ShardedGemm`` / ``HostShardedGemm`` (one process
    per GPU, NCCL).

    Single-process form (``tb_dgemm_mgpu``): ``c_rows[i] = a_rows[i] · B``
    with every ``a_rows[i]`` / ``c_rows[i]`` (and ``b_replicas[i]``, i >= 1)
    a contiguous float64 CUDA tensor on device i's GPU and B on the GPU of
    ``a_rows[0]``. B is forwarded down the device chain in K-panels by peer
    copies overlapped with the panel GEMMs; ``b_replicas`` defaults to fresh
    buffers. Returns ``(kernel_seconds_max, total_seconds)``."""
    import ctypes

    from . import _lib
    from .errors import ShapeError

    nd = len(a_rows)
    if nd < 1 or len(c_rows) != nd:
        raise ShapeError(f"need one C block per A block, got {nd} and {len(c_rows)}")
    k, n = b_root.shape
    for i, (a, c) in enumerate(zip(a_rows, c_rows)):
        for t, name in ((a, "a"), (c, "c")):
            if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
                raise ShapeError(f"{name}_rows[{i}] must be a contiguous float64 CUDA tensor")
        if a.shape[1] != k or tuple(c.shape) != (a.shape[0], n) or a.device != c.device:
            raise ShapeError(f"block {i}: {tuple(a.shape)} @ {k}x{n} -> {tuple(c.shape)} on {a.device}/{c.device}")
    if b_root.dtype != torch.float64 or not b_root.is_cuda or not b_root.is_contiguous() \
            or b_root.device != a_rows[0].device:
        raise ShapeError("b_root must be a contiguous float64 CUDA tensor on a_rows[0]'s device")
    if b_replicas is None:
        b_replicas = [None] + [torch.empty((k, n), dtype=torch.float64, device=a.device) for a in a_rows[1:]]
    for i in range(1, nd):
        r = b_replicas[i]
        if r is None or tuple(r.shape) != (k, n) or r.device != a_rows[i].device or not r.is_contiguous():
            raise ShapeError(f"b_replicas[{i}] must be a contiguous {k}x{n} tensor on {a_rows[i].device}")
    for d in {a.device.index for a in a_rows}:
        torch.cuda.synchronize(d)  # the call does not order itself after torch's streams
    devs = (ctypes.c_int32 * nd)(*[a.device.index for a in a_rows])
    ap = (ctypes.c_void_p * nd)(*[a.data_ptr() for a in a_rows])
    cp = (ctypes.c_void_p * nd)(*[c.data_ptr() for c in c_rows])
    bp = (ctypes.c_void_p * nd)(*([0] + [r.data_ptr() for r in b_replicas[1:]]))
    rows = (ctypes.c_int64 * nd)(*[a.shape[0] for a in a_rows])
    kmax, total = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.lib().tb_dgemm_mgpu(nd, devs, ap, b_root.data_ptr(), bp, cp, rows, k, n,
                                        _lib.variant_id(variant), ctypes.byref(kmax), ctypes.byref(total)))
    return kmax.value, total.value
