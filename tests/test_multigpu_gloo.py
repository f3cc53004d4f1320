"""The row-sharded multi-GPU driver's exchange logic, world_size 2 over gloo
on CPU: partitions (plan_partitions rule), the (K-panel) broadcast of B from
rank 0, per-panel accumulation and the row gather. The local multiply is a
torch CPU matmul here; on the GPU it is the sm_100a kernel."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_04594_b200.multigpu import (HostShardedGemm, ShardedGemm, gather_rows, gathered_panels, panel_bounds,
                                            ramp_panel_bounds, row_partitions)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cpu_matmul(a, b, out, accumulate):
    if accumulate:
        out += a @ b
    else:
        out.copy_(a @ b)


def _worker(rank, world, port, n, panels, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.Generator(np.random.PCG64(1))
        a = torch.from_numpy(rng.random((n, n)) * 3 + 2)
        b_full = torch.from_numpy(np.random.Generator(np.random.PCG64(2)).random((n, n)) * 3 + 2)
        parts = row_partitions(n, world)
        r0, r1 = parts[rank]
        b = b_full.clone() if rank == 0 else torch.full((n, n), float("nan"), dtype=torch.float64)
        out = torch.empty((r1 - r0, n), dtype=torch.float64)
        ShardedGemm(panels=panels, local_matmul=_cpu_matmul)(a[r0:r1].contiguous(), b, out)
        assert torch.equal(b, b_full), "broadcast did not deliver B"
        full = gather_rows(out, parts, dst=0)
        if rank == 0:
            ref = (a @ b_full).numpy()
            q.put(float(np.linalg.norm(full.numpy() - ref) / np.linalg.norm(ref)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,panels", [(37, 1), (64, 3), (5, 2), (700, None)])
def test_sharded_world2(n, panels):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, panels, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get() <= 1e-12


def test_row_partitions_rule():
    assert row_partitions(10000, 8) == [(i * 1250, (i + 1) * 1250) for i in range(8)]
    assert row_partitions(32768, 8)[-1] == (28672, 32768)
    assert row_partitions(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert row_partitions(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    for m in (1, 7, 10000):
        for w in (1, 2, 3, 8):
            p = row_partitions(m, w)
            assert p[0][0] == 0 and p[-1][1] == m and len(p) == w


def test_panel_bounds_even_and_covering():
    for k in (1, 2, 3, 100, 10000, 32768):
        for panels in (1, 2, 3, 4, 7, 16):
            b = panel_bounds(k, panels)
            assert b[0][0] == 0 and b[-1][1] == k
            assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
            assert all(k0 % 2 == 0 for k0, _ in b)


def _host_worker(rank, world, port, m, k, n, panels, chunks, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = torch.from_numpy(np.random.Generator(np.random.PCG64(3)).random((m, k)) * 3 + 2)
        b = torch.from_numpy(np.random.Generator(np.random.PCG64(4)).random((k, n)) * 3 + 2)
        parts = row_partitions(m, world)
        r0, r1 = parts[rank]
        c = torch.full((r1 - r0, n), float("nan"), dtype=torch.float64)
        g = HostShardedGemm(panels=panels, chunks=chunks, local_matmul=_cpu_matmul, device="cpu")
        for _ in range(2):  # cached buffers reused by the second call
            g(a[r0:r1].contiguous(), b, c)
        full = gather_rows(c, parts, dst=0)
        # the same product from only this rank's shares of B (packed in panel order)
        packed = torch.full((g.packed_rows(k, world), n), float("nan"), dtype=torch.float64)
        off = 0
        for (k0, k1), (s0, s1) in zip(g.plan(k, world), g.share_rows(k, world, rank)):
            packed[off:off + (k1 - k0) // world] = 0.0
            packed[off:off + s1 - s0] = b[s0:s1]
            off += (k1 - k0) // world
        c2 = torch.full((r1 - r0, n), float("nan"), dtype=torch.float64)
        g(a[r0:r1].contiguous(), packed, c2, b_packed=True)
        assert torch.equal(c, c2)
        if rank == 0:
            ref = (a @ b).numpy()
            q.put(float(np.linalg.norm(full.numpy() - ref) / np.linalg.norm(ref)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,k,n,panels,chunks", [(37, 41, 29, 3, 2), (64, 64, 64, 1, 4), (5, 3, 7, 2, 1),
                                                 (300, 200, 100, 4, 3), (300, 700, 90, None, None),
                                                 (7, 1001, 33, None, None)])
def test_host_sharded_world2(m, k, n, panels, chunks):
    """End-to-end multi-GPU form: B uploaded in equal per-rank shares per
    K-panel and rebuilt by all-gather, last panel in row chunks copied back."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_host_worker, args=(r, 2, port, m, k, n, panels, chunks, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get() <= 1e-12


def test_gathered_panels_cover_and_divide():
    for k in (1, 2, 3, 5, 37, 1000, 10000, 32768):
        for world in (1, 2, 3, 4, 8):
            for panels in (1, 2, 4, 7):
                b = gathered_panels(k, world, panels)
                assert b[0][0] == 0 and b[-1][1] >= k and b[-1][1] - k < 2 * world
                assert all(x1 == y0 for (_, x1), (y0, _) in zip(b, b[1:]))
                assert all((k1 - k0) % (2 * world) == 0 and k1 > k0 for k0, k1 in b)


def test_ramp_panel_bounds():
    for k in (1, 2, 3, 5, 37, 1000, 10000, 32768):
        for panels in (1, 2, 4, 7):
            b = ramp_panel_bounds(k, panels)
            assert b[0][0] == 0 and b[-1][1] == k and all(x1 == y0 for (_, x1), (y0, _) in zip(b, b[1:]))
            assert all(k1 > k0 and k0 % 2 == 0 for k0, k1 in b)
            if len(b) > 2 and k >= 1000:
                assert b[0][1] - b[0][0] <= (b[1][1] - b[1][0]) // 4  # short first panel


def test_geometric_panel_bounds():
    from paper_2509_04594_b200.multigpu import geometric_panel_bounds

    assert geometric_panel_bounds(10000) == [(0, 128), (128, 512), (512, 1664), (1664, 5120), (5120, 10000)]
    for k in (1, 2, 3, 5, 37, 127, 128, 129, 1000, 10000, 32768):
        b = geometric_panel_bounds(k)
        assert b[0][0] == 0 and b[-1][1] == k
        assert all(x1 == y0 for (_, x1), (y0, _) in zip(b, b[1:]))
        assert all(k1 > k0 for k0, k1 in b)
        assert all(k0 % 2 == 0 for k0, _ in b)          # TMA alignment of every panel start
        assert len(b) <= 8


def test_host_panel_bounds_and_chunks():
    from paper_2509_04594_b200.multigpu import host_panel_bounds, shrinking_chunks

    for world in (1, 2, 3, 4, 8):
        for k in (1, 2, 3, 5, 37, 1000, 4000, 10000, 32768):
            b = host_panel_bounds(k, world)
            assert b[0][0] == 0 and b[-1][1] >= k and b[-1][1] - k < 2 * world
            assert all(x1 == y0 for (_, x1), (y0, _) in zip(b, b[1:]))
            assert all((k1 - k0) % (2 * world) == 0 and k1 > k0 for k0, k1 in b)
            if len(b) > 1:
                assert b[-1][1] - b[-1][0] >= 3328 - 2 * world     # deep last panel hides C's D2H
    assert [y - x for x, y in host_panel_bounds(10000, 8)] == [128, 208, 336, 544, 880, 1408, 2256, 4240]
    for m in (0, 1, 127, 128, 129, 1250, 5000, 16384):
        c = shrinking_chunks(m)
        assert sum(r1 - r0 for r0, r1 in c) == m
        assert all(x1 == y0 for (_, x1), (y0, _) in zip(c, c[1:]))
        assert all(r0 % 128 == 0 for r0, _ in c)
        if c:
            assert c[-1][1] - c[-1][0] <= 128
