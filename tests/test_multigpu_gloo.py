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

from paper_2509_04594_b200.multigpu import ShardedGemm, gather_rows, panel_bounds, row_partitions


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


@pytest.mark.parametrize("n,panels", [(37, 1), (64, 3), (5, 2)])
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
