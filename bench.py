#!/usr/bin/env python
"""Benchmark of the FP64 square-GEMM hot path (arXiv 2509.04594, tilebench).

Metric (BASELINE.json): FP64 GFLOPS = (2N^3 - N^2) / kernel seconds at
N = 10000, with % of B200 FP64 peak. One step = one C = A·B over the whole
N x N problem (at N GPUs: B broadcast from rank 0 over NCCL + each rank's
row-block GEMM).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--size 10000] [--impl ours|reference]

Prints ONE JSON line on rank 0. Inputs (800 MB per matrix at N = 10000) are
larger than the 126 MB L2, so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from datetime import timedelta

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "FP64 GFLOPS ((2N^3−N^2)/kernel s) at N=10000; % of B200 FP64 peak"
UNIT = "GFLOPS"
SMS = 148
FP64_FMA_PER_CLK_PER_SM = 64


def flop_count(n: int) -> int:
    return 2 * n**3 - n**2


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def fp64_peak_tflops() -> tuple[float, str]:
    mhz = measured_peaks().get("sm_max_mhz")
    src = "MEASURED_PEAKS.json sm_max_mhz"
    if not mhz:
        mhz, src = 1965.0, "B200_PROFILING.md clocks.max.sm"
    return SMS * FP64_FMA_PER_CLK_PER_SM * 2 * mhz * 1e6 / 1e12, (
        f"nominal FP64 (DMMA/DFMA pipe): 148 SM x 64 FMA/clk x 2 x {mhz:.0f} MHz ({src}); "
        "measured DMMA register-only loop 37.15 TFLOPS (profiles/r01_pipe_microbench.txt)")


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        try:
            with open(self.path) as f:
                for line in f:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9:
                        rows.append(parts)
        except OSError:
            pass
        finally:
            if self.path:
                try:
                    os.unlink(self.path)
                except OSError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in rows if num(r[1])]
        mx = max((num(r[2]) or 0) for r in rows)
        power = [num(r[3]) for r in rows if num(r[3])]
        load = [s for s, r in zip(sm, rows) if (num(r[3]) or 0) > 300] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(power) if power else None}


def _cpu_operands(n: int, rows: int):
    import numpy as np

    b = np.random.Generator(np.random.PCG64(1)).random((n, n)) * 3.0 + 2.0
    a = np.random.Generator(np.random.PCG64(2)).random((rows, n)) * 3.0 + 2.0
    return a, b


def cpu_calibrate(n: int, threads: int, target_s: float) -> int:
    """Rows of the N x N product that take about target_s on the host cores."""
    from oracle import oracle as ref

    rows = max(threads, 16)
    a, b = _cpu_operands(n, rows)
    t0 = time.perf_counter()
    ref.tiled_parallel(a, b, 32, threads)
    dt = time.perf_counter() - t0
    return int(min(n, max(threads, rows * target_s / max(dt, 1e-3))))


def cpu_sample(n: int, threads: int, rows: int) -> dict:
    """The reference's CPU tiled path (oracle C port of tile_range_kernel +
    plan_partitions, pthreads) timed on a bounded row sample of the N x N
    workload; rows of tiled(A[rows], B) are bitwise rows of the full product."""
    from oracle import oracle as ref

    a, b = _cpu_operands(n, rows)
    t0 = time.perf_counter()
    ref.tiled_parallel(a, b, 32, threads)
    dt = time.perf_counter() - t0
    flops = rows * (2 * n * n - n)
    return {"value": flops / dt / 1e9, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"tiled-parallel K=32 (oracle/tb_oracle.c port of kernels.py:32-53 + backends.py:119-160) "
                      f"on {rows} of {n} rows of the N={n} product, {dt:.1f} s, {threads} threads",
            "seconds": dt}


def blas_sample(n: int, target_s: float = 3.0) -> dict:
    """The reference's BLAS backend (``a @ b`` through numpy's bundled
    OpenBLAS, demos/06_external_backends.py / SURVEY.md §8(d)) on a row
    sample of the N x N product, all host threads: reported beside the
    tiled-path baseline, not the reference arm's value."""
    import numpy as np

    a_full, b = _cpu_operands(n, 256)
    t0 = time.perf_counter()
    a_full @ b
    dt = max(time.perf_counter() - t0, 1e-3)
    rows = int(min(n, max(256, 256 * target_s / dt)))
    a, _ = _cpu_operands(n, rows) if rows > 256 else (a_full, b)
    t0 = time.perf_counter()
    a @ b
    dt = time.perf_counter() - t0
    threads = os.environ.get("OPENBLAS_NUM_THREADS") or os.cpu_count()
    return {"value": rows * (2 * n * n - n) / dt / 1e9, "unit": UNIT, "threads": threads,
            "sample": f"numpy {np.__version__} matmul (OpenBLAS) on {rows} of {n} rows, {dt:.2f} s"}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _ref_cpu_worker(n: int, threads: int, target_s: float) -> None:
    """Subprocess body (``bench.py --ref-cpu-worker``): the reference's OWN
    numba CPU backends, imported unmodified from baseline/_ref, timed on a
    row sample of the N x N product: ``tiled_parallel_multiply`` (the
    OpenMP-style static split, backends.py:139-160) and
    ``tiled_pool_multiply`` (the C++-threads-style task queue,
    backends.py:163-190), both with PoolConfig(threads) and TileConfig(32),
    timed with the reference's own perf_counter bracket (harness.py:163-172).
    Prints one JSON object."""
    import numba
    import numpy as np
    import tilebench
    from tilebench.backends import PoolConfig, TileConfig, tiled_parallel_multiply, tiled_pool_multiply

    out = {"tilebench": getattr(tilebench, "__version__", "?"), "numba": numba.__version__, "threads": threads,
           "from": REF_DIR}
    b = np.random.Generator(np.random.PCG64(1)).random((n, n)) * 3.0 + 2.0
    tile, pool = TileConfig(32), PoolConfig(threads)
    tiled_parallel_multiply(np.ones((2, 2)), np.ones((2, 2)), tile, pool)  # JIT (cache outside the tree)
    for name, fn in (("tiled-parallel", tiled_parallel_multiply), ("tiled-pool", tiled_pool_multiply)):
        rows = min(n, 8 * threads)  # enough tile rows to keep every thread busy while calibrating
        a = np.random.Generator(np.random.PCG64(2)).random((rows, n)) * 3.0 + 2.0
        t0 = time.perf_counter()
        fn(a, b, tile, pool)
        dt = max(time.perf_counter() - t0, 1e-3)
        rows = int(min(n, max(32, rows * target_s / dt))) // 32 * 32 or 32
        a = np.random.Generator(np.random.PCG64(2)).random((rows, n)) * 3.0 + 2.0
        t0 = time.perf_counter()
        fn(a, b, tile, pool)
        dt = time.perf_counter() - t0
        out[name] = {"value": rows * (2 * n * n - n) / dt / 1e9, "unit": UNIT, "cores": threads, "rows": rows,
                     "seconds": dt,
                     "sample": f"reference tilebench.backends.{fn.__name__} (numba {numba.__version__}, unmodified, "
                               f"baseline/_ref) on {rows} of {n} rows of the N={n} product, {dt:.1f} s, "
                               f"{threads} threads"}
    print(json.dumps(out), flush=True)


def reference_numba_cpu(n: int, threads: int, target_s: float = 8.0) -> dict:
    """The reference's own CPU code (numba ``tiled-parallel`` and
    ``tiled-pool``) timed in a clean subprocess with NUMBA_CACHE_DIR outside
    the tree; reported beside the C port (the reference arm's value)."""
    if not os.path.isdir(os.path.join(REF_DIR, "tilebench")):
        return {"unavailable": "baseline/_ref/tilebench not installed"}
    env = dict(os.environ, PYTHONPATH=REF_DIR, NUMBA_CACHE_DIR=os.path.join(tempfile.gettempdir(), "tb_numba_cache"),
               NUMBA_NUM_THREADS=str(threads))
    cmd = [sys.executable, os.path.abspath(__file__), "--ref-cpu-worker", "--size", str(n), "--ref-threads",
           str(threads), "--ref-seconds", str(target_s)]
    try:
        res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    except subprocess.TimeoutExpired:
        return {"unavailable": "reference numba run timed out"}
    if res.returncode != 0:
        return {"unavailable": f"reference numba run failed: {res.stderr.strip().splitlines()[-1:]}"}
    return json.loads(res.stdout.strip().splitlines()[-1])


def cpu_baselines(n: int, target_s: float) -> dict:
    """cpu_baseline: the C port of the reference's tiled-parallel path on all
    host threads (``value``), plus sub-records on the same N: the
    reference's own numba tiled-parallel and tiled-pool, and its BLAS
    backend (numpy matmul, demos/06_external_backends.py)."""
    threads = os.cpu_count() or 1
    cpu = cpu_sample(n, threads, cpu_calibrate(n, threads, target_s))
    cpu.pop("seconds", None)
    cpu["blas"] = blas_sample(n)
    cpu["reference_numba"] = reference_numba_cpu(n, threads)
    cpu["host_threads"] = threads
    return cpu


def run_reference(args) -> None:
    rank, world, _ = env_rank()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals = []
    # each step a bounded sample; the whole --steps/--warmup run stays within ~3 minutes
    per_step = min(args.ref_seconds, 150.0 / max(1, args.steps + args.warmup))
    rows = cpu_calibrate(args.n, threads, per_step)
    for i in range(args.warmup + args.steps):
        s = cpu_sample(args.n, threads, rows)
        if i >= args.warmup:
            vals.append(s)
    v = statistics.median([s["value"] for s in vals])
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic uniform[2,5] (numpy PCG64)",
            "config": {"workload": f"N={args.n} FP64 square GEMM, bounded row sample on host cores", "n": args.n},
            "cpu_baseline": {**{k: vals[-1][k] for k in ("unit", "cores", "kind", "sample")}, "value": v,
                             "blas": blas_sample(args.n), "reference_numba": reference_numba_cpu(args.n, threads)},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "ms_per_step": statistics.median([s["seconds"] for s in vals]) * 1e3}
    print(json.dumps(line), flush=True)


def run_ours(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2509_04594_b200 as tb
    from paper_2509_04594_b200 import _lib
    from paper_2509_04594_b200.harness import gpu_environment
    from paper_2509_04594_b200.multigpu import HostShardedGemm, ShardedGemm, row_partitions

    rank, world, local = env_rank()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 under torchrun")
    # TB_BENCH_SHARED_DEVICE=1 puts every rank on cuda:0 (exercises the N>1
    # code path on a 1-GPU box with --dist-backend gloo; not a measurement).
    local_dev = 0 if os.environ.get("TB_BENCH_SHARED_DEVICE") == "1" else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    n = args.n
    parts = row_partitions(n, world)
    r0, r1 = parts[rank]
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)
    a_loc = torch.rand((r1 - r0, n), dtype=torch.float64, device=dev, generator=g) * 3.0 + 2.0
    b = torch.empty((n, n), dtype=torch.float64, device=dev)
    if rank == 0:
        g.manual_seed(7)
        b.copy_(torch.rand((n, n), dtype=torch.float64, device=dev, generator=g) * 3.0 + 2.0)
    c_loc = torch.empty((r1 - r0, n), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    sharded = ShardedGemm(panels=args.panels or None) if world > 1 else None

    def step():
        if world > 1:
            sharded(a_loc, b, c_loc)
        else:
            tb.dgemm_launch(a_loc, b, c_loc, variant=args.variant)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    # kernel-only launch timing of the dominant kernel on its own stream (roofline achieved)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    launches0 = _lib.kernel_launches()
    with ClockSampler(local_dev) as clocks:
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(args.steps):
            if world > 1:
                step()
            else:
                ev[2 * i].record(stream)
                step()
                ev[2 * i + 1].record(stream)
        t1.record(stream)
        barrier()
    gpu_launches = _lib.kernel_launches() - launches0  # our kernels enqueued in the timed region
    total_s = t0.elapsed_time(t1) / 1e3
    if world > 1:
        t = torch.tensor([total_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_s = t.item()
    ms_per_step = total_s / args.steps * 1e3
    value = flop_count(n) * args.steps / total_s / 1e9
    clk = clocks.summary()

    # kernel-only per-launch durations (N=1: the timed launches themselves; N>1: a local-GEMM pass)
    if world == 1:
        launch_s = [ev[2 * i].elapsed_time(ev[2 * i + 1]) / 1e3 for i in range(args.steps)]
    else:
        launch_s = []
        for _ in range(max(3, args.steps // 2)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            tb.dgemm_launch(a_loc, b, c_loc)
            e1.record(stream)
            e1.synchronize()
            launch_s.append(e0.elapsed_time(e1) / 1e3)
    avg_launch = sum(launch_s) / len(launch_s)
    flops_per_launch = (r1 - r0) * (2 * n * n - n)
    peak, peak_src = fp64_peak_tflops()
    achieved = flops_per_launch / avg_launch / 1e12
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        try:
            traffic = json.load(open(tr_path)).get(str(n))
        except (OSError, ValueError):
            traffic = None

    # cuBLAS DGEMM on the same buffers (reported baseline, not the target)
    cub = []
    for i in range(3 + 1):
        _, sec = tb.cublas_dgemm(a_loc, b)
        if i:
            cub.append(sec)
    cublas_gflops = flop_count(n) / world / min(cub) / 1e9 if cub else None

    # correctness spot check of the timed result vs cuBLAS (normwise)
    c_ref, _ = tb.cublas_dgemm(a_loc, b)
    tb.dgemm_launch(a_loc, b, c_loc)
    torch.cuda.synchronize()
    rel = (torch.linalg.norm(c_loc - c_ref) / torch.linalg.norm(c_ref)).item()
    del c_ref

    # End to end from pinned HOST buffers. N = 1: the reference-facing flat C
    # ABI (gpuTiledMultiplyFlat shape). N > 1: HostShardedGemm — each rank
    # uploads its A rows and an equal share of every K-panel of B, NCCL
    # all-gathers the panels over NVLink, C rows come back as they finish.
    # Host buffers are pinned directly (no pageable intermediate). At N > 1 a
    # rank holds its A / C rows and only its own shares of B's K-panels
    # (HostShardedGemm.share_rows, packed in panel order): B crosses PCIe
    # once in total and no rank ever holds all of B in host memory.
    def pinned(rows, cols):
        return torch.empty((rows, cols), dtype=torch.float64, pin_memory=True)

    a_h = pinned(r1 - r0, n)
    a_h.copy_(a_loc)
    host_sharded = HostShardedGemm(panels=args.panels or None) if world > 1 else None
    if world > 1:
        dist.broadcast(b, 0)
        b_h = pinned(host_sharded.packed_rows(n, world), n)
        b_h.zero_()
        off = 0
        for (k0, k1), (s0, s1) in zip(host_sharded.plan(n, world), host_sharded.share_rows(n, world, rank)):
            b_h[off:off + s1 - s0].copy_(b[s0:s1])
            off += (k1 - k0) // world
    else:
        b_h = pinned(n, n)
        b_h.copy_(b)
    c_h = pinned(r1 - r0, n)
    out_s = np.zeros(1)
    e2e = np.zeros(1)
    e2e_times, e2e_dev = [], []
    for i in range(1 + max(2, args.steps // 3)):
        if world > 1:
            dist.barrier()
        t_call = time.perf_counter()
        if world > 1:
            host_sharded(a_h, b_h, c_h, b_packed=True)
            dist.barrier()  # the step ends when every rank's C rows are in host memory
        else:
            st = tb.gpu_tiled_multiply_flat(local_dev, a_h, b_h, r1 - r0, n, n, 32, c_h, out_s,
                                            variant=args.variant, out_e2e_seconds=e2e)
            if st != 0:
                raise RuntimeError(f"flat ABI status {st}: {_lib.last_error()}")
        t_call = time.perf_counter() - t_call  # synchronous: C is in host memory on return
        if i:
            e2e_times.append(t_call)
            e2e_dev.append(e2e[0] if world == 1 else t_call)
    del host_sharded
    e2e_s = statistics.median(e2e_times)
    e2e_dev_s = statistics.median(e2e_dev)
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = t.item()
    _lib.lib().tb_release()
    h2d = 16 * n * n  # whole job: A once (row shards) + B once (per-rank panel shares); N = 1: A + B
    d2h = 8 * n * n

    import resource

    # Peak host RSS of the GEMM path (pinned A/C rows + this rank's B shares,
    # before the CPU baselines allocate their own operands), max over ranks.
    rss_gb = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20  # KiB -> GiB
    if world > 1:
        t = torch.tensor([rss_gb], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rss_gb = t.item()
    pinned_gb = (a_h.numel() + b_h.numel() + c_h.numel()) * 8 / 2**30
    env_meta = gpu_environment([], device=local_dev)
    env_meta["launch_plan"] = _lib.launch_plan(r1 - r0, n, n, args.variant, sms=env_meta["gpu"].get("sm_count", SMS))

    # CPU baselines on rank 0 (any N). The other ranks wait in the rendezvous
    # store (a blocking socket read, not a spinning device sync), so every
    # host core is free for the measurement.
    cpu = None
    if not args.no_cpu:
        store = dist.distributed_c10d._get_default_store() if world > 1 else None
        if rank == 0:
            cpu = cpu_baselines(n, args.ref_seconds)
            if store is not None:
                store.set("tb_bench_cpu_done", "1")
        elif store is not None:
            store.wait(["tb_bench_cpu_done"], timedelta(minutes=15))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic uniform[2,5] (torch Philox on device; host e2e buffers copied from it)",
            "config": {"workload": f"N={n} FP64 square GEMM C=A*B (BASELINE configs[3], 1..8 GPUs)", "n": n,
                       "tile": "128x128x16 CTA, 8 DMMA warps + TMA producer warpgroup, 6 stages",
                       "variant": args.variant, "parallelism": f"row-shard{world}" + (
                           f" + NCCL broadcast of B ({args.panels or 'geometric'} K-panels)" if world > 1 else ""),
                       "l2": f"inputs ({8 * n * n / 1e6:.0f} MB/matrix) larger than L2 (126 MB); no flush"},
            "pct_fp64_peak": 100.0 * value / 1e3 / peak,
            "pct_fp64_peak_40tf": 100.0 * value / 1e3 / 40.0,
            "cublas_gflops": cublas_gflops,
            "vs_cublas": (value / world) / cublas_gflops if cublas_gflops else None,
            "check_vs_cublas_normwise": rel,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "dgemm_dmma_kernel<1, 6, TMA, DMMA, 128> (cross-stage prefetch) on the whole 128x128 "
                                   "tiles + edge-strip launches for ragged m / n on a side stream filling its tail; "
                                   "achieved over the whole GEMM call",
                         "flops_per_launch": flops_per_launch,
                         "avg_launch_ms": avg_launch * 1e3, "peak_source": peak_src},
            "e2e": {"value": flop_count(n) / e2e_s / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3,
                    "device_event_value": flop_count(n) / e2e_dev_s / 1e9 if world == 1 else None,
                    "path": ("HostShardedGemm (multigpu.py): pinned host A rows + per-rank shares of each K-panel of B "
                             "-> H2D -> NCCL all-gather of the panel over NVLink -> panel GEMMs -> C row chunks D2H as "
                             "they finish; max over ranks of the host wall clock, barrier-to-barrier") if world > 1 else
                            "gpu_tiled_multiply_flat -> tb_gpu_tiled_multiply_flat_ex (the reference's flat FFI shape): "
                            "pinned host A,B -> copy/compute pipeline (phase 1: K-panels of A[:Mq] and B, 2D copies, consumed by "
                            "one flag-driven persistent GEMM launch; phase 2: full-K row blocks; C row blocks back as they "
                            "finish) -> host C. value: host wall clock "
                            "around the synchronous call (median); device_event_value: CUDA events first H2D -> last D2H"},
            "gpu_launches": gpu_launches,
            "clocks": clk,
            "cpu_baseline": cpu,
            "library": _lib.version(),
            "host_memory": {"rss_gb_max_rank_gemm_path": rss_gb, "pinned_gb_rank0": pinned_gb,
                            "rss_gb_rank0_incl_cpu_baseline": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20},
            "env": env_meta,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    p = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--size", dest="n", type=int, default=10000, help="matrix order N")
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--variant", default="auto")
    p.add_argument("--panels", type=int, default=0,
                   help="K-panels of the B exchange at N>1 (0: the default plans, geometric_panel_bounds for the device "
                        "path and host_panel_bounds for the host path)")
    p.add_argument("--ref-seconds", type=float, default=10.0, help="CPU sample length per measurement (s)")
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--dist-backend", default="nccl", help="torch.distributed backend at N>1 (nccl; gloo for tests)")
    p.add_argument("--ref-cpu-worker", action="store_true", help=argparse.SUPPRESS)
    p.add_argument("--ref-threads", type=int, default=0, help=argparse.SUPPRESS)
    args = p.parse_args()
    if args.ref_cpu_worker:
        _ref_cpu_worker(args.n, args.ref_threads or os.cpu_count() or 1, args.ref_seconds)
        return
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
