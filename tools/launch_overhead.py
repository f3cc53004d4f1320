"""Launch overhead of a synchronous kernel-only call (tooling): for small
square N, the event-timed single call (tb.dgemm / cuBLAS through the same
tb_cublas_dgemm clock) against the per-launch time of back-to-back launches
(host work hidden behind the queue). The difference is host-side time inside
a synchronous call's kernel-only interval.

    python tools/launch_overhead.py [N ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2509_04594_b200 as tb  # noqa: E402
from paper_2509_04594_b200 import _lib  # noqa: E402

REPS = 50
for n in [int(x) for x in sys.argv[1:]] or [64, 256, 1024]:
    A = torch.rand((n, n), dtype=torch.float64, device="cuda")
    B = torch.rand((n, n), dtype=torch.float64, device="cuda")
    C = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ours = min(tb.dgemm(A, B, C)[1] for _ in range(REPS))
    cub = min(tb.cublas_dgemm(A, B, C)[1] for _ in range(REPS))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()
    for _ in range(3):
        tb.dgemm_launch(A, B, C)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(20):
        tb.dgemm_launch(A, B, C)
    e1.record(s)
    torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) * 1e-3 / 20
    t0 = time.perf_counter()
    for _ in range(200):
        _lib.launch_plan(n, n, n)
    plan_us = (time.perf_counter() - t0) / 200 * 1e6
    print(json.dumps({"n": n, "single_call_us": ours * 1e6, "cublas_single_call_us": cub * 1e6,
                      "back_to_back_us": b2b * 1e6, "launch_plan_dry_run_us": plan_us}), flush=True)
