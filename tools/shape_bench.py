"""Kernel-only TFLOP/s for explicit (m, k, n) shapes (tooling).
    python tools/shape_bench.py 1250x10000x10000 4096x32768x32768 ..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2509_04594_b200 as tb  # noqa: E402

variant = os.environ.get("VARIANT", "auto")
for spec in sys.argv[1:]:
    m, k, n = map(int, spec.split("x"))
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.rand((m, k), dtype=torch.float64, device="cuda", generator=g)
    B = torch.rand((k, n), dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty((m, n), dtype=torch.float64, device="cuda")
    best = 1e9
    for i in range(4):
        if os.environ.get("ACC") == "1":  # C += A·B through the async launch entry
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            tb.dgemm_launch(A, B, C, accumulate=True, variant=variant)
            e1.record()
            e1.synchronize()
            s = e0.elapsed_time(e1) / 1e3
        else:
            _, s = tb.dgemm(A, B, C, variant=variant)
        if i:
            best = min(best, s)
    cb = 1e9
    for i in range(3):
        _, s = tb.cublas_dgemm(A, B, C)
        if i:
            cb = min(cb, s)
    f = 2.0 * m * n * k
    print(json.dumps({"shape": spec, "ms": best * 1e3, "tflops": f / best / 1e12, "cublas_tflops": f / cb / 1e12}))
    del A, B, C
    torch.cuda.empty_cache()
