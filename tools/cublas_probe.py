"""cuBLAS DGEMM probe (torch.matmul on float64 CUDA tensors): the baseline the
hand-written kernels are compared against. Not part of the product."""
import json
import sys

import torch

for n in [int(x) for x in (sys.argv[1:] or ["4000", "10000"])]:
    a = torch.rand(n, n, dtype=torch.float64, device="cuda") * 3 + 2
    b = torch.rand(n, n, dtype=torch.float64, device="cuda") * 3 + 2
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(5):
        e0.record()
        c = a @ b
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    t = min(times)
    print(json.dumps({"probe": "cublas_dgemm", "n": n, "best_s": t,
                      "gflops": (2 * n**3 - n**2) / t / 1e9,
                      "median_s": sorted(times)[len(times) // 2]}))
