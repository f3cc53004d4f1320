"""Run the GEMM a few times at one size (ncu driver; not a bench)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2509_04594_b200 as tb  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=10000)
p.add_argument("--m", type=int, default=0, help="rows of A / C (default n): row shards, e.g. 1250 x 10000")
p.add_argument("--k", type=int, default=0, help="inner dimension (default n)")
p.add_argument("--variant", default="auto")
p.add_argument("--reps", type=int, default=3)
p.add_argument("--cublas", action="store_true")
a = p.parse_args()
g = torch.Generator(device="cuda").manual_seed(1)
m, k = a.m or a.n, a.k or a.n
A = torch.rand((m, k), dtype=torch.float64, device="cuda", generator=g) * 3 + 2
B = torch.rand((k, a.n), dtype=torch.float64, device="cuda", generator=g) * 3 + 2
C = torch.empty((m, a.n), dtype=torch.float64, device="cuda")
for _ in range(a.reps):
    if a.cublas:
        tb.cublas_dgemm(A, B, C)
    else:
        _, s = tb.dgemm(A, B, C, variant=a.variant)
        print(f"{a.variant} {m}x{k}x{a.n} {2 * m * k * a.n / s / 1e9:.1f} GFLOPS")
