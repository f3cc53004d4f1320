"""Kernel-only TFLOP/s of square GEMMs for one main-tile configuration
(tooling for the small/medium-N tile chooser).

    TB_TILE=64x64 python tools/tile_sweep.py 1000:3001:100 [--cublas]

One JSON line per size: best of REPS launches (CUDA events, fresh C), and
with --cublas the cuBLAS DGEMM time on the same operands."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2509_04594_b200 as tb  # noqa: E402

REPS = int(os.environ.get("REPS", "7"))


def sizes(spec):
    out = []
    for part in spec.split(","):
        if ":" in part:
            a, b, c = map(int, part.split(":"))
            out.extend(range(a, b, c))
        else:
            out.append(int(part))
    return out


def best(fn):
    t = []
    for i in range(REPS + 1):
        t.append(fn())
    return min(t[1:])


tile = os.environ.get("TB_TILE", "auto")
for n in sizes(sys.argv[1]):
    g = torch.Generator(device="cuda").manual_seed(n)
    A = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g)
    B = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ours = best(lambda: tb.dgemm(A, B, C)[1])
    ref = A @ B
    err = (torch.linalg.norm(C - ref) / torch.linalg.norm(ref)).item()
    f = 2.0 * n ** 3
    rec = {"tile": tile, "n": n, "us": ours * 1e6, "tflops": f / ours / 1e12, "normwise_vs_torch": err}
    if "--cublas" in sys.argv:
        cb = best(lambda: tb.cublas_dgemm(A, B, C)[1])
        rec["cublas_us"] = cb * 1e6
        rec["cublas_tflops"] = f / cb / 1e12
    print(json.dumps(rec), flush=True)
