"""Probe run by tests/test_gpu_mutations.py in a subprocess, with
TB_LIB_VARIANT selecting a mutant build of libtbgpu.so (or none: the product
build). Runs the parity checks of the GPU suite that exercise the consumer's
stage protocol on every kernel shape it has — the cross-stage-prefetch loop
(128 x 128 tiles), the plain loop (64-row tiles, edge strips), stream-K and
split-K fixups, and the accumulate epilogue that exposed the round-1 race —
with fresh operands per repetition (stale shared memory from an identical
earlier launch would otherwise mask a read-before-land), and prints the
largest normwise error per case as JSON. The reference: cuBLAS FP64 (torch)."""
import json
import os
import sys

import torch

import paper_2509_04594_b200 as tb

CASES = [  # (name, m, k, n, accumulate, env: TB_TILE forces a tile shape, TB_SPLIT=1 the edge strips)
    ("tiles128_streamk", 2048, 2048, 2048, False, {"TB_TILE": "128x128"}),
    ("tiles64_dataparallel", 1000, 1000, 1000, False, {"TB_TILE": "64x128"}),
    ("tiles64x64_streamk", 1300, 1300, 1300, False, {"TB_TILE": "64x64"}),
    ("tiles96x96_streamk", 2000, 1000, 2000, False, {"TB_TILE": "96x96"}),
    ("tiles128_edge_strips", 4000, 1000, 4000, False, {"TB_SPLIT": "1"}),
    ("splitk", 256, 4096, 256, False, {}),
    ("accumulate_epilogue", 4096, 512, 4096, True, {"TB_TILE": "128x128"}),
]


def main(reps: int) -> None:
    g = torch.Generator(device="cuda")
    out = {}
    for name, m, k, n, acc, env in CASES:
        for key in ("TB_TILE", "TB_SPLIT"):
            os.environ.pop(key, None)
        os.environ.update(env)
        worst = 0.0
        for r in range(reps):
            g.manual_seed(1000 * r + m + k + n)
            a = torch.rand((m, k), dtype=torch.float64, device="cuda", generator=g) + 2.0
            b = torch.rand((k, n), dtype=torch.float64, device="cuda", generator=g) + 2.0
            ref = a @ b
            if acc:
                c = torch.rand((m, n), dtype=torch.float64, device="cuda", generator=g)
                ref = ref + c
                tb.dgemm_launch(a, b, c, accumulate=True)
                torch.cuda.synchronize()
            else:
                c, _ = tb.dgemm(a, b)
            err = (torch.linalg.norm(c - ref) / torch.linalg.norm(ref)).item()
            worst = max(worst, err if err == err else float("inf"))
        out[name] = worst
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
