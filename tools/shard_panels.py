"""Per-rank compute of the row-sharded multi-GPU driver on one GPU (tooling):
the shard GEMM C_loc = A_loc · B as one launch vs as the K-panel launches
ShardedGemm issues (geometric panels; the earlier ramped even split), i.e.
the cost of splitting K so the broadcast can overlap.

    python tools/shard_panels.py [N ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2509_04594_b200 as tb  # noqa: E402
from paper_2509_04594_b200.multigpu import geometric_panel_bounds, ramp_panel_bounds, row_partitions  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


for n in [int(x) for x in sys.argv[1:]] or [10000, 32768]:
    g = torch.Generator(device="cuda").manual_seed(1)
    b = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g)
    for world in (2, 4, 8):
        r0, r1 = row_partitions(n, world)[0]
        a = torch.rand((r1 - r0, n), dtype=torch.float64, device="cuda", generator=g)
        c = torch.empty((r1 - r0, n), dtype=torch.float64, device="cuda")
        flops = 2.0 * (r1 - r0) * n * n
        res = {"n": n, "world": world, "rows": r1 - r0}

        def panels(bounds):
            def run():
                for i, (k0, k1) in enumerate(bounds):
                    tb.dgemm_launch(a[:, k0:k1], b[k0:k1], c, accumulate=i > 0)
            return run

        for name, fn in (("single", lambda: tb.dgemm_launch(a, b, c)),
                         ("geometric", panels(geometric_panel_bounds(n))),
                         ("ramp4", panels(ramp_panel_bounds(n, 4)))):
            ms = timed(fn)
            res[name + "_ms"] = round(ms, 3)
            res[name + "_tflops"] = round(flops / ms / 1e9, 2)
        print(json.dumps(res), flush=True)
        del a, c
