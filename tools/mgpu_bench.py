"""Time tb_dgemm_mgpu (single-process row-sharded GEMM, B forwarded down the
device chain in K-panels) on the visible GPUs (tooling).

    python tools/mgpu_bench.py N ENTRIES [reps]

ENTRIES device entries are assigned round-robin to the visible GPUs (with
one GPU they all share it: a panel-plan overhead check, not a scaling
number). Prints kernel-max / total seconds and TFLOP/s, plus tb.dgemm on the
whole product on GPU 0 for comparison.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2509_04594_b200 as tb  # noqa: E402
from paper_2509_04594_b200 import multigpu as mg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
entries = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
ng = torch.cuda.device_count()
devs = [torch.device("cuda", i % ng) for i in range(entries)]
parts = mg.row_partitions(n, entries)
g = torch.Generator(device="cuda:0").manual_seed(1)
a = torch.rand((n, n), dtype=torch.float64, device="cuda:0", generator=g) * 3 + 2
b = torch.rand((n, n), dtype=torch.float64, device="cuda:0", generator=g) * 3 + 2
a_rows = [a[r0:r1].to(d) for (r0, r1), d in zip(parts, devs)]
c_rows = [torch.empty((r1 - r0, n), dtype=torch.float64, device=d) for (r0, r1), d in zip(parts, devs)]
reps_b = [None] + [torch.empty_like(b, device=d) for d in devs[1:]]
flops = 2 * n**3 - n**2
res = []
for i in range(reps + 1):
    km, tot = mg.peer_sharded_dgemm(a_rows, b, c_rows, reps_b)
    if i:
        res.append((km, tot))
km = sorted(r[0] for r in res)[len(res) // 2]
tot = sorted(r[1] for r in res)[len(res) // 2]
c = torch.empty((n, n), dtype=torch.float64, device="cuda:0")
ks = []
for i in range(reps + 1):
    _, s = tb.dgemm(a, b, c)
    if i:
        ks.append(s)
k1 = sorted(ks)[len(ks) // 2]
err = max(((torch.cat([x.to("cuda:0") for x in c_rows]) - c).norm() / c.norm()).item(), 0.0)
print(json.dumps({"n": n, "entries": entries, "gpus": ng, "kernel_max_ms": km * 1e3, "total_ms": tot * 1e3,
                  "tflops_total": flops / tot / 1e12, "single_dgemm_ms": k1 * 1e3,
                  "single_tflops": flops / k1 / 1e12, "normwise_vs_single": err,
                  "panels": os.environ.get("TB_MGPU_PANEL", "1024")}))
