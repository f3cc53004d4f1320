"""Per-CTA phase timing of the persistent DMMA kernel (tooling): runs the
instrumented build (libtbgpu_timeline.so, -DTB_TIMELINE) on given shapes and
prints the TBTIMELINE summary lines (startup to first stage, main loop, stream-K
fixup, epilogue, end skew across CTAs).

    python -m paper_2509_04594_b200.build --timeline
    TB_LIB_VARIANT=timeline TB_TIMELINE=1 python tools/kernel_timeline.py 1000x1000x1000 ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2509_04594_b200 as tb  # noqa: E402

for spec in sys.argv[1:]:
    m, k, n = map(int, spec.split("x"))
    A = torch.rand((m, k), dtype=torch.float64, device="cuda")
    B = torch.rand((k, n), dtype=torch.float64, device="cuda")
    C = torch.empty((m, n), dtype=torch.float64, device="cuda")
    for _ in range(3):
        tb.dgemm(A, B, C)
    torch.cuda.synchronize()
    print(spec, "done", flush=True)
