"""Per-CTA timeline of the host pipeline's flag-driven phase-1 (PIPE) launch
(tooling): with the instrumented build, every host-buffer call prints a
TBPIPE line (span, CTA end skew, producer flag-wait time incl. the first
panel, epilogue time per CTA).

    python -m paper_2509_04594_b200.build --timeline
    TB_LIB_VARIANT=timeline TB_TIMELINE=1 python tools/pipe_timeline.py 10000
"""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2509_04594_b200 as tb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
g = torch.Generator().manual_seed(1)
a = (torch.rand((n, n), dtype=torch.float64, generator=g) * 3 + 2).pin_memory()
b = (torch.rand((n, n), dtype=torch.float64, generator=g) * 3 + 2).pin_memory()
c = torch.empty((n, n), dtype=torch.float64).pin_memory()
s, e = np.zeros(1), np.zeros(1)
for i in range(3):
    assert tb.gpu_tiled_multiply_flat(0, a, b, n, n, n, 32, c, s, out_e2e_seconds=e) == 0
    print("E2E", e[0] * 1e3, s[0] * 1e3, file=sys.stderr, flush=True)
