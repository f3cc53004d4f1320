"""Time the host-buffer pipeline (tb_gpu_tiled_multiply_flat_ex) for several
TB_PIPE=R,P,Q shapes in subprocesses (tooling)."""
import json
import os
import subprocess
import sys

CODE = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2509_04594_b200 as tb
n = int(sys.argv[1])
g = torch.Generator().manual_seed(1)
a = (torch.rand((n, n), dtype=torch.float64, generator=g) * 3 + 2).pin_memory()
b = (torch.rand((n, n), dtype=torch.float64, generator=g) * 3 + 2).pin_memory()
c = torch.empty((n, n), dtype=torch.float64).pin_memory()
s, e = np.zeros(1), np.zeros(1)
best = 1e9
for i in range(4):
    assert tb.gpu_tiled_multiply_flat(0, a, b, n, n, n, 32, c, s, out_e2e_seconds=e) == 0
    if i: best = min(best, e[0])
print(best, s[0])
'''
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
shapes = sys.argv[2:] or ["default", "8,8,2", "8,8,3", "8,16,2", "16,8,4", "8,4,2", "4,8,1", "16,16,4"]
for sh in shapes:
    env = dict(os.environ)
    if sh != "default":
        env["TB_PIPE"] = sh
    out = subprocess.run([sys.executable, "-c", CODE, str(n)], env=env, capture_output=True, text=True)
    try:
        e2e, ks = map(float, out.stdout.split())
        print(json.dumps({"pipe": sh, "n": n, "e2e_ms": e2e * 1e3, "kernel_ms": ks * 1e3,
                          "e2e_tflops": (2 * n**3 - n**2) / e2e / 1e12}))
    except ValueError:
        print(sh, out.stdout[-300:], out.stderr[-500:])
