"""Time the host-buffer pipeline (tb_gpu_tiled_multiply_flat_ex) under
several environment settings, each in its own subprocess, interleaved over
rounds (tooling).

    python tools/pipe_tune.py N ROUNDS spec ...
    spec = default | VAR=value[;VAR=value]      e.g. TB_TAIL=128,384,768
    TRACE_PAGEABLE=1 (as a spec or in the environment): numpy A and B; =2: numpy C too
"""
import json
import os
import statistics
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
import os
if os.environ.get("TRACE_PAGEABLE") in ("1", "2"):  # numpy A, B (staged), pinned C: the MultiplyFn's case
    a, b = a.numpy().copy(), b.numpy().copy()
if os.environ.get("TRACE_PAGEABLE") == "2":  # numpy C too (the ctypes binding of INTEGRATION.md §1)
    c = np.empty((n, n))
s, e = np.zeros(1), np.zeros(1)
es, ks = [], []
for i in range(9):
    assert tb.gpu_tiled_multiply_flat(0, a, b, n, n, n, 32, c, s, out_e2e_seconds=e) == 0
    if i: es.append(e[0]); ks.append(s[0])
es.sort(); ks.sort()
print(es[len(es) // 2], es[0], ks[len(ks) // 2])
'''
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 1
specs = sys.argv[3:] or ["default"]
res = {sp: [] for sp in specs}
for rd in range(rounds):
    for sp in specs:
        env = dict(os.environ)
        if sp != "default":
            for kv in sp.split(";"):
                k, v = kv.split("=", 1)
                env[k] = v
        out = subprocess.run([sys.executable, "-c", CODE, str(n)], env=env, capture_output=True, text=True)
        try:
            med, best, kmed = map(float, out.stdout.split())
        except ValueError:
            print(sp, out.stdout[-300:], out.stderr[-500:], flush=True)
            continue
        res[sp].append(med)
        print(json.dumps({"spec": sp, "round": rd, "n": n, "e2e_ms_median": med * 1e3, "e2e_ms_best": best * 1e3,
                          "kernel_ms": kmed * 1e3}), flush=True)
for sp, v in res.items():
    if v:
        m = statistics.median(v)
        print(f"{sp:40s} median-of-rounds {m * 1e3:8.3f} ms  {(2 * n**3 - n**2) / m / 1e12:6.2f} TFLOP/s")
