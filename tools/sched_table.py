"""Tabulate tools/sched_ab.sh output: best-of-reps TFLOP/s per shape and mode (tooling)."""
import json
import sys
from collections import defaultdict

r = defaultdict(list)
modes = []
for line in open(sys.argv[1]):
    m, j = line.split(" ", 1)
    try:
        d = json.loads(j)
    except ValueError:
        continue
    if m not in modes:
        modes.append(m)
    r[(d["shape"], m)].append(d["tflops"])
    r[(d["shape"], "cublas")].append(d["cublas_tflops"])
for sh in sorted({k[0] for k in r}, key=lambda x: int(x.split("x")[0])):
    print(sh, {m: round(max(r[(sh, m)]), 2) for m in modes + ["cublas"] if r[(sh, m)]})
