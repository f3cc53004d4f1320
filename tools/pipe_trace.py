"""Timeline of the host-buffer pipeline (tb_gpu_tiled_multiply_flat_ex) with
TB_PIPE_TRACE=1 (tooling): per shape, the device intervals of every H2D / GEMM
cell / D2H, the compute-idle gaps, and bare pinned-copy bandwidths.

    python tools/pipe_trace.py [N] [shape ...]      shape = default | R,P,Q
    TRACE_PAGEABLE=1: pageable (numpy) A and B, pinned C
"""
import json
import os
import subprocess
import sys

CODE = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2509_04594_b200 as tb
n = int(sys.argv[1])
g = torch.Generator().manual_seed(1)
a = (torch.rand((n, n), dtype=torch.float64, generator=g) * 3 + 2).pin_memory()
b = (torch.rand((n, n), dtype=torch.float64, generator=g) * 3 + 2).pin_memory()
c = torch.empty((n, n), dtype=torch.float64).pin_memory()
import os
if os.environ.get("TRACE_PAGEABLE") == "1":  # numpy A, B (staged), pinned C: the MultiplyFn's case
    a, b = a.numpy().copy(), b.numpy().copy()
s, e = np.zeros(1), np.zeros(1)
for i in range(3):
    print("CALL", i, file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    assert tb.gpu_tiled_multiply_flat(0, a, b, n, n, n, 32, c, s, out_e2e_seconds=e) == 0
    wall = time.perf_counter() - t0
    print("E2E", i, e[0] * 1e3, wall * 1e3, file=sys.stderr, flush=True)
'''

BW = r'''
import torch
x = torch.empty(200_000_000 // 8, dtype=torch.float64).pin_memory()
d = torch.empty_like(x, device="cuda")
out = {}
for name, fn in (("h2d", lambda: d.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record(); torch.cuda.synchronize()
    out[name] = 5 * x.numel() * 8 / (e0.elapsed_time(e1) / 1e3) / 1e9
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty_like(d); x2 = torch.empty_like(x).pin_memory()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    with torch.cuda.stream(s1):
        d.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        x2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
e1.record(); torch.cuda.synchronize()
out["duplex_each"] = 5 * x.numel() * 8 / (e0.elapsed_time(e1) / 1e3) / 1e9
print("BW", json.dumps(out))
'''


def analyse(lines, call):
    recs = []
    cur = None
    for ln in lines:
        p = ln.split()
        if p[0] == "CALL":
            cur = int(p[1])
        elif p[0] == "TBTRACE" and cur == call:
            recs.append((p[1], int(p[2]), float(p[3]), float(p[4]), float(p[5])))
    gem = sorted([r for r in recs if r[0] == "gemm"], key=lambda r: r[2])
    busy, last, gaps = 0.0, 0.0, []
    for r in gem:  # union of GEMM intervals
        if r[2] > last:
            gaps.append((round(last, 3), round(r[2], 3)))
            busy += r[3] - r[2]
            last = r[3]
        elif r[3] > last:
            busy += r[3] - last
            last = r[3]
    end = max(r[3] for r in recs)
    return recs, {"end_ms": end, "compute_busy_ms": busy, "idle_ms": end - busy,
                  "first_gemm_ms": gem[0][2], "last_gemm_end_ms": last, "gaps": gaps}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
    shapes = sys.argv[2:] or ["default"]
    bw = subprocess.run([sys.executable, "-c", "import json\n" + BW], capture_output=True, text=True)
    print(bw.stdout.strip(), bw.stderr[-300:])
    for sh in shapes:
        env = dict(os.environ, TB_PIPE_TRACE="1")
        if sh != "default":
            env["TB_PIPE"] = sh
        out = subprocess.run([sys.executable, "-c", CODE, str(n)], env=env, capture_output=True, text=True)
        lines = [ln for ln in out.stderr.splitlines() if ln.split() and ln.split()[0] in ("CALL", "TBTRACE", "E2E", "TBHOST")]
        e2e = [float(ln.split()[2]) for ln in lines if ln.startswith("E2E")]
        wall = [float(ln.split()[3]) for ln in lines if ln.startswith("E2E")]
        if not e2e:
            print(sh, out.stderr[-800:])
            continue
        recs, summ = analyse(lines, 2)
        summ["host"] = [ln for ln in lines if ln.startswith("TBHOST")][-1:]
        print(json.dumps({"pipe": sh, "n": n, "e2e_ms": e2e, "wall_ms": wall, **summ}))
        for r in sorted(recs, key=lambda r: r[2]):
            gbs = r[4] / ((r[3] - r[2]) * 1e-3) / 1e9 if r[4] else 0.0
            print(f"  {r[0]:6s} {r[1]:3d} {r[2]:9.3f} {r[3]:9.3f} {r[3] - r[2]:8.3f} ms" +
                  (f"  {gbs:6.1f} GB/s" if gbs else ""))


if __name__ == "__main__":
    main()
