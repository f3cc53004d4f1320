"""Wall time of the host-buffer entry points at N on pageable (numpy) vs
pinned buffers, and of the MultiplyFn (tooling)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_04594_b200 as tb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
rng = np.random.default_rng(1)
a = rng.random((n, n)) * 3 + 2
b = rng.random((n, n)) * 3 + 2
f = 2 * n**3 - n**2


def best(fn, reps=3):
    ts = []
    for _ in range(reps + 1):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts[1:])


c = np.empty(n * n)
s = np.zeros(1)
t = best(lambda: tb.gpu_tiled_multiply_flat(0, a, b, n, n, n, 32, c, s))
print(f"flat pageable      {t*1e3:8.1f} ms {f/t/1e12:6.2f} TFLOP/s")
ap, bp = torch.from_numpy(a).pin_memory(), torch.from_numpy(b).pin_memory()
cp = torch.empty((n, n), dtype=torch.float64).pin_memory()
t = best(lambda: tb.gpu_tiled_multiply_flat(0, ap, bp, n, n, n, 32, cp, s))
print(f"flat pinned        {t*1e3:8.1f} ms {f/t/1e12:6.2f} TFLOP/s")
t = best(lambda: tb.gpu_tiled_multiply(a, b), reps=2)
print(f"MultiplyFn (numpy) {t*1e3:8.1f} ms {f/t/1e12:6.2f} TFLOP/s")
held = []


def fn_held():  # a harness keeps the previous product while making the next one
    held.append(tb.gpu_tiled_multiply(a, b))
    del held[:-1]


t = best(fn_held, reps=3)
print(f"MultiplyFn, previous output held {t*1e3:8.1f} ms {f/t/1e12:6.2f} TFLOP/s")

# output page-fault cost: the MultiplyFn allocates a fresh output per call
import ctypes  # noqa: E402
libc = ctypes.CDLL("libc.so.6")


def fn_thp():
    out = np.empty((n, n))
    addr = out.ctypes.data
    page = 2 << 20
    start = (addr + page - 1) // page * page
    libc.madvise(ctypes.c_void_p(start), ctypes.c_size_t(out.nbytes - (start - addr)), 14)  # MADV_HUGEPAGE
    tb.gpu_tiled_multiply_flat(0, a, b, n, n, n, 32, out, s)
    return out


t = best(fn_thp, reps=2)
print(f"flat pageable, fresh THP output {t*1e3:8.1f} ms {f/t/1e12:6.2f} TFLOP/s")


def fn_fresh():
    out = np.empty((n, n))
    tb.gpu_tiled_multiply_flat(0, a, b, n, n, n, 32, out, s)


t = best(fn_fresh, reps=2)
print(f"flat pageable, fresh output     {t*1e3:8.1f} ms {f/t/1e12:6.2f} TFLOP/s")
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
