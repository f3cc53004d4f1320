"""Randomised stress (tooling): many random shapes / strides / variants /
buffer kinds through tb_dgemm, tb_dgemm_launch (accumulate, strided views)
and the host-buffer entry, each compared with cuBLAS on the same operands.
    python tools/fuzz.py [cases] [seed]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_04594_b200 as tb  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
worst = 0.0
for i in range(cases):
    big = rng.random() < 0.25
    hi = 6000 if big else 700
    m, k, n = (int(rng.integers(1, hi)) for _ in range(3))
    if rng.random() < 0.5:  # even leading dimensions: TMA-addressable, through the tile-shape chooser
        k, n = k + k % 2, n + n % 2
    mode = rng.choice(["dgemm", "launch_acc", "view", "flat_pinned", "flat_pageable"])
    variant = rng.choice(["auto", "auto", "dmma_tma", "dmma_cpasync", "dfma"]) if mode != "flat_pageable" else "auto"
    a = torch.from_numpy(rng.random((m, k)) * 3 + 2)
    b = torch.from_numpy(rng.random((k, n)) * 3 + 2)
    ref, _ = tb.cublas_dgemm(a.cuda(), b.cuda())
    if mode == "dgemm":
        got, _ = tb.dgemm(a.cuda(), b.cuda(), variant=variant)
    elif mode == "launch_acc":
        got = ref.clone()
        tb.dgemm_launch(a.cuda(), b.cuda(), got, accumulate=True, variant=variant)
        ref = 2 * ref
    elif mode == "view":
        pa, pb = int(rng.integers(0, 3)), int(rng.integers(0, 3))
        A = torch.zeros((m, k + pa), dtype=torch.float64, device="cuda")
        B = torch.zeros((k, n + pb), dtype=torch.float64, device="cuda")
        A[:, pa:] = a.cuda()
        B[:, pb:] = b.cuda()
        got = torch.empty((m, n), dtype=torch.float64, device="cuda")
        tb.dgemm_launch(A[:, pa:], B[:, pb:], got, variant=variant)
    else:
        pin = mode == "flat_pinned"
        ah = a.pin_memory() if pin else a.numpy()
        bh = b.pin_memory() if pin else b.numpy()
        c = torch.empty((m, n), dtype=torch.float64).pin_memory() if pin else np.empty(m * n)
        st = tb.gpu_tiled_multiply_flat(0, ah, bh, m, k, n, 32, c, np.zeros(1), variant=variant)
        assert st == 0, (st, tb._lib.last_error())
        got = torch.as_tensor(np.asarray(c).reshape(m, n)).cuda()
    torch.cuda.synchronize()
    rel = (torch.linalg.norm(got - ref) / torch.linalg.norm(ref)).item()
    worst = max(worst, rel)
    status = "ok" if rel <= 1e-12 else "FAIL"
    print(f"{i:4d} {mode:14s} {variant:13s} {m}x{k}x{n} normwise {rel:.2e} {status}", flush=True)
    assert rel <= 1e-12
print("all ok, worst", worst)
