"""GPU parity of the sm_100a kernels against the CPU oracle and the
reference-generated golden fixtures (run on a B200: pytest -m gpu).

Mirrors the reference's kernel suite (pkg/gpu/tests/kernel.test.ts:21-182)
and the backend pins (pkg/tests/test_backends.py:23-71,
test_acceptance.py:57-73). Bars (BASELINE.json north_star):
  normwise ||C_gpu - C_ref||_F / ||C_ref||_F <= 1e-12,
  max_abs_rel_diff <= 1e-10 (harness.py:41 ORACLE_RTOL),
  and BITWISE equality with the reference naive oracle for the paper variant
  (no FMA contraction, k-order running sum; kernel.ts:50-78).
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NORMWISE = 1e-12
ELEMWISE = 1e-10
FAST = ["dmma_tma", "dmma_cpasync", "dfma"]


@pytest.fixture(scope="module")
def tb():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (run with -m 'not gpu' on CPU)")
    import paper_2509_04594_b200 as tb

    assert tb._lib.device_count() >= 1
    return tb


def _gen(o, m, k, n, sa, sb):
    return o.generate(m, k, sa), o.generate(k, n, sb)


def _gpu(tb, a, b, variant, tile=32):
    out, sec = tb.gpu_tiled_multiply_timed(a, b, tb.TileConfig(tile), variant=variant)
    assert sec > 0.0
    return out


def test_one_by_one_is_twelve(tb):
    for v in ["auto", "paper"] + FAST:
        out = _gpu(tb, np.array([[3.0]]), np.array([[4.0]]), v)
        assert out.shape == (1, 1) and out[0, 0] == 12.0


def test_hand_checked_two_by_two(tb):
    a = np.array([[1.0, 2.0], [3.0, 4.0]])
    b = np.array([[5.0, 6.0], [7.0, 8.0]])
    for v in ["paper"] + FAST:
        assert np.array_equal(_gpu(tb, a, b, v), [[19.0, 22.0], [43.0, 50.0]])


@pytest.mark.parametrize("variant", ["paper"] + FAST)
def test_golden_grid(tb, golden, oracle, variant):
    meta, g = golden
    for c in meta["cases"]:
        a, b = _gen(oracle, c["m"], c["k"], c["n"], c["seed_a"], c["seed_b"])
        naive = g[c["tag"] + "_naive"]
        tiles = c["tiles"] if variant == "paper" else [32]
        for t in tiles:
            if t * t > 1024:
                continue
            got = _gpu(tb, a, b, variant, t)
            if variant == "paper":
                assert np.array_equal(got, naive), (c["tag"], t)
            assert tb.max_abs_rel_diff(got, naive) <= ELEMWISE, (c["tag"], variant, t)
            assert oracle.normwise_rel(got, naive) <= NORMWISE, (c["tag"], variant, t)
            assert oracle.normwise_rel(got, g[c["tag"] + "_tiled32"]) <= NORMWISE


@pytest.mark.parametrize("variant", ["paper"] + FAST)
def test_identity_with_hanging_column_is_bitwise(tb, oracle, variant):
    n = 33
    b = oracle.generate(n, n, 11)
    assert np.array_equal(_gpu(tb, np.eye(n), b, variant), b)


@pytest.mark.parametrize("variant", FAST)
def test_zero_fill_border_row(tb, oracle, variant):
    n = 33
    a, b = _gen(oracle, n, n, n, 9, 10)
    got = _gpu(tb, a, b, variant)
    want = oracle.naive(a, b)
    assert oracle.max_abs_rel_diff(got[n - 1], want[n - 1]) <= 1e-12
    assert oracle.max_abs_rel_diff(got[:, n - 1], want[:, n - 1]) <= 1e-12


@pytest.mark.parametrize("m,k,n", [(1, 1000, 1), (130, 17, 257), (255, 129, 127), (128, 16, 128), (7, 3, 300)])
@pytest.mark.parametrize("variant", FAST)
def test_ragged_shapes(tb, oracle, m, k, n, variant):
    a, b = _gen(oracle, m, k, n, m + 1, n + 2)
    got = _gpu(tb, a, b, variant)
    ref = oracle.tiled_parallel(a, b)
    assert oracle.normwise_rel(got, ref) <= NORMWISE
    assert oracle.max_abs_rel_diff(got, ref) <= ELEMWISE


def test_config0_n1000_full(tb, golden, oracle):
    """configs[0]: N = 1000, seeds (1, 2): GPU vs the reference's tiled CPU
    result (oracle reproduces its SHA-256, test_oracle.py)."""
    meta, g = golden
    a, b = oracle.generate(1000, 1000, 1), oracle.generate(1000, 1000, 2)
    ref = oracle.tiled_parallel(a, b)
    for v in ["auto"] + FAST:
        got = _gpu(tb, a, b, v)
        assert oracle.normwise_rel(got, ref) <= NORMWISE
        assert oracle.max_abs_rel_diff(got, ref) <= ELEMWISE
        rows = g["n1000_rows"]
        assert oracle.normwise_rel(got[rows], g["n1000_tiled32_rows"]) <= NORMWISE


@pytest.mark.parametrize("n", [4000, 10000])
def test_large_row_sampled(tb, golden, oracle, n):
    """configs[1] / [3] sizes: rows of the GPU product vs the reference's
    tiled result on the same rows (bitwise equal to the full CPU product's
    rows), plus a full-matrix check against cuBLAS."""
    import torch

    meta, g = golden
    a, b = oracle.generate(n, n, 1), oracle.generate(n, n, 2)
    ta, tb_ = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    c, sec = tb.dgemm(ta, tb_)
    rows = g[f"n{n}_rows"]
    got_rows = c[torch.from_numpy(rows).cuda()].cpu().numpy()
    assert oracle.normwise_rel(got_rows, g[f"n{n}_tiled32_rows"]) <= NORMWISE
    assert oracle.max_abs_rel_diff(got_rows, g[f"n{n}_tiled32_rows"]) <= ELEMWISE
    ref, _ = tb.cublas_dgemm(ta, tb_)
    rel = (torch.linalg.norm(c - ref) / torch.linalg.norm(ref)).item()
    assert rel <= NORMWISE


def test_full_size_checksums(tb, oracle):
    """Every element of a full-size product, in aggregate (algorithm-based
    fault tolerance): column sums e^T C = (e^T A) B and row sums C e =
    A (B e), the right-hand sides computed on the host (numpy, O(N^2)), for
    the device entry and the host-buffer pipeline at N = 10000 (configs[3]).
    A missing, doubled or misplaced tile, panel or strip moves a checksum by
    ~1e-4 relative; rounding moves it by ~1e-16."""
    import torch

    n = 10000
    a, b = oracle.generate(n, n, 11), oracle.generate(n, n, 12)
    col_ref, row_ref = a.sum(axis=0) @ b, a @ b.sum(axis=1)
    c, _ = tb.dgemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    for name, cc in (("device", c.cpu().numpy()), ("host", None)):
        if cc is None:
            cc = np.empty((n, n))
            sec = np.zeros(1)
            assert tb.gpu_tiled_multiply_flat(0, a, b, n, n, n, 32, cc, sec) == 0
        assert oracle.normwise_rel(cc.sum(axis=0), col_ref) <= NORMWISE, name
        assert oracle.normwise_rel(cc.sum(axis=1), row_ref) <= NORMWISE, name


def test_n32768_checksums(tb):
    """configs[4] size on one GPU: full-matrix column / row checksums of the
    N = 32768 product (8.6 GB per matrix) against fp64 matrix-vector products
    of the operands (cuBLAS DGEMV on the device; O(N^2))."""
    import torch

    n = 32768
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g) * 3 + 2
    b = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g) * 3 + 2
    c, _ = tb.dgemm(a, b)
    col = c.sum(0)
    row = c.sum(1)
    del c
    col_ref = a.sum(0) @ b
    row_ref = a @ b.sum(1)
    assert (torch.linalg.norm(col - col_ref) / torch.linalg.norm(col_ref)).item() <= NORMWISE
    assert (torch.linalg.norm(row - row_ref) / torch.linalg.norm(row_ref)).item() <= NORMWISE


def test_deterministic_bits(tb, oracle):
    a, b = _gen(oracle, 515, 515, 515, 3, 4)
    for v in FAST + ["paper"]:
        one, two = _gpu(tb, a, b, v), _gpu(tb, a, b, v)
        assert one.tobytes() == two.tobytes()


def test_inputs_not_mutated(tb, oracle):
    a, b = _gen(oracle, 64, 64, 64, 5, 6)
    a0, b0 = a.copy(), b.copy()
    tb.gpu_tiled_multiply(a, b)
    assert np.array_equal(a, a0) and np.array_equal(b, b0)


def test_variant_resolution(tb):
    import torch

    lib = tb._lib.lib()
    x = torch.empty(64, dtype=torch.float64, device="cuda")
    p = x.data_ptr()
    assert lib.tb_resolve_variant(ctypes.c_void_p(p), 10, ctypes.c_void_p(p), 10, 0) == tb._lib.VARIANT_DMMA_TMA
    assert lib.tb_resolve_variant(ctypes.c_void_p(p), 11, ctypes.c_void_p(p), 10, 0) == tb._lib.VARIANT_DMMA_CPASYNC
    assert lib.tb_resolve_variant(ctypes.c_void_p(p + 8), 10, ctypes.c_void_p(p), 10, 0) == tb._lib.VARIANT_DMMA_CPASYNC
    assert lib.tb_resolve_variant(ctypes.c_void_p(p), 10, ctypes.c_void_p(p), 10, 1) == tb._lib.VARIANT_PAPER


def test_launch_accumulate_and_strided_panels(tb, oracle):
    """tb_dgemm_launch: column-panel views of A (lda = k), row-panel views of
    B, C += A·B — the multi-GPU K-panel step."""
    import torch

    m, k, n = 300, 258, 190
    a, b = _gen(oracle, m, k, n, 21, 22)
    ta, tb_ = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    out = torch.zeros((m, n), dtype=torch.float64, device="cuda")
    for i, (k0, k1) in enumerate([(0, 100), (100, 202), (202, 258)]):
        tb.dgemm_launch(ta[:, k0:k1], tb_[k0:k1], out, accumulate=i > 0)
    torch.cuda.synchronize()
    ref = oracle.tiled_parallel(a, b)
    assert oracle.normwise_rel(out.cpu().numpy(), ref) <= NORMWISE
    # odd panel boundary -> unaligned base -> cp.async path
    out.zero_()
    for i, (k0, k1) in enumerate([(0, 101), (101, 258)]):
        tb.dgemm_launch(ta[:, k0:k1], tb_[k0:k1], out, accumulate=i > 0)
    torch.cuda.synchronize()
    assert oracle.normwise_rel(out.cpu().numpy(), ref) <= NORMWISE


def test_flat_abi_status_codes(tb, oracle):
    """kernel.test.ts:123-182: OK / NO_DEVICE / OVER_LIMITS / BAD_DIMS."""
    n = 16
    a, b = _gen(oracle, n, n, n, 12, 13)
    out_c = np.zeros(n * n)
    out_s = np.zeros(1)
    assert tb.gpu_tiled_multiply_flat(0, a, b, n, n, n, 16, out_c, out_s) == tb.STATUS_OK
    assert out_s[0] > 0
    assert oracle.max_abs_rel_diff(out_c.reshape(n, n), oracle.naive(a, b)) <= ELEMWISE
    assert tb.gpu_tiled_multiply_flat(None, a, b, n, n, n, 32, out_c, out_s) == tb.STATUS_NO_DEVICE
    assert tb.gpu_tiled_multiply_flat(4096, a, b, n, n, n, 32, out_c, out_s) == tb.STATUS_NO_DEVICE
    assert tb.gpu_tiled_multiply_flat(0, a, b, n, n, n, 64, out_c, out_s) == tb.STATUS_OVER_LIMITS
    assert tb.gpu_tiled_multiply_flat(0, a, b, n, n, n, 4, np.zeros(3), out_s) == tb.STATUS_BAD_DIMS
    assert tb.gpu_tiled_multiply_flat(0, a, b, n, n, n, 0, out_c, out_s) == tb.STATUS_BAD_DIMS
    assert tb.gpu_tiled_multiply_flat(0, a, b, 0, n, n, 32, out_c, out_s) == tb.STATUS_BAD_DIMS
    # executor.ts:86 / multiply.ts:71-73: buffers must match the dims; the
    # flat ABI reads dense row-major host memory only.
    import torch

    assert tb.gpu_tiled_multiply_flat(0, a[:-1], b, n, n, n, 32, out_c, out_s) == tb.STATUS_BAD_DIMS
    assert tb.gpu_tiled_multiply_flat(0, a, b[:, :-1], n, n, n, 32, out_c, out_s) == tb.STATUS_BAD_DIMS
    assert tb.gpu_tiled_multiply_flat(0, a.T, b, n, n, n, 32, out_c, out_s) == tb.STATUS_BAD_DIMS
    assert tb.gpu_tiled_multiply_flat(0, a.astype(np.float32), b, n, n, n, 32, out_c, out_s) == tb.STATUS_BAD_DIMS
    assert tb.gpu_tiled_multiply_flat(0, torch.from_numpy(a).cuda(), b, n, n, n, 32, out_c,
                                      out_s) == tb.STATUS_BAD_DIMS
    assert tb.gpu_tiled_multiply_flat(0, torch.from_numpy(a), torch.from_numpy(b), n, n, n, 32,
                                      torch.from_numpy(out_c), out_s) == tb.STATUS_OK
    for v in ("paper", "dmma_tma", "dmma_cpasync", "dfma"):
        out_c[:] = 0
        e2e = np.zeros(1)
        assert tb.gpu_tiled_multiply_flat(0, a, b, n, n, n, 16, out_c, out_s, variant=v,
                                          out_e2e_seconds=e2e) == tb.STATUS_OK
        assert e2e[0] >= out_s[0] > 0
        assert oracle.normwise_rel(out_c.reshape(n, n), oracle.naive(a, b)) <= NORMWISE


def test_exceptions_map_to_reference_kinds(tb, oracle):
    a, b = _gen(oracle, 4, 4, 4, 1, 2)
    with pytest.raises(tb.InvalidConfigError):
        tb.gpu_tiled_multiply(a, b, tb.TileConfig(64), variant="paper")
    with pytest.raises(tb.ShapeError):
        tb.gpu_tiled_multiply(np.ones((2, 3)), np.ones((2, 3)))


def test_registry_and_device_timed_runner(tb, oracle, tmp_path):
    reg = tb.BackendRegistry()
    assert reg.names() == [tb.GPU_BACKEND_NAME, tb.PAPER_BACKEND_NAME, tb.CUBLAS_BACKEND_NAME]
    cfg = tb.RunConfig(backends=(tb.GPU_BACKEND_NAME, tb.CUBLAS_BACKEND_NAME), sizes=(64, 129), trials=3,
                       verify=True)
    records, meta = tb.run_trials(cfg, reg, verifier=oracle.naive)
    assert len(records) == 2 * 2 * 3
    for r in records:
        assert r.seconds > 0 and abs(r.flops - tb.flop_count(r.n) / r.seconds) <= 1e-12 * r.flops
    path = tmp_path / "gpu.csv"
    tb.write_records(path, records, meta)
    lines = path.read_text().splitlines()
    assert lines[0] == "backend,n,trial,seconds,flops" and len(lines) == 13
    # host<->device copies timed separately, reported as metadata
    import json

    tr = json.loads((tmp_path / "gpu.csv.meta.json").read_text())["config"]["transfers"]
    for name in (tb.GPU_BACKEND_NAME, tb.CUBLAS_BACKEND_NAME):
        cell = tr[name]["129"]
        assert cell["trials"] == 3
        assert cell["h2d_bytes"] == 2 * 8 * 129 * 129 and cell["d2h_bytes"] == 8 * 129 * 129
        assert cell["h2d_seconds_median"] > 0 and cell["d2h_seconds_median"] > 0
    # run metadata (harness.py:126-142 + SURVEY.md §5): versions, loaded cuBLAS, pinned math mode, GPU, plan
    cfg_meta = json.loads((tmp_path / "gpu.csv.meta.json").read_text())["config"]
    gpu = cfg_meta["gpu"]
    for key in ("cublas_version", "cublas_path", "cuda_runtime_version", "cuda_driver_version", "gpu_name",
                "sm_count", "sm_clock_max_khz", "compute_capability"):
        assert gpu.get(key), key
    assert gpu["cublas_math_mode"] == 0 and gpu["cublas_math_mode_name"] == "CUBLAS_DEFAULT_MATH"
    assert gpu["compute_capability"] == 100 and gpu["sm_count"] >= 100
    assert cfg_meta["nccl_version"] and cfg_meta["torch"]
    assert cfg_meta["clocks_at_start"]["sm_max_mhz"]
    plan = cfg_meta["launch_plans"]["129"]
    assert plan and all(p["kernel"] == "dmma" for p in plan if "kernel" in p)


def test_liar_backend_caught_by_verify(tb, oracle):
    reg = tb.BackendRegistry()
    reg.register_external(tb.BackendDescriptor("liar"), lambda a, b: tb.gpu_tiled_multiply(a, b) + 1.0)
    cfg = tb.RunConfig(backends=("liar",), sizes=(16,), trials=1, verify=True)
    with pytest.raises(tb.TrialError):
        tb.run_trials(cfg, reg, verifier=oracle.naive)


def test_sharded_gemm_single_rank_nccl_panels(tb, oracle):
    """The multi-GPU driver on one rank over NCCL: K-panel broadcast + panel GEMMs."""
    import os

    import torch
    import torch.distributed as dist

    from paper_2509_04594_b200.multigpu import HostShardedGemm, ShardedGemm, row_partitions

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n = 1000
        a, b = oracle.generate(n, n, 1), oracle.generate(n, n, 2)
        (r0, r1), = row_partitions(n, 1)
        ta = torch.from_numpy(a[r0:r1]).cuda()
        tb_ = torch.from_numpy(b).cuda()
        ref = oracle.tiled_parallel(a, b)
        for panels in (None, 1, 4, 7):
            out = torch.empty((r1 - r0, n), dtype=torch.float64, device="cuda")
            ShardedGemm(panels=panels)(ta, tb_, out)
            torch.cuda.synchronize()
            assert oracle.normwise_rel(out.cpu().numpy(), ref) <= NORMWISE
        # end-to-end form from pinned host buffers (per-rank B shares + all-gather)
        a_h = torch.from_numpy(a[r0:r1]).pin_memory()
        b_h = torch.from_numpy(b).pin_memory()
        for panels, chunks in ((1, 1), (4, 3), (7, 4)):
            c_h = torch.full((r1 - r0, n), float("nan"), dtype=torch.float64).pin_memory()
            g = HostShardedGemm(panels=panels, chunks=chunks)
            for _ in range(2):
                g(a_h, b_h, c_h)
            assert oracle.normwise_rel(c_h.numpy(), ref) <= NORMWISE
        # default plan on a deeper product: panel ramp + deep last panel, A
        # uploaded per panel by 2D copies (odd k: the padded last panel)
        m2, k2, n2 = 700, 5001, 300
        a2, b2 = oracle.generate(m2, k2, 5), oracle.generate(k2, n2, 6)
        ref2 = oracle.tiled_parallel(a2, b2)
        c2 = torch.full((m2, n2), float("nan"), dtype=torch.float64).pin_memory()
        g = HostShardedGemm()
        for _ in range(2):
            g(torch.from_numpy(a2).pin_memory(), torch.from_numpy(b2).pin_memory(), c2)
        assert oracle.normwise_rel(c2.numpy(), ref2) <= NORMWISE
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,k,n", [(4000, 4000, 4000), (3001, 2999, 2500), (7000, 4999, 6000), (7000, 4000, 6032),
                                   (5100, 3000, 9999)])
def test_flat_pipelined_host_path(tb, golden, oracle, m, k, n):
    """Large host-buffer calls run the copy/compute pipeline (phase 1: K-panels
    of the first Mq rows with 2D copies of A's panel slices; phase 2: full-K
    row blocks); results must match the single-launch device path. 7000 x
    4999 x 6000 has an odd k (cp.async loader on panel views) and both phases."""
    import torch

    meta, g = golden
    a, b = oracle.generate(m, k, 1), oracle.generate(k, n, 2)
    a_h = torch.from_numpy(a).pin_memory()
    b_h = torch.from_numpy(b).pin_memory()
    c_h = torch.empty((m, n), dtype=torch.float64).pin_memory()
    out_s, e2e = np.zeros(1), np.zeros(1)
    assert tb.gpu_tiled_multiply_flat(0, a_h, b_h, m, k, n, 32, c_h, out_s, out_e2e_seconds=e2e) == tb.STATUS_OK
    assert e2e[0] > 0 and out_s[0] > 0
    ref, _ = tb.cublas_dgemm(a_h.cuda(), b_h.cuda())
    got = c_h.cuda()
    assert (torch.linalg.norm(got - ref) / torch.linalg.norm(ref)).item() <= NORMWISE
    if (m, k, n) == (4000, 4000, 4000):
        rows = g["n4000_rows"]
        assert oracle.normwise_rel(c_h.numpy()[rows], g["n4000_tiled32_rows"]) <= NORMWISE
    # pageable host buffers take the same path
    c2 = np.zeros(m * n)
    assert tb.gpu_tiled_multiply_flat(0, a, b, m, k, n, 32, c2, out_s) == tb.STATUS_OK
    assert oracle.normwise_rel(c2.reshape(m, n), c_h.numpy()) <= NORMWISE


@pytest.mark.parametrize("m,k,n", [(1000, 777, 1000), (500, 1000, 500), (640, 1010, 384), (1500, 1500, 1500),
                                   (1100, 900, 1100)])
@pytest.mark.parametrize("variant", FAST)
def test_schedule_shapes(tb, oracle, m, k, n, variant):
    """Each host-side schedule shape against the oracle: split-K with k-slabs
    padded past K (1000x777x1000: 64 tiles, s = 2, 49 -> 50 slabs), split-K
    without padding (500x1000x500, 640x1010x384), a >= 90 % single wave run
    data-parallel (1500^3: 144 tiles) and plain stream-K (1100^3: 81 tiles)."""
    a, b = oracle.generate(m, k, 11), oracle.generate(k, n, 12)
    got, sec = tb.gpu_tiled_multiply_timed(a, b, variant=variant)
    assert sec > 0
    assert oracle.normwise_rel(got, oracle.tiled_parallel(a, b)) <= NORMWISE


@pytest.mark.parametrize("variant", ["dmma_tma", "dmma_cpasync", "dfma"])
def test_accumulate_epilogue_many_tiles_per_cta(tb, variant):
    """C += A·B with several tiles per persistent CTA (4096^2 outputs = 1024
    tiles on 148 SMs), repeated: must equal the fp64 reference and be bitwise
    reproducible. Regression test for a stage-release race (fragment loads
    overtaken by the next TMA into the stage while the accumulate epilogue's
    global loads back up the LSU queue) fixed with a proxy fence before the
    empty-barrier arrive."""
    import torch

    g = torch.Generator(device="cuda").manual_seed(5)
    m, k, n = 4096, 512, 4096
    a = torch.rand((m, 2 * k), dtype=torch.float64, device="cuda", generator=g) + 2
    b = torch.rand((2 * k, n), dtype=torch.float64, device="cuda", generator=g) + 2
    ref = a @ b
    first = a[:, :k] @ b[:k]
    outs = []
    for _ in range(3):
        c = first.clone()
        tb.dgemm_launch(a[:, k:], b[k:], c, accumulate=True, variant=variant)
        torch.cuda.synchronize()
        assert (torch.linalg.norm(c - ref) / torch.linalg.norm(ref)).item() <= NORMWISE
        outs.append(c)
    assert all(torch.equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("shape", ["1024,128,640,384", "256,2,4000,4000", "100000,512,512,1"])
def test_flat_pipeline_shapes(tb, oracle, monkeypatch, shape, fused):
    """Forced pipeline shapes (TB_PIPE=mq,kp0,kp,blk): many small panels and
    blocks, a 2-wide first panel, all rows panelised — with phase 1 as the
    fused flag-driven launch and as a launch per panel — all equal the
    single-launch result to the normwise bound."""
    import torch

    m, k, n = 4000, 3998, 4000
    a, b = oracle.generate(m, k, 3), oracle.generate(k, n, 4)
    monkeypatch.setenv("TB_PIPE", shape)
    monkeypatch.setenv("TB_PIPE_FUSED", fused)
    c = np.zeros(m * n)
    out_s = np.zeros(1)
    assert tb.gpu_tiled_multiply_flat(0, a, b, m, k, n, 32, c, out_s) == tb.STATUS_OK
    ref, _ = tb.cublas_dgemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    got = torch.from_numpy(c.reshape(m, n)).cuda()
    assert (torch.linalg.norm(got - ref) / torch.linalg.norm(ref)).item() <= NORMWISE


@pytest.mark.parametrize("m,k,n", [(1000, 1000, 1000), (1001, 999, 1003), (129, 40000, 257), (2047, 1500, 3001)])
@pytest.mark.parametrize("kind", ["pinned", "numpy"])
def test_flat_small_no_phase_one(tb, oracle, m, k, n, kind):
    """Calls between 1e9 and 2e10 flops skip phase 1 (B first, full-K row
    blocks with overlapped copies): odd and skinny shapes, pinned and
    pageable buffers, against the oracle's rows and cuBLAS."""
    import torch

    assert tb._lib.pipeline_plan(m, k, n, staged=kind == "numpy")["mq"] == 0
    a, b = oracle.generate(m, k, 81), oracle.generate(k, n, 82)
    if kind == "pinned":
        ah, bh = torch.from_numpy(a).pin_memory(), torch.from_numpy(b).pin_memory()
        c = torch.full((m, n), float("nan"), dtype=torch.float64).pin_memory()
        cn = c.numpy()
    else:
        ah, bh, c = a, b, np.full((m, n), np.nan)
        cn = c
    s = np.zeros(1)
    assert tb.gpu_tiled_multiply_flat(0, ah, bh, m, k, n, 32, c, s) == tb.STATUS_OK
    ref, _ = tb.cublas_dgemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    assert oracle.normwise_rel(cn, ref.cpu().numpy()) <= NORMWISE
    rows = np.r_[0:2, m // 2, m - 2:m]
    assert oracle.normwise_rel(cn[rows], oracle.tiled_parallel(a[rows], b)) <= NORMWISE


@pytest.mark.parametrize("m,k,n", [(2320, 600, 2320), (2336, 500, 2368), (2368, 300, 2340), (2320, 400, 2334),
                                   (4001, 257, 3999)])
def test_edge_strip_split(tb, oracle, monkeypatch, m, k, n):
    """TMA products with ragged m / n run as a whole-tile launch plus edge
    strips (16/32/64-row and 16/32/64-column strip shapes; TB_SPLIT=1 takes
    the split wherever the shape allows, the cost model would pick one
    launch for some of these); C, plain and accumulated, equals the oracle's
    rows and cuBLAS normwise."""
    import torch

    monkeypatch.setenv("TB_SPLIT", "1")
    a, b = oracle.generate(m, k, 41), oracle.generate(k, n, 42)
    ta, tbm = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    c, sec = tb.dgemm(ta, tbm)
    rows = np.r_[0:3, m - 70:m]  # first rows and the bottom strip
    assert oracle.normwise_rel(c.cpu().numpy()[rows], oracle.tiled_parallel(a[rows], b)) <= NORMWISE
    ref, _ = tb.cublas_dgemm(ta, tbm)
    assert (torch.linalg.norm(c - ref) / torch.linalg.norm(ref)).item() <= NORMWISE
    out = ref.clone()
    tb.dgemm_launch(ta, tbm, out, accumulate=True)
    torch.cuda.synchronize()
    assert (torch.linalg.norm(out - 2 * ref) / torch.linalg.norm(2 * ref)).item() <= NORMWISE


def test_side_stream_strips_match_serial(tb, monkeypatch):
    """The edge strips run on a side stream joined back to the caller's
    stream (tb_launch.cuh launch()): bitwise the same C as all launches on
    one stream, on the default stream and on a user stream, plain and
    accumulate, and the caller's stream sees the strips' results."""
    import torch

    monkeypatch.setenv("TB_SPLIT", "1")
    g = torch.Generator(device="cuda").manual_seed(9)
    a = torch.rand((2320, 400), dtype=torch.float64, device="cuda", generator=g)
    b = torch.rand((400, 2334), dtype=torch.float64, device="cuda", generator=g)
    outs = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("TB_STRIP_CONCURRENT", mode)
        c, _ = tb.dgemm(a, b)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            c2 = torch.ones_like(c)
            tb.dgemm_launch(a, b, c2, accumulate=True, stream=s)
            # consumed on the user stream right after: must include the strips
            col = c2[:, -30:].sum()
        s.synchronize()
        outs[mode] = (c, c2, col.item())
    assert torch.equal(outs["0"][0], outs["1"][0]) and torch.equal(outs["0"][1], outs["1"][1])
    assert outs["0"][2] == outs["1"][2]
    ref = a @ b
    assert (torch.linalg.norm(outs["1"][0] - ref) / torch.linalg.norm(ref)).item() <= NORMWISE


TILES = ["128x128", "128x64", "128x96", "96x96", "96x96t", "64x64", "64x64d", "64x128", "64x128d", "96x128", "64x96"]


@pytest.mark.parametrize("tile", TILES)
@pytest.mark.parametrize("m,k,n", [(1000, 1000, 1000), (1300, 700, 1700), (250, 3000, 130), (4096, 96, 4096)])
def test_every_main_tile_shape(tb, oracle, monkeypatch, tile, m, k, n):
    """Every main-tile shape the cost model can pick (TB_TILE forces it):
    ragged tile grids, stream-K / split-K / data-parallel schedules; plain C
    against the oracle's rows and cuBLAS, then C += A·B."""
    import torch

    monkeypatch.setenv("TB_TILE", tile)
    a, b = oracle.generate(m, k, 51), oracle.generate(k, n, 52)
    ta, tbm = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    c, sec = tb.dgemm(ta, tbm)
    rows = np.r_[0:3, m // 2, m - 3:m]
    assert oracle.normwise_rel(c.cpu().numpy()[rows], oracle.tiled_parallel(a[rows], b)) <= NORMWISE
    ref, _ = tb.cublas_dgemm(ta, tbm)
    assert (torch.linalg.norm(c - ref) / torch.linalg.norm(ref)).item() <= NORMWISE
    out = ref.clone()
    tb.dgemm_launch(ta, tbm, out, accumulate=True)
    torch.cuda.synchronize()
    assert (torch.linalg.norm(out - 2 * ref) / torch.linalg.norm(2 * ref)).item() <= NORMWISE
    again, _ = tb.dgemm(ta, tbm)
    assert torch.equal(again, c)  # deterministic stream-K reduction


# Square sizes at which the cost model (tb_launch.cuh choose_tile) picks each
# (shape, schedule) it uses in N = 200..5000, found with the host-only plan;
# the test re-derives the plan, so a model refit that moves a pick still
# tests the launch it makes.
CHOOSER_SIZES = [200, 230, 330, 490, 650, 810, 840, 1090, 1110, 1290, 1350, 1370, 1480, 1890, 2070, 2500]


@pytest.mark.parametrize("n", CHOOSER_SIZES)
def test_chooser_picks_match_cublas(tb, oracle, n):
    """Whatever (tile shape, schedule) the cost model picks — data-parallel on
    min(T, 148) CTAs, stream-K, split-K — the default dgemm equals cuBLAS
    normwise and the oracle on sampled rows, repeatably."""
    import torch

    from paper_2509_04594_b200 import _lib

    plan = _lib.launch_plan(n, n, n)
    assert len(plan) == 1 and plan[0]["kernel"] == "dmma" and plan[0]["loader"] == "tma", plan
    a, b = oracle.generate(n, n, 61), oracle.generate(n, n, 62)
    ta, tbm = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    c, _ = tb.dgemm(ta, tbm)
    ref, _ = tb.cublas_dgemm(ta, tbm)
    assert (torch.linalg.norm(c - ref) / torch.linalg.norm(ref)).item() <= NORMWISE, plan[0]
    rows = np.r_[0:2, n // 2, n - 2:n]
    assert oracle.normwise_rel(c.cpu().numpy()[rows], oracle.tiled_parallel(a[rows], b)) <= NORMWISE
    again, _ = tb.dgemm(ta, tbm)
    assert torch.equal(again, c)


def test_staged_tma_for_misaligned_operands(tb, oracle):
    """AUTO on operands TMA cannot address (odd leading dimension; base off a
    16-byte boundary) above the staging threshold copies them to even-pitch
    workspace and runs the TMA kernel: results equal the oracle's rows and
    cuBLAS normwise; the caller's buffers are untouched."""
    import torch

    m = k = n = 2223  # odd: lda = ldb = 2223; 2.2e10 flops >= the staging threshold
    a, b = oracle.generate(m, k, 31), oracle.generate(k, n, 32)
    ta, tbm = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    c, sec = tb.dgemm(ta, tbm)
    rows = np.arange(0, m, 97)
    want = oracle.tiled_parallel(a[rows], b)
    assert oracle.normwise_rel(c.cpu().numpy()[rows], want) <= NORMWISE
    assert torch.equal(ta.cpu(), torch.from_numpy(a))
    # even leading dims, but the bases are 8 bytes past a 16-byte boundary (column views)
    big_a = torch.from_numpy(oracle.generate(m, k + 3, 33)).cuda()
    big_b = torch.from_numpy(oracle.generate(k, n + 3, 34)).cuda()
    va, vb = big_a[:, 1:k + 1], big_b[:, 1:n + 1]
    assert va.stride(0) % 2 == 0 and (va.data_ptr() % 16) == 8
    out = torch.empty((m, n), dtype=torch.float64, device="cuda")
    tb.dgemm_launch(va, vb, out)
    ref, _ = tb.cublas_dgemm(va.contiguous(), vb.contiguous())
    torch.cuda.synchronize()
    assert (torch.linalg.norm(out - ref) / torch.linalg.norm(ref)).item() <= NORMWISE


@pytest.mark.parametrize("m,k,n", [(4000, 4000, 4032), (333, 129, 257), (7001, 3000, 5000)])
def test_pageable_staging_matches_direct_copies(tb, oracle, monkeypatch, m, k, n):
    """Pageable (numpy) host buffers go through the pinned staging ring and
    the copy-thread pool; the product matches the plain pageable copies
    (TB_STAGE=0, which also takes the launch-per-panel phase 1, so a
    different k-split: normwise) and is bitwise the same when a pinned output
    with pageable inputs (and the reverse) mixes both paths. The plan's
    phase-1 rows depend on which buffers are staged, so TB_PIPE pins one
    shape for the bitwise comparisons."""
    import torch

    monkeypatch.setenv("TB_PIPE", "2048,256,2048,1536")
    a, b = oracle.generate(m, k, 51), oracle.generate(k, n, 52)
    s = np.zeros(1)
    outs = []
    for stage in ("1", "0"):
        monkeypatch.setenv("TB_STAGE", stage)
        c = np.full(m * n, np.nan)
        assert tb.gpu_tiled_multiply_flat(0, a, b, m, k, n, 32, c, s) == tb.STATUS_OK
        outs.append(c)
    assert oracle.normwise_rel(outs[0].reshape(m, n), outs[1].reshape(m, n)) <= NORMWISE
    monkeypatch.setenv("TB_STAGE", "1")
    c_pin = torch.full((m, n), float("nan"), dtype=torch.float64).pin_memory()
    assert tb.gpu_tiled_multiply_flat(0, a, b, m, k, n, 32, c_pin, s) == tb.STATUS_OK
    assert np.array_equal(c_pin.numpy().ravel(), outs[0])
    a_pin = torch.from_numpy(a).pin_memory()
    c = np.full(m * n, np.nan)
    assert tb.gpu_tiled_multiply_flat(0, a_pin, b, m, k, n, 32, c, s) == tb.STATUS_OK
    assert np.array_equal(c, outs[0])
    rows = np.r_[0:2, m - 2:m]
    assert oracle.normwise_rel(outs[0].reshape(m, n)[rows], oracle.tiled_parallel(a[rows], b)) <= NORMWISE


def test_multiplyfn_through_host_pipeline(tb, oracle):
    """The registered MultiplyFn (what the reference harness times) returns a
    fresh product equal to the oracle, inputs untouched."""
    for m, k, n in ((1000, 1000, 1000), (2501, 1999, 3003)):
        a, b = oracle.generate(m, k, 61), oracle.generate(k, n, 62)
        a0, b0 = a.copy(), b.copy()
        c = tb.gpu_tiled_multiply(a, b)
        assert c.shape == (m, n) and c.dtype == np.float64
        assert np.array_equal(a, a0) and np.array_equal(b, b0)
        rows = np.r_[0:3, m - 3:m]
        assert oracle.normwise_rel(c[rows], oracle.tiled_parallel(a[rows], b)) <= NORMWISE


def test_multiplyfn_outputs_are_fresh_and_independent(tb, oracle):
    """The MultiplyFn's product arrays come from a pinned-block cache: each
    call returns a new, writable, C-contiguous array that the caller owns; a
    held product is never reused or overwritten by later calls, and a
    dropped one may be (backends.py:17-19: fresh output per call)."""
    import torch

    m = k = n = 1200
    a, b = oracle.generate(m, k, 71), oracle.generate(k, n, 72)
    ref = tb.gpu_tiled_multiply_timed(a, b)[0]
    first = tb.gpu_tiled_multiply(a, b)
    snap = first.copy()
    assert first.flags["C_CONTIGUOUS"] and first.flags["WRITEABLE"] and first.dtype == np.float64
    assert torch.from_numpy(first).is_pinned()
    outs = [tb.gpu_tiled_multiply(a * (i + 2), b) for i in range(3)]
    assert np.array_equal(first, snap), "a held product was overwritten by a later call"
    ptrs = {o.ctypes.data for o in outs + [first]}
    assert len(ptrs) == 4, "live products share memory"
    for i, o in enumerate(outs):
        assert oracle.normwise_rel(o, (i + 2) * ref) <= NORMWISE
    first[:] = 0.0  # the caller may write its own array
    del outs
    again = tb.gpu_tiled_multiply(a, b)
    assert oracle.normwise_rel(again, ref) <= NORMWISE


def test_flat_repeated_varied_calls(tb, oracle):
    """Back-to-back host-buffer calls of varying size and buffer kind (pinned
    / pageable, pipelined / single-shot, ragged / aligned) reuse and regrow
    the cached workspaces, event pool, staging ring and pipeline tables:
    every result equals cuBLAS on the same operands."""
    import torch

    rng = np.random.default_rng(7)
    shapes = [(4000, 4000, 4032), (700, 300, 900), (5003, 2999, 4500), (128, 64, 128), (4100, 4000, 4000),
              (6000, 3000, 2000), (333, 1000, 77)]
    for i, (m, k, n) in enumerate(shapes * 2):
        a = rng.random((m, k)) * 3 + 2
        b = rng.random((k, n)) * 3 + 2
        pinned = i % 3 == 0
        ah = torch.from_numpy(a).pin_memory() if pinned else a
        bh = torch.from_numpy(b).pin_memory() if i % 2 == 0 else b
        c = torch.empty((m, n), dtype=torch.float64).pin_memory() if pinned else np.empty(m * n)
        assert tb.gpu_tiled_multiply_flat(0, ah, bh, m, k, n, 32, c, np.zeros(1)) == tb.STATUS_OK
        got = torch.as_tensor(np.asarray(c).reshape(m, n)).cuda()
        ref, _ = tb.cublas_dgemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
        assert (torch.linalg.norm(got - ref) / torch.linalg.norm(ref)).item() <= NORMWISE, (m, k, n, i)


def test_concurrent_host_threads(tb, oracle):
    """The registered MultiplyFn and the flat host entry called from several
    host threads at once (the reference's CPU backends are thread-safe,
    test_backends.py:136-149; the GPU library serialises per device)."""
    from concurrent.futures import ThreadPoolExecutor

    shapes = [(300, 200, 100), (129, 257, 65), (640, 64, 512), (1000, 300, 700)] * 2
    ops = [(oracle.generate(m, k, 20 + i), oracle.generate(k, n, 40 + i)) for i, (m, k, n) in enumerate(shapes)]

    def via_fn(i):
        a, b = ops[i]
        return tb.gpu_tiled_multiply(a, b)

    def via_flat(i):
        a, b = ops[i]
        c = np.zeros(a.shape[0] * b.shape[1])
        assert tb.gpu_tiled_multiply_flat(0, a, b, a.shape[0], a.shape[1], b.shape[1], 32, c,
                                          np.zeros(1)) == tb.STATUS_OK
        return c.reshape(a.shape[0], b.shape[1])

    with ThreadPoolExecutor(max_workers=4) as ex:
        futs = [ex.submit(via_fn if i % 2 else via_flat, i) for i in range(len(ops))]
        for i, f in enumerate(futs):
            a, b = ops[i]
            assert oracle.normwise_rel(f.result(), oracle.tiled_parallel(a, b)) <= NORMWISE


def test_cli_run_writes_reference_csv(tb, tmp_path):
    from paper_2509_04594_b200.__main__ import main

    out = tmp_path / "gpu.csv"
    assert main(["run", "--backends", "gpu-tiled,cublas-dgemm", "--sizes", "64,200", "--trials", "2",
                 "--verify", "--out", str(out)]) == 0  # host CPU product as the --verify reference
    lines = out.read_text().splitlines()
    assert lines[0] == "backend,n,trial,seconds,flops" and len(lines) == 1 + 2 * 2 * 2
    assert (tmp_path / "gpu.csv.meta.json").exists()
    out2 = tmp_path / "gpu2.csv"
    assert main(["run", "--backends", "gpu-tiled", "--sizes", "333", "--trials", "1", "--verify",
                 "--verify-with", "cublas", "--out", str(out2)]) == 0


def test_n32768_sampled_exact_oracle(tb, oracle):
    """configs[4] size (8.6 GB per matrix) on one B200: C[rows][:, cols] vs
    the reference's tiled product on the same rows and columns
    (tiled(A[rows], B[:, cols]) is entrywise bitwise equal to the full tiled
    product: the k0 phases depend on k only), plus a full-matrix normwise
    check of a row block against cuBLAS."""
    import torch

    n = 32768
    g = torch.Generator(device="cuda").manual_seed(32768)
    A = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g).mul_(3.0).add_(2.0)
    B = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g).mul_(3.0).add_(2.0)
    C, sec = tb.dgemm(A, B)
    assert tb.flop_count(n) / sec / 1e12 > 20.0  # sanity: full-size run is on the fast path
    rows = torch.tensor([0, 127, 128, 16383, 16384, 32639, 32640, 32767], device="cuda")
    cols = torch.tensor(list(range(0, 16)) + list(range(16376, 16392)) + list(range(32752, 32768)), device="cuda")
    a_rows = A[rows].cpu().numpy()
    b_cols = B[:, cols].contiguous().cpu().numpy()
    want = oracle.tiled_parallel(a_rows, b_cols)
    got = C[rows][:, cols].cpu().numpy()
    assert oracle.normwise_rel(got, want) <= NORMWISE
    assert oracle.max_abs_rel_diff(got, want) <= ELEMWISE
    # A 1024-row block of the full product against cuBLAS (keeps memory bounded).
    ref, _ = tb.cublas_dgemm(A[8192:9216].contiguous(), B)
    rel = (torch.linalg.norm(C[8192:9216] - ref) / torch.linalg.norm(ref)).item()
    assert rel <= NORMWISE
    del A, B, C, ref
    torch.cuda.empty_cache()


@pytest.mark.parametrize("seed", range(6))
def test_random_shapes_property(tb, oracle, seed):
    """Seeded random (m, k, n) in [1, 400]^3 x every variant: normwise and
    elementwise bars vs the reference tiled oracle; the paper variant bitwise
    vs the naive oracle."""
    rng = np.random.Generator(np.random.PCG64(9000 + seed))
    for _ in range(4):
        m, k, n = (int(x) for x in rng.integers(1, 401, size=3))
        a, b = oracle.generate(m, k, seed * 7 + m), oracle.generate(k, n, seed * 11 + n)
        ref = oracle.tiled_parallel(a, b)
        for v in FAST:
            got = _gpu(tb, a, b, v)
            assert oracle.normwise_rel(got, ref) <= NORMWISE, (m, k, n, v)
            assert oracle.max_abs_rel_diff(got, ref) <= ELEMWISE, (m, k, n, v)
        assert np.array_equal(_gpu(tb, a, b, "paper"), oracle.naive(a, b)), (m, k, n)


def test_dimension_limits(tb):
    lib = tb._lib.lib()
    big = 2**31
    assert lib.tb_validate_launch(big, 4, 4, 32, 0, 0) == tb.STATUS_OVER_LIMITS
    assert lib.tb_validate_launch(4, big, 4, 32, 0, 0) == tb.STATUS_OVER_LIMITS
    assert lib.tb_validate_launch(4, 4, 4, 33, 1, 0) == tb.STATUS_OVER_LIMITS  # 1089 threads (limits.test.ts)
    assert lib.tb_validate_launch(4, 4, 4, 0, 0, 0) == tb.STATUS_BAD_DIMS
    assert lib.tb_validate_launch(4, 4, 4, 32, 9, 0) == tb.STATUS_BAD_DIMS
    assert lib.tb_validate_launch(4, 4, 4, 32, 0, 0) == tb.STATUS_OK
    assert lib.tb_validate_launch(4, 4, 4, 32, 0, 999) == tb.STATUS_NO_DEVICE


def test_performance_floor(tb):
    """Loose guard against silent slow paths (a wrong loader, a lost
    schedule, a CPU detour): kernel-only N = 4096 >= 25 TFLOP/s (measured
    ~35), pinned host-buffer N = 6000 end to end >= 15 TFLOP/s (measured
    ~23, PCIe-bound at this size)."""
    import torch

    n = 4096
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g)
    b = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g)
    c = torch.empty_like(a)
    best = min(tb.dgemm(a, b, c)[1] for _ in range(4))
    assert tb.flop_count(n) / best / 1e12 >= 25.0, best
    n = 6000
    ah = torch.rand((n, n), dtype=torch.float64).pin_memory()
    bh = torch.rand((n, n), dtype=torch.float64).pin_memory()
    ch = torch.empty((n, n), dtype=torch.float64).pin_memory()
    e2e = np.zeros(1)
    times = []
    for _ in range(3):
        assert tb.gpu_tiled_multiply_flat(0, ah, bh, n, n, n, 32, ch, np.zeros(1), out_e2e_seconds=e2e) == 0
        times.append(e2e[0])
    assert tb.flop_count(n) / min(times) / 1e12 >= 15.0, times
