"""Host-buffer pipeline planner (tb_pipeline_plan, the shape
tb_gpu_tiled_multiply_flat_ex runs) — pure host logic, no device needed."""
import random

import pytest

from paper_2509_04594_b200 import _lib


def _check(m, k, n, sms=148, fused_ok=True):
    p = _lib.pipeline_plan(m, k, n, sms, fused_ok)
    pan, blk, mq = p["panels"], p["blocks"], p["mq"]
    assert pan[0] == 0 and pan[-1] == k and all(a < b for a, b in zip(pan, pan[1:]))
    assert blk[0] == mq and blk[-1] == m and all(a < b for a, b in zip(blk, blk[1:]))
    assert mq == m or (mq % 128 == 0 and 0 <= mq < m)  # mq = 0: no phase 1 (small problems)
    align = 16 if p["fused"] else 2  # k-stage bounds for the fused PIPE launch, TMA (even k0) otherwise
    assert all(x % align == 0 for x in pan[1:-1])
    assert all(x % 128 == 0 for x in blk[1:-1])  # only the last row block may be ragged
    if not fused_ok:
        assert not p["fused"]
    if 2.0 * m * n * k < 1e9:
        assert (mq, pan, blk, p["fused"]) == (m, [0, k], [m], False)
    if p["fused"]:
        assert 2 <= len(pan) - 1 <= 120
    return p


def test_n10000_shape():
    p = _check(10000, 10000, 10000)
    # 34 tile rows cover the compute/transfer balance; 41 rows give 3239
    # tiles = 21.89 per CTA on 148 SMs (least imbalance within +8 rows).
    assert p["mq"] == 41 * 128 and p["fused"]
    assert p["panels"][1] == 256  # small first panel: the GEMM starts after 0.56 ms of copies
    assert p["blocks"][-1] - p["blocks"][-2] <= 512  # short final D2H


def test_small_problems_are_single_shot():
    for s in [(1, 1, 1), (700, 700, 700), (100, 1000, 100)]:
        _check(*s)


def test_small_problems_have_no_phase_one():
    """Below 2e10 flops, B lands first and all rows come from row blocks."""
    for s in [(1000, 1000, 1000), (2000, 2000, 2000), (1001, 999, 1500)]:
        p = _check(*s)
        assert p["mq"] == 0 and p["panels"] == [0, s[1]] and not p["fused"] and len(p["blocks"]) > 2
    p = _check(3001, 2999, 2500)
    assert p["mq"] > 0


def test_unfused_form():
    p = _check(10000, 10000, 10000, fused_ok=False)
    assert not p["fused"]


@pytest.mark.parametrize("seed", range(8))
def test_random_shapes(seed):
    rng = random.Random(seed)
    for _ in range(60):
        m, k, n = (rng.randint(1, 40000) for _ in range(3))
        _check(m, k, n, sms=rng.choice([148, 132, 8]), fused_ok=rng.random() < 0.8)


def test_bad_arguments():
    with pytest.raises(Exception):
        _lib.pipeline_plan(0, 10, 10)


def test_staged_inputs_plan_more_phase1_rows():
    """Staged (pageable) operands land at ~42 instead of 55 GB/s, so phase 1
    must cover more rows to outlast its transfers (up to the D2H-bound cap)."""
    from paper_2509_04594_b200 import _lib

    for n in (8000, 10000, 12000, 16384):
        pinned = _lib.pipeline_plan(n, n, n)
        staged = _lib.pipeline_plan(n, n, n, staged=True)
        # N = 8000: both hit the D2H-bound cap (tb_pipeline.cuh), which does not depend on the inputs
        assert staged["mq"] > pinned["mq"] or (n == 8000 and staged["mq"] == pinned["mq"])
        assert staged["blocks"][0] == staged["mq"] and staged["blocks"][-1] == n
        assert staged["panels"][0] == 0 and staged["panels"][-1] == n
    assert _lib.pipeline_plan(10000, 10000, 10000, staged=True)["mq"] == 7168


def test_d2h_bound_cap():
    """Where all of C's D2H would outlast phase 2's compute (N ~ 3000-7000
    pinned), phase 1 is capped at m(1 - 4F/(D·k)) rows, phase-2 blocks are
    >= 256 rows of ~0.3 ms, and the first K-panel is 512 deep."""
    from paper_2509_04594_b200 import _lib

    p = _lib.pipeline_plan(4000, 4000, 4000)
    assert p["mq"] == 1280 and p["panels"][1] == 512
    sizes = [b - a for a, b in zip(p["blocks"], p["blocks"][1:])]
    assert sizes.count(256) >= 8 and max(sizes) <= 256
    big = _lib.pipeline_plan(10000, 10000, 10000)
    assert big["mq"] > 4000 and big["panels"][1] == 256  # the cap does not bind at N = 10000
