"""The CPU oracle is pinned BITWISE to vectors the reference itself produced
(tests/golden/make_golden.py imports /root/reference's tilebench). CPU-only."""
import hashlib

import numpy as np
import pytest


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


def test_hand_checked_vectors(golden, oracle):
    meta, _ = golden
    kat = meta["kat"]
    assert oracle.naive(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[5.0, 6.0], [7.0, 8.0]])).tolist() == \
        kat["two_by_two"] == [[19.0, 22.0], [43.0, 50.0]]
    assert oracle.naive(np.array([[2.0]]), np.array([[5.0]]))[0, 0] == kat["one_by_one"] == 10.0
    assert oracle.paper_kernel(np.array([[3.0]]), np.array([[4.0]]))[0, 0] == kat["three_by_four"] == 12.0
    for n, v in kat["flop_count"].items():
        assert oracle.flop_count(int(n)) == v
    assert oracle.max_abs_rel_diff(np.array([[1.0]]), np.array([[2.0]])) == kat["max_abs_rel_diff_1_2"] == 0.5


def test_generator_pinned(golden, oracle):
    meta, g = golden
    assert np.array_equal(oracle.generate(4, 4, 0), g["gen_4x4_seed0"])
    for key, digest in meta["gen_digest"].items():
        n, s = map(int, key.split("_"))
        assert sha(oracle.generate(n, n, s)) == digest


def test_grid_bitwise(golden, oracle):
    meta, g = golden
    for c in meta["cases"]:
        a, b = oracle.generate(c["m"], c["k"], c["seed_a"]), oracle.generate(c["k"], c["n"], c["seed_b"])
        naive = g[c["tag"] + "_naive"]
        assert np.array_equal(oracle.naive(a, b), naive), c["tag"]
        # the paper's GPU order (kernel.ts:50-78) is bitwise the naive order
        assert np.array_equal(oracle.paper_kernel(a, b, 32), naive), c["tag"]
        for t in c["tiles"]:
            want = g[f"{c['tag']}_tiled{t}"]
            assert np.array_equal(oracle.tiled_seq(a, b, t), want), (c["tag"], t)
            for threads in (1, 2, 7):
                assert np.array_equal(oracle.tiled_parallel(a, b, t, threads), want), (c["tag"], t, threads)


def test_config0_n1000_sha(golden, oracle):
    meta, g = golden
    a, b = oracle.generate(1000, 1000, 1), oracle.generate(1000, 1000, 2)
    c = oracle.tiled_parallel(a, b)
    assert sha(c) == meta["large"]["1000"]["tiled32_sha256"]
    assert np.array_equal(c[g["n1000_rows"]], g["n1000_tiled32_rows"])


def test_row_sampling_is_bitwise(golden, oracle):
    """tiled(A[rows], B) == tiled(A, B)[rows] — the basis of the large-N row-sampled oracle."""
    a, b = oracle.generate(203, 203, 3), oracle.generate(203, 203, 4)
    rows = np.array([0, 5, 31, 32, 100, 202])
    assert np.array_equal(oracle.tiled_seq(a[rows], b), oracle.tiled_seq(a, b)[rows])


@pytest.mark.parametrize("n", [4000, 10000])
def test_large_full_products(golden, oracle, n):
    """configs[1] / configs[3]: the oracle's FULL N x N tiled product is
    bitwise the reference's (SHA-256 of its tiled_parallel_multiply output,
    tests/golden/make_golden.py), and so are the 64 sampled rows kept
    verbatim. ~2 s / ~35 s on 8 host threads."""
    meta, g = golden
    assert sha(oracle.generate(min(n, 4000), min(n, 4000), 1)) == meta["gen_digest"]["4000_1"]
    a, b = oracle.generate(n, n, 1), oracle.generate(n, n, 2)
    c = oracle.tiled_parallel(a, b)
    assert sha(c) == meta["large"][str(n)]["tiled32_sha256"]
    rows = g[f"n{n}_rows"]
    assert len(rows) >= 64
    assert np.array_equal(c[rows], g[f"n{n}_tiled32_rows"])
    assert np.array_equal(oracle.tiled_parallel(a[rows[:4]], b), g[f"n{n}_tiled32_rows"][:4])


def test_plan_partitions(oracle):
    """backends.py:119-136 and test_backends.py partition coverage."""
    assert oracle.plan_partitions(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert oracle.plan_partitions(2, 5) == [(0, 1), (1, 2)]
    assert oracle.plan_partitions(0, 4) == []
    for tiles in (1, 7, 100):
        for w in (1, 2, 3, 48):
            ch = oracle.plan_partitions(tiles, w)
            assert ch[0][0] == 0 and ch[-1][1] == tiles
            assert all(x[1] == y[0] for x, y in zip(ch, ch[1:]))


def test_normwise_metric(oracle):
    x = np.array([[3.0, 4.0]])
    assert oracle.normwise_rel(x, x) == 0.0
    assert abs(oracle.normwise_rel(np.array([[3.0, 4.0 + 5e-12]]), x) - 1e-12) < 1e-15
