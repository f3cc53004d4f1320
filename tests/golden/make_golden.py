"""Generate the golden parity fixtures by importing the REFERENCE package.

Run here (the container with /root/reference), never on the GPU box:

    python tests/golden/make_golden.py

It copies /root/reference/pkg/src to a temp dir (numba's cache=True would
otherwise write into the read-only reference tree), imports ``tilebench`` from
there and records, for identical seeded inputs:

* the reference's hand-checked vectors (test_backends.py:23-34,
  kernel.test.ts:22-28, test_matrices.py:68-76, :99-100);
* naive / tiled-seq outputs on the oracle grid (test_acceptance.py:57-73,
  kernel.test.ts:30-62, test_backends.py:53-71);
* SHA-256 digests of generate() output and of the FULL tiled products at
  N = 1000 (configs[0]), N = 4000 (configs[1]) and N = 10000 (configs[3]),
  computed by the reference's own ``tiled_parallel_multiply`` (numba, all
  host threads; bitwise equal to ``tiled_seq``, backends.py:21-24), plus
  64-row samples at N = 4000 and N = 10000 kept verbatim
  (tiled_seq(A[rows], B) is bitwise equal to those rows of the full product,
  SURVEY.md §7 step 1; the row samples are recomputed with ``tiled_seq`` on
  the sampled rows and cross-checked against the full product's rows).

Outputs: tests/golden/golden_small.npz, tests/golden/golden_meta.json.
"""
from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"

GRID = [1, 2, 31, 32, 33, 64, 65, 100]  # test_acceptance.py:57-73 DIMS
SQUARE_EXTRA = [129]  # kernel.test.ts:56-62
RECT = [(21, 47, 9), (37, 41, 29), (3, 5, 2)]  # kernel.test.ts:46-54, test_backends.py:66-71, :36-39
ROW_SAMPLE = {4000: 64, 10000: 64}  # SURVEY.md §8(d) parity gate: >= 64 rows


def sha(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


def main() -> None:
    tmp = tempfile.mkdtemp(prefix="tbref_")
    shutil.copytree(REF, os.path.join(tmp, "src"))
    os.environ["NUMBA_CACHE_DIR"] = os.path.join(tmp, "numba_cache")
    sys.path.insert(0, os.path.join(tmp, "src"))
    import tilebench as tb  # noqa: E402
    from tilebench.backends import (PoolConfig, TileConfig, naive_multiply,  # noqa: E402
                                    tiled_parallel_multiply, tiled_seq_multiply)
    from tilebench.matrices import GenSpec, flop_count, generate, max_abs_rel_diff  # noqa: E402

    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"reference": "tilebench " + getattr(tb, "__version__", "?"),
                  "numpy": np.__version__, "cases": []}

    # Hand-checked vectors.
    meta["kat"] = {
        "two_by_two": naive_multiply(np.array([[1.0, 2.0], [3.0, 4.0]]),
                                     np.array([[5.0, 6.0], [7.0, 8.0]])).tolist(),
        "one_by_one": float(naive_multiply(np.array([[2.0]]), np.array([[5.0]]))[0, 0]),
        "three_by_four": float(naive_multiply(np.array([[3.0]]), np.array([[4.0]]))[0, 0]),
        "flop_count": {str(n): flop_count(n) for n in (1, 2, 3, 64, 1000, 4000, 10000, 32768, 100000)},
        "max_abs_rel_diff_1_2": max_abs_rel_diff(np.array([[1.0]]), np.array([[2.0]])),
    }

    # Generator pin: first values and digests of generate().
    g = generate(GenSpec(4, 4, 2.0, 5.0, 0))
    arrays["gen_4x4_seed0"] = g
    meta["gen_digest"] = {}
    for n, s in [(1000, 1), (1000, 2), (4000, 1), (4000, 2)]:
        meta["gen_digest"][f"{n}_{s}"] = sha(generate(GenSpec(n, n, 2.0, 5.0, s)))

    def case(tag, m, k, n, sa, sb, tiles=(32,)):
        a = generate(GenSpec(m, k, 2.0, 5.0, sa))
        b = generate(GenSpec(k, n, 2.0, 5.0, sb))
        arrays[f"{tag}_naive"] = naive_multiply(a, b)
        for t in tiles:
            arrays[f"{tag}_tiled{t}"] = tiled_seq_multiply(a, b, TileConfig(t))
        meta["cases"].append({"tag": tag, "m": m, "k": k, "n": n, "seed_a": sa, "seed_b": sb,
                              "tiles": list(tiles)})

    for n in GRID + SQUARE_EXTRA:
        case(f"sq{n}", n, n, n, 100 + n, 200 + n, tiles=(8, 16, 32))
    for (m, k, n) in RECT:
        case(f"rect{m}x{k}x{n}", m, k, n, 7, 8, tiles=(1, 2, 3, 16, 32, 64))

    # configs[0]: N = 1000 full product (digest + a few rows kept verbatim).
    full = {}
    for n in (1000,):
        a = generate(GenSpec(n, n, 2.0, 5.0, 1))
        b = generate(GenSpec(n, n, 2.0, 5.0, 2))
        c = tiled_seq_multiply(a, b, TileConfig(32))
        rows = np.array([0, 1, 31, 32, 499, 998, 999])
        arrays[f"n{n}_rows"] = rows
        arrays[f"n{n}_tiled32_rows"] = c[rows]
        full[str(n)] = {"seed_a": 1, "seed_b": 2, "tiled32_sha256": sha(c),
                        "tiled32_fro": float(np.linalg.norm(c))}
    # configs[1] / configs[3]: N = 4000, 10000 full products (the reference's
    # own tiled-parallel path on every host thread: ~15 s and ~4 min here)
    # -> SHA-256 + Frobenius norm, and 64-row samples kept verbatim.
    threads = os.cpu_count() or 1
    for n, r in ROW_SAMPLE.items():
        a = generate(GenSpec(n, n, 2.0, 5.0, 1))
        b = generate(GenSpec(n, n, 2.0, 5.0, 2))
        c = tiled_parallel_multiply(a, b, TileConfig(32), PoolConfig(threads))
        rows = np.sort(np.random.Generator(np.random.PCG64(n)).choice(n, r, replace=False))
        sampled = tiled_seq_multiply(a[rows], b, TileConfig(32))
        assert np.array_equal(sampled, c[rows]), "row sampling must be bitwise"
        arrays[f"n{n}_rows"] = rows
        arrays[f"n{n}_tiled32_rows"] = sampled
        full[str(n)] = {"seed_a": 1, "seed_b": 2, "tiled32_sha256": sha(c),
                        "tiled32_fro": float(np.linalg.norm(c)), "threads": threads}
        del c
    meta["large"] = full

    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **arrays)
    with open(os.path.join(HERE, "golden_meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    shutil.rmtree(tmp, ignore_errors=True)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
