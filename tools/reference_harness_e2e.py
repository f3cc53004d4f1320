"""Drop-in check with the REFERENCE's own harness (tooling, GPU box).

Imports the unmodified reference package installed under baseline/_ref
(`pip install --no-index --no-build-isolation --find-links /opt/wheelhouse
--target baseline/_ref <copy of /root/reference/pkg> --no-deps`), registers
this repo's `gpu-tiled` / `cublas-dgemm` MultiplyFns into a reference
`BackendRegistry` with `register_into`, adds the
reference demos' `blas-numpy` backend (`a @ b`), and runs the reference's
`run_trials`: its operand generation, its wall clock around `fn(a, b)`
(harness.py:163-172, i.e. end to end incl. host<->device copies), its
TrialRecord invariants and, at N = 1000, its `--verify` oracle check. The
records are written with the reference's `write_records`.

    python tools/reference_harness_e2e.py out.csv [trials] [--paper]

--paper: the paper's grid N = 1000..10000 step 1000 (after the N = 1000
verified run) instead of 2000 / 4000 / 10000.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "tilebench")):
    raise SystemExit(f"reference package not installed under {REF} (see module docstring)")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_refharness")

from tilebench.backends import BackendDescriptor, BackendRegistry  # noqa: E402
from tilebench.harness import RunConfig, run_trials  # noqa: E402
from tilebench.records import write_records  # noqa: E402

import paper_2509_04594_b200 as tb  # noqa: E402


def main():
    args = [x for x in sys.argv[1:] if not x.startswith("--")]
    out = args[0] if args else "ref_harness.csv"
    trials = int(args[1]) if len(args) > 1 else 5
    sizes = tuple(range(2000, 10001, 1000)) if "--paper" in sys.argv else (2000, 4000, 10000)
    reg = BackendRegistry()
    names = [d.name for d in tb.register_into(reg, BackendDescriptor)]
    assert names, "no CUDA device: register_into is a no-op"
    reg.register_external(BackendDescriptor("blas-numpy", parallel=True, requires_external=True),
                          lambda a, b: a @ b)
    records = []
    # N = 1000 with the reference's own verification (naive oracle, max_abs_rel_diff <= 1e-10)
    r1, meta = run_trials(RunConfig(backends=("gpu-tiled", "cublas-dgemm"), sizes=(1000,), trials=trials,
                                    verify=True), registry=reg)
    records += r1
    r2, _ = run_trials(RunConfig(backends=("gpu-tiled", "cublas-dgemm", "blas-numpy"), sizes=sizes,
                                 trials=trials), registry=reg)
    records += r2
    write_records(out, records, meta)
    by = {}
    for r in records:
        by.setdefault((r.backend, r.n), []).append(r.flops)
    for (name, n), v in sorted(by.items(), key=lambda x: (x[0][1], x[0][0])):
        print(f"{n:6d} {name:14s} mean {sum(v) / len(v) / 1e9:10.1f} GFLOPS  best {max(v) / 1e9:10.1f}")


if __name__ == "__main__":
    main()
