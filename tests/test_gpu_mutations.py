"""Barrier-discipline mutants must be caught (run on a B200: pytest -m gpu).

The reference proves its two-barrier discipline by deleting each barrier
from the kernel and showing the product goes wrong on its shuffled simulator
(/root/reference/pkg/gpu/tests/barriers.test.ts:37-82). The sm_100a kernel's
discipline is the full/empty mbarrier protocol of its stage ring
(dgemm_dmma.cuh); each mutant build (-DTB_MUTATE=n, see the header of
dgemm_dmma.cuh) breaks one rule of it:

  1  read a stage's fragments before its full-barrier wait   (missing load barrier)
  2  release a stage (empty arrive) before reading it        (missing reuse barrier)
  3  drop fence.proxy.async before the empty arrive          (the round-1 race)

and the probe (tests/_mutation_probe.py: the parity checks that exercise the
stage protocol on every kernel shape) must report an error above the 1e-12
bar for it, while the product build passes the same probe. A mutant that
crashes or hangs the probe also counts as caught (the suite fails loudly).
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2509_04594_b200")
PROBE = os.path.join(ROOT, "tests", "_mutation_probe.py")
MUTANTS = {1: "fragment loads before the full-barrier wait", 2: "empty arrive before the stage is read",
           3: "no fence.proxy.async before the empty arrive"}


@pytest.fixture(scope="module")
def mutant_libs():
    """Build the mutant libraries (in parallel; ~15 s) unless present and current."""
    from paper_2509_04594_b200 import build

    srcs = [os.path.join(build.CSRC, d) for d in build.DEPS]
    newest = max(os.path.getmtime(x) for x in srcs if os.path.exists(x))
    procs = {}
    for n in MUTANTS:
        lib = os.path.join(PKG, f"libtbgpu_mut{n}.so")
        if not os.path.exists(lib) or os.path.getmtime(lib) < newest:
            procs[n] = subprocess.Popen([sys.executable, os.path.join(ROOT, "tools", "build_variant.py"), f"mut{n}",
                                         f"-DTB_MUTATE={n}"], stdout=subprocess.PIPE, stderr=subprocess.PIPE)
    for n, p in procs.items():
        _, err = p.communicate(timeout=600)
        assert p.returncode == 0, err.decode()[-2000:]
    return {n: f"mut{n}" for n in MUTANTS}


def _probe(variant: str | None, reps: int = 4) -> dict:
    env = dict(os.environ, PYTHONPATH=ROOT)
    env.pop("TB_LIB_VARIANT", None)
    if variant:
        env["TB_LIB_VARIANT"] = variant
    try:
        res = subprocess.run([sys.executable, PROBE, str(reps)], env=env, capture_output=True, text=True,
                             timeout=180)
    except subprocess.TimeoutExpired:
        return {"outcome": "hang (killed after 180 s)"}
    if res.returncode != 0:
        return {"outcome": f"crash (rc={res.returncode}): {res.stderr.strip()[-300:]}"}
    return json.loads(res.stdout.strip().splitlines()[-1])


def test_product_build_passes_probe():
    errs = _probe(None)
    assert all(v <= 1e-12 for v in errs.values()), errs


@pytest.mark.parametrize("n", sorted(MUTANTS))
def test_mutant_is_caught(mutant_libs, n):
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import sass_lint

    errs = _probe(mutant_libs[n])
    lint = sass_lint.lint(os.path.join(PKG, f"libtbgpu_{mutant_libs[n]}.so"))
    print(f"mutant {n} ({MUTANTS[n]}): probe {errs}; sass lint: {len(lint['violations'])} of "
          f"{lint['arrives']} consumer arrives unfenced")
    if "outcome" in errs:
        return  # crashed or hung: caught
    assert max(errs.values()) > 1e-12 or lint["violations"], \
        f"mutant {n} ({MUTANTS[n]}) survived the probe and the SASS check: {errs}"
