"""compute-sanitizer over the C ABI on a B200 (SURVEY.md §5 race detection):
memcheck (out-of-bounds TMA/cp.async/epilogue), racecheck (shared-memory
hazards between the producer ring and the consumers), synccheck (barrier
misuse). The reference checks races with barrier-mutation tests on its
shuffled simulator (barriers.test.ts:84-118); on hardware the sanitizer is
the equivalent."""
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2509_04594_b200")


@pytest.fixture(scope="module")
def driver(tmp_path_factory):
    from paper_2509_04594_b200 import _lib

    _lib.lib()
    out = str(tmp_path_factory.mktemp("san") / "sanitize_driver")
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    subprocess.run([nvcc, "-O2", "-I", os.path.join(ROOT, "include"), "-o", out,
                    os.path.join(ROOT, "tools", "sanitize_driver.cu"), "-L", PKG, "-ltbgpu",
                    "-Xlinker", f"-rpath,{PKG}"], check=True)
    return out


def _sanitizer():
    for cand in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if cand and os.path.exists(cand):
            return cand
    pytest.fail("compute-sanitizer not found")


def test_driver_plain(driver):
    res = subprocess.run([driver, "--pipeline", "--mgpu"], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr


@pytest.mark.parametrize("bm", ["", "128"])
@pytest.mark.parametrize("tool,args", [("memcheck", ["--pipeline", "--mgpu"]), ("synccheck", ["--mgpu"]), ("racecheck", ["--tma-only"])])
def test_sanitizer_clean(driver, tool, args, bm):
    """racecheck runs on the TMA-fed variants and the paper kernel only: it
    tracks 8-byte cp.async shared writes but not the mbarrier arrive/wait that
    orders them against the consumers' reads, so the cp.async loader (ordered
    by cp.async.wait_group + mbarrier release/acquire, dgemm_dmma.cuh) shows
    false hazards. Its correctness is covered by memcheck/synccheck here and by
    the bitwise-repeatability and parity tests."""
    env = dict(os.environ, TB_BM=bm)  # "": choose_bm picks 64-row tiles for these shapes; "128" forces 128
    res = subprocess.run([_sanitizer(), "--tool", tool, "--error-exitcode", "3", driver, *args],
                         capture_output=True, text=True, timeout=900, env=env)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-2000:]


@pytest.mark.parametrize("tile", ["128x64", "128x96", "96x128", "96x96", "96x96t", "64x64", "64x64d", "64x96",
                                  "64x128d"])
@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_sanitizer_clean_every_tile_shape(driver, tool, tile):
    """Every tile shape the cost model can pick (TB_TILE forces it on the
    driver's TMA-fed calls: split-K fixups on these small shapes, ragged
    edges, early stage release): memcheck and racecheck clean."""
    env = dict(os.environ, TB_TILE=tile)
    res = subprocess.run([_sanitizer(), "--tool", tool, "--error-exitcode", "3", driver, "--tma-only"],
                         capture_output=True, text=True, timeout=900, env=env)
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-2000:]
