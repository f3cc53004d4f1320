"""The shipped library keeps the consumer's stage-release rule in SASS: every
consumer empty-barrier arrive of every dgemm_dmma_kernel instantiation is
preceded by FENCE.VIEW.ASYNC.S after its last fragment LDS (tools/sass_lint.py;
the -DTB_MUTATE=3 build breaks it, tests/test_gpu_mutations.py). CPU-only:
cuobjdump reads the sm_100a cubins without a device."""
import os
import shutil
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


@pytest.mark.skipif(shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"),
                    reason="cuobjdump not available")
def test_every_consumer_arrive_is_fenced():
    import sass_lint
    from paper_2509_04594_b200 import _lib

    os.environ["PATH"] = os.environ.get("PATH", "") + ":/usr/local/cuda/bin"
    _lib.lib()  # builds it if missing
    res = sass_lint.lint(_lib.LIB_PATH)
    assert res["kernels"] >= 10 and res["arrives"] >= res["kernels"] - 2, res
    assert not res["violations"], res["violations"][:3]
