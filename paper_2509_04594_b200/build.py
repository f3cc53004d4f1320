"""In-tree build of the CUDA C-ABI library ``libtbgpu.so`` for sm_100a.

    python -m paper_2509_04594_b200.build        # or __graft_entry__.build()

The .so is written next to this file so it travels to the GPU box with the
repo snapshot (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtbgpu.so")
SOURCES = ["tb_capi.cu"]
DEPS = ["tb_capi.cu", "tb_state.cuh", "tb_launch.cuh", "tb_pipeline.cuh", "tb_staging.cuh", "tb_mgpu.cuh", "dgemm_dmma.cuh", "dgemm_paper.cuh", "ptx.cuh"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; set NVCC")


def nvcc_flags() -> list[str]:
    return [
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-std=c++17", "-lineinfo",
        "-Xptxas", "-v",
        "-Xcompiler", "-fPIC,-fvisibility=hidden",
        "-shared",
        "-I", os.path.join(ROOT, "include"),
    ]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, d) for d in DEPS] + [os.path.join(ROOT, "include", "tbgpu.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, timeline: bool = False) -> str:
    """Build libtbgpu.so; ``timeline=True`` builds the instrumented tooling
    variant libtbgpu_timeline.so (-DTB_TIMELINE: per-CTA %globaltimer stamps)."""
    lib = LIB.replace("libtbgpu.so", "libtbgpu_timeline.so") if timeline else LIB
    if not force and not timeline and not stale():
        return LIB
    cmd = [nvcc(), *nvcc_flags(), *(["-DTB_TIMELINE"] if timeline else []), *[os.path.join(CSRC, s) for s in SOURCES],
           "-o", lib + ".tmp", "-lcublas", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = res.stdout + res.stderr
    with open(os.path.join(HERE, "build_timeline.log" if timeline else "build.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + log)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{log}")
    os.replace(lib + ".tmp", lib)
    if verbose:
        print(log)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, timeline="--timeline" in sys.argv))
