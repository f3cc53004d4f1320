"""Build an A/B variant of libtbgpu.so with extra nvcc defines (tooling):

    python tools/build_variant.py NAME [-DX=Y ...]   -> paper_2509_04594_b200/libtbgpu_NAME.so

Load it with TB_LIB_VARIANT=NAME (tools/ab_bench.sh, tools/pipe_tune.py).
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04594_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = b.LIB.replace("libtbgpu.so", f"libtbgpu_{name}.so")
cmd = [b.nvcc(), *b.nvcc_flags(), *defs, *[os.path.join(b.CSRC, s) for s in b.SOURCES], "-o", out, "-lcublas",
       "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
res = subprocess.run(cmd, capture_output=True, text=True)
if res.returncode:
    sys.exit(res.stdout + res.stderr)
print(out)
