"""Static check of the consumer's stage-release rule in the shipped SASS
(tooling + tests/test_sass_lint.py, tests/test_gpu_mutations.py).

Rule (dgemm_dmma.cuh, "Release the stage to the producer"): every consumer
empty-barrier arrive must be preceded by fence.proxy.async (SASS
FENCE.VIEW.ASYNC.S) issued after the last shared-memory fragment load (LDS)
before it, so the producer's next TMA into the stage cannot overtake a
fragment read still in flight. Walks each dgemm_dmma_kernel backwards from
every consumer arrive (the lane-0-predicated `SYNCS.ARRIVE.TRANS64.A1T0 RZ,
[Rx+URZ+off]`) and reports arrives that reach an LDS before a fence.

    python tools/sass_lint.py paper_2509_04594_b200/libtbgpu.so   -> JSON summary, rc 1 on a violation
"""
import json
import re
import subprocess
import sys

ARRIVE = re.compile(r"@!?P\d\s+SYNCS\.ARRIVE\.TRANS64\.A1T0 RZ, \[R\d+\+URZ\+0x[0-9a-f]+\]")
FENCE = re.compile(r"\bFENCE\.VIEW\.ASYNC\.S\b")
LDS = re.compile(r"\bLDS(\.\w+)*\b")


def functions(so_path: str) -> dict:
    out = subprocess.run(["cuobjdump", "-sass", so_path], capture_output=True, text=True, check=True).stdout
    funcs, name = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            name = m.group(1)
            funcs[name] = []
        elif name and re.search(r"/\*[0-9a-f]{4,}\*/", line):
            funcs[name].append(line)
    return funcs


def lint(so_path: str) -> dict:
    """{"kernels": n, "arrives": n, "violations": [(kernel, sass line), ...]}"""
    kernels = arrives = 0
    bad = []
    for name, lines in functions(so_path).items():
        if "dgemm_dmma_kernel" not in name:
            continue
        kernels += 1
        for i, line in enumerate(lines):
            if not ARRIVE.search(line):
                continue
            arrives += 1
            for j in range(i - 1, -1, -1):
                if FENCE.search(lines[j]):
                    break
                if LDS.search(lines[j]):
                    bad.append((name, line.strip()))
                    break
    return {"kernels": kernels, "arrives": arrives, "violations": bad}


if __name__ == "__main__":
    res = lint(sys.argv[1])
    print(json.dumps({"kernels": res["kernels"], "arrives": res["arrives"],
                      "violations": len(res["violations"]), "first": res["violations"][:3]}))
    sys.exit(1 if res["violations"] else 0)
