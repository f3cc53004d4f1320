"""Per-kernel SASS comparison of two builds (tooling): lists kernels whose
SASS differs (ignoring addresses/file identifiers), to confirm a change did
not perturb the production kernels.   python tools/sass_diff.py old.so new.so"""
import re
import subprocess
import sys


def kernels(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    funcs, name = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            name = re.sub(r"_GLOBAL__N__[0-9a-f]+_", "G_", m.group(1))
            funcs[name] = []
            continue
        if name:
            funcs[name].append(re.sub(r"/\*[0-9a-f]{4,}\*/", "", line).rstrip())
    return funcs


a, b = kernels(sys.argv[1]), kernels(sys.argv[2])
same = [k for k in a if k in b and a[k] == b[k]]
diff = [k for k in a if k in b and a[k] != b[k]]
print(f"{len(same)} identical, {len(diff)} differ, {len(set(a) ^ set(b))} only in one")
for k in diff:
    print("DIFF", k[:160])
for k in set(a) ^ set(b):
    print("ONLY", k[:160])
