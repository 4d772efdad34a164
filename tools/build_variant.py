#!/usr/bin/env python
"""Build a variant of libagcn.so for an A/B (loaded with AGCN_LIBRARY=...): copies csrc/ to a
scratch dir, applies literal replacements, compiles with the library's own nvcc flags.

    python tools/build_variant.py NAME FILE 'old' 'new' [FILE 'old' 'new' ...]
    -> ab_libs/libagcn_NAME.so
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2308_11825_b200 import _build  # noqa: E402

name, edits = sys.argv[1], sys.argv[2:]
tmp = tempfile.mkdtemp(prefix=f"agcn_{name}_")
src = os.path.join(tmp, "pkg", "csrc")            # internal.h includes ../../include/agcn.h
shutil.copytree(_build.CSRC, src)
shutil.copytree(_build.INCLUDE, os.path.join(tmp, "include"))
for i in range(0, len(edits), 3):
    f, old, new = edits[i:i + 3]
    p = os.path.join(src, f)
    s = open(p).read()
    assert old in s, (f, old)
    open(p, "w").write(s.replace(old, new))
out = os.path.join(ROOT, "ab_libs", f"libagcn_{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
from concurrent.futures import ThreadPoolExecutor


def one(cu):
    o = os.path.join(tmp, cu[:-3] + ".o")
    subprocess.check_call([_build._nvcc()] + _build.NVCC_FLAGS + ["-I", src, "-c", os.path.join(src, cu), "-o", o])
    return o


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(one, sorted(c for c in os.listdir(src) if c.endswith(".cu"))))
subprocess.check_call([_build._nvcc()] + _build.ARCH + ["-shared", "-o", out] + objs +
                      ["-lcudart_static", "-lrt", "-ldl", "-lpthread"])
print(out)
