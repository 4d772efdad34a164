"""CPU-only checks of the C-ABI library: it builds for sm_100a, loads, exports every symbol
declared in include/agcn.h, and rejects bad arguments before touching a device."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "agcn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(agcn_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for want in ("agcn_plan", "agcn_spmm", "agcn_plan_ex", "agcn_plan_destroy", "agcn_plan_stats",
                 "agcn_plan_copy", "agcn_shard_bounds", "agcn_propagate_host", "agcn_last_error"):
        assert want in names


def test_library_exports_every_declared_symbol():
    from paper_2308_11825_b200 import _lib
    L = _lib.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", L._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (agcn_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    assert set(_lib.EXPORTS) == set(_declared())


def test_library_is_sm100a():
    from paper_2308_11825_b200 import _lib
    L = _lib.lib()
    out = subprocess.run(["cuobjdump", "--list-elf", L._name], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_counter():
    import paper_2308_11825_b200 as A
    assert "sm_100a" in A.version()
    assert A.launch_count() >= 0


def test_argument_errors_without_device():
    from paper_2308_11825_b200 import _lib
    L = _lib.lib()
    assert not L.agcn_plan(None, None, -1, 0)
    assert L.agcn_last_status() == 1            # AGCN_ERR_INVALID_ARG
    assert b"n and nnz" in L.agcn_last_error()
    assert not L.agcn_plan(None, None, 4, 3)
    assert L.agcn_last_status() == 1            # rowptr NULL
    assert not L.agcn_plan(ctypes.c_void_p(16), ctypes.c_void_p(16), 4, 1 << 31)
    assert L.agcn_last_status() == 1            # nnz >= 2^31
    o = _lib.Opts()
    L.agcn_default_opts(ctypes.byref(o))
    assert (o.max_block_warps, o.max_warp_nzs, o.partition, o.validate) == (12, 32, 0, 1)
    o.max_block_warps, o.max_warp_nzs = 64, 64                     # deg_bound 4096 > 2048
    assert not L.agcn_plan_ex(ctypes.c_void_p(16), ctypes.c_void_p(16), 4, 4, ctypes.byref(o))
    assert L.agcn_last_status() == 6                               # AGCN_ERR_UNSUPPORTED
    o.max_block_warps = 70000                                      # 16-bit info half overflows
    assert not L.agcn_plan_ex(ctypes.c_void_p(16), ctypes.c_void_p(16), 4, 4, ctypes.byref(o))
    assert L.agcn_last_status() == 5                               # AGCN_ERR_OVERFLOW
    assert L.agcn_spmm(None, None, None, 4, None, None) == 1
    assert L.agcn_plan_destroy(None) == 0
    assert L.agcn_pipe_submit(None, None, None, None, 4, 3, None, 4, 1, None) == 1
    assert L.agcn_pipe_wait(None) == 1
    assert L.agcn_pipe_destroy(None) == 0
    assert not L.agcn_graph_create(None, None, None, 4, 2, None, None)
    assert L.agcn_last_status() == 1
    assert L.agcn_graph_launch(None, None) == 1
    assert L.agcn_graph_destroy(None) == 0


def test_auto_partition_rule():
    """agcn_auto_partition (host-only): the per-graph Alg. 1 parameters of DESIGN.md 9 at the
    five BASELINE configs on a 148-SM B200, the rule's branch edges, and argument errors."""
    import paper_2308_11825_b200 as A
    from paper_2308_11825_b200 import _lib
    cfg = {"c1": (2708, 10556, (12, 32)), "c2": (19717, 88648, (4, 16)),
           "c3": (169343, 1166243, (8, 16)), "c4": (232965, 114615891, (8, 32)),
           "c5": (8388608, 134217728, (32, 16))}
    for name, (n, nnz, want) in cfg.items():
        assert A.auto_partition(n, nnz, 148) == want, name
    slots = 148 * 24
    assert A.auto_partition(10 ** 6, 8 * slots - 1, 148) == (12, 32)     # launch-bound: paper's
    assert A.auto_partition(10 ** 6, 8 * slots, 148) == (4, 16)
    assert A.auto_partition(10 ** 6, 320 * slots, 148) == (8, 16)        # share / 2.5 = 128
    assert A.auto_partition(10 ** 6, 640 * slots, 148) == (8, 32)        # share / 2.5 = 256
    assert A.auto_partition(10 ** 6, 960 * slots, 148) == (32, 16)       # large, mean degree < 64
    assert A.auto_partition(10 ** 4, 960 * slots, 148) == (8, 32)        # large, mean degree >= 64
    assert A.auto_partition(1000, 256 * 1000, 148) == (4, 16)             # dense but small: share rule
    assert A.auto_partition(0, 0, 148) == (12, 32)
    L = _lib.lib()
    assert L.agcn_auto_partition(-1, 0, 148, None, None) == 1


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2308_11825_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
                assert not re.search(r"#include\s+[<\"].*oracle", txt), f
                assert "liboracle" not in txt and "agcn_inputs" not in txt, f


def _build_c_example(out):
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.dirname(A_lib_path())
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", os.path.join(root, "examples", "spmm_c.c"),
           "-I", os.path.join(root, "include"), "-I", "/usr/local/cuda/include", "-L", lib, "-lagcn",
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-lm", f"-Wl,-rpath,{lib}:/usr/local/cuda/lib64", "-o", out]
    return subprocess.run(cmd, capture_output=True, text=True)


def A_lib_path():
    import paper_2308_11825_b200 as A
    return A.library_path()


def test_c_example_compiles(tmp_path):
    """examples/spmm_c.c: the C ABI used from plain C (gcc, include/agcn.h, libagcn.so)."""
    r = _build_c_example(str(tmp_path / "spmm_c"))
    assert r.returncode == 0, r.stderr
