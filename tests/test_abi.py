"""The C-ABI boundary (include/gr.h) without a GPU: the library loads, exports
every declared symbol, rejects bad arguments on the host, and is a native
sm_100a build whose SASS shows the bulk-copy (TMA) path.  No compute call."""
import ctypes as C
import os
import re
import shutil
import subprocess

import pytest

from paper_2011_08373_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gr.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"//[^\n]*", "", src)
    names = set(re.findall(r"\b(gr_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


def test_header_declares_the_boundary():
    names = declared_functions()
    for f in ("gr_solve_pms", "gr_mhs_exact", "gr_mhs_greedy", "gr_mhs_greedy_matrix"):
        assert f in names
    assert sorted(names) == sorted(N.EXPORTED)


def test_library_loads_and_exports_every_symbol():
    L = N.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    if shutil.which("nm"):
        out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True,
                             text=True).stdout
        for name in declared_functions():
            assert re.search(rf"\bT {name}\b", out), name


def test_version_and_host_validation():
    L = N.lib()
    assert N.version().startswith("grsolve")
    assert L.gr_workspace_bytes(None, 0) == 0
    assert L.gr_solve_pms(None, None, None, 0, None) == N.GR_EINVAL
    assert L.gr_mhs_exact(None, None, None, 0, None) == N.GR_EINVAL
    assert L.gr_mhs_greedy(None, None, None, 0, None) == N.GR_EINVAL
    assert L.gr_mhs_greedy_matrix(None, None, None, None, None, None, 0, None) == N.GR_EINVAL
    # the column-sharded greedy protocol rejects a missing shard
    assert L.gr_greedy_shard_workspace_bytes(None) == 0
    assert L.gr_greedy_shard_begin(None, None, None, 0, None) == N.GR_EINVAL
    assert L.gr_greedy_shard_step(None, None, None, 0, None) == N.GR_EINVAL
    assert L.gr_greedy_shard_state(None, None, 0, None, None, None, None) == N.GR_EINVAL
    assert L.gr_greedy_shard_private(None, -1, None, None, 0, None) == N.GR_EINVAL
    assert L.gr_greedy_shard_remove(None, 0, None, 0, None) == N.GR_EINVAL
    assert L.gr_greedy_shard_finalize(None, None, None, None, None, 0, None) == N.GR_EINVAL
    assert L.gr_last_error()
    b = N.GrBatch(0, 1, 0, 0, 0, None, None, None, None, None, 0, None)
    assert L.gr_workspace_bytes(C.byref(b), 0) == 0  # B < 1
    b = N.GrBatch(4, 3, 0, 0, 0, 1, 1, 1, 1, None, 0, None)
    assert L.gr_workspace_bytes(C.byref(b), 0) == 0  # W = 3
    b = N.GrBatch(4, 1, 100, 10, 0, 1, 1, 1, 1, None, 0, None)
    assert L.gr_workspace_bytes(C.byref(b), 0) > 0
    assert L.gr_workspace_bytes(C.byref(b), 2) > 0
    # max_clauses beyond the exact solvers' limit is a call-level error
    b = N.GrBatch(4, 1, 100, 5000, 0, 1, 1, 1, 1, None, 0, None)
    r = N.GrResult(1, 1, 1, None)
    assert L.gr_solve_pms(C.byref(b), C.byref(r), 1, 1 << 40, None) == N.GR_ETOOBIG
    # workspace too small
    b = N.GrBatch(4, 1, 100, 10, 0, 1, 1, 1, 1, None, 0, None)
    assert L.gr_solve_pms(C.byref(b), C.byref(r), 1, 8, None) == N.GR_EWORKSPACE
    assert N.bitmatrix_ld(1) == 64
    assert N.bitmatrix_ld(64 * 64) == 64
    assert N.bitmatrix_ld(64 * 64 + 1) == 128


def test_product_path_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2011_08373_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
                assert "oracle.c" not in src and "liboracle" not in src, f


@pytest.mark.skipif(not shutil.which("cuobjdump"), reason="cuobjdump not available")
def test_native_sm100a_build_with_bulk_copies():
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass  # cp.async.bulk (TMA bulk copy) in the greedy count pass
    assert "POPC" in sass
