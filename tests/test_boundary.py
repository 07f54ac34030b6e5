"""CPU-side checks of the C-ABI boundary: the library loads and exports every
symbol include/bbmm.h declares; the header and the binding agree.  No compute
calls (no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "bbmm.h")
LIB = os.path.join(ROOT, "paper_1809_11165_b200", "lib", "libbbmm.so")


def declared_symbols():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:bbmm_status_t|const char \*)\s*(bbmm_\w+)\s*\(", src, re.M)))


def test_header_declares_the_north_star_entry_points():
    syms = declared_symbols()
    for s in ("bbmm_pivchol", "bbmm_mbcg", "bbmm_mll_and_grad", "bbmm_kernel_matmul",
              "bbmm_ctx_create", "bbmm_ctx_destroy", "bbmm_ctx_set_comm", "bbmm_nccl_unique_id"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        from paper_1809_11165_b200 import _build
        _build.build()
    lib = ctypes.CDLL(LIB)
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_binding_loads_and_reports_version():
    import paper_1809_11165_b200 as b
    assert "sm_100a" in b.version()


def test_library_is_sm100a_native():
    """The .so carries sm_100a SASS (no PTX-JIT fallback for another arch)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_binding_fails_loudly_without_gpu():
    import torch
    import paper_1809_11165_b200 as b
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(b.BBMMError):
        b.Context()


def test_oracle_not_imported_by_product():
    pkg = os.path.join(ROOT, "paper_1809_11165_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "bbmm_oracle" not in txt and "liboracle" not in txt, f


def test_row_partition_matches_python_mirror():
    # the C partition (bbmm_row_partition, used by every multi-rank call) == the binding's
    # row_partition used by the gloo multi-rank tests: contiguous, disjoint, covering,
    # 128-aligned rank boundaries
    lib = ctypes.CDLL(LIB)
    lib.bbmm_row_partition.restype = ctypes.c_int
    from paper_1809_11165_b200 import row_partition
    r0, r1, nb = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    for n in (0, 1, 127, 128, 129, 1000, 3338, 45730, 200000, 1000000, 1000003):
        for G in (1, 2, 3, 4, 7, 8):
            end = 0
            for r in range(G):
                st = lib.bbmm_row_partition(ctypes.c_int64(n), G, r, ctypes.byref(r0), ctypes.byref(r1),
                                            ctypes.byref(nb))
                assert st == 0
                assert (r0.value, r1.value, nb.value) == tuple(row_partition(n, G, r))
                assert r0.value == end and r1.value >= r0.value
                assert r0.value % 128 == 0 or r0.value == n
                end = r1.value
            assert end == n
    assert lib.bbmm_row_partition(ctypes.c_int64(10), 2, 2, ctypes.byref(r0), ctypes.byref(r1), None) != 0
