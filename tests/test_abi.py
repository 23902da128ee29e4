"""C-ABI boundary checks that need no GPU: libsofa.so builds, loads, exports every entry point
include/sofa.h declares, the ctypes struct layouts match the C compiler's, and argument
validation returns the documented error codes before touching the device."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2411_17483_b200 import build, sofa

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sofa.h")


@pytest.fixture(scope="module")
def L():
    build.build_library()
    return sofa.lib()


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sofa_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(L):
    names = declared_functions()
    assert len(names) >= 13
    for n in names:
        assert hasattr(L, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", build.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sofa_\w+)", out))
    assert set(names) <= exported


def test_struct_layouts_match_c(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text("""
#include <stdio.h>
#include <stddef.h>
#include "sofa.h"
int main(void){
  printf("%zu %zu %zu %zu %zu\\n", sizeof(sofa_model), sizeof(sofa_build_opts), sizeof(sofa_knn_stats),
         sizeof(sofa_index_info), offsetof(sofa_model, edges));
  printf("%zu %zu\\n", offsetof(sofa_build_opts, model), offsetof(sofa_build_opts, global_n));
  return 0; }
""")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    a, b = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")[:2]
    sizes = list(map(int, a.split()))
    assert sizes == [ctypes.sizeof(sofa.sofa_model), ctypes.sizeof(sofa.sofa_build_opts),
                     ctypes.sizeof(sofa.sofa_knn_stats), ctypes.sizeof(sofa.sofa_index_info),
                     sofa.sofa_model.edges.offset]
    assert list(map(int, b.split())) == [sofa.sofa_build_opts.model.offset, sofa.sofa_build_opts.global_n.offset]


def test_default_opts(L):
    o = sofa.sofa_default_opts()
    assert o.sample_ratio == 0.01 and o.block_size == 256 and o.binning == 0 and not o.model


@pytest.mark.parametrize("len_,l,a,msg", [(3, 2, 4, "len"), (10, 2, 4, "len"), (2048, 16, 256, "len"),
                                          (256, 0, 256, "l must"), (256, 65, 256, "l must"), (8, 8, 4, "l must"),
                                          (256, 16, 3, "alphabet"), (256, 16, 512, "alphabet"),
                                          (256, 16, 1, "alphabet")])
def test_build_rejects_bad_shapes(L, len_, l, a, msg):
    h = ctypes.c_void_p()
    rc = L.sofa_build(None, 10, len_, l, a, None, None, ctypes.byref(h))
    assert rc == -1 and msg in sofa.sofa_last_error() and not h.value


def test_build_rejects_bad_opts(L):
    o = sofa.sofa_default_opts()
    o.block_size = 100
    h = ctypes.c_void_p()
    assert L.sofa_build(ctypes.c_void_p(16), 10, 256, 16, 256, ctypes.byref(o), None, ctypes.byref(h)) == -1
    assert "block_size" in sofa.sofa_last_error()
    o = sofa.sofa_default_opts()
    assert L.sofa_build(None, 0, 256, 16, 256, ctypes.byref(o), None, ctypes.byref(h)) == -1
    assert "model" in sofa.sofa_last_error()
    m = sofa.sofa_model()
    m.len, m.l, m.alphabet = 128, 16, 256
    o.model = ctypes.pointer(m)
    assert L.sofa_build(None, 0, 256, 16, 256, ctypes.byref(o), None, ctypes.byref(h)) == -1
    assert "disagrees" in sofa.sofa_last_error()
    o = sofa.sofa_default_opts()
    o.binning = sofa.BINNING["isax"]  # iSAX segments need n % l == 0
    assert L.sofa_build(ctypes.c_void_p(16), 10, 248, 16, 256, ctypes.byref(o), None, ctypes.byref(h)) == -1
    assert "iSAX" in sofa.sofa_last_error()
    o.binning = 7
    assert L.sofa_build(ctypes.c_void_p(16), 10, 256, 16, 256, ctypes.byref(o), None, ctypes.byref(h)) == -1
    assert "binning" in sofa.sofa_last_error()


def test_knn_and_merge_reject_bad_args(L):
    assert L.sofa_knn(None, None, 1, 1, None, None, None, None, None) == -1
    assert L.sofa_merge_topk(None, None, 0, 1, 1, None, None, None) == -1
    assert "parts" in sofa.sofa_last_error()
    assert L.sofa_merge_topk(ctypes.c_void_p(16), ctypes.c_void_p(16), 2, 1, 129, ctypes.c_void_p(16),
                             ctypes.c_void_p(16), None) == -1
    with pytest.raises(sofa.SofaError):
        sofa.sofa_merge_topk(None, None, 0, 1, 1, None, None, stream=0)
    m = sofa.sofa_model()
    assert L.sofa_transform(None, 5, ctypes.byref(m), None, None, None) == -1
    assert L.sofa_kernel_timing(None, 1, None, None) == -1 and "NULL" in sofa.sofa_last_error()
