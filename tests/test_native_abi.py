"""The C-ABI library loads and exports every symbol include/tvstencil.h
declares, and the ctypes struct layouts match the C compiler's (CPU only —
no compute calls)."""

from __future__ import annotations

import ctypes
import os
import re
import subprocess
import tempfile

from paper_2010_04868_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tvstencil.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tvs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.library_path())
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_native._SIGS), set(names) ^ set(_native._SIGS)


def test_struct_layouts_match_c():
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "tvstencil.h"
int main(void) {
  printf("%zu %zu %zu %zu\n", sizeof(tvs_stencil), sizeof(tvs_layout), sizeof(tvs_exec), sizeof(tvs_geometry));
  printf("%zu %zu %zu\n", offsetof(tvs_stencil, coeffs), offsetof(tvs_stencil, boundary), offsetof(tvs_geometry, origin));
  printf("%zu %zu %zu\n", sizeof(tvs_life_rule), offsetof(tvs_life_rule, birth_mask), offsetof(tvs_life_rule, boundary));
  printf("%zu %zu %zu %zu\n", sizeof(tvs_problem), offsetof(tvs_problem, boundary), offsetof(tvs_problem, coeffs),
         offsetof(tvs_problem, offset));
  printf("%zu %zu %zu\n", sizeof(tvs_exec), offsetof(tvs_exec, n_gpus), offsetof(tvs_exec, flags));
  printf("%zu\n", sizeof(tvs_shard_handle));
  return 0;
}
'''
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "s.c")
        exe = os.path.join(d, "s")
        open(src, "w").write(prog)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, src], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.split()
    sizes = [int(x) for x in out]
    assert sizes[:4] == [ctypes.sizeof(_native.Stencil), ctypes.sizeof(_native.Layout),
                         ctypes.sizeof(_native.Exec), ctypes.sizeof(_native.Geometry)]
    assert sizes[4:7] == [_native.Stencil.coeffs.offset, _native.Stencil.boundary.offset,
                          _native.Geometry.origin.offset]
    assert sizes[7:10] == [ctypes.sizeof(_native.LifeRule), _native.LifeRule.birth_mask.offset,
                           _native.LifeRule.boundary.offset]
    assert sizes[10:14] == [ctypes.sizeof(_native.Problem), _native.Problem.boundary.offset,
                            _native.Problem.coeffs.offset, _native.Problem.offset.offset]
    assert sizes[14:17] == [ctypes.sizeof(_native.Exec), _native.Exec.n_gpus.offset, _native.Exec.flags.offset]
    assert sizes[17] == ctypes.sizeof(_native.ShardHandle)


def test_host_only_entry_points():
    lib = _native.lib()
    assert b"sm_100a" in lib.tvs_version()
    g = _native.geometry(2, (100, 37))
    assert g.strides[1] == 1 and g.strides[0] % 32 == 0 and g.origin % 32 == 0
    assert g.alloc_elems == 102 * g.strides[0]
    g3 = _native.geometry(3, (4, 5, 6), axis0_offset=-2, axis0_global=10)
    assert g3.axis0_offset == -2 and g3.axis0_global == 10 and g3.strides[0] == 7 * g3.strides[1]
    assert _native.device_count() >= 0


def test_product_path_never_imports_oracle():
    """No CPU fallback: nothing under the package references oracle/."""
    pkg = os.path.join(ROOT, "paper_2010_04868_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
