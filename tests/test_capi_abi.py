"""The C-ABI library (CPU-only checks: no kernel is launched here).

* libvdi_b200.so loads and exports every entry point include/vdi_b200.h
  declares;
* the ctypes structures in _capi.py have exactly the C layout (a probe
  compiled against the header prints sizeof/offsetof);
* argument validation fails with the documented status codes before any
  device work is enqueued.
"""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2206_08660_b200 import _capi
from paper_2206_08660_b200 import build as vbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vdi_b200.h")


@pytest.fixture(scope="module")
def lib():
    vbuild.build()
    return _capi.load()


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(vdi_\w+)\(", src, re.M)))


def test_header_declares_entry_points():
    assert set(declared_functions()) == set(_capi.EXPORTS)


def test_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (vdi_\w+)", out))
    for name in declared_functions():
        assert name in exported, name
        assert hasattr(lib, name)


def test_every_entry_point_has_a_prototype(lib):
    """ctypes passes arguments by its declared prototype: an entry point with
    parameters but no argtypes would pass a struct by value (a crash)."""
    no_params = {"vdi_last_error", "vdi_abi_version"}
    for name in _capi.EXPORTS:
        if name in no_params:
            continue
        assert getattr(lib, name).argtypes, name


def test_abi_version(lib):
    assert lib.vdi_abi_version() == 8


PROBE = r"""
#include <stdio.h>
#include <stddef.h>
#include "vdi_b200.h"
#define F(T, f) printf(#T "." #f " %zu\n", offsetof(T, f));
int main(void) {
  printf("VdiGenArgs %zu\nVdiGridArgs %zu\nVdiRenderArgs %zu\n",
         sizeof(VdiGenArgs), sizeof(VdiGridArgs), sizeof(VdiRenderArgs));
  %FIELDS%
  return 0;
}
"""


def test_struct_layouts_match_header(tmp_path):
    structs = {"VdiGenArgs": _capi.VdiGenArgs, "VdiGridArgs": _capi.VdiGridArgs,
               "VdiRenderArgs": _capi.VdiRenderArgs}
    fields = "\n".join(f"F({n}, {f})" for n, s in structs.items() for f, _ in s._fields_)
    c = tmp_path / "probe.c"
    c.write_text(PROBE.replace("%FIELDS%", fields))
    exe = tmp_path / "probe"
    subprocess.run(["/usr/bin/gcc", "-I", os.path.dirname(HEADER), str(c), "-o", str(exe)],
                   check=True)
    lines = dict(l.rsplit(" ", 1) for l in
                 subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n")
                 if l)
    for n, s in structs.items():
        assert int(lines[n]) == ctypes.sizeof(s), n
        for f, _ in s._fields_:
            assert int(lines[f"{n}.{f}"]) == getattr(s, f).offset, (n, f)


def test_invalid_args_rejected_without_launch(lib):
    a = _capi.VdiGenArgs()
    assert lib.vdi_gen_launch(a, None) == -1          # null pointers
    assert b"null" in lib.vdi_last_error()
    r = _capi.VdiRenderArgs()
    assert lib.vdi_render_launch(r, None) == -1
    assert lib.vdi_segs_to_aos(None, None, 1, 0, None) == -1
    assert lib.vdi_find_first_batch(None, None, None, 0, None, None, None, None, None, 1,
                                    None) == -1


def test_size_queries_are_64_bit(lib):
    """Byte-count queries return size_t: C5-sized answers exceed 2^32 and
    must not be truncated by the binding (_capi.load sets the restypes)."""
    from paper_2206_08660_b200 import _capi
    L = _capi.load()
    assert L.vdi_lz4_workspace_bytes(10_000_000_000) > 2 ** 34
    assert L.vdi_vdi1_max_bytes(3840, 2160, 40, 240, 135, 32) == (
        160 + 2 * 3840 * 2160 + 24 * 3840 * 2160 * 40 + 4 * 240 * 135 * 32)
    assert L.vdi_lz4_max_bytes(2 ** 33) == 2 ** 33 + 2 ** 33 // 255 + 16
    assert L.vdi_volume_cells_bytes(0, 2048, 2048, 1920) == 8 * 2048 * 2048 * 1920


def test_integration_stub_matches_binding():
    """The ctypes stub INTEGRATION.md hands a maintainer has the binding's
    VdiGenArgs layout (a stale copy would pass misaligned arguments)."""
    text = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                             "INTEGRATION.md")).read()
    code = text[text.index("import ctypes\n"):text.index('lib = ctypes.CDLL("libvdi_b200.so")')]
    ns = {}
    exec(code, ns)
    stub = ns["VdiGenArgs"]
    assert [f[0] for f in stub._fields_] == [f[0] for f in _capi.VdiGenArgs._fields_]
    assert ctypes.sizeof(stub) == ctypes.sizeof(_capi.VdiGenArgs)
