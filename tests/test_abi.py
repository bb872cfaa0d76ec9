"""The C-ABI library loads and exports every symbol include/ta.h declares; the ctypes binding's
struct layouts equal the C compiler's (no GPU needed; no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2405_14866_b200 as tb
from paper_2405_14866_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ta.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^[A-Za-z_][\w \*]*?\b(ta_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    L = tb.lib(build_if_stale=True)
    names = declared_functions()
    assert len(names) >= 12, names
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_lib.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib._build.LIB], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", out, flags=re.M), n


def test_struct_layouts_match_c(tmp_path):
    structs = {"ta_intrinsics": _lib.Intrinsics, "ta_extrinsics": _lib.Extrinsics, "ta_source_view": _lib.SourceView,
               "ta_gaussians": _lib.Gaussians, "ta_raster_params": _lib.RasterParams, "ta_debug_view": _lib.DebugView,
               "ta_blend_params": _lib.BlendParams}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-o", str(exe), str(c)])
    got = dict(l.split() for l in subprocess.check_output([str(exe)], text=True).splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, (cname, f)


def test_defaults_and_status_strings():
    p = tb.default_params()
    assert abs(p.dilation - 0.3) < 1e-7 and abs(p.alpha_max - 0.99) < 1e-7
    assert p.alpha_min == ctypes.c_float(1.0 / 255.0).value and p.t_eps == ctypes.c_float(1e-4).value
    assert p.cull_sigma == 3.0 and p.flags == 0 and p.exact_exp == 1
    L = tb.lib()
    assert L.ta_status_string(0) == b"TA_OK" and L.ta_status_string(5) == b"TA_ERR_CAPACITY"
    assert b"sm_100a" in L.ta_build_info()


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(tb.TaError):
        tb.Context(0)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2405_14866_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                s = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in s and "from oracle" not in s and "taoracle" not in s, f
