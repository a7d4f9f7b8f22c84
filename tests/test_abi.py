"""The C-ABI library: builds for sm_100a, loads without a GPU, exports every
symbol include/predgen_b200.h declares, and the product path refuses to run
without it (no CPU fallback)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2506_15556_b200 import _native

HEADER = Path(__file__).resolve().parent.parent / "include" / "predgen_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(ps_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _native.SIGNATURES, s


def test_struct_layouts_match_the_c_compiler(tmp_path):
    """ctypes mirrors of ps_config / ps_stats agree with gcc on every offset."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc unavailable")
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for struct, cls in (("ps_config", _native.PsConfig), ("ps_stats", _native.PsStats)):
        lines.append(f'printf("{struct} size %zu\\n", sizeof({struct}));')
        for name, _ in cls._fields_:
            lines.append(f'printf("{struct} {name} %zu\\n", offsetof({struct}, {name}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l}
    for struct, cls in (("ps_config", _native.PsConfig), ("ps_stats", _native.PsStats)):
        assert got[(struct, "size")] == ctypes.sizeof(cls)
        for name, _ in cls._fields_:
            assert got[(struct, name)] == getattr(cls, name).offset, (struct, name)


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(_native.NativeLibraryError):
        _native.load(tmp_path / "nope.so")


def test_sass_has_tcgen05_and_tma():
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists():
        pytest.skip("cuobjdump unavailable")
    sass = subprocess.run([tool, "-sass", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass
