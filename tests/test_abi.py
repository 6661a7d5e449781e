"""The C-ABI library loads and exports every symbol include/akv.h declares
(no compute calls: CPU only)."""

import ctypes
import os
import re
import subprocess

from paper_2310_01801_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "akv.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(akv_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_bound_symbols():
    assert _declared() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    for name in _declared():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header():
    """Compile a tiny C program against include/akv.h and compare sizeof /
    offsetof with the ctypes mirrors."""
    import tempfile

    fields = {
        "akv_profile_args": _lib.ProfileArgs,
        "akv_compact_args": _lib.CompactArgs,
        "akv_decode_args": _lib.DecodeArgs,
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "akv.h"', "int main(){"]
    for cname, cls in fields.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "t.c")
        exe = os.path.join(d, "t")
        open(src, "w").write("\n".join(lines))
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        got = dict(l.split() for l in subprocess.run([exe], capture_output=True, text=True,
                                                     check=True).stdout.splitlines())
    for cname, cls in fields.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for f, _ in cls._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(cls, f).offset, f"{cname}.{f}"


def test_compute_entry_points_fail_loudly_without_device():
    import torch

    if torch.cuda.is_available():
        return
    rc = _lib.lib.akv_device_check()
    assert rc != _lib.AKV_OK
    assert _lib.lib.akv_last_error()


def test_smoke_reference_covers_every_compared_field():
    """smoke() builds its reference from the oracle; it must carry every
    field test_gpu_parity._compare reads (a missing key only shows on the
    GPU box at round end)."""
    import ast
    import inspect

    import smoke_check
    import test_gpu_parity

    src = inspect.getsource(test_gpu_parity._compare)
    used = {n.slice.value for n in ast.walk(ast.parse(src))
            if isinstance(n, ast.Subscript) and isinstance(n.value, ast.Name) and n.value.id == "g"
            and isinstance(n.slice, ast.Constant)}
    smoke_src = inspect.getsource(smoke_check.run_smoke)
    missing = [k for k in used if f"{k}=" not in smoke_src]
    assert not missing, missing
