"""The C-ABI library builds, loads without a GPU and exports every entry
point include/bp_b200.h declares (no compute calls here)."""

import ctypes
import os
import re

from conftest import ROOT


def _declared():
    text = open(os.path.join(ROOT, "include", "bp_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|long long|const char\*)\s+(bp_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = _declared()
    assert "bp_fused_span" in names and "bp_sort_by_cell" in names
    from paper_2008_04397_b200 import _lib
    assert sorted(_lib.EXPORTS) == names


def test_library_exports_every_declared_symbol():
    from paper_2008_04397_b200 import _lib
    lib = _lib.load()
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(raw, name), name
    assert lib.bp_version() >= 100
    assert lib.bp_last_error() == b""


def test_kernel_objects_are_sm100a():
    # the fatbin carries sm_100a SASS (cuobjdump lists the ELF arch)
    import shutil
    import subprocess
    from paper_2008_04397_b200 import _lib
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        return
    out = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _param_counts():
    """Parameter count of every declaration in include/bp_b200.h."""
    text = open(os.path.join(ROOT, "include", "bp_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    out = {}
    for m in re.finditer(r"^\s*(?:int|int64_t|long long|const char\*)\s+(bp_\w+)\s*\(([^)]*)\)\s*;",
                         text, re.M):
        args = m.group(2).strip()
        out[m.group(1)] = 0 if args in ("", "void") else args.count(",") + 1
    return out


def test_ctypes_signatures_match_header():
    # a wrong argtypes length silently shifts every later argument
    from paper_2008_04397_b200 import _lib
    counts = _param_counts()
    assert set(counts) == set(_lib.EXPORTS)
    for name, (_res, argtypes) in _lib._SIGS.items():
        assert len(argtypes) == counts[name], (name, len(argtypes), counts[name])
