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


def test_bins_abi_argument_checks_without_gpu():
    """The binned layout's entry points validate their dtype arguments before
    any CUDA call: 48- / 80-byte leaver records for f32 / f64 particles, and
    only the (4, 4), (4, 8), (8, 8) particle / field pairs."""
    import numpy as np
    from paper_2008_04397_b200 import _lib
    L = _lib.load()
    assert L.bp_bins_leaver_bytes(4) == 48
    assert L.bp_bins_leaver_bytes(8) == 80
    assert L.bp_bins_leaver_bytes(2) == _lib.EINVAL
    gi = np.array([4, 4, 4, 0, 1, 0], np.int64)
    gg = np.zeros(6, np.float64)
    gf = np.zeros(9, np.float64)
    p = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    total = ctypes.c_int64(0)
    rc = L.bp_bins_plan(8, 4, None, None, None, 0, p(gf), p(gg), p(gi), 1.0, 64, None, None,
                        ctypes.byref(total), None)
    assert rc == _lib.EINVAL and b"binned layout" in L.bp_last_error()
    rc = L.bp_bins_export(3, None, None, None, None, 64, None, 0, None, None, None, None,
                          ctypes.byref(total), None)
    assert rc == _lib.EINVAL
