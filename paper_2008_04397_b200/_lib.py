"""ctypes binding of libbp_b200.so (the C ABI declared in include/bp_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2008_04397_b200/csrc``).  There is no fallback: if the
library is missing or CUDA is unavailable every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbp_b200.so")

OK = 0
ERR_RUNAWAY = 1
ERR_MIDPOINT = 2
ERR_DOMAIN = 3
EINVAL = -1
ECUDA = -2
ARITH_PARITY = 0
ARITH_FAST = 1

# every symbol include/bp_b200.h declares (checked by tests/test_capi_symbols.py)
EXPORTS = (
    "bp_version", "bp_last_error", "bp_kernel_launches", "bp_fused_span", "bp_push_span",
    "bp_deposit_span", "bp_gather_span", "bp_fused_span_ex",
    "bp_fused_span_host", "bp_sort_by_cell", "bp_sort_by_cell_into", "bp_cell_keys",
    "bp_fold_periodic_i64", "bp_moments_total", "bp_susceptibility",
    "bp_field_records_bytes", "bp_field_records_build", "bp_fused_span_rec",
    "bp_timing_enable", "bp_timing_read",
    "bp_bins_leaver_bytes", "bp_bins_plan", "bp_bins_fill", "bp_bins_cycle", "bp_bins_export",
    "bp_bins_reslack", "bp_init_maxwellian",
)

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_INT = ctypes.c_int

_SIGS = {
    "bp_version": (_INT, []),
    "bp_last_error": (ctypes.c_char_p, []),
    "bp_kernel_launches": (ctypes.c_longlong, []),
    "bp_fused_span": (_INT, [_INT, _INT] + [_P] * 7 + [_I64, _I64] + [_P] * 4
                      + [_P, _P, _P] + [_D] * 5 + [_INT, _D, _INT, _P, _P]),
    "bp_fused_span_ex": (_INT, [_INT, _INT, _INT] + [_P] * 7 + [_I64, _I64]
                         + [_P] * 4 + [_P, _P, _P] + [_D] * 5
                         + [_INT, _D, _INT, _P, _P]),
    "bp_fused_span_rec": (_INT, [_INT, _INT, _INT] + [_P] * 7 + [_I64, _I64]
                          + [_P] * 4 + [_P, _P, _P] + [_D] * 5
                          + [_INT, _D, _INT, _P, _P, _P]),
    "bp_field_records_bytes": (_I64, [_INT, _P]),
    "bp_timing_enable": (_INT, [_INT]),
    "bp_timing_read": (_INT, [_P, _P, _INT]),
    "bp_field_records_build": (_INT, [_INT, _INT, _P, _P, _P, _P, _P]),
    "bp_push_span": (_INT, [_INT, _INT] + [_P] * 6 + [_I64, _I64, _P, _P]
                     + [_P, _P, _P] + [_D] * 5 + [_INT, _INT, _INT, _P, _P]),
    "bp_deposit_span": (_INT, [_INT, _INT] + [_P] * 7 + [_I64, _I64, _P, _P,
                                                        _P, _P, _D, _D, _P, _P]),
    "bp_gather_span": (_INT, [_INT, _INT, _P, _P, _P, _I64, _I64, _P, _P, _P,
                              _P, _D, _P, _P, _P]),
    "bp_fused_span_host": (_INT, [_INT, _INT, _INT] + [_P] * 7 + [_I64, _I64]
                           + [_P] * 4 + [_P, _P, _P] + [_D] * 5
                           + [_INT, _D, _INT, _I64]),
    "bp_sort_by_cell": (_INT, [_INT] + [_P] * 7 + [_P, _I64, _P, _P, _P, _P]),
    "bp_sort_by_cell_into": (_INT, [_INT, _P, _P, _P, _P, _I64, _P, _P, _P, _P]),
    "bp_cell_keys": (_INT, [_INT, _P, _P, _P, _I64, _P, _P, _P, _P, _P]),
    "bp_fold_periodic_i64": (_INT, [_P, _I64, _P, _P]),
    "bp_moments_total": (_INT, [_P, _INT, _I64, _P, _P]),
    "bp_susceptibility": (_INT, [_P, _P, _INT, _INT, _D, _D, _I64, _P, _P]),
    "bp_bins_leaver_bytes": (_INT, [_INT]),
    "bp_bins_plan": (_INT, [_INT, _INT, _P, _P, _P, _I64, _P, _P, _P, _D, _INT, _P, _P, _P, _P]),
    "bp_bins_fill": (_INT, [_INT, _INT] + [_P] * 8 + [_I64, _P, _P, _P, _P, _P, _P, _P]),
    "bp_bins_cycle": (_INT, [_INT, _INT] + [_P] * 4 + [_I64, _P, _I64, _P, _I64, _P, _I64, _P, _P,
                                                  _P, _P]
                      + [_P, _P, _P] + [_D] * 5 + [_INT, _D, _P, _P]),
    "bp_init_maxwellian": (_INT, [_INT, ctypes.c_uint64, ctypes.c_uint64] + [_P] * 3
                           + [_INT] + [_P] * 3 + [_I64, _I64] + [_P] * 10 + [_I64, _P, _P]),
    "bp_bins_export": (_INT, [_INT, _P, _P, _P, _P, _I64, _P, _I64, _P, _P, _P, _P, _P, _P]),
    "bp_bins_reslack": (_INT, [_INT, _P, _P, _P, _P, _I64, _P, _I64, _P, _D, _INT, _P, _P, _P, _P, _P,
                               _P]),
}

_lib = None


class BackendError(RuntimeError):
    """The CUDA library is missing or a call failed at the CUDA level."""


def load():
    """Load libbp_b200.so (no GPU needed to load; calls need one)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise BackendError(
            f"{LIB_PATH} is not built; run __graft_entry__.build() or "
            f"make -C {os.path.join(_HERE, 'csrc')}")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


TIMED_KERNELS = ("mover", "deposit", "records", "span")


def timing_read():
    """{class: (ms, launches)} of the library's timed kernels since the last
    read (bp_timing_enable(1) first)."""
    ms = (ctypes.c_double * len(TIMED_KERNELS))()
    cnt = (ctypes.c_longlong * len(TIMED_KERNELS))()
    load().bp_timing_read(ms, cnt, len(TIMED_KERNELS))
    return {k: (ms[i], cnt[i]) for i, k in enumerate(TIMED_KERNELS)}


def last_error():
    return load().bp_last_error().decode(errors="replace")


def check(rc, what):
    """Raise for negative (call-level) return codes; pass statuses through."""
    if rc < 0:
        kind = "invalid argument" if rc == EINVAL else "CUDA failure"
        raise BackendError(f"{what}: {kind}: {last_error()}")
    return rc
