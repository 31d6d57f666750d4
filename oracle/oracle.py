"""TEST INFRASTRUCTURE ONLY — ctypes front-end of the CPU oracle (oracle.cpp).

Exposes the reference kernel signatures of ``batchpic.kernels``
(``pkg/src/batchpic/kernels.py:82,310,385,458``) on top of the C++
restatement so parity tests can call the oracle and the CUDA path with the
same arguments.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU legs may import this module.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

OK = 0
ERR_RUNAWAY = 1
ERR_MIDPOINT = 2

_P = ctypes.c_void_p
_I = ctypes.c_int64
_D = ctypes.c_double
_INT = ctypes.c_int


def build(force=False):
    """Compile liboracle.so with the committed Makefile (gcc, no FMA)."""
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(src) > os.path.getmtime(_LIB_PATH)):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.or_span.restype = _INT
        L.or_span.argtypes = [_INT, _INT] + [_P] * 7 + [_I, _I] + [_P] * 4 + [
            _P, _P, _P] + [_D] * 5 + [_INT, _D, _INT, _INT, _INT, _INT]
        L.or_gather.restype = _INT
        L.or_gather.argtypes = [_INT, _INT, _P, _P, _P, _I, _I, _P, _P, _P, _P, _P]
        L.or_fused_parallel.restype = _INT
        L.or_fused_parallel.argtypes = [_INT, _INT] + [_P] * 7 + [_I, _I] + [
            _P] * 4 + [_P, _P, _P] + [_D] * 5 + [_INT, _D, _INT, _INT]
        L.or_cell_keys.restype = _INT
        L.or_cell_keys.argtypes = [_INT, _P, _P, _P, _I, _P, _P, _P, _P]
        L.or_stable_order.restype = _INT
        L.or_stable_order.argtypes = [_P, _I, _I, _P]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data if a is not None else None


def _c(a, dtype=None):
    a = np.asarray(a)
    if dtype is not None and a.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {a.dtype}")
    if not a.flags.c_contiguous:
        raise ValueError("oracle arrays must be C-contiguous")
    return a


def _geo_d(geo):
    return np.ascontiguousarray(np.asarray(geo, dtype=np.float64))


def _modes(xs, E):
    pb = np.asarray(xs).dtype.itemsize
    fb = np.asarray(E).dtype.itemsize
    return pb, fb


def fused_span(xs, ys, zs, us, vs, ws, qs, start, count, E, B, acc, invvol,
               geo_f, geo_g, geo_i, dt, dth, qdt2m, beta, one, n_iters, scale,
               mixed, scratch=None):
    """kernels.fused_span (kernels.py:458-735) restated in C++."""
    pb, fb = _modes(xs, E)
    arrs = [_c(a) for a in (xs, ys, zs, us, vs, ws, qs)]
    gf, gg = _geo_d(geo_f), _geo_d(geo_g)
    gi = _c(np.asarray(geo_i, dtype=np.int64))
    acc = _c(acc, np.int64)
    return lib().or_span(pb, fb, *[_ptr(a) for a in arrs], int(start), int(count),
                         _ptr(_c(E)), _ptr(_c(B)), _ptr(acc), _ptr(_c(invvol)),
                         _ptr(gf), _ptr(gg), _ptr(gi), float(dt), float(dth),
                         float(qdt2m), float(beta), float(one), int(n_iters),
                         float(scale), int(mixed), 1, 1, 1)


def push_span(xs, ys, zs, us, vs, ws, start, count, E, B, geo_f, geo_g, geo_i,
              dt, dth, qdt2m, beta, one, n_iters, apply_bc, mixed, scratch=None):
    """kernels.push_span (kernels.py:82-307)."""
    pb, fb = _modes(xs, E)
    arrs = [_c(a) for a in (xs, ys, zs, us, vs, ws)]
    gf, gg = _geo_d(geo_f), _geo_d(geo_g)
    gi = _c(np.asarray(geo_i, dtype=np.int64))
    return lib().or_span(pb, fb, *[_ptr(a) for a in arrs], None, int(start),
                         int(count), _ptr(_c(E)), _ptr(_c(B)), None, None,
                         _ptr(gf), _ptr(gg), _ptr(gi), float(dt), float(dth),
                         float(qdt2m), float(beta), float(one), int(n_iters),
                         0.0, int(mixed), 1, 0, int(apply_bc))


def deposit_span(xs, ys, zs, us, vs, ws, qs, start, count, acc, invvol, geo_g,
                 geo_i, one, scale):
    """kernels.deposit_span (kernels.py:310-382)."""
    pb = np.asarray(xs).dtype.itemsize
    fb = np.asarray(invvol).dtype.itemsize
    arrs = [_c(a) for a in (xs, ys, zs, us, vs, ws, qs)]
    gg = _geo_d(geo_g)
    gi = _c(np.asarray(geo_i, dtype=np.int64))
    acc = _c(acc, np.int64)
    return lib().or_span(pb, fb, *[_ptr(a) for a in arrs], int(start), int(count),
                         None, None, _ptr(acc), _ptr(_c(invvol)), _ptr(gg),
                         _ptr(gg), _ptr(gi), 0.0, 0.0, 0.0, 0.0, float(one), 0,
                         float(scale), 0, 0, 1, 0)


def gather_span(xs, ys, zs, start, count, E, B, geo_g, geo_i, one, out):
    """kernels.gather_span (kernels.py:385-455); ``out`` rows in xs dtype."""
    pb, fb = _modes(xs, E)
    out = _c(out)
    if out.dtype.itemsize != pb:
        raise TypeError("oracle gather writes rows in particle precision")
    gg = _geo_d(geo_g)
    gi = _c(np.asarray(geo_i, dtype=np.int64))
    return lib().or_gather(pb, fb, _ptr(_c(xs)), _ptr(_c(ys)), _ptr(_c(zs)),
                           int(start), int(count), _ptr(_c(E)), _ptr(_c(B)),
                           _ptr(gg), _ptr(gi), _ptr(out))


def fused_parallel(xs, ys, zs, us, vs, ws, qs, start, count, E, B, acc, invvol,
                   geo_f, geo_g, geo_i, dt, dth, qdt2m, beta, one, n_iters,
                   scale, mixed, nthreads):
    """Fused pass on ``nthreads`` host threads (private grids, integer merge)."""
    pb, fb = _modes(xs, E)
    arrs = [_c(a) for a in (xs, ys, zs, us, vs, ws, qs)]
    gf, gg = _geo_d(geo_f), _geo_d(geo_g)
    gi = _c(np.asarray(geo_i, dtype=np.int64))
    return lib().or_fused_parallel(
        pb, fb, *[_ptr(a) for a in arrs], int(start), int(count), _ptr(_c(E)),
        _ptr(_c(B)), _ptr(_c(acc, np.int64)), _ptr(_c(invvol)), _ptr(gf),
        _ptr(gg), _ptr(gi), float(dt), float(dth), float(qdt2m), float(beta),
        float(one), int(n_iters), float(scale), int(mixed), int(nthreads))


def cell_keys(x, y, z, origin, spacing, counts):
    """geometry.cell_index_of (geometry.py:152-159), f64 arithmetic."""
    x = _c(x)
    n = x.shape[0]
    keys = np.empty(n, np.int64)
    o = np.asarray(origin, np.float64)
    d = np.asarray(spacing, np.float64)
    c = np.asarray(counts, np.int64)
    rc = lib().or_cell_keys(x.dtype.itemsize, _ptr(x), _ptr(_c(y)), _ptr(_c(z)),
                            n, _ptr(o), _ptr(d), _ptr(c), _ptr(keys))
    if rc != 0:
        raise ValueError("positions below the box origin")
    return keys


def stable_order(keys, nkeys):
    """np.argsort(keys, kind='stable') for keys in [0, nkeys)."""
    keys = _c(np.asarray(keys, np.int64))
    order = np.empty(keys.shape[0], np.int64)
    if lib().or_stable_order(_ptr(keys), keys.shape[0], int(nkeys), _ptr(order)):
        raise ValueError("key out of range")
    return order
