"""Drop-in replacement of ``batchpic.kernels`` running on the B200.

Same names, positional signatures, status codes and in-place semantics as
the reference module (``pkg/src/batchpic/kernels.py``):

* ``fused_span``  (kernels.py:458-735)  mover + boundary + 10-moment deposit
* ``push_span``   (kernels.py:82-307)   mover only
* ``deposit_span``(kernels.py:310-382)  deposit only
* ``gather_span`` (kernels.py:385-455)  E/B samples
* ``make_geo_arrays`` (:57-67), ``kernel_scalars`` (:70-79), ``OK``,
  ``ERR_RUNAWAY``, ``ERR_MIDPOINT``, ``BC_PERIODIC``, ``BC_REFLECTING``.

Arrays may be numpy arrays (host; the call stages them through the device
and writes results back in place — for ``fused_span`` this is the C ABI's
batched host pipeline ``bp_fused_span_host``) or CUDA torch tensors
(device-resident; no copies, launched on the tensor's current stream).  The
return value is the worst particle status, as in the reference.  The
``scratch`` argument exists for signature compatibility; the GPU rounds the
mixed-mode sample in registers.

``arith`` (keyword-only, default "parity") selects the bitwise-reference
arithmetic or the FMA / native-f32 "fast" kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

OK = _lib.OK
ERR_RUNAWAY = _lib.ERR_RUNAWAY
ERR_MIDPOINT = _lib.ERR_MIDPOINT
ERR_DOMAIN = _lib.ERR_DOMAIN

BC_PERIODIC = 0
BC_REFLECTING = 1

_ARITH = {"parity": _lib.ARITH_PARITY, "fast": _lib.ARITH_FAST}


def make_geo_arrays(geom, dtype):
    """Pack geometry: (dx dy dz ox oy oz Lx Ly Lz) in ``dtype`` and
    (nx ny nz bcx bcy bcz) int64 — the layout of kernels.py:57-67."""
    geo_f = np.array([geom.dx, geom.dy, geom.dz,
                      geom.origin[0], geom.origin[1], geom.origin[2],
                      geom.Lx, geom.Ly, geom.Lz], dtype=dtype)
    bc = [BC_PERIODIC if k == "periodic" else BC_REFLECTING for k in geom.bc]
    geo_i = np.array([geom.nx, geom.ny, geom.nz] + bc, dtype=np.int64)
    return geo_f, geo_i


def kernel_scalars(species, dt, c, particle_dtype):
    """dt, dt/2, qom*dt/2, qom*dt/(2c), 1 — computed in f64, cast to the
    particle dtype (kernels.py:70-79)."""
    pd = particle_dtype
    return {"dt": pd(dt), "dth": pd(dt / 2.0), "qdt2m": pd(species.qom * dt / 2.0),
            "beta": pd(species.qom * dt / (2.0 * c)), "one": pd(1.0)}


# ----------------------------------------------------------------- helpers

def _torch():
    import torch
    return torch


def _is_dev(a):
    if isinstance(a, np.ndarray) or a is None:
        return False
    t = _torch()
    return isinstance(a, t.Tensor) and a.is_cuda


def _nbytes_of(a):
    if isinstance(a, np.ndarray):
        return a.dtype.itemsize
    return a.element_size()


def _dptr(t):
    if not t.is_contiguous():
        raise ValueError("device arrays must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream_of(t):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _geo(g):
    return np.ascontiguousarray(np.asarray(g, dtype=np.float64))


def _geoi(g):
    return np.ascontiguousarray(np.asarray(g, dtype=np.int64))


def _hp(a):
    return ctypes.c_void_p(a.ctypes.data)


def _check_host(*arrs):
    for a in arrs:
        if not isinstance(a, np.ndarray):
            raise TypeError("mix of host and device arrays")
        if not a.flags.c_contiguous:
            raise ValueError("host arrays must be C-contiguous")


def _check_dev(*arrs):
    for a in arrs:
        if not _is_dev(a):
            raise TypeError("mix of host and device arrays")


def _span_ok(n, start, count):
    if start < 0 or count < 0 or start + count > n:
        raise IndexError(f"span ({start}, {count}) outside array of {n}")


class _Staged:
    """Host numpy arrays staged onto the current CUDA device (torch owns the
    memory); ``back`` copies the named arrays' span into the originals."""

    def __init__(self):
        self.torch = _torch()
        self.dev = self.torch.device("cuda", self.torch.cuda.current_device())

    def put(self, a, sl=None):
        src = a if sl is None else a[sl]
        return self.torch.from_numpy(np.ascontiguousarray(src)).to(self.dev)

    def back(self, host, dev, sl=None):
        out = dev.cpu().numpy()
        if sl is None:
            host[...] = out
        else:
            host[sl] = out


# ----------------------------------------------------------------- kernels

def fused_span(xs, ys, zs, us, vs, ws, qs, start, count, E, B, acc, invvol,
               geo_f, geo_g, geo_i, dt, dth, qdt2m, beta, one, n_iters, scale,
               mixed, scratch=None, *, arith="parity", d_status=None,
               batch_particles=0):
    """Fused mover + interpolation over [start, start+count) (in place)."""
    L = _lib.load()
    pb, fb = _nbytes_of(xs), _nbytes_of(E)
    gf, gg, gi = _geo(geo_f), _geo(geo_g), _geoi(geo_i)
    mode = _ARITH[arith]
    start, count = int(start), int(count)
    if _is_dev(xs):
        _check_dev(ys, zs, us, vs, ws, qs, E, B, acc, invvol)
        _span_ok(xs.shape[0], start, count)
        rc = L.bp_fused_span_ex(
            mode, pb, fb, *[_dptr(a) for a in (xs, ys, zs, us, vs, ws, qs)],
            start, count, _dptr(E), _dptr(B), _dptr(acc), _dptr(invvol),
            _hp(gf), _hp(gg), _hp(gi), float(dt), float(dth), float(qdt2m),
            float(beta), float(one), int(n_iters), float(scale), int(mixed),
            None if d_status is None else _dptr(d_status), _stream_of(xs))
        return _lib.check(rc, "fused_span")
    _check_host(xs, ys, zs, us, vs, ws, qs, E, B, acc, invvol)
    _span_ok(xs.shape[0], start, count)
    if acc.dtype != np.int64:
        raise TypeError("acc must be int64")
    rc = L.bp_fused_span_host(
        mode, pb, fb, *[_hp(a) for a in (xs, ys, zs, us, vs, ws, qs)], start, count,
        _hp(E), _hp(B), _hp(acc), _hp(invvol), _hp(gf), _hp(gg), _hp(gi),
        float(dt), float(dth), float(qdt2m), float(beta), float(one),
        int(n_iters), float(scale), int(mixed), int(batch_particles))
    return _lib.check(rc, "fused_span")


def push_span(xs, ys, zs, us, vs, ws, start, count, E, B, geo_f, geo_g, geo_i,
              dt, dth, qdt2m, beta, one, n_iters, apply_bc, mixed, scratch=None,
              *, d_status=None):
    """Implicit mover over a span; boundaries only with ``apply_bc``."""
    L = _lib.load()
    pb, fb = _nbytes_of(xs), _nbytes_of(E)
    gf, gg, gi = _geo(geo_f), _geo(geo_g), _geoi(geo_i)
    start, count = int(start), int(count)
    if count == 0:
        return OK
    if _is_dev(xs):
        _check_dev(ys, zs, us, vs, ws, E, B)
        _span_ok(xs.shape[0], start, count)
        rc = L.bp_push_span(pb, fb, *[_dptr(a) for a in (xs, ys, zs, us, vs, ws)],
                            start, count, _dptr(E), _dptr(B), _hp(gf), _hp(gg),
                            _hp(gi), float(dt), float(dth), float(qdt2m),
                            float(beta), float(one), int(n_iters),
                            int(apply_bc), int(mixed),
                            None if d_status is None else _dptr(d_status),
                            _stream_of(xs))
        return _lib.check(rc, "push_span")
    _check_host(xs, ys, zs, us, vs, ws, E, B)
    _span_ok(xs.shape[0], start, count)
    st = _Staged()
    sl = slice(start, start + count)
    d = [st.put(a, sl) for a in (xs, ys, zs, us, vs, ws)]
    dE, dB = st.put(E), st.put(B)
    rc = L.bp_push_span(pb, fb, *[_dptr(a) for a in d], 0, count, _dptr(dE),
                        _dptr(dB), _hp(gf), _hp(gg), _hp(gi), float(dt), float(dth),
                        float(qdt2m), float(beta), float(one), int(n_iters),
                        int(apply_bc), int(mixed), None, _stream_of(dE))
    _lib.check(rc, "push_span")
    for h, dv in zip((xs, ys, zs, us, vs, ws), d):
        st.back(h, dv, sl)
    return rc


def deposit_span(xs, ys, zs, us, vs, ws, qs, start, count, acc, invvol, geo_g,
                 geo_i, one, scale, *, d_status=None):
    """Deposit the 10 moments of a span onto ``acc`` (int64, +=)."""
    L = _lib.load()
    pb, fb = _nbytes_of(xs), _nbytes_of(invvol)
    gg, gi = _geo(geo_g), _geoi(geo_i)
    start, count = int(start), int(count)
    if count == 0:
        return OK
    if _is_dev(xs):
        _check_dev(ys, zs, us, vs, ws, qs, acc, invvol)
        _span_ok(xs.shape[0], start, count)
        rc = L.bp_deposit_span(pb, fb, *[_dptr(a) for a in (xs, ys, zs, us, vs, ws, qs)],
                               start, count, _dptr(acc), _dptr(invvol), _hp(gg),
                               _hp(gi), float(one), float(scale),
                               None if d_status is None else _dptr(d_status),
                               _stream_of(xs))
        return _lib.check(rc, "deposit_span")
    _check_host(xs, ys, zs, us, vs, ws, qs, acc, invvol)
    _span_ok(xs.shape[0], start, count)
    st = _Staged()
    sl = slice(start, start + count)
    d = [st.put(a, sl) for a in (xs, ys, zs, us, vs, ws, qs)]
    dacc, dinv = st.put(acc), st.put(invvol)
    rc = L.bp_deposit_span(pb, fb, *[_dptr(a) for a in d], 0, count, _dptr(dacc),
                           _dptr(dinv), _hp(gg), _hp(gi), float(one), float(scale),
                           None, _stream_of(dacc))
    _lib.check(rc, "deposit_span")
    st.back(acc, dacc)
    return rc


def gather_span(xs, ys, zs, start, count, E, B, geo_g, geo_i, one, out, *,
                d_status=None):
    """E, B at in-domain points into ``out[p - start, 0:6]``."""
    L = _lib.load()
    pb, fb = _nbytes_of(xs), _nbytes_of(E)
    gg, gi = _geo(geo_g), _geoi(geo_i)
    start, count = int(start), int(count)
    if count == 0:
        return OK
    if _nbytes_of(out) != pb:
        raise TypeError("gather rows are written in the particle dtype")
    if _is_dev(xs):
        _check_dev(ys, zs, E, B, out)
        _span_ok(xs.shape[0], start, count)
        rc = L.bp_gather_span(pb, fb, _dptr(xs), _dptr(ys), _dptr(zs), start, count,
                              _dptr(E), _dptr(B), _hp(gg), _hp(gi), float(one),
                              _dptr(out), None if d_status is None else _dptr(d_status),
                              _stream_of(xs))
        return _lib.check(rc, "gather_span")
    _check_host(xs, ys, zs, E, B, out)
    _span_ok(xs.shape[0], start, count)
    st = _Staged()
    sl = slice(start, start + count)
    d = [st.put(a, sl) for a in (xs, ys, zs)]
    dE, dB = st.put(E), st.put(B)
    dout = st.torch.empty((count, 6), dtype=d[0].dtype, device=st.dev)
    rc = L.bp_gather_span(pb, fb, *[_dptr(a) for a in d], 0, count, _dptr(dE), _dptr(dB),
                          _hp(gg), _hp(gi), float(one), _dptr(dout), None,
                          _stream_of(dE))
    _lib.check(rc, "gather_span")
    out[:count] = dout.cpu().numpy()
    return rc


def install(module=None):
    """Rebind the reference kernel seam onto this module.

    ``module`` defaults to ``batchpic.kernels`` (the reference package, when
    importable).  Every reference caller resolves ``kernels.<name>`` at call
    time (mover.py:85,135,154,179,194,221; pipeline.py:206), so afterwards the
    reference mover, pipeline and tests run on the GPU.  Returns the previous
    bindings so they can be restored.
    """
    if module is None:
        import batchpic.kernels as module  # noqa: F811
    names = ("fused_span", "push_span", "deposit_span", "gather_span")
    prev = {n: getattr(module, n) for n in names}
    for n in names:
        setattr(module, n, globals()[n])
    return prev
