"""Cell-binned device layout of one species (csrc/bp_bins.cu for f32
particles, csrc/bp_bins64.cu for f64; C ABI ``bp_bins_*``): the fast-arithmetic
layout of :class:`pipeline.DeviceSimulation`.

The reference restores cell order with a stable sort every ``sort_period``
cycles (particles.py:157-167, pipeline.py:300-304).  Here cell ``c`` owns
slots ``[start[c], start[c + 1])`` of particle records (the reference's
ParticleBuffer columns x y z u v w q_p, then 0: 32 bytes in f32, 64 in f64)
and of the int64 ids, the first
``count[c]`` of them live, and every cycle (``bp_bins_cycle``: mover, leaver
migration, deposit) leaves each particle in its cell's bin — cell-sorted at
every cycle.  ``flat()`` exports the live particles (cell order) as a
:class:`particles.DeviceParticles`; ``rebuild()`` re-bins after a bin
overflowed.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import DomainError, IntegrityError
from .particles import ARRAYS, DeviceParticles

STAT_LEAVERS, STAT_OVERFLOW, STAT_MISPLACED, STAT_LOST = 0, 1, 2, 3


def layout_bytes(n_cells, ppcs, slack, pbytes, world=1):
    """Device bytes of the binned layout of a deck on one rank: two buffer
    sets (live + the re-slack's destination) of records (8 scalars of
    pbytes) + int64 ids, count + max(slack_min, slack_frac x count) slots per
    cell and species, 3% headroom (BinnedSpecies._alloc_set)."""
    frac, smin = slack
    slots = sum(n_cells * (p + max(smin, frac * p)) for p in ppcs) / max(1, world)
    return 2 * 1.03 * slots * (8 * pbytes + 8)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


class BinnedSpecies:
    """One species' particles in per-cell bins on one device."""

    def __init__(self, parts, geom, geo_f, geo_g, geo_i, fbytes, slack=(0.5, 64),
                 overflow_frac=1.0 / 16, stream=None):
        import torch
        if parts.dtype not in (torch.float32, torch.float64):
            raise TypeError("the binned layout holds f32 or f64 particles")
        if parts.dtype == torch.float64 and int(fbytes) != 8:
            raise TypeError("f64 particles need f64 fields")
        self.torch = torch
        self.dtype = parts.dtype
        self.pbytes = parts.x.element_size()
        self.geom = geom
        self.geo_f = np.ascontiguousarray(geo_f, np.float64)
        self.geo_g = np.ascontiguousarray(geo_g, np.float64)
        self.geo_i = np.ascontiguousarray(geo_i, np.int64)
        self.fbytes = int(fbytes)
        self.slack = (float(slack[0]), int(slack[1]))
        self.species_id = parts.species_id
        self.device = parts.x.device
        self.ncell = int(geom.n_cells)
        self.n = parts.n
        dev = self.device
        self.count = torch.zeros(self.ncell, dtype=torch.int32, device=dev)
        self.start = torch.zeros(self.ncell + 1, dtype=torch.int64, device=dev)
        self.stat = torch.zeros(8, dtype=torch.int64, device=dev)
        # this species' overflow list: leavers whose bin was full (deposited
        # on their own, merged back by the rebuild after the cycle)
        rb = int(_lib.load().bp_bins_leaver_bytes(self.pbytes))
        self.overflow_cap = max(4096, int(parts.n * overflow_frac))
        self.overflow = torch.empty(self.overflow_cap * rb, dtype=torch.uint8, device=dev)
        self.rebuilds = 0
        self.last_stats = None
        self._build(parts, stream)

    # ------------------------------------------------------------ layout
    def _stream(self, stream):
        return stream if stream is not None else self.torch.cuda.current_stream(self.device)

    def _build(self, parts, stream=None):
        torch = self.torch
        L = _lib.load()
        s = self._stream(stream)
        total = ctypes.c_int64(0)
        gf, gg, gi = (ctypes.c_void_p(a.ctypes.data) for a in (self.geo_f, self.geo_g, self.geo_i))
        rc = L.bp_bins_plan(self.pbytes, self.fbytes, _ptr(parts.x), _ptr(parts.y), _ptr(parts.z), parts.n,
                            gf, gg, gi, self.slack[0], self.slack[1], _ptr(self.count),
                            _ptr(self.start), ctypes.byref(total), ctypes.c_void_p(s.cuda_stream))
        _lib.check(rc, "bins_plan")
        if rc == _lib.ERR_DOMAIN:
            raise DomainError("positions below the box origin")
        cap = int(total.value)
        self.cap = cap
        self.rec, self.ids = self._alloc_set(cap)
        # the re-slack's destination: allocated after the first cycle (when the
        # caller's flat input and the build's scratch are gone), so that a
        # re-slack inside a run only copies
        self._spare = None
        rc = L.bp_bins_fill(self.pbytes, self.fbytes, *[_ptr(a) for a in parts.arrays()],
                            _ptr(parts.ids),
                            parts.n, gf, gg, gi, _ptr(self.start), _ptr(self.rec), _ptr(self.ids),
                            ctypes.c_void_p(s.cuda_stream))
        _lib.check(rc, "bins_fill")
        self.n = parts.n

    def _alloc_set(self, cap):
        """One buffer set (records x y z u | v w q 0 of the particle dtype,
        int64 ids) for `cap` slots plus headroom (3% + 64k slots), so that the
        slightly larger layouts of later re-slacks fit."""
        torch = self.torch
        n = int(cap * 1.03) + (1 << 16)
        return (torch.empty(8 * n, dtype=self.dtype, device=self.device),
                torch.empty(n, dtype=torch.int64, device=self.device))

    def flat(self, stream=None):
        """The live particles (bins in cell order, then the overflow list of
        the last cycle) as DeviceParticles."""
        torch = self.torch
        L = _lib.load()
        s = self._stream(stream)
        off = torch.empty(self.ncell + 1, dtype=torch.int64, device=self.device)
        total = ctypes.c_int64(0)
        args = (self.pbytes, _ptr(self.rec), _ptr(self.ids), _ptr(self.start), _ptr(self.count),
                self.ncell, _ptr(self.overflow), self.overflow_cap, _ptr(self.stat))
        rc = L.bp_bins_export(*args, _ptr(off), None, None, ctypes.byref(total),
                              ctypes.c_void_p(s.cuda_stream))
        _lib.check(rc, "bins_export")
        n = int(total.value)
        out = [torch.empty(n, dtype=self.dtype, device=self.device) for _ in ARRAYS]
        ids = torch.empty(n, dtype=torch.int64, device=self.device)
        if n:
            dst = (ctypes.c_void_p * 7)(*[a.data_ptr() for a in out])
            rc = L.bp_bins_export(*args, _ptr(off), dst, _ptr(ids), ctypes.byref(total),
                                  ctypes.c_void_p(s.cuda_stream))
            _lib.check(rc, "bins_export")
        return DeviceParticles(*out, ids, species_id=self.species_id)

    def rebuild(self, stream=None):
        """Re-bin (fresh slack) from the current bins plus the overflow list:
        a full rebuild (export + sort) — needed when particles sit in a bin
        that is not their cell."""
        self._build(self.flat(stream), stream)
        self.stat.zero_()
        self.rebuilds += 1

    def reslack(self, stream=None):
        """The cheap rebuild after bins overflowed (bp_bins_reslack): new
        capacities from the live counts plus the overflow list, every bin
        copied to its new place (into the spare buffer set), no sort."""
        torch = self.torch
        L = _lib.load()
        s = self._stream(stream)
        ncount = torch.empty(self.ncell, dtype=torch.int32, device=self.device)
        nstart = torch.empty(self.ncell + 1, dtype=torch.int64, device=self.device)
        total = ctypes.c_int64(0)
        args = (self.pbytes, _ptr(self.rec), _ptr(self.ids), _ptr(self.start), _ptr(self.count),
                self.ncell, _ptr(self.overflow), self.overflow_cap, _ptr(self.stat),
                self.slack[0], self.slack[1], _ptr(ncount), _ptr(nstart))
        rc = L.bp_bins_reslack(*args, None, None, ctypes.byref(total),
                               ctypes.c_void_p(s.cuda_stream))
        _lib.check(rc, "bins_reslack")
        cap = int(total.value)
        spare = self._spare
        if spare is None or spare[1].numel() < cap:
            spare = self._alloc_set(cap)
        rc = L.bp_bins_reslack(*args, _ptr(spare[0]), _ptr(spare[1]), ctypes.byref(total),
                               ctypes.c_void_p(s.cuda_stream))
        _lib.check(rc, "bins_reslack")
        self._spare = (self.rec, self.ids)
        self.rec, self.ids = spare
        self.start, self.count, self.cap = nstart, ncount, cap
        self.stat.zero_()
        self.rebuilds += 1

    def stats(self):
        return [int(v) for v in self.stat.cpu()]

    # ------------------------------------------------------------ cycle
    def cycle(self, lists, records, acc, invvol, sc, n_iters, scale, d_status, stream):
        """Mover + migration + deposit of this species (asynchronous, on
        `stream`, which must be the stream `lists` is used on)."""
        L = _lib.load()
        gf, gg, gi = (ctypes.c_void_p(x.ctypes.data) for x in (self.geo_f, self.geo_g, self.geo_i))
        rc = L.bp_bins_cycle(self.pbytes, self.fbytes, _ptr(self.rec), _ptr(self.ids), _ptr(self.start),
                             _ptr(self.count), self.ncell, _ptr(lists.leavers), lists.leaver_cap,
                             _ptr(self.overflow), self.overflow_cap,
                             # the late list (misplaced particles the deposit
                             # meets) reuses the leaver list: the migration
                             # drained it before the deposit runs
                             _ptr(lists.leavers), lists.slots, _ptr(self.stat),
                             ctypes.c_void_p(records), _ptr(acc), _ptr(invvol), gf, gg, gi,
                             float(sc["dt"]), float(sc["dth"]), float(sc["qdt2m"]),
                             float(sc["beta"]), float(sc["one"]), int(n_iters), float(scale),
                             _ptr(d_status), ctypes.c_void_p(stream.cuda_stream))
        _lib.check(rc, "bins_cycle")

    def check_after_cycle(self, stats=None):
        """Host check after a synchronised cycle: lost particles are fatal,
        an overflow or a misplaced particle triggers a rebuild."""
        st = self.stats() if stats is None else stats
        self.last_stats = list(st)
        if self._spare is None:
            self._spare = self._alloc_set(self.cap)
        if st[STAT_LOST]:
            raise IntegrityError(f"{st[STAT_LOST]} particles lost: bin overflow / late list too "
                                 f"small (stats {st})")
        if st[STAT_MISPLACED]:
            self.rebuild()
            return True
        if st[STAT_OVERFLOW]:
            self.reslack()
            return True
        return False


class TransitLists:
    """The leaver list shared by the species of a simulation: filled by one
    species' mover and drained by its migration, inside one bp_bins_cycle on
    one stream (species on other streams need their own); the deposit then
    reuses it as the late list."""

    def __init__(self, device, n_max, leaver_frac=0.25, pbytes=4):
        import torch
        self.pbytes = int(pbytes)
        rb = int(_lib.load().bp_bins_leaver_bytes(self.pbytes))
        # + the warps' partly used 128-slot chunks (bp_bins.cu kLvChunk)
        self.leaver_cap = int(n_max * leaver_frac) + (1 << 20)
        self.leavers = torch.empty(self.leaver_cap * rb, dtype=torch.uint8, device=device)
        # the buffer's records: the late list's capacity
        self.slots = self.leaver_cap
