"""Device-resident cycle driver: phases 1-4 and 6 of the reference
``pipeline.run_cycle`` (``pkg/src/batchpic/pipeline.py:228-324``) on B200s.

  phase 1  E/B from the host solver -> HBM (rank 0), NCCL broadcast to ranks
  phase 2  zero the per-species int64 accumulators
  phase 3  fused mover + deposition per species over this rank's particle
           shard (``bp_fused_span_ex``), optionally in batches; per-species
           NCCL all-reduce (int64 sum, exact) issued as soon as the species'
           kernels are queued so it overlaps the next species
  phase 4  periodic fold of the moment grids on device, copy to the host
  phase 6  on-device stable cell sort every ``sort_period`` cycles

Particle decomposition (paper §III.A, re-targeted at GPUs): every species'
particles are split into contiguous spans, one per rank (``shard_span``);
every rank holds a full E/B copy and a full accumulator per species.  Integer
moments make the result bit-identical for any rank count.

The host field solve (phase 5) stays outside, as in the paper; a caller
passes the new E/B in every cycle (``set_fields``).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .config import PrecisionMode
from .errors import ConfigurationError, IntegrityError
from .fields import MOMENT_SCALE, N_MOMENTS
from .particles import DeviceParticles, partition_batches


def shard_span(n, rank, world):
    """Contiguous span (start, count) of rank ``rank`` out of ``world`` for a
    species of ``n`` particles (the reference's partition rule,
    particles.py:97-114: the first n % world ranks take one extra)."""
    return partition_batches(n, world).spans[rank]


def reduce_moments(accs, group=None, async_op=False, root=None):
    """Exact int64 SUM of per-species moment grids across the ranks of
    ``group`` (NCCL for CUDA tensors, gloo for CPU tensors): an all-reduce, or
    with ``root`` a reduce onto that rank only (the host field solve runs on
    one rank; the other ranks' grids are then unspecified).  Returns the work
    handles when ``async_op``."""
    import torch.distributed as dist
    if root is None:
        works = [dist.all_reduce(a, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
                 for a in accs]
    else:
        dst = root if group is None else dist.get_global_rank(group, root)
        works = [dist.reduce(a, dst, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
                 for a in accs]
    return works if async_op else None


def broadcast_fields(E, B, src=0, group=None):
    import torch.distributed as dist
    dist.broadcast(E, src, group=group)
    dist.broadcast(B, src, group=group)


@dataclass
class CycleTiming:
    cycle: int
    phase3_ms: float            # device time of phase 3 (kernels + reduce)
    kernel_ms: float            # device time of the fused kernels alone
    sort_ms: float = 0.0
    particles: int = 0          # particles advanced by ALL ranks
    sorted_this_cycle: bool = False

    @property
    def mpa_s(self):
        return self.particles / (self.phase3_ms * 1e-3) / 1e6 if self.phase3_ms > 0 else 0.0


@dataclass
class DeviceSimulation:
    """One rank's view of a device-resident simulation."""

    geom: object
    species: tuple
    dt: float
    c: float = 1.0
    precision: PrecisionMode = field(default_factory=PrecisionMode)
    arith: str = "parity"
    sort_period: int = 10
    batches: int = 1
    device: object = None
    group: object = None          # torch.distributed process group (None = default)
    distributed: bool = False
    # "all": every rank ends the cycle with the summed moments (all-reduce);
    # "root": only rank 0 (where the host solve runs) gets them (reduce)
    reduce: str = "all"
    # particle layout: "flat" (the reference's SoA, sorted every sort_period
    # cycles) or "bins" (per-cell bins kept sorted every cycle, bins.py; the
    # fast arithmetic, f32 or f64 particles); "auto" picks bins where they apply
    layout: str = "auto"
    # bin capacity = count + max(slack[1], slack[0] * count), rounded to 8
    # slots: a bin that fills up forces a re-slack of the species (a copy of
    # all bins, ~1.6 ms at C3).  None: the largest of slack fractions 3, 2, 1
    # (min 64) whose two buffer sets fit half the device — at C3 3.0 (86 GB):
    # over 100 cycles 1 re-slack per electron species instead of 7 with 1.0
    # (26.3 against 25.8 G particles/s)
    bin_slack: tuple = None

    def __post_init__(self):
        import torch
        self.torch = torch
        if self.device is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        pd = torch.float32 if self.precision.particle_dtype == np.float32 else torch.float64
        fd = torch.float32 if self.precision.field_dtype == np.float32 else torch.float64
        self.pdt, self.fdt = pd, fd
        shp = (3,) + self.geom.node_shape
        self.E = torch.zeros(shp, dtype=fd, device=self.device)
        self.B = torch.zeros(shp, dtype=fd, device=self.device)
        self.invvol = torch.from_numpy(
            self.geom.inv_node_volume(self.precision.field_dtype)).to(self.device)
        self.acc = [torch.zeros((N_MOMENTS,) + self.geom.node_shape, dtype=torch.int64,
                                device=self.device) for _ in self.species]
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._flat = [None] * len(self.species)
        self._bins = [None] * len(self.species)
        self._lists = None
        self._flat_cache = None
        binnable = self.arith == "fast"
        if self.layout not in ("auto", "flat", "bins"):
            raise ConfigurationError(f"layout must be auto, flat or bins, not {self.layout!r}")
        if self.layout == "bins" and not binnable:
            raise ConfigurationError("the binned layout needs the fast arithmetic")
        if self.bin_slack is None:
            from .bins import layout_bytes
            half = 0.5 * torch.cuda.get_device_properties(self.device).total_memory
            pbytes = 4 if pd == torch.float32 else 8
            world = self._world_hint()
            ppcs = [sp.ppc for sp in self.species]
            self.bin_slack = (1.0, 64)
            for frac in (3.0, 2.0):
                if layout_bytes(int(self.geom.n_cells), ppcs, (frac, 64), pbytes, world) <= half:
                    self.bin_slack = (frac, 64)
                    break
        if self.layout == "auto" and binnable:
            # the bins hold two buffer sets (live + the re-slack's destination)
            # of (1 + slack) slots per particle: decks whose sets would not fit
            # the device (f64 C5 at 1e9 particles: ~300 GB) stay flat
            binnable = self.bins_bytes_estimate() <= 0.92 * torch.cuda.get_device_properties(
                self.device).total_memory
        self.binned = self.layout == "bins" or (self.layout == "auto" and binnable)
        self.cycle = 0
        from .kernels import make_geo_arrays, kernel_scalars
        npd, nfd = self.precision.particle_dtype, self.precision.field_dtype
        self.geo_f, self.geo_i = make_geo_arrays(self.geom, npd)
        self.geo_g, _ = make_geo_arrays(self.geom, nfd)
        self.geo_f = np.ascontiguousarray(self.geo_f, np.float64)
        self.geo_g = np.ascontiguousarray(self.geo_g, np.float64)
        self.scalars = [kernel_scalars(s, self.dt, self.c, npd) for s in self.species]
        self.mixed = 1 if npd != nfd else 0
        self.scale = float(nfd(MOMENT_SCALE))
        self._arith = {"parity": _lib.ARITH_PARITY, "fast": _lib.ARITH_FAST}[self.arith]
        # fast arithmetic: per-cell coefficient records of E/B in the particle
        # precision (bp_field_records_build), built once per field update and
        # shared by every species' call (f32, mixed, and f64 with f64 fields)
        self.records = None
        # run_cycle(stream_moments=True): the copy stream still writing the
        # pinned moment buffers, and whether the last cycle streamed them
        self._moments_copy_pending = None
        self._moments_streamed = False
        self._records_fresh = False
        self._records_pbytes = 4 if pd == torch.float32 else 8
        if self.arith == "fast":
            gi = np.ascontiguousarray(self.geo_i, np.int64)
            nbytes = int(_lib.load().bp_field_records_bytes(self._records_pbytes,
                                                            ctypes.c_void_p(gi.ctypes.data)))
            self.records = torch.empty(nbytes // 4 + 64, dtype=torch.float32, device=self.device)
        if self.reduce not in ("all", "root"):
            raise ConfigurationError(f"reduce must be 'all' or 'root', not {self.reduce!r}")
        if self.distributed:
            import torch.distributed as dist
            self.rank, self.world = dist.get_rank(self.group), dist.get_world_size(self.group)
        else:
            self.rank, self.world = 0, 1

    def _world_hint(self):
        if not self.distributed:
            return 1
        import torch.distributed as dist
        return dist.get_world_size(self.group)

    def bins_bytes_estimate(self, world=None):
        """Device bytes of the binned layout for this deck on one rank
        (bins.layout_bytes)."""
        if world is None:
            world = self._world_hint()
        from .bins import layout_bytes
        pbytes = 4 if self.pdt == self.torch.float32 else 8
        return layout_bytes(int(self.geom.n_cells), [sp.ppc for sp in self.species],
                            self.bin_slack, pbytes, world)

    # ------------------------------------------------------------ loading
    def load_species(self, sid, parts):
        """Install this rank's shard (a DeviceParticles) of species ``sid``."""
        if parts.dtype != self.pdt:
            raise ConfigurationError("particle dtype does not match the precision mode")
        self._flat_cache = None
        if not self.binned:
            self._flat[sid] = parts
            return
        from .bins import BinnedSpecies, TransitLists
        self._bins[sid] = BinnedSpecies(parts, self.geom, self.geo_f, self.geo_g, self.geo_i,
                                        self.E.element_size(), slack=self.bin_slack)
        n_max = max(b.n for b in self._bins if b is not None)
        pb = parts.x.element_size()
        if (self._lists is None or self._lists.pbytes != pb
                or self._lists.leaver_cap < int(n_max * 0.25) + (1 << 20)):
            self._lists = TransitLists(self.device, n_max, pbytes=pb)
            self._side_lists = None

    @property
    def particles(self):
        """Per-species DeviceParticles of this rank (the binned layout exports
        its live particles in cell order; cached until the next cycle)."""
        if not self.binned:
            return self._flat
        if self._flat_cache is None:
            self._flat_cache = [b.flat() if b is not None else None for b in self._bins]
        return self._flat_cache

    def _species_n(self):
        if self.binned:
            return [0 if b is None else b.n for b in self._bins]
        return [0 if p is None else p.n for p in self._flat]

    def load_host_buffers(self, buffers):
        """Shard full host buffers (reference ParticleBuffers) onto this rank."""
        for sid, buf in enumerate(buffers):
            start, count = shard_span(buf.n, self.rank, self.world)
            self.load_species(sid, DeviceParticles.from_host(buf, self.device, start, count))

    def total_particles(self):
        n = sum(self._species_n())
        if self.distributed:
            import torch.distributed as dist
            t = self.torch.tensor([n], dtype=self.torch.int64, device=self.device)
            dist.all_reduce(t, group=self.group)
            n = int(t.item())
        return n

    # ------------------------------------------------------------ phases
    def set_fields(self, E=None, B=None):
        """Phase 1: host E/B (numpy, rank 0) -> HBM, broadcast to all ranks
        (collective: all ranks call it; only rank 0's arrays are used)."""
        # staged through persistent pinned buffers: one DMA each, in stream
        # order, no pageable bounce copy
        for name, src in (("E", E), ("B", B)):
            if src is None:
                continue
            dst = getattr(self, name)
            stage = self._pinned(f"_stage_{name}", dst)
            done = getattr(self, f"_stage_{name}_done", None)
            if done is not None:
                done.synchronize()  # the previous DMA out of this buffer
            if isinstance(src, np.ndarray):
                stage.numpy()[...] = src
            else:
                stage.copy_(src)
            dst.copy_(stage, non_blocking=True)
            done = self.torch.cuda.Event()
            done.record(self.torch.cuda.current_stream(self.device))
            setattr(self, f"_stage_{name}_done", done)
        if self.distributed:
            broadcast_fields(self.E, self.B, src=0, group=self.group)
        self._records_fresh = False

    def _records_ptr(self, stream):
        """Device address of the cell records for the current E/B (built on
        first use after a field update), or None off the fast arithmetic."""
        if self.records is None:
            return None
        base = self.records.data_ptr()
        ptr = (base + 255) & ~255
        if not self._records_fresh:
            L = _lib.load()
            gi = np.ascontiguousarray(self.geo_i, np.int64)
            rc = L.bp_field_records_build(self._records_pbytes, self.E.element_size(),
                                          ctypes.c_void_p(self.E.data_ptr()),
                                          ctypes.c_void_p(self.B.data_ptr()),
                                          ctypes.c_void_p(gi.ctypes.data), ctypes.c_void_p(ptr),
                                          ctypes.c_void_p(stream.cuda_stream))
            _lib.check(rc, "field_records_build")
            self._records_fresh = True
        return ptr

    def _fused(self, sid, start, count, stream):
        p = self._flat[sid]
        sc = self.scalars[sid]
        L = _lib.load()
        ptr = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        hp = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
        rec = self._records_ptr(stream)
        rc = L.bp_fused_span_rec(
            self._arith, p.x.element_size(), self.E.element_size(),
            *[ptr(a) for a in p.arrays()], int(start), int(count), ptr(self.E), ptr(self.B),
            ptr(self.acc[sid]), ptr(self.invvol), hp(self.geo_f), hp(self.geo_g),
            hp(self.geo_i), float(sc["dt"]), float(sc["dth"]), float(sc["qdt2m"]),
            float(sc["beta"]), float(sc["one"]), int(self.species[sid].mover_iters),
            self.scale, self.mixed, None if rec is None else ctypes.c_void_p(rec),
            ptr(self.status), ctypes.c_void_p(stream.cuda_stream))
        _lib.check(rc, "fused_span")

    def _side_streams(self, s):
        """Species on alternating side streams (env BP_SPECIES_STREAMS=2 on
        the flat layout, BP_BIN_STREAMS=2 on the bins, each stream with its
        own leaver list): one species' deposit may then share the SMs with
        the next one's mover.  The side streams start after everything
        queued on `s`."""
        import os
        n = int(os.environ.get("BP_BIN_STREAMS" if self.binned else "BP_SPECIES_STREAMS", "0"))
        if n <= 1:
            return []
        if self.binned and (getattr(self, "_side_lists", None) is None
                            or len(self._side_lists) != n):
            from .bins import TransitLists
            n_max = max(b.n for b in self._bins if b is not None)
            self._side_lists = [TransitLists(self.device, n_max, pbytes=self._lists.pbytes)
                                for _ in range(n)]
        torch = self.torch
        if getattr(self, "_side", None) is None or len(self._side) != n:
            self._side = [torch.cuda.Stream(device=self.device) for _ in range(n)]
        for ss in self._side:
            ss.wait_stream(s)
        return self._side

    def phase3(self, reduce=True, stream_moments=False):
        """Phases 2-3 for every species; returns (phase3_ms, kernel_ms) of
        device time on the compute stream (events), reduce included.

        ``stream_moments`` (single rank): each species' grid is folded right
        after its kernels and copied to its pinned host buffer on a copy
        stream while the next species runs (moments_host(reuse=True) then
        only waits for the last copy)."""
        torch = self.torch
        s = torch.cuda.current_stream(self.device)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        stream_moments = stream_moments and not self.distributed
        cs = self._copy_stream() if stream_moments else None
        if self._moments_copy_pending is not None:
            # the previous cycle's host copies read the grids zeroed below
            s.wait_stream(self._moments_copy_pending)
        self._moments_copy_pending = None
        self.status.zero_()
        ev[0].record(s)
        for a in self.acc:
            a.zero_()
        ev[1].record(s)
        works = []
        # the cell records are built on `s` before any side stream forks off
        # it (side streams wait on everything queued on `s` so far)
        rec = self._records_ptr(s)
        side = self._side_streams(s)
        self._flat_cache = None
        for sid, n in enumerate(self._species_n()):
            if n == 0:
                continue
            ss = side[sid % len(side)] if side else s
            if self.binned:
                sp = self.species[sid]
                lists = self._side_lists[sid % len(side)] if side else self._lists
                self._bins[sid].cycle(lists, rec, self.acc[sid], self.invvol,
                                      self.scalars[sid], sp.mover_iters, self.scale, self.status,
                                      ss)
            else:
                for (b0, bn) in partition_batches(n, self.batches).spans:
                    if bn:
                        self._fused(sid, b0, bn, ss)
            if reduce and self.distributed:
                if side:
                    s.wait_stream(ss)
                works += reduce_moments([self.acc[sid]], self.group, async_op=True,
                                        root=0 if self.reduce == "root" else None)
            if cs is not None:
                self._fold_one(self.acc[sid], ss)
                cs.wait_stream(ss)
                h = self._pinned(f"_mom_host_{sid}", self.acc[sid])
                with torch.cuda.stream(cs):
                    h.copy_(self.acc[sid], non_blocking=True)
        for ss in side:
            s.wait_stream(ss)
        ev[2].record(s)
        for w in works:
            w.wait()
        ev[3].record(s)
        if self.distributed:
            # every rank raises together (a one-sided raise would strand the
            # others in the next collective)
            import torch.distributed as dist
            dist.all_reduce(self.status, op=dist.ReduceOp.MAX, group=self.group)
        if cs is not None:
            # species without particles: zero grids, nothing to fold
            for sid, n in enumerate(self._species_n()):
                if n == 0:
                    h = self._pinned(f"_mom_host_{sid}", self.acc[sid])
                    cs.wait_stream(s)
                    with torch.cuda.stream(cs):
                        h.copy_(self.acc[sid], non_blocking=True)
            self._moments_copy_pending = cs
        ev[3].synchronize()
        st = int(self.status.item())
        if self.binned:
            self._bins_after_cycle()
        if st == _lib.ERR_RUNAWAY:
            raise IntegrityError("runaway particle (moved a full box length)")
        if st == _lib.ERR_MIDPOINT:
            raise IntegrityError("mover midpoint not mappable into the domain")
        if st == _lib.ERR_DOMAIN:
            raise IntegrityError("particle outside the domain at deposition")
        return ev[0].elapsed_time(ev[3]), ev[1].elapsed_time(ev[2])

    def _bins_after_cycle(self):
        """Overflowed or misplaced particles: re-bin that species (host
        decision after the synchronised cycle; the moments are complete)."""
        live = [b for b in self._bins if b is not None]
        if not live:
            return
        stats = self.torch.stack([b.stat for b in live]).cpu().tolist()
        for b, st in zip(live, stats):
            b.check_after_cycle(st)

    def bin_stats(self):
        """Per species: leavers, overflowed, misplaced, lost of the last
        cycle and the number of rebuilds so far (binned layout)."""
        return [None if b is None else (b.last_stats or b.stats())[:4] + [b.rebuilds]
                for b in self._bins]

    def fold_moments(self):
        """Phase 4 on device: merge duplicated periodic planes (exact)."""
        s = self.torch.cuda.current_stream(self.device)
        for a in self.acc:
            self._fold_one(a, s)

    def _fold_one(self, a, stream):
        L = _lib.load()
        gi = np.ascontiguousarray(self.geo_i, np.int64)
        rc = L.bp_fold_periodic_i64(ctypes.c_void_p(a.data_ptr()), N_MOMENTS,
                                    ctypes.c_void_p(gi.ctypes.data),
                                    ctypes.c_void_p(stream.cuda_stream))
        _lib.check(rc, "fold_periodic")

    def _copy_stream(self):
        cs = getattr(self, "_mom_copy_stream", None)
        if cs is None:
            cs = self.torch.cuda.Stream(device=self.device)
            self._mom_copy_stream = cs
        return cs

    def _pinned(self, attr, like):
        """Persistent pinned host tensor shaped like ``like`` (lazily made)."""
        t = getattr(self, attr, None)
        if t is None or t.shape != like.shape or t.dtype != like.dtype:
            t = self.torch.empty(like.shape, dtype=like.dtype, pin_memory=True)
            setattr(self, attr, t)
        return t

    def moments_host(self, reuse=False):
        """The per-species int64 moment grids on the host.  ``reuse=True``
        returns views of persistent pinned buffers (one DMA each, overwritten
        by the next call) instead of fresh arrays."""
        if not reuse:
            return [a.cpu().numpy() for a in self.acc]
        if self._moments_streamed:
            # run_cycle(stream_moments=True) already queued the copies
            self._moments_copy_pending.synchronize()
            return [self._pinned(f"_mom_host_{sid}", a).numpy()
                    for sid, a in enumerate(self.acc)]
        out = []
        for sid, a in enumerate(self.acc):
            h = self._pinned(f"_mom_host_{sid}", a)
            h.copy_(a, non_blocking=True)
            out.append(h)
        self.torch.cuda.current_stream(self.device).synchronize()
        return [h.numpy() for h in out]

    def total_moments(self):
        """Exact int64 sum of the species grids on device (fields.total_moments)."""
        torch = self.torch
        L = _lib.load()
        total = torch.empty_like(self.acc[0])
        rows = (ctypes.c_void_p * len(self.acc))(*[a.data_ptr() for a in self.acc])
        s = torch.cuda.current_stream(self.device)
        _lib.check(L.bp_moments_total(rows, len(self.acc), total.numel(),
                                      ctypes.c_void_p(total.data_ptr()),
                                      ctypes.c_void_p(s.cuda_stream)), "moments_total")
        return total

    def susceptibility(self, theta):
        """maxwell.plasma_susceptibility of the current (folded) moments,
        computed on device (bitwise the reference); returns a float64 device
        tensor of node shape."""
        torch = self.torch
        L = _lib.load()
        chi = torch.empty(self.geom.node_shape, dtype=torch.float64, device=self.device)
        rows = (ctypes.c_void_p * len(self.acc))(*[a.data_ptr() for a in self.acc])
        qom = np.ascontiguousarray([s.qom for s in self.species], np.float64)
        s = torch.cuda.current_stream(self.device)
        single = 1 if self.precision.fields == "single" else 0
        _lib.check(L.bp_susceptibility(rows, ctypes.c_void_p(qom.ctypes.data), len(self.acc),
                                       single, float(theta), float(self.dt), chi.numel(),
                                       ctypes.c_void_p(chi.data_ptr()),
                                       ctypes.c_void_p(s.cuda_stream)), "susceptibility")
        return chi

    def sort(self):
        """Phase 6.  The binned layout is cell-sorted after every cycle, so
        only the flat layout sorts."""
        if self.binned:
            return
        for p in self._flat:
            if p is not None:
                p.sort_by_cell(self.geom)

    def run_cycle(self, E=None, B=None, stream_moments=False):
        """One cycle on device: phases 1-4 and (when due) 6.  The host solve
        (phase 5) is the caller's; moments for it are in ``self.acc``.

        ``stream_moments=True`` (single rank): each species' folded grid is
        copied to pinned host memory while the next species runs;
        ``moments_host(reuse=True)`` returns those buffers.

        Distributed: every rank calls this collectively; rank 0 passes the new
        E/B (others may pass None) and the broadcast runs on all ranks."""
        torch = self.torch
        if E is not None or B is not None or self.distributed:
            self.set_fields(E, B)
        # phase 1 always refreshes the cell records (a cycle's fields are new
        # in a real run, even when the caller updated self.E / self.B in place)
        self._records_fresh = False
        streamed = stream_moments and not self.distributed
        self._moments_streamed = False
        p3, kt = self.phase3(stream_moments=streamed)
        self._moments_streamed = streamed
        if not streamed:
            self.fold_moments()
        sort_ms, sorted_now = 0.0, False
        if (not self.binned and self.sort_period > 0
                and (self.cycle + 1) % self.sort_period == 0):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            self.sort()
            e1.record()
            e1.synchronize()
            sort_ms, sorted_now = e0.elapsed_time(e1), True
        t = CycleTiming(self.cycle, p3, kt, sort_ms, self.total_particles(), sorted_now)
        self.cycle += 1
        return t

    # ------------------------------------------------------- diagnostics
    def kinetic_energy(self):
        """Per-species sum of (q_p / qom) |v|^2 / 2 in f64 over all ranks
        (diagnostics.kinetic_energy, diagnostics.py:64-73)."""
        torch = self.torch
        out = []
        for sp, p in zip(self.species, self.particles):
            if p is None or p.n == 0:
                k = torch.zeros((), dtype=torch.float64, device=self.device)
            else:
                u, v, w = (a.to(torch.float64) for a in (p.u, p.v, p.w))
                m = p.q_p.to(torch.float64) / sp.qom
                k = 0.5 * torch.sum(m * (u * u + v * v + w * w))
            out.append(k)
        t = torch.stack(out)
        if self.distributed:
            import torch.distributed as dist
            dist.all_reduce(t, group=self.group)
        return [float(x) for x in t.cpu()]


def field_energy(E, B, geom):
    """Sum of (|E|^2 + |B|^2) w V / 8 pi over unique nodes, f64
    (diagnostics.field_energy, diagnostics.py:52-61)."""
    sl = (slice(None),) + geom.unique_slices()
    E = np.asarray(E, np.float64)[sl]
    B = np.asarray(B, np.float64)[sl]
    w = geom.node_weights()[geom.unique_slices()]
    dens = (E * E).sum(axis=0) + (B * B).sum(axis=0)
    return float(np.sum(dens * w)) * geom.cell_volume / (8.0 * np.pi)
