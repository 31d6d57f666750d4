"""Particle storage, batching, boundaries, sorting and loading on the path
(reference ``pkg/src/batchpic/particles.py``).

``ParticleBuffer`` is the reference's host SoA buffer (x y z u v w q_p +
int64 ids).  ``DeviceParticles`` holds the same arrays as CUDA tensors —
the layout the kernels stream — and converts to/from a host buffer.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from .config import PrecisionMode
from .errors import ConfigurationError, DomainError, IntegrityError
from .geometry import PERIODIC

COMPONENTS = ("x", "y", "z", "u", "v", "w")
ARRAYS = COMPONENTS + ("q_p",)


@dataclass
class ParticleBuffer:
    """One species in SoA layout (particles.py:23-81)."""

    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    u: np.ndarray
    v: np.ndarray
    w: np.ndarray
    q_p: np.ndarray
    ids: np.ndarray
    species_id: int = 0

    @classmethod
    def empty(cls, n, species_id=0, dtype=np.float64):
        z = lambda: np.zeros(n, dtype=dtype)  # noqa: E731
        return cls(x=z(), y=z(), z=z(), u=z(), v=z(), w=z(), q_p=z(),
                   ids=np.arange(n, dtype=np.int64), species_id=species_id)

    @property
    def n(self):
        return self.x.shape[0]

    @property
    def dtype(self):
        return self.x.dtype

    def components(self):
        return tuple(getattr(self, c) for c in COMPONENTS)

    def copy(self):
        return ParticleBuffer(*(getattr(self, a).copy() for a in ARRAYS + ("ids",)),
                              species_id=self.species_id)

    def permute(self, order):
        for a in ARRAYS + ("ids",):
            setattr(self, a, np.ascontiguousarray(getattr(self, a)[order]))
        return self

    def validate(self, geom=None):
        for a in ARRAYS + ("ids",):
            if getattr(self, a).shape != (self.n,):
                raise IntegrityError("particle component arrays disagree in length")
        if geom is not None and self.n:
            for q, o, L in zip((self.x, self.y, self.z), geom.origin, geom.lengths):
                if q.min() < o or q.max() > o + L:
                    raise IntegrityError("particle positions outside the domain")
        return self


@dataclass
class BatchPlan:
    spans: tuple
    batches: int
    group_of: tuple = field(default=())

    def __post_init__(self):
        if not self.group_of:
            self.group_of = tuple(0 for _ in self.spans)


def partition_batches(n_p, m):
    """``m`` contiguous spans differing by at most one; the first
    ``n_p % m`` take the extra particle (particles.py:97-114)."""
    if m < 1:
        raise ConfigurationError(f"batch count must be >= 1, got {m}")
    if n_p < 0:
        raise ConfigurationError(f"negative particle count {n_p}")
    q, r = divmod(n_p, m)
    spans, start = [], 0
    for b in range(m):
        ln = q + 1 if b < r else q
        spans.append((start, ln))
        start += ln
    return BatchPlan(spans=tuple(spans), batches=m)


def apply_boundaries(buf, geom):
    """Vectorised boundary map with the kernel's exact branch semantics:
    periodic wrap with snap-to-origin, reflecting mirror + velocity flip,
    runaway -> IntegrityError (particles.py:117-154)."""
    for pos, vel, o, L, kind in zip((buf.x, buf.y, buf.z), (buf.u, buf.v, buf.w),
                                    geom.origin, geom.lengths, geom.bc):
        if pos.size == 0:
            continue
        t = pos.dtype.type
        Lc, oc = t(L), t(o)
        hi = oc + Lc
        if kind == PERIODIC:
            below, above = pos < oc, pos >= hi
            pos[below] += Lc
            pos[below & (pos >= hi)] = oc
            pos[above] -= Lc
        else:
            below, above = pos < oc, pos > hi
            pos[below] = oc + (oc - pos[below])
            vel[below] = -vel[below]
            pos[above] = hi + hi - pos[above]
            vel[above] = -vel[above]
        if (pos < oc).any() or (pos > hi).any():
            raise IntegrityError("particle left the domain by a full box length (runaway)")
    return buf


def sort_by_cell(buf, geom):
    """Stable reorder by linear cell index (particles.py:157-167).  Host
    buffers are sorted with numpy; use ``DeviceParticles.sort_by_cell`` for
    device-resident particles."""
    if buf.n == 0:
        return buf
    keys = geom.cell_index_of(buf.x, buf.y, buf.z)
    return buf.permute(np.argsort(keys, kind="stable"))


def cell_sequence(buf, geom):
    if buf.n == 0:
        return np.zeros(0, np.int64)
    return geom.cell_index_of(buf.x, buf.y, buf.z)


# --------------------------------------------------------------- loading

def _species_rng(seed, species_id):
    key = np.array([np.uint64(seed), np.uint64(species_id)], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def cell_charges(species, geom, density_fn=None):
    """Per-cell charge weight q n(cell centre) V_cell / ppc over all cells,
    x fastest (particles.py:222-230, the same array expressions)."""
    nc = geom.n_cells
    lin = np.arange(nc)
    ci = lin % geom.nx
    cj = (lin // geom.nx) % geom.ny
    ck = lin // (geom.nx * geom.ny)
    if density_fn is None:
        dens = np.ones(nc)
    else:
        cx, cy, cz = (geom.cell_centers(a) for a in range(3))
        dens = np.asarray(density_fn(cx[ci], cy[cj], cz[ck]), dtype=np.float64)
        if (dens <= 0.0).any():
            raise ConfigurationError("density profile must be positive")
    return species.charge * dens * geom.cell_volume / species.ppc


# numpy random_standard_normal's tail strip (distributions.c): r and 1/r
_ZIG_R, _ZIG_INV_R = 3.6541528853610087963519472518, 0.27366123732975827203338247596


def init_maxwellian_device(species, geom, device, density_fn=None, seed=1, precision=None,
                           drift=None, cells=None):
    """init_maxwellian generated in HBM (csrc/bp_init.cu, bp_init_maxwellian):
    the same Philox(key=[seed, species]) draws, cell-major order and
    arithmetic, so the buffers are bit-identical to the reference's
    (particles.py:177-241).  ``cells`` = (first, count) loads only that
    contiguous cell range (a rank's shard; ids stay the global indices).
    The ziggurat's tail-strip normals (~0.03%) are finished here with the host
    libm's log1p, as numpy computes them."""
    import ctypes
    import math
    import torch
    from . import _lib
    mode = precision or PrecisionMode()
    pd = mode.particle_dtype
    tdt = torch.float32 if pd == np.float32 else torch.float64
    ppc = species.ppc
    c0, nc = (0, geom.n_cells) if cells is None else (int(cells[0]), int(cells[1]))
    n = nc * ppc
    n_p = geom.n_cells * ppc
    q_cell = torch.from_numpy(
        np.ascontiguousarray(cell_charges(species, geom, density_fn)[c0:c0 + nc])).to(device)
    arrs = [torch.empty(n, dtype=tdt, device=device) for _ in ARRAYS]
    ids = torch.empty(n, dtype=torch.int64, device=device)
    dv = species.drift if drift is None else tuple(drift)
    cap = max(4096, (3 * n) // 1000)
    tk = torch.empty(cap, dtype=torch.int64, device=device)
    tu = torch.empty(cap, dtype=torch.float64, device=device)
    ntail = ctypes.c_int64(0)
    d3 = lambda v: (ctypes.c_double * 3)(*[float(x) for x in v])  # noqa: E731
    geo_i = (ctypes.c_int64 * 3)(geom.nx, geom.ny, geom.nz)
    ptr = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    L = _lib.load()
    rc = L.bp_init_maxwellian(
        np.dtype(pd).itemsize, int(seed), int(species.species_id), geo_i, d3(geom.origin),
        d3(geom.spacings), ppc, d3(dv), d3(species.vth), ptr(q_cell), c0, nc,
        *[ptr(a) for a in arrs], ptr(ids), ptr(tk), ptr(tu), cap, ctypes.byref(ntail),
        ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream))
    _lib.check(rc, "init_maxwellian")
    nt = int(ntail.value)
    if nt > cap:
        raise IntegrityError(f"init_maxwellian: {nt} tail normals exceed the list ({cap})")
    if nt:
        ks, us = tk[:nt].cpu().numpy(), tu[:nt].cpu().numpy()
        per = [([], []) for _ in range(3)]
        for kk, u in zip(ks.tolist(), us.tolist()):
            k, neg = kk >> 1, kk & 1
            xx = -_ZIG_INV_R * math.log1p(-u)
            val = -(_ZIG_R + xx) if neg else _ZIG_R + xx
            a, p = divmod(k, n_p)
            per[a][0].append(p - c0 * ppc)
            per[a][1].append(dv[a] + species.vth[a] * val)
        for a in range(3):
            if per[a][0]:
                idx = torch.tensor(per[a][0], dtype=torch.int64, device=device)
                val = torch.from_numpy(np.asarray(per[a][1], np.float64).astype(pd)).to(device)
                arrs[3 + a].index_copy_(0, idx, val)
    return DeviceParticles(*arrs, ids, species_id=species.species_id)


def init_maxwellian(species, geom, density_fn=None, seed=1, precision=None, drift=None):
    """Cell-major loading of ``ppc`` particles per cell, drifting Maxwellian
    velocities, charge weights from the density at cell centres — the same
    Philox(seed, species) draw sequence as particles.py:182-241, so buffers are
    bit-identical to the reference's."""
    mode = precision or PrecisionMode()
    pd = mode.particle_dtype
    ppc = species.ppc
    nc = geom.n_cells
    n_p = nc * ppc
    rng = _species_rng(seed, species.species_id)
    lin = np.arange(nc)
    ci = lin % geom.nx
    cj = (lin // geom.nx) % geom.ny
    ck = lin // (geom.nx * geom.ny)
    # positions are drawn before velocities
    jit = rng.random((3, n_p))
    pos = []
    for a, cidx in enumerate((ci, cj, ck)):
        d, o = geom.spacings[a], geom.origin[a]
        corner = o + d * np.repeat(cidx, ppc)
        pos.append(corner + d * jit[a])
    dv = species.drift if drift is None else tuple(drift)
    nrm = rng.standard_normal((3, n_p))
    vel = [dv[a] + species.vth[a] * nrm[a] for a in range(3)]
    q_p = np.repeat(cell_charges(species, geom, density_fn), ppc)
    buf = ParticleBuffer(*(a.astype(pd) for a in pos + vel + [q_p]),
                         ids=np.arange(n_p, dtype=np.int64), species_id=species.species_id)
    return buf.validate(geom)


# ------------------------------------------------------------ checkpoint

CHECKPOINT_MAGIC = b"BPIC"
CHECKPOINT_VERSION = 1
CHECKPOINT_VERSION_FULL = 2
_HEADER = "<4sIQB"


def write_particles(buf, path, version=CHECKPOINT_VERSION):
    """Particle checkpoint.  Version 1 is the reference format byte for byte
    (particles.py:244-255: little-endian ``<4sIQB`` header — magic, version,
    count, item size — then x y z u v w).  Version 2 appends q_p (same item
    size), the int64 ids and the species id, so a run can resume deposition
    (the reference's v1 drops them)."""
    import struct
    item = buf.dtype.itemsize
    with open(path, "wb") as fh:
        fh.write(struct.pack(_HEADER, CHECKPOINT_MAGIC, version, buf.n, item))
        for arr in buf.components():
            fh.write(np.ascontiguousarray(arr, dtype=f"<f{item}").tobytes())
        if version >= CHECKPOINT_VERSION_FULL:
            fh.write(np.ascontiguousarray(buf.q_p, dtype=f"<f{item}").tobytes())
            fh.write(np.ascontiguousarray(buf.ids, dtype="<i8").tobytes())
            fh.write(struct.pack("<q", int(buf.species_id)))


def read_particles(path, species_id=0):
    """Read a v1 (reference: q_p zero-filled, fresh ids, particles.py:258-274)
    or v2 checkpoint."""
    import struct
    with open(path, "rb") as fh:
        raw = fh.read(struct.calcsize(_HEADER))
        magic, version, n, item = struct.unpack(_HEADER, raw)
        if magic != CHECKPOINT_MAGIC:
            raise IntegrityError(f"bad checkpoint magic {magic!r}")
        if version not in (CHECKPOINT_VERSION, CHECKPOINT_VERSION_FULL):
            raise IntegrityError(f"unsupported checkpoint version {version}")
        dt = np.float32 if item == 4 else np.float64
        comps = [np.frombuffer(fh.read(n * item), dtype=f"<f{item}").astype(dt)
                 for _ in range(6)]
        if version >= CHECKPOINT_VERSION_FULL:
            q = np.frombuffer(fh.read(n * item), dtype=f"<f{item}").astype(dt)
            ids = np.frombuffer(fh.read(n * 8), dtype="<i8").astype(np.int64)
            species_id = struct.unpack("<q", fh.read(8))[0]
        else:
            q = np.zeros(n, dt)
            ids = np.arange(n, dtype=np.int64)
    return ParticleBuffer(*comps, q_p=q, ids=ids, species_id=species_id)


# ------------------------------------------------------- device residency

class DeviceParticles:
    """One species' SoA arrays resident in HBM (CUDA torch tensors)."""

    def __init__(self, x, y, z, u, v, w, q_p, ids, species_id=0):
        self.x, self.y, self.z, self.u, self.v, self.w = x, y, z, u, v, w
        self.q_p, self.ids, self.species_id = q_p, ids, species_id

    @classmethod
    def from_host(cls, buf, device, start=0, count=None):
        import torch
        count = buf.n - start if count is None else count
        sl = slice(start, start + count)
        t = [torch.from_numpy(np.ascontiguousarray(getattr(buf, a)[sl])).to(device)
             for a in ARRAYS + ("ids",)]
        return cls(*t, species_id=buf.species_id)

    def to_host(self):
        return ParticleBuffer(*(getattr(self, a).cpu().numpy() for a in ARRAYS + ("ids",)),
                              species_id=self.species_id)

    @property
    def n(self):
        return self.x.shape[0]

    @property
    def dtype(self):
        return self.x.dtype

    def arrays(self):
        return tuple(getattr(self, a) for a in ARRAYS)

    def nbytes(self):
        return sum(getattr(self, a).numel() * getattr(self, a).element_size()
                   for a in ARRAYS + ("ids",))

    def sort_by_cell(self, geom, stream=None):
        """On-device stable cell sort (bp_sort_by_cell_into): cell keys in f64
        as geometry.cell_index_of, stable radix sort, one fused gather of all
        eight arrays into a spare buffer set, which is then swapped in (the
        spare is kept for the next sort)."""
        import torch
        from . import _lib
        if self.n <= 1:
            return self
        L = _lib.load()
        o = np.ascontiguousarray(geom.origin, np.float64)
        d = np.ascontiguousarray(geom.spacings, np.float64)
        c = np.ascontiguousarray(geom.counts, np.int64)
        s = stream if stream is not None else torch.cuda.current_stream(self.x.device)
        spare = getattr(self, "_spare", None)
        if spare is None or spare[0].shape != self.x.shape:
            spare = [torch.empty_like(a) for a in self.arrays()] + [torch.empty_like(self.ids)]
        src = (ctypes.c_void_p * 7)(*[a.data_ptr() for a in self.arrays()])
        dst = (ctypes.c_void_p * 7)(*[a.data_ptr() for a in spare[:7]])
        rc = L.bp_sort_by_cell_into(self.x.element_size(), src,
                                    ctypes.c_void_p(self.ids.data_ptr()), dst,
                                    ctypes.c_void_p(spare[7].data_ptr()), self.n,
                                    ctypes.c_void_p(o.ctypes.data), ctypes.c_void_p(d.ctypes.data),
                                    ctypes.c_void_p(c.ctypes.data),
                                    ctypes.c_void_p(s.cuda_stream))
        _lib.check(rc, "sort_by_cell")
        if rc == _lib.ERR_DOMAIN:
            self._spare = spare
            raise DomainError("positions below the box origin")
        old = list(self.arrays()) + [self.ids]
        for name, t in zip(ARRAYS + ("ids",), spare):
            setattr(self, name, t)
        self._spare = old
        return self

    def sort_by_cell_inplace(self, geom, stream=None):
        """In-place variant (bp_sort_by_cell): no spare buffers, one scratch
        array, eight gathers with copy back."""
        import torch
        from . import _lib
        if self.n <= 1:
            return self
        L = _lib.load()
        o = np.ascontiguousarray(geom.origin, np.float64)
        d = np.ascontiguousarray(geom.spacings, np.float64)
        c = np.ascontiguousarray(geom.counts, np.int64)
        s = stream if stream is not None else torch.cuda.current_stream(self.x.device)
        ptr = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        rc = L.bp_sort_by_cell(self.x.element_size(), *[ptr(a) for a in self.arrays()],
                               ptr(self.ids), self.n, ctypes.c_void_p(o.ctypes.data),
                               ctypes.c_void_p(d.ctypes.data), ctypes.c_void_p(c.ctypes.data),
                               ctypes.c_void_p(s.cuda_stream))
        _lib.check(rc, "sort_by_cell")
        if rc == _lib.ERR_DOMAIN:
            raise DomainError("positions below the box origin")
        return self
