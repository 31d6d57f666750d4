"""GEM reconnection initial condition (reference ``pkg/src/batchpic/gem.py``):
Harris sheet with flux perturbation, two current-carrying and two background
species.

``init_gem_host`` reproduces the reference loader bit for bit on the host
(same numpy Philox streams and expression order); ``init_gem_device``
generates the same buffers bit for bit directly in HBM (csrc/bp_init.cu), the
loader of the device-resident runs and benchmarks (1e8-1e9 particles).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .config import PrecisionMode, SpeciesParams
from .errors import ConfigurationError
from .fields import FieldGrid, sync_periodic
from .geometry import GridGeometry, REFLECTING, PERIODIC
from .particles import DeviceParticles, init_maxwellian

SHEET_ELECTRON, SHEET_ION, BG_ELECTRON, BG_ION = 0, 1, 2, 3

# decks/gem_full.deck values
VTH_E = 0.02240119044455748
VTH_I = 0.006261323076368657


@dataclass(frozen=True)
class GemInit:
    seed: int = 20250809
    n0: float = 0.07957747154594767
    b0: float = 0.0097
    sheet_thickness: float = 0.5
    perturbation: float = 0.1
    background_fraction: float = 0.2


def gem_species(ppc, mover_iters=3):
    me = 1.0 / 64.0
    return (
        SpeciesParams(0, -1.0, me, ppc, vth=(VTH_E,) * 3, mover_iters=mover_iters,
                      name="sheet_electrons"),
        SpeciesParams(1, 1.0, 1.0, ppc, vth=(VTH_I,) * 3, mover_iters=mover_iters,
                      name="sheet_ions"),
        SpeciesParams(2, -1.0, me, ppc, vth=(VTH_E,) * 3, mover_iters=mover_iters,
                      name="background_electrons"),
        SpeciesParams(3, 1.0, 1.0, ppc, vth=(VTH_I,) * 3, mover_iters=mover_iters,
                      name="background_ions"),
    )


def gem_geometry(cells, lengths=None):
    """GEM box 25.6 x 12.8 x 12.8 (gem_full.deck); a 2D grid (one cell in z)
    takes lz = dx as the reference's 2D decks do."""
    if lengths is None:
        lz = 25.6 / cells[0] if cells[2] == 1 else 12.8
        lengths = (25.6, 12.8, lz)
    return GridGeometry.from_box(cells, lengths, bc=(PERIODIC, REFLECTING, PERIODIC))


def sheet_drifts(species, init, c):
    """Out-of-plane drifts splitting the sheet current c b0 / (4 pi lambda)
    by temperature (gem.py:46-61)."""
    t_e = species[SHEET_ELECTRON].mass * species[SHEET_ELECTRON].vth[2] ** 2
    t_i = species[SHEET_ION].mass * species[SHEET_ION].vth[2] ** 2
    if t_e <= 0.0 or t_i <= 0.0:
        raise ConfigurationError("sheet species need nonzero thermal velocity")
    e = abs(species[SHEET_ION].charge)
    jz = -c * init.b0 / (4.0 * np.pi * init.sheet_thickness)
    dv = jz / (init.n0 * e)
    return -dv * t_e / (t_i + t_e), dv * t_i / (t_i + t_e)


def _check(species):
    if len(species) != 4 or [np.sign(s.charge) for s in species] != [-1.0, 1.0, -1.0, 1.0]:
        raise ConfigurationError("GEM needs 4 species: sheet e-, sheet i+, bg e-, bg i+")


def gem_fields(geom, init, precision=None):
    """E = 0; B = Harris tanh profile + flux perturbation (gem.py:104-113)."""
    mode = precision or PrecisionMode()
    f = FieldGrid.zeros(geom, mode)
    yc = geom.origin[1] + 0.5 * geom.Ly
    lam = init.sheet_thickness
    X, Y = np.meshgrid(geom.node_coords(0), geom.node_coords(1), indexing="ij")
    bx = init.b0 * np.tanh((Y - yc) / lam)
    psi0 = init.perturbation * init.b0
    carg = 2.0 * np.pi * X / geom.Lx
    sarg = np.pi * (Y - yc) / geom.Ly
    dbx = -psi0 * (np.pi / geom.Ly) * np.cos(carg) * np.sin(sarg)
    dby = psi0 * (2.0 * np.pi / geom.Lx) * np.sin(carg) * np.cos(sarg)
    f.E[:] = 0
    f.B[0] = ((bx + dbx)[:, :, None]).astype(f.dtype)
    f.B[1] = (dby[:, :, None]).astype(f.dtype)
    sync_periodic(f.B, geom)
    f.check_finite()
    return f


def smooth_e_field(geom, amp, dtype=np.float64):
    """A smooth, periodic, non-zero E of amplitude ``amp`` on the nodes (the
    GEM start has E = 0; benchmarks and tests use this so the E gather and
    the boundary-skip test see a real field)."""
    X, Y, Z = np.meshgrid(geom.node_coords(0), geom.node_coords(1), geom.node_coords(2),
                          indexing="ij")
    kx, ky, kz = (2 * np.pi / L for L in geom.lengths)
    return (amp * np.stack([np.sin(kx * X + 0.3) * np.cos(ky * Y),
                            np.cos(kz * Z) * np.sin(kx * X),
                            np.sin(ky * Y + 0.7) * np.cos(kz * Z - 0.2)])).astype(dtype)


def init_gem_host(geom, species, init=GemInit(), precision=None, c=1.0):
    """Bit-identical restatement of the reference loader (gem.py:64-115)."""
    _check(species)
    yc = geom.origin[1] + 0.5 * geom.Ly
    lam = init.sheet_thickness
    u_e, u_i = sheet_drifts(species, init, c)

    def sheet(x, y, z):
        return init.n0 / np.cosh((y - yc) / lam) ** 2

    def bg(x, y, z):
        return np.full_like(np.asarray(y, dtype=np.float64), init.background_fraction * init.n0)

    drifts = {SHEET_ELECTRON: (0.0, 0.0, u_e), SHEET_ION: (0.0, 0.0, u_i),
              BG_ELECTRON: (0.0, 0.0, 0.0), BG_ION: (0.0, 0.0, 0.0)}
    bufs = [init_maxwellian(s, geom, density_fn=sheet if s.species_id < 2 else bg,
                            seed=init.seed, precision=precision, drift=drifts[s.species_id])
            for s in species]
    return bufs, gem_fields(geom, init, precision)


def init_gem_device(geom, species, device, init=GemInit(), precision=None, c=1.0,
                    cells=None, id_offset=0):
    """The reference loader (gem.py:64-115 -> particles.py:177-241) generated
    in HBM, bit-identical to it (particles.init_maxwellian_device: the same
    Philox(seed, species) draws, ziggurat normals, expression order; sheet /
    background densities at the cell centres).

    ``cells`` = (first, count) restricts the load to a contiguous range of
    cells (x-fastest order), which is how ranks get their particle shard;
    ``id_offset`` is added to the (global) particle ids."""
    from .particles import init_maxwellian_device
    _check(species)
    yc = geom.origin[1] + 0.5 * geom.Ly
    lam = init.sheet_thickness
    u_e, u_i = sheet_drifts(species, init, c)

    def sheet(x, y, z):
        return init.n0 / np.cosh((y - yc) / lam) ** 2

    def bg(x, y, z):
        return np.full_like(np.asarray(y, dtype=np.float64), init.background_fraction * init.n0)

    drifts = {SHEET_ELECTRON: (0.0, 0.0, u_e), SHEET_ION: (0.0, 0.0, u_i),
              BG_ELECTRON: (0.0, 0.0, 0.0), BG_ION: (0.0, 0.0, 0.0)}
    out = []
    for s in species:
        p = init_maxwellian_device(s, geom, device, density_fn=sheet if s.species_id < 2 else bg,
                                   seed=init.seed, precision=precision,
                                   drift=drifts[s.species_id], cells=cells)
        if id_offset:
            p.ids += id_offset
        out.append(p)
    return out


def gem_deck_sizes(cells, ppc, species=4):
    return math.prod(cells) * ppc * species


def sample_host(geom, species, cells, init=GemInit(), precision=None, c=1.0, seed=1):
    """GEM-shaped particles of a contiguous cell range (x-fastest), drawn on
    the host with numpy — the CPU legs of the benchmark time the reference
    arithmetic on such a bounded sample of the same workload."""
    from .particles import ParticleBuffer
    _check(species)
    mode = precision or PrecisionMode()
    pd = mode.particle_dtype
    c0, nc = cells
    yc = geom.origin[1] + 0.5 * geom.Ly
    lam = init.sheet_thickness
    u_e, u_i = sheet_drifts(species, init, c)
    drift_z = {SHEET_ELECTRON: u_e, SHEET_ION: u_i, BG_ELECTRON: 0.0, BG_ION: 0.0}
    out = []
    for s in species:
        rng = np.random.default_rng([seed, s.species_id, c0])
        lin = np.arange(c0, c0 + nc)
        ci, cj, ck = lin % geom.nx, (lin // geom.nx) % geom.ny, lin // (geom.nx * geom.ny)
        n = nc * s.ppc
        pos = [geom.origin[a] + geom.spacings[a] * (np.repeat(ix, s.ppc) + rng.random(n))
               for a, ix in enumerate((ci, cj, ck))]
        vel = [(drift_z[s.species_id] if a == 2 else 0.0) + s.vth[a] * rng.standard_normal(n)
               for a in range(3)]
        ycell = geom.origin[1] + geom.dy * (cj + 0.5)
        dens = (init.n0 / np.cosh((ycell - yc) / lam) ** 2 if s.species_id < 2
                else np.full(nc, init.background_fraction * init.n0))
        q = np.repeat(s.charge * dens * geom.cell_volume / s.ppc, s.ppc)
        out.append(ParticleBuffer(*(a.astype(pd) for a in pos + vel + [q]),
                                  ids=np.arange(n, dtype=np.int64), species_id=s.species_id))
    return out


def init_uniform_device(geom, species, device, n0=1.0, precision=None, cells=None, seed=1):
    """The reference's uniform loader (make_state for init.kind != "gem",
    pipeline.py:140-151: init_maxwellian with density n0) generated in HBM,
    bit-identical to it (particles.init_maxwellian_device)."""
    from .particles import init_maxwellian_device

    def uniform(x, y, z):
        return np.full_like(np.asarray(y, dtype=np.float64), n0)

    return [init_maxwellian_device(s, geom, device, density_fn=uniform, seed=seed,
                                   precision=precision, cells=cells) for s in species]
