"""Node-grid geometry — the subset of the reference ``GridGeometry``
(``pkg/src/batchpic/geometry.py:24-207``) the mover/deposit path consumes:
box, spacings, boundary kinds, node extents, the cell sort key and the
control volumes used by deposition.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError, DomainError

PERIODIC = "periodic"
REFLECTING = "reflecting"


@dataclass(frozen=True)
class GridGeometry:
    """nx*ny*nz cells, nodes (nx+1, ny+1, nz+1); ``L = n * d`` exactly."""

    nx: int
    ny: int
    nz: int
    dx: float
    dy: float
    dz: float
    Lx: float
    Ly: float
    Lz: float
    origin: tuple = (0.0, 0.0, 0.0)
    bc: tuple = (PERIODIC, PERIODIC, PERIODIC)

    def __post_init__(self):
        for n in self.counts:
            if not isinstance(n, int) or n < 1:
                raise ConfigurationError(f"cell counts must be positive integers, got {n}")
        for kind in self.bc:
            if kind not in (PERIODIC, REFLECTING):
                raise ConfigurationError(f"unknown boundary kind {kind!r}")
        for n, d, L, ax in zip(self.counts, self.spacings, self.lengths, "xyz"):
            if d <= 0.0 or L <= 0.0:
                raise ConfigurationError(f"non-positive spacing/length on axis {ax}")
            if n * d != L:
                raise ConfigurationError(f"L{ax} = {L!r} is not exactly n{ax} * d{ax}")

    @classmethod
    def from_box(cls, counts, lengths, origin=(0.0, 0.0, 0.0),
                 bc=(PERIODIC, PERIODIC, PERIODIC)):
        nx, ny, nz = (int(c) for c in counts)
        Lx, Ly, Lz = (float(v) for v in lengths)
        return cls(nx=nx, ny=ny, nz=nz, dx=Lx / nx, dy=Ly / ny, dz=Lz / nz,
                   Lx=Lx, Ly=Ly, Lz=Lz, origin=tuple(float(v) for v in origin),
                   bc=tuple(bc))

    @property
    def counts(self):
        return (self.nx, self.ny, self.nz)

    @property
    def spacings(self):
        return (self.dx, self.dy, self.dz)

    @property
    def lengths(self):
        return (self.Lx, self.Ly, self.Lz)

    @property
    def node_shape(self):
        return (self.nx + 1, self.ny + 1, self.nz + 1)

    @property
    def n_nodes(self):
        return (self.nx + 1) * (self.ny + 1) * (self.nz + 1)

    @property
    def n_cells(self):
        return self.nx * self.ny * self.nz

    @property
    def cell_volume(self):
        return self.dx * self.dy * self.dz

    def node_coords(self, axis):
        return self.origin[axis] + self.spacings[axis] * np.arange(
            self.counts[axis] + 1, dtype=np.float64)

    def cell_centers(self, axis):
        return self.origin[axis] + self.spacings[axis] * (
            np.arange(self.counts[axis], dtype=np.float64) + 0.5)

    def cell_index_of(self, x, y, z):
        """Linear cell index, x fastest, upper faces clamped; f64 arithmetic
        (geometry.py:152-159)."""
        idx = []
        for q, o, d, n in zip((x, y, z), self.origin, self.spacings, self.counts):
            i = ((np.asarray(q, np.float64) - o) / d).astype(np.int64)
            idx.append(np.minimum(i, n - 1))
        i, j, k = idx
        if (i < 0).any() or (j < 0).any() or (k < 0).any():
            raise DomainError("positions below the box origin")
        return i + self.nx * (j + self.ny * k)

    def axis_weights(self, axis):
        """Control-volume share per node: reflecting walls 1/2, duplicate
        periodic plane 0 (geometry.py:161-174)."""
        n = self.counts[axis]
        w = np.ones(n + 1)
        if self.bc[axis] == PERIODIC:
            w[n] = 0.0
        else:
            w[0] = w[n] = 0.5
        return w

    def node_weights(self):
        wx, wy, wz = (self.axis_weights(a) for a in range(3))
        return wx[:, None, None] * wy[None, :, None] * wz[None, None, :]

    def inv_node_volume(self, dtype=np.float64):
        """1/(control volume) per node, the deposit divisor: walls double it
        (geometry.py:186-203; product of factors, then / cell volume)."""
        f = []
        for a in range(3):
            v = np.ones(self.counts[a] + 1)
            if self.bc[a] == REFLECTING:
                v[0] = v[-1] = 2.0
            f.append(v)
        inv = (f[0][:, None, None] * f[1][None, :, None] * f[2][None, None, :]) / self.cell_volume
        return np.ascontiguousarray(inv.astype(dtype))

    def unique_slices(self):
        """Slices dropping the duplicated periodic planes (fields.unique_view)."""
        return tuple(slice(0, n if k == PERIODIC else n + 1)
                     for n, k in zip(self.counts, self.bc))
