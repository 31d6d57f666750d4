"""Precision modes and species parameters consumed by the path
(reference ``pkg/src/batchpic/config.py:19-81``)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError

SINGLE = "single"
DOUBLE = "double"


@dataclass(frozen=True)
class PrecisionMode:
    """Particle / field storage precision; "mixed" = single particles with
    double fields.  Double particles with single fields is rejected."""

    particles: str = DOUBLE
    fields: str = DOUBLE

    def __post_init__(self):
        for v in (self.particles, self.fields):
            if v not in (SINGLE, DOUBLE):
                raise ConfigurationError(f"precision must be single or double, got {v!r}")
        if self.particles == DOUBLE and self.fields == SINGLE:
            raise ConfigurationError("double particles with single fields is not supported")

    @classmethod
    def from_label(cls, label):
        return {"double": cls(DOUBLE, DOUBLE), "single": cls(SINGLE, SINGLE),
                "mixed": cls(SINGLE, DOUBLE)}[label]

    @property
    def label(self):
        if self.particles == SINGLE and self.fields == DOUBLE:
            return "mixed"
        return self.particles

    @property
    def particle_dtype(self):
        return np.float32 if self.particles == SINGLE else np.float64

    @property
    def field_dtype(self):
        return np.float32 if self.fields == SINGLE else np.float64


@dataclass(frozen=True)
class SpeciesParams:
    species_id: int
    charge: float
    mass: float
    ppc: int
    drift: tuple = (0.0, 0.0, 0.0)
    vth: tuple = (0.0, 0.0, 0.0)
    mover_iters: int = 3
    name: str = ""

    def __post_init__(self):
        if self.mass <= 0.0:
            raise ConfigurationError(f"species {self.species_id}: mass must be positive")
        if self.charge == 0.0:
            raise ConfigurationError(f"species {self.species_id}: charge must be nonzero")
        if self.ppc < 1:
            raise ConfigurationError(f"species {self.species_id}: ppc must be >= 1")
        if self.mover_iters < 1:
            raise ConfigurationError(f"species {self.species_id}: mover_iters must be >= 1")

    @property
    def qom(self):
        return self.charge / self.mass
