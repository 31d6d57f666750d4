"""Exception types raised on the path (same names and bases as the
reference's ``pkg/src/batchpic/errors.py:4-24``)."""


class ConfigurationError(ValueError):
    """Invalid run configuration."""


class DomainError(ValueError):
    """A position that should be inside the simulation box is not."""


class IntegrityError(RuntimeError):
    """Runaway particle, unmappable midpoint, non-finite field."""
