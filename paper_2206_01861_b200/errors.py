"""Exception taxonomy of the reference (pkg/src/lowbit/errors.py:1-13), preserved
at the boundary: UsageError for caller mistakes, ShapeError for inconsistent
operand shapes, plain ValueError for non-finite inputs."""


class ShapeError(ValueError):
    """Operand shapes are inconsistent (pkg/src/lowbit/errors.py:8)."""


class UsageError(ValueError):
    """Invalid arguments or state (pkg/src/lowbit/errors.py:12)."""
