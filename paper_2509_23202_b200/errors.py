"""Exception types of the reference API (/root/reference/pkg/src/microfp/errors.py:8-13).

Same names and bases so ``except DataError`` code written against the reference
keeps working: shape / non-finite / unsupported-configuration problems raise
``DataError`` (a ``ValueError``); numerical failures ``NumericalError``.
"""


class DataError(ValueError):
    """Invalid input data: bad shapes, non-finite elements, unsupported formats."""


class NumericalError(RuntimeError):
    """A numerical procedure failed."""
