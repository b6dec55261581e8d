"""Exception taxonomy of the reference (errors.py:4-31), reproduced for the drop-in API.

``StructuralError`` is a ``ValueError``; ``FactorizationError`` a
``RuntimeError`` carrying ``.row``; ``SingularBlockError`` subclasses it.
"""


class StructuralError(ValueError):
    """A matrix, pattern, or schedule violates a structural requirement."""


class FactorizationError(RuntimeError):
    """Numeric factorization could not proceed (zero or unusable pivot)."""

    def __init__(self, message, row=None):
        super().__init__(message)
        self.row = row


class SingularBlockError(FactorizationError):
    """A diagonal block was singular to working precision."""


class MatrixMarketError(ValueError):
    """A Matrix Market file could not be parsed (reference errors.py MatrixMarketError).

    ``line`` holds the 1-based physical line number of the problem; the
    message starts with ``"line <n>: "`` when it is known.
    """

    def __init__(self, message, line=None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")
