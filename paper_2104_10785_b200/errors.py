"""Exception types of the drop-in API (reference linops.py:26-35)."""


class ShapeMismatchError(ValueError):
    """Operand shapes are incompatible. The message names both shapes."""


class ConfigError(ValueError):
    """Bad configuration value (CLI exit code 2 in the reference)."""


class NumericalError(RuntimeError):
    """NaN/Inf encountered or a result is numerically undefined (exit code 3)."""
