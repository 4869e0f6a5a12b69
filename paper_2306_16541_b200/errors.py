"""Exception types of the reference interface (``ad:26-31``, ``fu:35-36``)."""


class DimensionError(ValueError):
    """Raised when operand shapes are incompatible (reference: autodiff.DimensionError)."""


class TrainingError(RuntimeError):
    """Raised on non-finite values in a training-critical computation (autodiff.TrainingError)."""


class BenchmarkGateError(RuntimeError):
    """Correctness gate failed; timings are refused (fused.BenchmarkGateError)."""
