"""B200-native TT-circuit expectation/gradient engine (TensorLy-Quantum hot path)."""

__version__ = "0.1.0"
