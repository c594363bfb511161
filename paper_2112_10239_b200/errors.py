"""Exception taxonomy, mirroring the reference (``tnsim/errors.py:10-161``).

``InputError`` maps to CLI exit code 2, ``NumericalError`` to exit code 1
(reference ``errors.py:1-8``).  The engine's C status codes are mapped onto
these classes in :mod:`paper_2112_10239_b200._lib`.
"""


class TnsimError(Exception):
    """Base class for all errors raised by this package (reference errors.py:10)."""


class InputError(TnsimError):
    """Invalid arguments or shapes supplied by the caller (reference errors.py:14)."""


class NumericalError(TnsimError):
    """A computation produced values outside its numerical contract (reference errors.py:18)."""


class NotFinite(NumericalError):
    """NaN or Inf in an output."""


class UnknownGate(InputError):
    """Gate name is not in the standard set."""


class ArityMismatch(InputError):
    """Number of wires does not match the gate."""


class MissingParam(InputError):
    """A parameterised gate was constructed without a parameter."""


class TooManyQubits(InputError):
    """Qubit count exceeds a dense guard."""


class WireOutOfRange(InputError):
    """A gate references a wire outside the register."""


class UnsupportedArity(InputError):
    """The engine only handles one- and two-qubit gates."""


class SizeMismatch(InputError):
    """Operands describe registers of different sizes."""


class NonHermitianResidue(NumericalError):
    """An expectation value had an imaginary part above tolerance."""


class QubitOutOfRange(InputError):
    """A qubit index is outside the register."""


class ParamCountMismatch(InputError):
    """Parameter vector length does not match the circuit's trainable slots."""


class UnsupportedGateForShift(InputError):
    """No shift rule is registered for this gate."""


class DivergenceDetected(NumericalError):
    """The optimiser encountered a non-finite loss or gradient."""


class ParseError(InputError):
    """A text input could not be parsed."""


class SelfLoop(InputError):
    """Graph edge connects a vertex to itself."""


class DuplicateEdge(InputError):
    """The same undirected edge appears twice."""


class InvalidLabel(InputError):
    """A vertex index is negative or out of range."""


class BondTooLarge(InputError):
    """The gate-factored bond dimension exceeds what the B200 kernels support.

    New in this engine: the reference's SVD engine has no such limit (it
    re-factorises); the factored exact path supports chi <= 32 (complex64) and
    chi <= 16 (complex128 parity mode)."""


class EngineUnavailable(NumericalError):
    """The CUDA engine library is missing or no CUDA device is present.

    There is no CPU fallback: the product path fails loudly instead."""


class EngineError(NumericalError):
    """A CUDA launch or runtime call failed inside the engine."""


class TooManyVertices(InputError):
    """Brute force enumeration is capped; the graph is too big."""
