"""B200-native TT-circuit expectation-value / gradient engine.

The hot path of TensorLy-Quantum (arXiv 2112.10239): <psi(theta)|H|psi(theta)>
and d/dtheta for tensor-train factorised variational circuits, evaluated by
hand-written sm_100a kernels (``csrc/tq_engine.cu``) behind the C ABI of
``include/tq_engine.h``.  Parity is defined against the reference package
``tnsim`` (``/root/reference/pkg``), whose public names this package mirrors.
"""

__version__ = "0.1.0"

from .circuits import (  # noqa: F401
    Circuit,
    Gate,
    custom_gate,
    gate_matrix,
    gate_matrix_derivative,
    standard_gate,
    with_params,
)
from .errors import *  # noqa: F401,F403
from .hamiltonians import PAULI_MATRICES, PauliHamiltonian, PauliTerm, term, tfim  # noqa: F401
from .seeding import generator, spawn  # noqa: F401

_LAZY = {
    "grad_expval": "autodiff", "evaluate_expval": "autodiff", "expectation_values": "autodiff",
    "parameter_shift_grad": "autodiff", "finite_diff_grad": "autodiff", "init_params": "autodiff",
    "minimize": "autodiff", "energy": "autodiff", "MinimizeResult": "autodiff",
    "compile_chain": "chain", "layered_circuit": "workloads",
}


def __getattr__(name):  # torch-dependent modules load on first use
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    return getattr(importlib.import_module(f".{mod}", __name__), name)
