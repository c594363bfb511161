"""The real-path sweeps (tq_chain.real_path, csrc/tq_engine.cu gmac<RE>): for a real problem
(ry rotations, CZ / CNOT splits, TFIM X/Z terms) the complex arithmetic has exactly-zero
imaginary parts, so the real-part instantiations must reproduce the complex ones BIT FOR BIT.
Checked by running the same device plan with the flag on and forced off, at chi = 4 ... 32."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_2112_10239_b200 import chain as C  # noqa: E402
from paper_2112_10239_b200 import engine as E  # noqa: E402
from paper_2112_10239_b200.hamiltonians import tfim  # noqa: E402
from paper_2112_10239_b200.workloads import layered_circuit, theta_sets  # noqa: E402


@pytest.mark.parametrize("n,layers,ent", [(40, 20, "cz"), (36, 14, "cnot"), (30, 20, "cz"), (24, 10, "cz"),
                                          (16, 4, "cnot")])
def test_real_path_bit_identical_to_complex(n, layers, ent):
    c = layered_circuit(n, layers, "ry", ent)
    terms = C.normalize_terms(tfim(n))
    B = 6
    dp = E.device_plan(c, terms, "energy", B, "cuda:0", segments=2)
    assert dp.chain.real_path == 1
    th = torch.tensor(theta_sets(c.n_params, B, seed=n), dtype=torch.float32, device="cuda:0")
    coef = torch.tensor([[t[0].real for t in terms]], dtype=torch.float32, device="cuda:0")
    e1, g1 = E.energy_grad_raw(dp, th, coef, True, "complex64")
    dp.chain.real_path = 0
    try:
        e0, g0 = E.energy_grad_raw(dp, th, coef, True, "complex64")
    finally:
        dp.chain.real_path = 1
    assert torch.equal(e1, e0)
    assert torch.equal(g1, g0)


def test_real_path_flag_follows_the_problem():
    for rot, ent, ham, want in (("ry", "cz", tfim(12), 1), ("ry", "cnot", tfim(12), 1), ("rx", "cz", tfim(12), 0),
                                ("rz", "cz", tfim(12), 0)):
        c = layered_circuit(12, 6, rot, ent)
        dp = E.device_plan(c, C.normalize_terms(ham), "energy", 2, "cuda:0")
        assert dp.chain.real_path == want, (rot, ent)
