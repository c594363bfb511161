"""GPU tests of the wider API surface: MBE MaxCut (cfg3), inner products,
product-state inputs, tlquantum-style TTCircuit, residue checks."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import oracle as O  # noqa: E402
from helpers_engine import grad_ok64, to_circuit  # noqa: E402
from paper_2112_10239_b200 import autodiff as AD  # noqa: E402
from paper_2112_10239_b200 import maxcut as MC  # noqa: E402
from paper_2112_10239_b200 import tlq  # noqa: E402
from paper_2112_10239_b200.errors import NonHermitianResidue, SizeMismatch  # noqa: E402
from paper_2112_10239_b200.hamiltonians import PauliHamiltonian, term, tfim  # noqa: E402
from paper_2112_10239_b200.workloads import layered_circuit, theta_sets  # noqa: E402


def test_mbe_objective_matches_reference(golden_small):
    d = golden_small["mbe10"]
    g = MC.Graph(10, tuple(tuple(e) for e in d["edges"]))
    c = MC.brickwork_ansatz(5, d["depth"])
    th = np.array(d["theta"])
    for dtype, tol in (("complex128", 1e-10), ("complex64", 2e-5)):
        loss, grad = MC.mbe_objective(c, g, alpha=d["alpha"], dtype=dtype)(th)
        assert abs(loss - d["loss"]) < tol * max(1, abs(d["loss"])), dtype
        assert np.max(np.abs(grad - np.array(d["grad"]))) < tol * max(1, np.max(np.abs(d["grad"]))), dtype
    ev = MC.vertex_expectations(c, th, g)
    np.testing.assert_allclose(ev, d["vertex"], atol=1e-12)
    asg = MC.round_cut(ev)
    assert list(asg) == d["assignment"] and MC.cut_value(g, asg) == d["cut"]


def test_mbe_cfg3_bit_exact_cut(golden_large):
    pairs = golden_large["cfg3_edges"]
    g = MC.Graph(2048, tuple((int(u), int(v), 1.0) for u, v in pairs))
    c = MC.brickwork_ansatz(1024, 4)
    th = golden_large["cfg3_theta"]
    ev = MC.vertex_expectations(c, th, g)  # complex128 readouts
    np.testing.assert_allclose(ev, golden_large["cfg3_vertex"], atol=1e-11)
    asg = np.array(MC.round_cut(ev), dtype=np.int8)
    np.testing.assert_array_equal(asg, golden_large["cfg3_assignment"])
    assert MC.cut_value(g, asg) == float(golden_large["cfg3_cut"])
    ref = float(golden_large["cfg3_loss"])
    for dtype in ("complex128", "complex64"):   # the drop-in default and the fast path
        loss, grad = MC.mbe_objective(c, g, dtype=dtype)(th)
        assert abs(loss - ref) < 1e-5 * max(1.0, abs(ref)), dtype
        assert grad_ok64(grad, golden_large["cfg3_grad"]), dtype


def test_solve_maxcut_small_graphs():
    tri = MC.Graph(3, ((0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0)))
    assert MC.solve_maxcut(tri, restarts=3, max_iters=80, seed=1).cut_value == 2.0
    c4 = MC.Graph(4, ((0, 1, 1.0), (1, 2, 1.0), (2, 3, 1.0), (3, 0, 1.0)))
    assert MC.solve_maxcut(c4, restarts=3, max_iters=80, seed=1).cut_value == 4.0
    a = MC.solve_maxcut(c4, restarts=2, max_iters=30, seed=7)
    b = MC.solve_maxcut(c4, restarts=2, max_iters=30, seed=7, threads=2)
    assert a == b


def test_inner_product_matches_reference(golden_small):
    d = golden_small["inner8"]
    c = to_circuit(d["circuit"])
    for dtype, tol in (("complex128", 1e-12), ("complex64", 2e-6)):
        ip = AD.state_inner_product(c, d["theta_b"], c, d["theta_a"], dtype=dtype)
        assert abs(ip - complex(d["re"], d["im"])) < tol, dtype


def test_product_state_inputs_against_oracle():
    rng = np.random.default_rng(5)
    n = 6
    vecs = rng.normal(size=(n, 2)) + 1j * rng.normal(size=(n, 2))
    vecs /= np.linalg.norm(vecs, axis=1, keepdims=True)
    c = layered_circuit(n, 6, "ry", "cz")
    th = theta_sets(c.n_params, 1, seed=3)[0]
    oc = O.ry_cz_layers(n, 6)
    ov, og = O.grad_expval_tt(oc, O.tfim_terms(n), th, init_vectors=vecs)
    circ = tlq.ansatz(n, 6, dtype="complex128")
    with torch.no_grad():
        for p, t in zip(circ._params, th):
            p.fill_(float(t))
    state = tlq.ProductState(vecs)
    e = circ.forward_expectation_value(state, tfim(n))
    e.backward()
    g = np.array([float(p.grad) for p in circ._params])
    assert abs(float(e.detach()) - ov) < 1e-10
    np.testing.assert_allclose(g, og, atol=1e-10)
    # <compare|U|state> for product states against the dense oracle
    psi = O.simulate_dense(oc, th).reshape(-1)
    comp = tlq.spins_to_tt_state([1, 0, 1, 1, 0, 0])
    idx = int("101100", 2)
    ip = circ.state_inner_product(tlq.spins_to_tt_state([0] * n), comp)
    assert abs(ip - psi[idx]) < 1e-12


def test_ttcircuit_matches_reference_circuit(golden_small):
    circ = tlq.ansatz(10, 4, rot="y", ent="cnot")
    case = golden_small["cases"][0]
    with torch.no_grad():
        for p, t in zip(circ._params, case["theta"]):
            p.fill_(float(t))
    assert circ.to_circuit().structure_key() == to_circuit(case["circuit"]).structure_key()
    e = circ.forward_expectation_value(tlq.spins_to_tt_state([0] * 10), tlq.ising_hamiltonian(10))
    e.backward()
    assert abs(float(e) - case["value"]) < 1e-5 * max(1, abs(case["value"]))
    g = np.array([float(p.grad) for p in circ._params])
    assert grad_ok64(g, case["grad"])


def test_non_hermitian_residue_raises():
    c = layered_circuit(4, 3)
    th = theta_sets(c.n_params, 1, seed=2)[0]
    ham = PauliHamiltonian(4, (term(1.0 + 0.3j, {0: "Z"}),))
    with pytest.raises(NonHermitianResidue):
        AD.evaluate_expval(c, ham, th)
    with pytest.raises(SizeMismatch):
        MC.mbe_objective(MC.brickwork_ansatz(3, 2), MC.Graph(3, ((0, 1, 1.0),)))


def test_expectation_values_batched_against_oracle():
    c = layered_circuit(12, 8, "rx", "cz")
    th = theta_sets(c.n_params, 3, seed=8)
    groups = [{0: "X"}, {5: "Y", 6: "Z"}, {2: "Z", 9: "X"}]
    vals = AD.expectation_values(c, th, groups, dtype="complex128")
    oc = O.ry_cz_layers(12, 8, "rx", "cz")
    for b in range(3):
        ref = O.taped_term_values(oc, th[b], [tuple(sorted(g.items())) for g in groups])
        np.testing.assert_allclose(vals[b], ref, atol=1e-12)


def test_inner_product_gradients_exact():
    """d<bra(tb)|ket(tk)>/dtheta through InnerFunction (batched shift rule) against central
    differences of the oracle's dense states, on both sides and for a batch."""
    from paper_2112_10239_b200.circuits import Circuit, standard_gate

    n = 6
    gk = [standard_gate(("ry", "rx", "rz")[q % 3], (q,), 0.0) for q in range(n)]
    gk += [standard_gate("cnot", (q, q + 1)) for q in range(0, n - 1, 2)]
    gk += [standard_gate("crz", (1, 2), 0.0), standard_gate("ry", (4,), 0.0)]
    ck = Circuit(n, tuple(gk), tuple(i for i, g in enumerate(gk) if g.param is not None))
    gb = [standard_gate("rx", (q,), 0.0) for q in range(n)] + [standard_gate("cz", (q, q + 1)) for q in range(1, n - 1, 2)]
    cb = Circuit(n, tuple(gb), tuple(range(n)))
    rng = np.random.default_rng(8)
    tk = rng.uniform(-np.pi, np.pi, (3, ck.n_params))
    tb = rng.uniform(-np.pi, np.pi, (3, cb.n_params))
    thk = torch.tensor(tk, dtype=torch.float64, device="cuda", requires_grad=True)
    thb = torch.tensor(tb, dtype=torch.float64, device="cuda", requires_grad=True)
    z = AD.inner(ck, thk, cb, thb)
    w = torch.tensor([0.3 - 0.2j, -0.5 + 0.1j, 0.25 + 0.6j], dtype=torch.complex128, device="cuda")
    loss = (w * z).real.sum() + (z.abs() ** 2).sum()
    loss.backward()

    def oc(c):
        return O.OCircuit(c.n_qubits, [(g.name, tuple(g.wires), g.param) for g in c.gates], list(c.trainable))

    def zval(b, a, bb):
        return np.vdot(O.simulate_dense(oc(cb), bb).reshape(-1), O.simulate_dense(oc(ck), a).reshape(-1))

    wn = w.cpu().numpy()
    for b in range(3):
        zz = zval(b, tk[b], tb[b])
        assert abs(complex(z[b].detach().cpu()) - zz) < 1e-12

        def lossb(a, bb):
            v = zval(b, a, bb)
            return (wn[b] * v).real + abs(v) ** 2

        h = 1e-6
        for k in range(ck.n_params):
            e = np.zeros(ck.n_params)
            e[k] = h
            fd = (lossb(tk[b] + e, tb[b]) - lossb(tk[b] - e, tb[b])) / (2 * h)
            assert abs(float(thk.grad[b, k]) - fd) < 1e-7, (b, k)
        for k in range(cb.n_params):
            e = np.zeros(cb.n_params)
            e[k] = h
            fd = (lossb(tk[b], tb[b] + e) - lossb(tk[b], tb[b] - e)) / (2 * h)
            assert abs(float(thb.grad[b, k]) - fd) < 1e-7, (b, k)


def test_adam_graph_matches_eager_iterations():
    """maxcut.AdamGraph (captured iteration, flags checked every 16 replays) against the eager
    per-restart loop it replaces, including per-restart freezing and the final no-update step."""
    from paper_2112_10239_b200 import maxcut as MC
    from paper_2112_10239_b200.seeding import generator

    rng = generator(7)
    graph = MC.pairing_graph(24, 3, rng)
    circuit = MC.brickwork_ansatz(12, 3)
    theta0 = np.stack([rng.uniform(-np.pi, np.pi, circuit.n_params) for _ in range(4)])
    obj = MC.MBEObjective(circuit, graph, 1.0, batch=4)
    th_g, val_g, it_g = MC.AdamGraph(obj, theta0, 0.1, max_iters=37, tol=0.05).run(check_every=5)

    dev = obj.device
    theta = torch.tensor(theta0, dtype=torch.float64, device=dev)
    m = torch.zeros_like(theta)
    v = torch.zeros_like(theta)
    active = torch.ones(4, dtype=torch.bool, device=dev)
    value = torch.zeros(4, dtype=torch.float64, device=dev)
    iters = torch.zeros(4, dtype=torch.int64, device=dev)
    for it in range(38):
        loss, grad = obj(theta.to(obj.tdt))
        grad = grad.double()
        value = torch.where(active, loss, value)
        iters = torch.where(active, torch.full_like(iters, it), iters)
        active = active & (torch.linalg.vector_norm(grad, dim=1) >= 0.05)
        if it == 37 or not bool(active.any()):
            break
        m = torch.where(active[:, None], 0.9 * m + 0.1 * grad, m)
        v = torch.where(active[:, None], 0.999 * v + 0.001 * grad * grad, v)
        upd = 0.1 * (m / (1 - 0.9 ** (it + 1))) / (torch.sqrt(v / (1 - 0.999 ** (it + 1))) + 1e-8)
        theta = torch.where(active[:, None], theta - upd, theta)
    np.testing.assert_allclose(th_g, theta.cpu().numpy(), atol=1e-12)
    np.testing.assert_allclose(val_g, value.cpu().numpy(), atol=1e-12)
    np.testing.assert_array_equal(it_g, iters.cpu().numpy())


def test_expval_program_serving_paths():
    """program.ExpvalProgram (the serving path bench.py times): eager, captured device graph
    and the captured host-buffer graph (H2D, kernels, D2H in one launch) all give the same
    energies and gradients as grad_expval, and repeated calls see each new batch."""
    from paper_2112_10239_b200.program import ExpvalProgram

    c, h = layered_circuit(24, 6, "ry", "cz"), tfim(24)
    B = 16
    th = [theta_sets(c.n_params, B, seed=s).astype(np.float32) for s in (1, 2)]
    ref = [AD.grad_expval(c, h, t.astype(np.float64), device="cuda:0") for t in th]
    prog = ExpvalProgram(c, h, B)
    e, g = prog(th[0])                                    # eager
    np.testing.assert_allclose(e, ref[0][0], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(g, ref[0][1], rtol=1e-4, atol=1e-5)
    prog.capture()
    for k in (0, 1, 0):
        e, g = prog(th[k])                                # numpy input -> staging buffer -> io graph
        np.testing.assert_allclose(e, ref[k][0], rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(g, ref[k][1], rtol=1e-4, atol=1e-5)
    pinned = torch.tensor(th[1]).pin_memory()
    e, g = prog(pinned)                                   # foreign pinned tensor
    np.testing.assert_allclose(e, ref[1][0], rtol=1e-5, atol=1e-5)
    prog.theta_dev.copy_(torch.tensor(th[0], device="cuda:0"))
    energy, grad = prog.replay()                          # device-resident path
    np.testing.assert_allclose(energy[:, 0].double().cpu().numpy(), ref[0][0], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(grad.cpu().numpy(), ref[0][1], rtol=1e-4, atol=1e-5)


def test_mbe_objective_captured_calls_track_inputs(golden_small):
    """mbe_objective's fun replays a captured graph from the second call on: every call must
    still see its own theta (against the eager batched objective), and bad inputs raise."""
    from paper_2112_10239_b200.errors import InputError, ParamCountMismatch

    d = golden_small["mbe10"]
    g = MC.Graph(10, tuple(tuple(e) for e in d["edges"]))
    c = MC.brickwork_ansatz(5, d["depth"])
    fun = MC.mbe_objective(c, g, alpha=d["alpha"], dtype="complex128")
    obj = MC.MBEObjective(c, g, d["alpha"], dtype="complex128", device="cuda:0")
    rng = np.random.default_rng(3)
    for _ in range(4):
        th = rng.uniform(-np.pi, np.pi, c.n_params)
        loss, grad = fun(th)
        rl, rg = obj(torch.tensor(th[None], device="cuda:0"))
        assert abs(loss - float(rl[0])) < 1e-10
        np.testing.assert_allclose(grad, rg[0].cpu().numpy(), atol=1e-10)
    with pytest.raises(ParamCountMismatch):
        fun(np.zeros(c.n_params + 1))
    with pytest.raises(InputError):
        fun(np.full(c.n_params, np.nan))


def test_mbe_host_evaluator_batched_matches_per_restart(golden_small):
    """MBEObjective.host_evaluator(B): B restarts per captured host round trip (the cfg3 bench
    e2e path) equal B single-restart calls of the reference-shaped mbe_objective fun."""
    from paper_2112_10239_b200.errors import ParamCountMismatch, SizeMismatch

    d = golden_small["mbe10"]
    g = MC.Graph(10, tuple(tuple(e) for e in d["edges"]))
    c = MC.brickwork_ansatz(5, d["depth"])
    fun = MC.mbe_objective(c, g, alpha=d["alpha"], dtype="complex128")
    obj = MC.MBEObjective(c, g, d["alpha"], dtype="complex128", device="cuda:0", batch=3)
    hev = obj.host_evaluator(3)
    rng = np.random.default_rng(5)
    for _ in range(3):   # eager, capture, replay
        th = rng.uniform(-np.pi, np.pi, (3, c.n_params))
        loss, grad = hev(th)
        for r in range(3):
            l1, g1 = fun(th[r])
            assert abs(loss[r] - l1) < 1e-10
            np.testing.assert_allclose(grad[r], g1, atol=1e-10)
    assert hev.h2d_bytes == 3 * c.n_params * 8 and hev.d2h_bytes == 3 * (c.n_params + 1) * 8
    with pytest.raises(SizeMismatch):
        hev(np.zeros((2, c.n_params)))
    with pytest.raises(ParamCountMismatch):
        hev(np.zeros((3, c.n_params + 1)))
