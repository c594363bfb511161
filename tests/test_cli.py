"""Row f4 on CPU: JSON documents, the tfim_workload generator, CLI argument handling, exit
codes and report formats.  Document parity is against the reference's own writer output
(tests/golden/golden_cli.json, made by make_golden_cli.py).  The commands themselves need
the GPU engine and are checked in test_gpu_cli.py."""

import csv
import io
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2112_10239_b200 import cli
from paper_2112_10239_b200.circuits import circuit_from_dict, circuit_to_dict, custom_gate, Circuit
from paper_2112_10239_b200.errors import NumericalError, ParseError, UnknownGate
from paper_2112_10239_b200.hamiltonians import hamiltonian_from_dict, hamiltonian_to_dict
from paper_2112_10239_b200.report import RunReport, bond_profile, tfim_workload

HERE = os.path.dirname(os.path.abspath(__file__))
SCHEMA = os.path.join(os.path.dirname(HERE), "paper_2112_10239_b200", "schemas", "runreport.schema.json")


@pytest.fixture(scope="module")
def golden_cli():
    with open(os.path.join(HERE, "golden", "golden_cli.json")) as f:
        return json.load(f)


def test_documents_round_trip_reference_writer(golden_cli):
    for doc in golden_cli["circuits"].values():
        c = circuit_from_dict(doc)
        assert circuit_to_dict(c) == doc
        assert json.dumps(circuit_to_dict(c)) == json.dumps(doc)
    for doc in golden_cli["hams"].values():
        h = hamiltonian_from_dict(doc)
        assert hamiltonian_to_dict(h) == doc


def test_document_errors():
    for bad in ({}, {"n_qubits": 2}, {"n_qubits": 2, "gates": [{"wires": [0]}]}, {"n_qubits": 2, "gates": 5}):
        with pytest.raises(ParseError):
            circuit_from_dict(bad)
    with pytest.raises(UnknownGate):
        circuit_to_dict(Circuit(1, (custom_gate("u", (0,), np.eye(2)),), ()))
    bads = [[], {"terms": []}, {"n_qubits": 2, "terms": {}}, {"n_qubits": 2, "terms": [{"coeff": 1.0}]},
            {"n_qubits": 2, "terms": [{"coeff": True, "ops": {}}]}, {"n_qubits": 2, "terms": [{"coeff": 1, "ops": []}]},
            {"n_qubits": 2, "terms": [{"coeff": 1, "ops": {"a": "X"}}]},
            {"n_qubits": 2, "terms": [{"coeff": 1, "ops": {"0": "Q"}}]},
            {"n_qubits": 2, "terms": [{"coeff": 1, "ops": {"5": "X"}}]}]
    for bad in bads:
        with pytest.raises(ParseError):
            hamiltonian_from_dict(bad)


def test_tfim_workload_matches_reference_generator(golden_cli):
    for n, g in ((3, 7), (4, 25), (5, 1), (2, 0), (6, 100), (6, 60)):
        c = tfim_workload(n, g)
        o = O.tfim_workload_gates(n, g)
        assert len(c.gates) == g
        assert [(x.name, x.wires) for x in c.gates] == [(x[0], tuple(x[1])) for x in o.gates]
        assert list(c.trainable) == list(o.trainable)
    for bad in ((0, 5), (3, -1)):
        with pytest.raises(Exception):
            tfim_workload(*bad)
    # the factored bond bounds the Schmidt rank of the state at every cut (dense oracle)
    rng = np.random.default_rng(0)
    for n, g in ((4, 25), (6, 60), (5, 47)):
        prof = bond_profile(tfim_workload(n, g))
        assert len(prof) == n + 1 and prof[0] == prof[-1] == 1
        o = O.tfim_workload_gates(n, g)
        psi = O.simulate_dense(o, rng.uniform(-np.pi, np.pi, len(o.trainable)))
        for k in range(1, n):
            s = np.linalg.svd(psi.reshape(2 ** k, -1), compute_uv=False)
            assert int(np.sum(s > 1e-12 * s[0])) <= prof[k]


def _run(argv, capsys):
    code = cli.run_cli(argv)
    cap = capsys.readouterr()
    return code, cap.out, cap.err


def test_exit_codes_without_engine(tmp_path, capsys, monkeypatch, golden_cli):
    (tmp_path / "bell.json").write_text(json.dumps(golden_cli["circuits"]["bell"]))
    (tmp_path / "z0.json").write_text(json.dumps(golden_cli["hams"]["z0"]))
    (tmp_path / "bad.json").write_text("{not json")
    b, z = str(tmp_path / "bell.json"), str(tmp_path / "z0.json")
    code, _, err = _run(["expval", "--circuit", str(tmp_path / "nope.json"), "--ham", z], capsys)
    assert code == 2 and "nope.json" in err
    assert _run(["expval", "--circuit", str(tmp_path / "bad.json"), "--ham", z], capsys)[0] == 2
    assert _run(["expval", "--circuit", b], capsys)[0] == 2          # --ham is required
    assert _run(["ptrace", "--n", "4"], capsys)[0] == 2               # outside the hot path
    assert _run(["expval", "--circuit", b, "--ham", z, "--engine", "tt", "--eps", "-1"], capsys)[0] == 2
    assert _run(["expval", "--circuit", b, "--ham", z, "--engine", "tt", "--chi", "0"], capsys)[0] == 2
    assert _run(["expval", "--circuit", b, "--ham", z, "--engine", "mps"], capsys)[0] == 2
    code, out, _ = _run(["--version"], capsys)
    assert code == 0 and out.strip() == cli.__version__

    def boom(*a, **k):
        raise NumericalError("synthetic instability")

    monkeypatch.setattr(cli, "evaluate_expval", boom)
    code, _, err = _run(["expval", "--circuit", b, "--ham", z], capsys)
    assert code == 1 and "synthetic" in err


def test_report_formats_and_schema():
    jsonschema = pytest.importorskip("jsonschema")
    rep = RunReport("expval", 3, {"circuit": "c.json"}, {"value": -0.5, "gradient": [1.0, 2.0], "nested": {"a": 1}},
                    {"wall_ms": {"expval": 1.5}, "peak_bytes": 1024, "device": {"name": "B200"}})
    with open(SCHEMA) as f:
        schema = json.load(f)
    jsonschema.validate(rep.to_dict(), schema)
    buf = io.StringIO()
    cli.emit(rep, "csv", buf)
    rows = list(csv.DictReader(io.StringIO(buf.getvalue())))
    assert len(rows) == 1 and rows[0]["command"] == "expval" and float(rows[0]["value"]) == -0.5
    assert json.loads(rows[0]["gradient"]) == [1.0, 2.0] and rows[0]["nested.a"] == "1"
    buf = io.StringIO()
    cli.emit(rep, "json", buf)
    assert json.loads(buf.getvalue()) == rep.to_dict()
