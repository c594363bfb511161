"""Row f4 on the GPU: the CLI subcommands and ``bench tfim`` through the B200 engine,
against the reference CLI's own RunReports (tests/golden/golden_cli.json) and the oracle."""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_2112_10239_b200 import cli  # noqa: E402
from paper_2112_10239_b200.report import bench_tfim  # noqa: E402
from paper_2112_10239_b200.errors import InputError  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SCHEMA = os.path.join(os.path.dirname(HERE), "paper_2112_10239_b200", "schemas", "runreport.schema.json")


@pytest.fixture(scope="module")
def golden_cli():
    with open(os.path.join(HERE, "golden", "golden_cli.json")) as f:
        return json.load(f)


@pytest.fixture()
def files(tmp_path, golden_cli):
    for k, v in {**golden_cli["circuits"], **golden_cli["hams"]}.items():
        (tmp_path / f"{k}.json").write_text(json.dumps(v))
    (tmp_path / "tri.txt").write_text("# triangle\n0 1\n1 2\n0 2\n")
    return tmp_path


def _report(argv, capsys):
    code = cli.run_cli(argv)
    cap = capsys.readouterr()
    assert code == 0, cap.err
    rep = json.loads(cap.out)
    jsonschema = pytest.importorskip("jsonschema")
    with open(SCHEMA) as f:
        jsonschema.validate(rep, json.load(f))
    return rep


def _ref(golden_cli, kind, key):
    for r in golden_cli["runs"]:
        if r["kind"] == kind and r["key"] == list(key):
            return r["report"]["outputs"]
    raise KeyError(key)


def test_expval_matches_reference_cli(files, capsys, golden_cli):
    for c, h in (("bell", "z0"), ("mixed", "h5")):
        rep = _report(["expval", "--circuit", str(files / f"{c}.json"), "--ham", str(files / f"{h}.json")], capsys)
        ref = _ref(golden_cli, "expval", (c, h))
        assert abs(rep["outputs"]["value"] - ref["value"]) < 1e-12
        assert rep["outputs"]["n_terms"] == ref["n_terms"] and rep["command"] == "expval"


def test_grad_methods_match_reference_cli(files, capsys, golden_cli):
    for c, h, methods in (("ry", "z0", ("ad", "shift", "fd")), ("mixed", "h5", ("ad", "shift"))):
        for m in methods:
            rep = _report(["grad", "--circuit", str(files / f"{c}.json"), "--ham", str(files / f"{h}.json"),
                           "--method", m], capsys)
            ref = _ref(golden_cli, "grad", (c, h, m))
            assert abs(rep["outputs"]["value"] - ref["value"]) < 1e-12
            tol = 1e-7 if m == "fd" else 1e-11
            np.testing.assert_allclose(rep["outputs"]["gradient"], ref["gradient"], atol=tol)
    rep = _report(["grad", "--circuit", str(files / "ry.json"), "--ham", str(files / "z0.json")], capsys)
    assert abs(rep["outputs"]["gradient"][0] + np.sin(0.7)) < 1e-12   # reference test_cli.py:106-118


def test_truncating_runs_match_reference_cli(files, capsys, golden_cli):
    c, h = str(files / "mixed.json"), str(files / "h5.json")
    rep = _report(["expval", "--circuit", c, "--ham", h, "--engine", "tt", "--chi", "2"], capsys)
    assert abs(rep["outputs"]["value"] - _ref(golden_cli, "expval", ("mixed", "h5", "chi2"))["value"]) < 1e-12
    rep = _report(["grad", "--circuit", c, "--ham", h, "--engine", "tt", "--chi", "2", "--method", "shift"], capsys)
    ref = _ref(golden_cli, "grad", ("mixed", "h5", "shift", "chi2"))
    np.testing.assert_allclose(rep["outputs"]["gradient"], ref["gradient"], atol=1e-11)
    # the reference's default engine is 'dense': --chi is ignored and the gradient is exact
    rep = _report(["grad", "--circuit", c, "--ham", h, "--chi", "2"], capsys)
    ref = _ref(golden_cli, "grad", ("mixed", "h5", "ad"))
    np.testing.assert_allclose(rep["outputs"]["gradient"], ref["gradient"], atol=1e-11)
    for key, extra in ((("mixed", "chi2"), ["--chi", "2"]), (("mixed", "tt"), [])):
        rep = _report(["simulate", "--circuit", c, "--engine", "tt"] + extra, capsys)
        ref = _ref(golden_cli, "simulate", key)
        assert rep["outputs"]["bond_dims"] == ref["bond_dims"], key
        assert abs(rep["outputs"]["norm"] - ref["norm"]) < 1e-12
        assert abs(rep["outputs"]["discarded_weight"] - ref["discarded_weight"]) < 1e-14
        np.testing.assert_allclose(rep["outputs"]["amplitudes"], ref["amplitudes"], atol=1e-12)


def test_simulate_amplitudes_match_reference_dense(files, capsys, golden_cli):
    for c in ("bell", "mixed"):
        rep = _report(["simulate", "--circuit", str(files / f"{c}.json")], capsys)
        ref = _ref(golden_cli, "simulate", (c,))
        assert abs(rep["outputs"]["norm"] - 1.0) < 1e-12
        np.testing.assert_allclose(rep["outputs"]["amplitudes"], ref["amplitudes"], atol=1e-12)
        assert rep["outputs"]["bond_dims"][0] == 1 and len(rep["outputs"]["bond_dims"]) == rep["outputs"]["n_qubits"] + 1


def test_bench_tfim_matches_reference(capsys, golden_cli):
    refs = [r for r in golden_cli["runs"] if r["kind"] == "bench"]
    for r in refs:
        i, ref = r["report"]["inputs"], r["report"]["outputs"]
        argv = ["bench", "tfim", "--n", str(i["n"]), "--gates", str(i["gates"]), "--seed", str(r["report"]["seed"])]
        argv += ["--chi", str(i["chi_max"]), "--eps", str(i["eps"])] + ([] if i["grad"] else ["--no-grad"])
        rep = _report(argv, capsys)
        out = rep["outputs"]
        for k in ("gate_count", "n_qubits", "n_params", "chi_max", "max_bond", "bond_histogram"):
            assert out[k] == ref[k], k
        assert abs(out["discarded_weight"] - ref["discarded_weight"]) < 1e-12
        assert abs(out["expval"] - ref["expval"]) < 1e-10
        if i["grad"]:
            assert abs(out["grad_value"] - ref["grad_value"]) < 1e-10
            assert abs(out["grad_norm"] - ref["grad_norm"]) < 1e-9
            assert out["grad_finite"] is True
        assert sum(out["bond_histogram"].values()) == i["n"] + 1
        again = _report(argv, capsys)
        rep.pop("measured"), again.pop("measured")
        assert rep == again


def test_maxcut_subcommand(files, capsys):
    rep = _report(["maxcut", "--graph", str(files / "tri.txt"), "--restarts", "2", "--max-iters", "40"], capsys)
    assert rep["outputs"]["cut"] == 2.0 and rep["outputs"]["optimal"] == 2.0


@pytest.fixture(scope="module")
def golden_st():
    with open(os.path.join(HERE, "golden", "golden_st.json")) as f:
        return json.load(f)


def test_straight_through_cli_matches_reference(files, capsys, golden_st):
    """``grad --engine tt --chi/--eps`` (method ad) and ``bench tfim --grad --chi``: the reference's
    straight-through gradient of its taped truncated state (autodiff.py:315-363, bench.py:136-141),
    against the reference CLI's own reports (make_golden_st.py)."""
    for run in golden_st["cli"]:
        argv = list(run["argv"])
        ref = run["report"]["outputs"]
        if argv[0] == "grad":
            argv[argv.index("--circuit") + 1] = str(files / "mixed.json")
            argv[argv.index("--ham") + 1] = str(files / "h5.json")
            out = _report(argv, capsys)["outputs"]
            if run["well_posed"]:   # see test_gpu_trunc.test_straight_through_gradient_matches_reference
                assert abs(out["value"] - ref["value"]) < 1e-10, argv
                np.testing.assert_allclose(out["gradient"], ref["gradient"], atol=1e-9, err_msg=str(argv))
        else:
            out = _report(argv, capsys)["outputs"]
            for k in ("gate_count", "n_params", "max_bond", "bond_histogram"):
                assert out[k] == ref[k], (argv, k)
            assert abs(out["expval"] - ref["expval"]) < 1e-10
            if run["well_posed"]:
                assert abs(out["grad_value"] - ref["grad_value"]) < 1e-9, argv
                assert abs(out["grad_norm"] - ref["grad_norm"]) < 1e-8 * max(1.0, ref["grad_norm"]), argv
            assert out["grad_finite"] is True
