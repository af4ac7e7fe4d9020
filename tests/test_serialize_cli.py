"""Circuit JSON and the ``qsim``-style CLI.

tests/golden/circuit_doc.json was written by the reference serializer
(tests/golden/make_golden.py); these tests load it with ours, check that we
write the identical document back, that the CLI optimizer passes give the
reference's gate counts, and (GPU) that ``run`` reproduces the reference's
amplitudes and classical registers for the same seed.
"""

import json
import os

import numpy as np
import pytest
from click.testing import CliRunner

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
DOC = os.path.join(GOLDEN, "circuit_doc.json")


def _meta():
    with open(os.path.join(GOLDEN, "serialize.json")) as fh:
        return json.load(fh)


def test_reference_document_round_trips_identically(tmp_path):
    from paper_2011_13524_b200 import serialize
    circ = serialize.load_circuit(DOC)
    with open(DOC) as fh:
        ref = json.load(fh)
    assert serialize.circuit_to_dict(circ) == ref
    out = tmp_path / "again.json"
    serialize.dump_circuit(circ, out)
    assert json.loads(out.read_text()) == ref


def test_format_errors():
    from paper_2011_13524_b200 import serialize
    with pytest.raises(serialize.CircuitFormatError):
        serialize.circuit_from_dict({"gates": []})
    with pytest.raises(serialize.CircuitFormatError, match="gate 0"):
        serialize.circuit_from_dict({"num_qubits": 2, "gates": [{"kind": "named", "name": "NOPE",
                                                                  "qubits": [0]}]})
    with pytest.raises(serialize.CircuitFormatError):
        serialize.circuit_from_dict({"num_qubits": 2, "gates": [
            {"kind": "diagonal", "targets": [0], "diag": [[1, 0], "x"]}]})
    with pytest.raises(ValueError):
        serialize.circuit_from_dict({"num_qubits": 2, "gates": [{"kind": "teleport"}]})


@pytest.mark.parametrize("opt,block,key", [("light", 2, "light"), ("heavy", 2, "heavy2"),
                                           ("heavy", 3, "heavy3")])
def test_cli_optimize_matches_reference_counts(tmp_path, opt, block, key):
    from paper_2011_13524_b200 import cli, serialize
    out = tmp_path / "opt.json"
    res = CliRunner().invoke(cli.main, ["optimize", DOC, "--opt", opt, "--block-size", str(block),
                                        "--output", str(out)])
    assert res.exit_code == 0, res.output
    assert serialize.load_circuit(out).get_gate_count() == _meta()["optimizer_counts"][key]


def test_cli_rejects_bad_input(tmp_path):
    from paper_2011_13524_b200 import cli
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    res = CliRunner().invoke(cli.main, ["optimize", str(bad), "--output", str(tmp_path / "o")])
    assert res.exit_code == 1
    res = CliRunner().invoke(cli.main, ["bench", "--repeats", "0"])
    assert res.exit_code == 1


@pytest.mark.gpu
def test_cli_run_matches_reference(tmp_path):
    from paper_2011_13524_b200 import cli
    out = tmp_path / "result.json"
    res = CliRunner().invoke(cli.main, ["run", DOC, "--seed", "7", "--output", str(out)])
    assert res.exit_code == 0, res.output
    doc = json.loads(out.read_text())
    amps = np.array([complex(r, i) for r, i in doc["amplitudes"]])
    ref = np.load(os.path.join(GOLDEN, "serialize.npz"))["amplitudes"]
    assert np.max(np.abs(amps - ref)) <= 1e-12
    assert doc["classical_registers"] == _meta()["cregs"]
    res = CliRunner().invoke(cli.main, ["run", DOC, "--seed", "7", "--samples", "16"])
    assert res.exit_code == 0 and len(json.loads(res.output)["samples"]) == 16


@pytest.mark.gpu
def test_cli_bench_report(tmp_path):
    from paper_2011_13524_b200 import cli
    out = tmp_path / "report.csv"
    res = CliRunner().invoke(cli.main, ["bench", "--family", "cnot-ring", "--nqubits", "6,8",
                                        "--opt", "heavy", "--block-size", "3",
                                        "--format", "csv", "--output", str(out)])
    assert res.exit_code == 0, res.output
    lines = out.read_text().strip().splitlines()
    assert lines[0].startswith("family,num_qubits") and len(lines) == 3
    out = tmp_path / "report.json"
    res = CliRunner().invoke(cli.main, ["bench", "--nqubits", "10-12", "--depth", "3",
                                        "--output", str(out)])
    assert res.exit_code == 0, res.output
    rep = json.loads(out.read_text())
    assert [p["num_qubits"] for p in rep["results"]] == [10, 11, 12]
    assert rep["environment"]["device"]["sm_count"] > 0
