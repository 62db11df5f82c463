"""Experiment harness and CLI (experiments.py / cli.py; reference experiments.py:46-296 and
cli.py:1-114): configuration validation messages, count-only rows, report formatting and
exit codes on the host; a full run on the GPU operator against the reference fixtures."""
import json
import os

import numpy as np
import pytest
import yaml

from conftest import load_golden
from paper_2001_07289_b200 import cli
from paper_2001_07289_b200.experiments import (CSV_COLUMNS, ExperimentConfig, ExperimentError, ReportRow,
                                               emit_report, run)


@pytest.mark.parametrize("data,msg", [
    ({"subdomains": [2, 2], "mesh": [8, 8], "foo": 1}, "unknown config keys"),
    ({"subdomains": [2, 2], "mesh": [8, 8], "preconditioner": "x"}, "unknown preconditioner"),
    ({"subdomains": [2, 2], "mesh": [8, 8], "weighting": "x"}, "unknown weighting"),
    ({"subdomains": [3, 2], "mesh": [8, 8]}, "3 subdomains do not divide 8 cells"),
    ({"subdomains": [2, 2], "mesh": [8, 8], "preconditioner": "bddc-so", "split": 3}, "split 3 does not divide"),
    ({"subdomains": [2, 2]}, "a mesh is required"),
    ({"subdomains": [2, 2], "mesh": [8]}, "same dimension"),
    ({"subdomains": [2, 2], "mesh": [8, 8], "coefficient": {"kind": "x"}}, "unknown coefficient kind"),
    ({"subdomains": [2, 2], "mesh": [8, 8], "element": "p2"}, "unknown element"),
])
def test_config_validation(data, msg):
    with pytest.raises(ValueError, match=msg):
        ExperimentConfig.from_dict(data)


def test_count_only_row_and_report():
    cfg = ExperimentConfig.from_dict({"subdomains": [10, 10, 10], "preconditioner": "bddc-so", "split": 4,
                                      "solve": False})
    row = run(cfg)
    assert row.coarse_size == 150039 and row.iters is None and row.dofs is None
    text = emit_report([row])
    lines = text.splitlines()
    assert lines[0] == ",".join(CSV_COLUMNS)
    assert lines[1] == ",10x10x10,4,bddc-so,vef,counting,,150039,,,,,"
    js = json.loads(emit_report([row], fmt="json"))
    assert js[0]["coarse_size"] == 150039 and js[0]["converged"] is None
    with pytest.raises(ValueError, match="unknown report format"):
        emit_report([row], fmt="xml")


def test_report_float_and_bool_formatting():
    row = ReportRow("4x4", "2x2", "1", "bddc", "vef", "counting", 9, 4, 3, 1.23456789, 0.5, 0.25, True)
    assert emit_report([row]).splitlines()[1] == "4x4,2x2,1,bddc,vef,counting,9,4,3,1.23457,0.5,0.25,true"


def test_cli_count_and_errors(tmp_path, capsys):
    assert cli.main(["count", "10x10x10", "2", "vef"]) == 0
    assert capsys.readouterr().out.strip() == "32319"
    bad = tmp_path / "bad.yaml"
    bad.write_text(yaml.safe_dump({"subdomains": [3, 2], "mesh": [8, 8]}))
    assert cli.main(["run", str(bad)]) == 1
    assert "do not divide" in capsys.readouterr().err
    assert cli.main(["preset", "nope", "--preset-dir", str(tmp_path)]) == 1
    count_only = tmp_path / "c.yaml"
    count_only.write_text(yaml.safe_dump({"runs": [{"subdomains": [4, 4, 4], "preconditioner": "bddc-so",
                                                     "split": 2, "solve": False}]}))
    assert cli.main(["run", str(count_only), "--format", "json"]) == 0
    assert json.loads(capsys.readouterr().out)[0]["coarse_size"] == 1647


@pytest.mark.gpu
def test_run_matches_reference_fixture(cuda_ok, tmp_path):
    """run() on the GPU operator reproduces the reference's cfg1 Q1 run (6 iterations, κ)."""
    g = load_golden("cfg1_q1_ref")
    cfg = {"mesh": [int(c) for c in g["cells"]], "subdomains": [int(s) for s in g["subs"]],
           "preconditioner": "bddc-so", "split": int(g["split"]), "recipe": str(g["recipe"]),
           "weighting": str(g["weighting"]), "tol": float(g["tol"]), "element": "q1"}
    row = run(ExperimentConfig.from_dict(cfg))
    assert row.converged and abs(row.iters - int(g["iterations"])) <= 1
    assert abs(row.kappa - float(g["kappa"])) <= 1e-6 * float(g["kappa"])
    assert row.coarse_size == int(g["coarse_size"]) and row.dofs == int(g["n"])
    p = tmp_path / "one.yaml"
    p.write_text(yaml.safe_dump(cfg))
    assert cli.main(["run", str(p), "--out", str(tmp_path / "r.csv")]) == 0
    assert (tmp_path / "r.csv").read_text().splitlines()[0] == ",".join(CSV_COLUMNS)
