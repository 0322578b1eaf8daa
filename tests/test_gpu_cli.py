"""The reference's command line routed to the device path (cli.py, SURVEY.md
§8(f) f4). Mirrors the reference's test_cli.py on its own pair
(test_cli.py:26-32) and compares every number with the output of the
reference's CLI on the same files (tests/golden/io/, make_io_golden.py)."""

import csv
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2404_09459_b200 import cli

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "io")
G1, G2 = os.path.join(GOLD, "g1.mtx"), os.path.join(GOLD, "g2.mtx")
PAIR = ["--g1", G1, "--g2", G2]


def _json(path):
    with open(path) as fh:
        return json.load(fh)


def _close(ours, ref, tol):
    a, b = np.asarray(ours, dtype=float), np.asarray(ref, dtype=float)
    assert a.shape == b.shape
    fin = np.isfinite(b)
    assert np.array_equal(fin, np.isfinite(a)) and np.array_equal(a[~fin], b[~fin])
    assert np.max(np.abs(a[fin] - b[fin]), initial=0.0) <= tol, np.max(np.abs(a[fin] - b[fin]))


def test_gsv_direct_csv_matches_reference(tmp_path, capsys):
    assert cli.main(["gsv", *PAIR, "--method", "direct"]) == 0
    lines = capsys.readouterr().out.splitlines()
    ref = open(os.path.join(GOLD, "gsv_direct.csv")).read().splitlines()
    assert lines[0] == "index,alpha,beta" == ref[0] and len(lines) == len(ref) == 1 + 12 + 2
    assert lines[-2:] == ref[-2:]  # r, s
    ours = np.array([[float(x) for x in ln.split(",")[1:]] for ln in lines[1:13]])
    theirs = np.array([[float(x) for x in ln.split(",")[1:]] for ln in ref[1:13]])
    _close(ours, theirs, 1e-13)


def test_gsv_randomized_matches_reference(tmp_path):
    out = tmp_path / "gsv.csv"
    assert cli.main(["gsv", *PAIR, "--seed", "9", "-o", str(out)]) == 0
    ours = list(csv.reader(open(out)))
    ref = list(csv.reader(open(os.path.join(GOLD, "gsv_seed9.csv"))))
    assert [r[0] for r in ours] == [r[0] for r in ref] and ours[-2:] == ref[-2:]
    _close([r[1:] for r in ours[1:13]], [r[1:] for r in ref[1:13]], 1e-12)


def test_compare_json_matches_reference(tmp_path):
    out = tmp_path / "report.json"
    assert cli.main(["compare", *PAIR, "--seed", "7", "-o", str(out), "--format", "json"]) == 0
    rep, ref = _json(out), _json(os.path.join(GOLD, "compare_seed7.json"))
    assert rep["kind"] == "comparative_report" and rep["meta"] == ref["meta"]
    assert (rep["r"], rep["s"], rep["n"]) == (ref["r"], ref["s"], ref["n"])
    for key in ("alphas", "betas", "theta", "p1", "p2"):
        _close(rep[key], ref[key], 1e-12)
    _close(rep["rho"], ref["rho"], 1e-9)  # rho = alpha / beta amplifies by 1 / beta
    _close([rep["d1"], rep["d2"]], [ref["d1"], ref["d2"]], 1e-12)


def test_identical_invocations_and_seed_env(tmp_path, monkeypatch):
    texts = []
    for name in ("a.csv", "b.csv"):
        assert cli.main(["gsv", *PAIR, "--seed", "33", "-o", str(tmp_path / name)]) == 0
        texts.append((tmp_path / name).read_text())
    monkeypatch.setenv("RGSV_SEED", "33")
    assert cli.main(["gsv", *PAIR, "-o", str(tmp_path / "env.csv")]) == 0
    assert texts[0] == texts[1] == (tmp_path / "env.csv").read_text()
    monkeypatch.setenv("RGSV_SEED", "x")
    assert cli.main(["gsv", *PAIR]) == 5


def test_extract_history_matches_reference(tmp_path):
    out = tmp_path / "basis.json"
    assert cli.main(["extract", "--input", G1, "--blocksize", "4", "-o", str(out), "--format",
                     "json"]) == 0
    res, ref = _json(out), _json(os.path.join(GOLD, "extract_bs4.json"))
    for key in ("kind", "columns", "converged", "iterations", "block_widths"):
        assert res[key] == ref[key], key
    assert len(res["residual_history"]) == res["iterations"] + 1
    # the last residuals sit at the rounding floor of ||G||^2 - captured
    _close(res["residual_history"], ref["residual_history"], 1e-7 * ref["residual_history"][0])
    _close(res["residual_history"][:2], ref["residual_history"][:2], 1e-11)


def test_bounds_certificate_matches_reference(tmp_path, capsys):
    out = tmp_path / "cert.json"
    assert cli.main(["bounds", *PAIR, "--k", "4", "--oversample", "3", "--tol", "1e-12", "-o",
                     str(out), "--format", "json"]) == 0
    err = capsys.readouterr().err
    cert, ref = _json(out), _json(os.path.join(GOLD, "bounds_k4.json"))
    assert cert["kind"] == "bound_certificate" and cert["vacuous"] == ref["vacuous"]
    assert abs(cert["eta"] - ref["eta"]) <= 1e-12 * ref["eta"]
    # e_script is the norm of a difference at the rounding level of the pair
    assert 0 <= cert["e_script"] <= 1e-12 and ref["e_script"] <= 1e-12
    assert err.splitlines() == open(os.path.join(GOLD, "bounds_k4.stderr")).read().splitlines()


def test_error_exits(tmp_path, capsys):
    bad = tmp_path / "bad.csv"
    bad.write_text("1,x\n")
    ok = tmp_path / "ok.csv"
    ok.write_text("1,0\n0,1\n")
    assert cli.main(["gsv", "--g1", str(bad), "--g2", str(ok)]) == 3
    assert "category=parse" in capsys.readouterr().err
    assert cli.main(["gsv", "--g1", str(tmp_path / "no.mtx"), "--g2", str(ok)]) == 3
    rank1 = tmp_path / "rank1.csv"
    rank1.write_text("1,2\n2,4\n")
    assert cli.main(["gsv", "--g1", str(rank1), "--g2", str(rank1)]) == 6
    assert "category=rank" in capsys.readouterr().err
    col = tmp_path / "col.csv"
    col.write_text("1\n2\n")
    assert cli.main(["gsv", "--g1", str(ok), "--g2", str(col)]) == 4
    assert "category=dimension" in capsys.readouterr().err
    cplx = tmp_path / "c.csv"
    cplx.write_text("1+2j,0\n0,1\n")
    assert cli.main(["gsv", "--g1", str(cplx), "--g2", str(ok)]) == 5  # no complex device path
    # synth with the reference's default field (complex): validation error
    assert cli.main(["synth", "--m", "20", "--p", "20", "--n", "8", "--out-dir",
                     str(tmp_path / "s")]) == 5
    with pytest.raises(SystemExit) as exc:
        cli.main(["gsv"])
    assert exc.value.code == 2  # argparse usage failure


def test_module_entry_point(tmp_path):
    out = tmp_path / "s.json"
    proc = subprocess.run([sys.executable, "-m", "paper_2404_09459_b200", "gsv", *PAIR, "--method",
                           "direct", "--format", "json", "-o", str(out)], capture_output=True,
                          text=True, cwd=os.path.dirname(os.path.dirname(__file__)))
    assert proc.returncode == 0, proc.stderr
    assert _json(out)["kind"] == "spectrum"
