"""CLI parity with the reference `fntdsp` CLI (cli.py): byte-identical stdout for
selftest (incl. the --fault-inject negative control) and complexity --measure,
identical output files for transform / convolve, identical exit codes."""

import contextlib
import io
import json

import pytest

from conftest import GOLDEN

REF = json.loads((GOLDEN / "cli.json").read_text())


def _run(argv):
    from paper_2405_04253_b200 import cli
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(argv)
    return rc, buf.getvalue()


def test_cli_host_commands(tmp_path):
    rc, _ = _run(["write-config", "--output", str(tmp_path / "link.ini")])
    assert rc == 0 and "[link]" in (tmp_path / "link.ini").read_text()
    rc, text = _run(["complexity"])
    assert (rc, text) == (REF["complexity"]["rc"], REF["complexity"]["stdout"])


@pytest.mark.gpu
def test_cli_selftest_and_fault_injection():
    for key, argv in (("selftest", ["selftest"]), ("selftest_fault", ["selftest", "--fault-inject"])):
        rc, text = _run(argv)
        assert rc == REF[key]["rc"]
        assert text == REF[key]["stdout"]


@pytest.mark.gpu
def test_cli_complexity_measure_counts():
    rc, text = _run(["complexity", "--measure"])
    assert rc == 0 and text == REF["complexity_measure"]["stdout"]


@pytest.mark.gpu
def test_cli_transform_convolve(tmp_path):
    for k, v in REF["files"].items():
        (tmp_path / f"{k}.txt").write_text(v)
    d = tmp_path
    cases = {
        "fnt": ["transform", "--plan", "cdc64", "--input", str(d / "x.txt"), "--output", str(d / "o.txt")],
        "ifnt": ["transform", "--plan", "aeq32", "--inverse", "--input", str(d / "x32.txt"), "--output", str(d / "o.txt")],
        "conv": ["convolve", "--plan", "cdc64", "--x", str(d / "x.txt"), "--h", str(d / "h.txt"), "--output", str(d / "o.txt")],
        "convc": ["convolve", "--plan", "cdc64", "--mode", "complex", "--x", str(d / "xc.txt"), "--h", str(d / "hc.txt"), "--output", str(d / "o.txt")],
        "overflow": ["convolve", "--plan", "cdc64", "--x", str(d / "big.txt"), "--h", str(d / "h.txt"), "--output", str(d / "o2.txt")],
    }
    for key, argv in cases.items():
        rc, _ = _run(argv)
        assert rc == REF["runs"][key]["rc"], key
        if rc == 0:
            assert (d / "o.txt").read_text() == REF["runs"][key]["out"], key


@pytest.mark.gpu
def test_cli_sweep_matches_reference(tmp_path, monkeypatch):
    """`sweep` on a small link config (tests/golden/make_sweep_golden.py): the host
    link simulator + GPU receiver + GPU metrology give the reference CLI's
    sweep.csv, summary and stdout byte for byte (same relative paths, so the
    manifest digest matches)."""
    g = json.loads((GOLDEN / "sweep.json").read_text())
    (tmp_path / "link.ini").write_text(g["ini"])
    monkeypatch.chdir(tmp_path)
    rc, text = _run(g["argv"])
    assert rc == g["rc"] and text == g["stdout"]
    assert (tmp_path / "sweep_out" / "sweep.csv").read_text() == g["csv"]
    assert (tmp_path / "sweep_out" / "summary.txt").read_text() == g["summary"]
