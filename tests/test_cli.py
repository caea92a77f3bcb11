"""The `ph0b` CLI (paper_2203_02527_b200/cli/ph0b_cli.cpp) against the text the reference's
own `ph0` CLI prints (tests/golden/ref_cli_text.json, generated from the reference sources by
tests/golden/make_text_golden.py): byte-identical stdout, the same "error: ..." stderr and
exit codes.  Cases that run the pipeline need the GPU; parsing, generation and argument
errors run on the CPU."""
import json
import subprocess

import pytest

import oracle_bridge as ob

CLI = ob.ROOT / "paper_2203_02527_b200" / "ph0b"
CASES = json.loads((ob.ROOT / "tests" / "golden" / "ref_cli_text.json").read_text())["cases"]


def params():
    for c in CASES:
        yield pytest.param(c, id=c["name"], marks=[pytest.mark.gpu] if c["gpu"] else [])


@pytest.mark.parametrize("case", list(params()))
def test_cli_matches_reference_text(case, tmp_path):
    if not CLI.exists():
        pytest.fail(f"{CLI} missing: run __graft_entry__.build()")
    argv = list(case["argv"])
    if case["input"] is not None:
        f = tmp_path / "points.txt"
        f.write_text(case["input"])
        argv = [a.replace("{in}", str(f)) for a in argv]
    res = subprocess.run([str(CLI), *argv], capture_output=True, text=True, timeout=600)
    assert res.returncode == case["rc"], res.stderr
    assert res.stdout == case["stdout"]
    if case["rc"] != 0:
        assert res.stderr == case["stderr"]


def test_cli_out_file_and_unknown_option(tmp_path):
    out = tmp_path / "pts.txt"
    res = subprocess.run([str(CLI), "generate", "--n", "37", "--dim", "3", "--seed", "2024",
                          "--out", str(out)], capture_output=True, text=True)
    assert res.returncode == 0 and res.stdout == ""
    ref = next(c for c in CASES if c["name"] == "generate_37_3_2024")
    assert out.read_text() == ref["stdout"]
    bad = subprocess.run([str(CLI), "compute", "--bogus"], capture_output=True, text=True)
    assert bad.returncode != 0 and "--bogus" in bad.stderr
    assert subprocess.run([str(CLI)], capture_output=True).returncode != 0
