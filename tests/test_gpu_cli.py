"""`helix` command line on the B200 backend (SPEC.md:611-627 examples):
matvec row / diag / bsgs correctness and counters, matmul counters and the
modelled cost trend over the input level, JSON and CSV outputs."""
import csv
import io
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "build", "helix")


def run(*args, rc=0):
    p = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=300)
    assert p.returncode == rc, (args, p.returncode, p.stderr)
    return p.stdout


def row(*args):
    return json.loads(run(*args, "--json", "--repeats", "1"))["rows"][0]


def test_matvec_bsgs_16x16():
    """bsgs 16 x 16 -> correct, rotations = (n1 - 1) + (n2 - 1) = 6, 1 level"""
    r = row("matvec", "--method", "bsgs", "--rows", "16", "--cols", "16")
    assert r["correct"] and r["rotations"] == 6 and r["levels_consumed"] == 1


def test_matvec_row_4x4_two_levels():
    """the packed-row method consumes two levels"""
    r = row("matvec", "--method", "row", "--rows", "4", "--cols", "4")
    assert r["correct"] and r["levels_consumed"] == 2


def test_matvec_diag_and_csv(tmp_path):
    out = tmp_path / "m.csv"
    run("matvec", "--method", "diag", "--rows", "8", "--cols", "8", "--repeats", "1", "--csv", str(out))
    t = list(csv.DictReader(io.StringIO(out.read_text())))
    assert t[0]["correct"] == "true" and t[0]["rotations"] == "7" and t[0]["method"] == "diag"


def test_matmul_counts_and_level_trend():
    """d = 2 -> 6 rotations; d = 4 at levels 2 and 5: same
    rotation count, larger modelled bytes at level 5"""
    r2 = row("matmul", "--d", "2")
    assert r2["correct"] and r2["rotations"] == 6 and r2["levels_consumed"] == 2
    a, b = row("matmul", "--d", "4", "--level", "2"), row("matmul", "--d", "4", "--level", "5")
    assert a["correct"] and b["correct"]
    assert a["rotations"] == b["rotations"] == 22
    assert b["modeled_bytes"] > a["modeled_bytes"] > 0
