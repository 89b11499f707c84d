"""CLI (paper_2407_20205_b200/cli.py): file format, records and errors on CPU;
the GPU-routed subcommands under -m gpu."""

import json

import numpy as np
import pytest

from paper_2407_20205_b200 import cli
from conftest import load_golden


def test_matrix_file_round_trip_and_both_conventions(tmp_path):
    a = cli.parse_matrix_text("3\n0 1 2\n2 2 0\n1 0 1\n")
    b = cli.parse_matrix_text("3\n0 1 -1\n-1 -1 0\n1 0 1\n")
    assert a == b
    assert cli.parse_matrix_text(cli.format_matrix_text(a)) == a
    assert cli.format_matrix_text(a, classes=True).splitlines()[1] == "0 1 2"


@pytest.mark.parametrize("text", ["", "x\n1", "0\n", "2\n1 0\n", "2\n1 0\n0\n", "2\n1 a\n0 1\n"])
def test_matrix_file_errors(text):
    with pytest.raises(ValueError):
        cli.parse_matrix_text(text)


def test_pi_matrix_command_matches_reference(capsys):
    assert cli.main(["pi-matrix", "--n", "3", "--mod3-classes"]) == 0
    out = capsys.readouterr().out.split()
    rec = next(r for r in load_golden("pi.json")["pi_matrix"] if r["n"] == 3 and not r["skip_integer_part"])
    assert "".join(out[1:]) == rec["a"]


def test_errors_exit_1(tmp_path, capsys):
    bad = tmp_path / "m.txt"
    bad.write_text("2\n1 0\n")
    assert cli.main(["perm", str(bad)]) == 1
    assert capsys.readouterr().err.startswith("error: ")
    good = tmp_path / "g.txt"
    good.write_text("1\n1\n")
    assert cli.main(["perm", str(good), "--method", "naive"]) == 1
    assert cli.main(["count-exact", "--n", "7"]) == 1


@pytest.mark.gpu
def test_gpu_subcommands(gpu, tmp_path, capsys):
    f = tmp_path / "m.txt"
    f.write_text("2\n1 1\n1 1\n")
    assert cli.main(["perm", str(f), "--mod3-classes"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[0] == "2"
    rec = json.loads(lines[1])
    assert rec["schema"] == cli.PERM_SCHEMA and rec["value"] == 2 and rec["n"] == 2
    assert cli.main(["count-exact", "--n", "3"]) == 0
    assert "z: 8163" in capsys.readouterr().out
    case = load_golden("anchors.json")["montecarlo"][3]
    assert cli.main(["montecarlo", "--n", str(case["n"]), "--trials", str(case["trials"]),
                     "--seed", str(case["seed"])]) == 0
    rows = capsys.readouterr().out.splitlines()
    assert rows[0].split(",") == cli.MC_COLUMNS
    assert rows[1].split(",")[4] == str(case["zero_count"])
    stack = tmp_path / "b.npy"
    np.save(stack, np.ones((4, 5, 5), dtype=np.uint8))
    assert cli.main(["perm-batch", str(stack)]) == 0
    rec = json.loads(capsys.readouterr().out)
    assert rec["classes"] == "0000" and rec["hist"] == [4, 0, 0]  # 5! = 120 = 0 mod 3
