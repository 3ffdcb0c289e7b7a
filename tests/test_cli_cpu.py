"""CPU: the hodlr-bench harness -- config grammar, diagnostics,
exit codes and the result formats (no GPU needed for these layers)."""

from __future__ import annotations

import pytest

from paper_2208_06290_b200 import cli

REC = {"problem": "laplace", "N": 4096, "L": 6, "leaf_size": 64, "tol": 0.0, "precision": "double",
       "variant": "pivoted_standard", "t_f_seconds": 0.001, "t_s_seconds": 0.0002, "mem_bytes": 123456,
       "relres": 1.5e-15, "flops_factor": 987654321, "flops_solve": 12345, "ranks": "32/32/32/32/32/32"}


def test_config_grammar_and_overrides():
    cells = cli.parse_config("# two cells\n[cell]\nproblem = standin\nn=1024\nleaf_size=32\n[cell]\nprecision=single\n")
    assert len(cells) == 2 and cells[0].kv["problem"] == "standin"
    c = cli.validate(cells[0])
    assert (c["n"], c["m"], c["L"], c["runs"]) == (1024, 32, 5, 5)
    assert cli.validate(cells[1])["precision"] == "single"
    assert len(cli.parse_config("")) == 1  # defaults-only cell


@pytest.mark.parametrize("text,msg", [
    ("problem\n", "line 1: expected key=value"),
    ("colour=red\n", "line 1: unknown key 'colour'"),
    ("n=abc\n", "key 'n': not a int"),
    ("problem=rpy\n", "key 'problem'"),
    ("tol=1e-8\n", "fixed-rank"),
    ("n=1000\n", "n = leaf_size \\* 2\\^L"),
])
def test_config_errors_carry_line_and_key(text, msg):
    with pytest.raises(cli.ConfigError, match=msg):
        [cli.validate(c) for c in cli.parse_config(text)]


def test_results_formats_round_trip():
    assert cli.emit([], "csv") == ",".join(cli.COLUMNS) + "\n"  # header-only CSV
    out = cli.emit([REC], "csv")
    lines = out.splitlines()
    assert len(lines) == 2 and len(lines[1].split(",")) == 14
    assert cli.parse_results(out, "csv") == [REC]
    assert cli.parse_results(cli.emit([REC, REC], "jsonl"), "jsonl") == [REC, REC]


def test_main_exit_code_on_config_error(tmp_path, capsys):
    p = tmp_path / "bad.txt"
    p.write_text("leaf_size=0\n")
    assert cli.main(["--config", str(p)]) == 2
    assert "config error" in capsys.readouterr().err
    assert cli.main(["--set", "nonsense"]) == 2
