"""CPU: the command-line front end's configuration / usage-error paths (no kernel runs)."""

import json

from paper_2307_04688_b200.cli import main


def test_custom_without_config_is_usage_error(tmp_path, capsys):
    assert main(["solve", "--out", str(tmp_path / "x")]) == 2
    assert "config" in capsys.readouterr().err


def test_bad_blocks_is_usage_error(tmp_path, capsys):
    rc = main(["solve", "--preset", "example1", "--np", "2", "--blocks", "4", "--out", str(tmp_path / "x")])
    assert rc == 2 and "block" in capsys.readouterr().err


def test_simulate_without_policy_is_error(tmp_path, capsys):
    assert main(["simulate", "--out", str(tmp_path / "nothing")]) == 2
    assert "solve" in capsys.readouterr().err


def test_compare_refuses_three_players(tmp_path, capsys):
    assert main(["compare", "--preset", "example3", "--out", str(tmp_path / "x")]) == 2
    assert "no oracle" in capsys.readouterr().err


def test_bad_config_file_and_p0(tmp_path, capsys):
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert main(["solve", "--config", str(bad), "--out", str(tmp_path / "x")]) == 2
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps({"preset": "example1", "p0": [0.1]}))
    assert main(["solve", "--config", str(cfg), "--out", str(tmp_path / "y")]) == 2
    assert "p0" in capsys.readouterr().err
