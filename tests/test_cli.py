"""CLI host logic without a GPU: sweep parsing (cli.py:11-21) and the
bench CSV layout (bench/runner.py:218-223)."""

from __future__ import annotations

from paper_2605_20577_b200 import cli


def test_parse_sweep():
    assert cli.parse_sweep("2..16") == [2, 4, 8, 16]
    assert cli.parse_sweep("1024..5000") == [1024, 2048, 4096]
    assert cli.parse_sweep("3,7,9") == [3, 7, 9]


def test_report_to_csv_layout():
    rep = cli.BenchReport((cli.BenchRow(4096, 0.0025, 163840000.0, 17), cli.BenchRow(8, 1.5, 533.3333, 0)),
                          {"seed": 0, "rule": "red"})
    assert cli.report_to_csv(rep) == ("# rule=red\n# seed=0\nbatch,wall_seconds,steps_per_second,games_completed\n"
                                      "4096,0.002500,163840000.00,17\n8,1.500000,533.33,0\n")
