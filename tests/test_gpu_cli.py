"""The command line (`paper_2605_20577_b200.cli`) against the reference's
(cli.py): selfplay logs and render SVGs byte for byte (sha256), and the
bench rows' games_completed equal to bench/runner.py's for the same
(rule, mode, seed, batch, steps) — fixtures from tests/golden/make_golden.py
make_cli.  Needs a B200."""

from __future__ import annotations

import gzip
import hashlib
import json
from pathlib import Path

import pytest

from paper_2605_20577_b200 import cli

pytestmark = pytest.mark.gpu

GOLD = json.loads(gzip.open(Path(__file__).resolve().parent / "golden" / "cli.json.gz").read())


def _sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def test_selfplay_and_render_match_reference():
    logs = []
    for g in GOLD["selfplay"]:
        text, scores = cli.selfplay_log(g["rule"], g["mode"], g["seed"], g["policy"])
        assert (_sha(text), len(text)) == (g["sha256"], g["len"]), g
        assert scores == json.loads(text)["final_scores"]
        logs.append(json.loads(text))
    for r in GOLD["render"]:
        svg = cli.render_log(logs[r["log"]], r["step"], r["viewer"], r["locale"])
        assert (_sha(svg), len(svg)) == (r["sha256"], r["len"]), r


def test_bench_rows_match_reference_games(tmp_path):
    for b in GOLD["bench"]:
        row = cli.rollout(b["rule"], b["mode"], b["batch"], b["steps"], b["seed"], min_duration=0.0)
        assert row.games_completed == b["games_completed"], b
        assert row.batch == b["batch"] and row.wall_seconds > 0
        assert abs(row.steps_per_second - b["batch"] * b["steps"] / row.wall_seconds) < 1e-6 * row.steps_per_second
    # the CLI end to end: the reference's CSV layout
    out = tmp_path / "bench.csv"
    assert cli.main(["bench", "--rule", "no-red", "--sweep", "64,256", "--steps", "50", "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    meta = dict(line[2:].split("=", 1) for line in lines if line.startswith("# "))
    assert {"rule", "mode", "steps", "seed", "threads", "cpu_count", "platform", "python"} <= set(meta)
    assert meta["rule"] == "no-red" and meta["steps"] == "50"
    rows = [line for line in lines if not line.startswith("#")]
    assert rows[0] == "batch,wall_seconds,steps_per_second,games_completed"
    assert [int(r.split(",")[0]) for r in rows[1:]] == [64, 256]
