"""mjlog-lite-v1 logs from device games (paper_2605_20577_b200.mjlog) against
the reference's own logs (tests/golden/logs.json.gz, made by the reference
GameRecorder): byte-identical canonical JSON."""

from __future__ import annotations

import gzip
import json
from pathlib import Path

import pytest

from paper_2605_20577_b200 import mjlog
from paper_2605_20577_b200.env import EnvConfig

GOLD = Path(__file__).resolve().parent / "golden"


def _logs():
    return json.loads(gzip.open(GOLD / "logs.json.gz").read())


def test_config_dict_round_trip_and_ranks():
    cfg = EnvConfig(rule="no-red", mode="half", kazoe=True, renchan_cap=8)
    d = mjlog.config_to_dict(cfg)
    assert d == {"rule": "no-red", "mode": "half", "kazoe": True, "double_yakuman": False,
                 "agari_yame": True, "max_steps": 10000, "renchan_cap": 8}
    assert mjlog.config_from_dict(d) == cfg
    # engine.py:885-891: ties break toward the earlier seat
    assert mjlog.final_ranks([25000, 30000, 25000, 20000]) == [1, 0, 2, 3]


def test_golden_logs_are_canonical():
    for item in _logs():
        log = json.loads(item["log"])
        assert mjlog.log_to_json(log) == item["log"]


@pytest.mark.gpu
@pytest.mark.parametrize("group", [("no-red", "single", 3, 4, 260), ("red", "single", 4, 4, 260),
                                   ("red", "east", 5, 1, 700)])
def test_rollout_logs_equal_reference(group):
    rule, mode, seed, n, steps = group
    want = [g["log"] for g in _logs() if (g["rule"], g["mode"], g["seed"]) == (rule, mode, seed)]
    got = [mjlog.log_to_json(x) for x in mjlog.logs_from_rollout(seed, 0, n, steps, EnvConfig(rule=rule, mode=mode))]
    assert len(got) == len(want)
    for i, (a, b) in enumerate(zip(got, want)):
        assert a == b, f"game {i}"


@pytest.mark.gpu
def test_replay_log_and_partial_replay():
    item = _logs()[0]
    log = json.loads(item["log"])
    final = mjlog.replay_log(log)
    assert final.fingerprint() == log["fingerprint"]
    mid = mjlog.replay_log(log, upto=10)
    assert int(mid.record.step_count) == 10
    bad = dict(log, actions=[[(log["actions"][0][0] + 1) % 4, log["actions"][0][1]]] + log["actions"][1:])
    with pytest.raises(ValueError):
        mjlog.replay_log(bad)
