"""The reference's own crafted engine scenarios (every apply_action made by
its tests/test_engine.py and tests/test_engine_rounds.py: calls priority,
chankan, multi-ron, triple-ron abort, four-riichi / nine-terminals aborts,
riichi kans, furiten, renchan cap, agari-yame, bankruptcy, ...), harvested
by tests/golden/make_golden.py as (pre-state, action, post-state
projection | exception).  Replayed on the CPU oracle here and on the GPU
(marked gpu).

wins.json.gz: the same format for tsumo / ron transitions of states
crafted around the scoring fixtures' hands (make_golden.make_wins): the
engine's win path end to end — _win_context (engine.py:345-375), score_win,
settle, the result record's win details, kazoe / double-yakuman configs,
haitei / houtei / rinshan / chankan / first-draw flags, honba and deposits,
and the next deal in half mode; NoYaku / furiten wins are rejected as
IllegalActionError."""

from __future__ import annotations

import gzip
import json
from pathlib import Path

import pytest

from oracle import mjoracle as O
from paper_2605_20577_b200 import abi
from paritylib import diff, normalize, projection, record_from_dict

GOLD = Path(__file__).resolve().parent / "golden"


def _scenarios(name="scenarios.json.gz"):
    return json.loads(gzip.open(GOLD / name).read())


def _check(kind, status, rec, sc):
    where = f"{sc['test']} action {sc['action']}"
    if sc["error"] == "IllegalActionError":
        assert status & abi.STATUS_ILLEGAL, where
        return
    if sc["error"] == "ContractError":
        assert status & abi.STATUS_CONTRACT, where
        return
    got = normalize(projection(rec))
    want = normalize(sc["post"])
    d = diff(got, want)
    assert not d, f"{kind}: {where}: {d[:5]}"


@pytest.mark.parametrize("name", ["scenarios.json.gz", "wins.json.gz"])
def test_scenarios_on_oracle(name):
    scs = _scenarios(name)
    assert len({s["test"] for s in scs}) >= (30 if name == "scenarios.json.gz" else 3)
    for sc in scs:
        pre = record_from_dict(sc["pre"])
        env = O.OracleEnv(pre.cfg)
        env.load(pre)
        status = env.step(sc["action"])
        _check("oracle", status, env.record(), sc)


def test_wins_cover_the_rare_branches():
    """the crafted wins reach the branches random play almost never does"""
    scs = _scenarios("wins.json.gz")
    wins = [sc for sc in scs if sc["post"] and sc["post"]["last_result"]]
    assert len(wins) >= 300
    assert sum(1 for sc in scs if sc["error"] == "IllegalActionError") >= 50
    details = [w for sc in wins for w in sc["post"]["last_result"]["win_details"]]
    kinds = {sc["post"]["last_result"]["kind"] for sc in wins}
    assert kinds == {"tsumo", "ron"}
    assert sum(1 for sc in wins if sc["pre"]["cfg"]["kazoe"] and sc["pre"]["cfg"]["double_yakuman"]) >= 20
    assert sum(1 for d in details if d["yakuman"]) >= 40
    assert any(y[1] == 2 for d in details if d["yakuman"] for y in d["yaku"])  # a double yakuman


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["scenarios.json.gz", "wins.json.gz"])
def test_scenarios_on_gpu(name):
    import torch

    from paper_2605_20577_b200.env import BatchEnv, EnvConfig

    scs = _scenarios(name)
    envs = {}
    for sc in scs:
        pre = record_from_dict(sc["pre"])
        key = (pre.cfg.rule, pre.cfg.mode, pre.cfg.max_steps, pre.cfg.agari_yame, pre.cfg.renchan_cap,
               pre.cfg.kazoe, pre.cfg.double_yakuman)
        if key not in envs:
            envs[key] = BatchEnv(1, EnvConfig(rule="red" if pre.cfg.rule == 0 else "no-red",
                                              mode=("single", "east", "half")[pre.cfg.mode],
                                              max_steps=pre.cfg.max_steps, agari_yame=bool(pre.cfg.agari_yame),
                                              renchan_cap=pre.cfg.renchan_cap, kazoe=bool(pre.cfg.kazoe),
                                              double_yakuman=bool(pre.cfg.double_yakuman)))
        env = envs[key]
        env.load(0, pre)
        env.step(torch.tensor([sc["action"]], dtype=torch.int32))
        torch.cuda.synchronize()
        _check("gpu", int(env.status[0]), env.export(0), sc)
