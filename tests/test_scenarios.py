"""The reference's own crafted engine scenarios (every apply_action made by
its tests/test_engine.py and tests/test_engine_rounds.py: calls priority,
chankan, multi-ron, triple-ron abort, four-riichi / nine-terminals aborts,
riichi kans, furiten, renchan cap, agari-yame, bankruptcy, ...), harvested
by tests/golden/make_golden.py as (pre-state, action, post-state
projection | exception).  Replayed on the CPU oracle here and on the GPU
(marked gpu)."""

from __future__ import annotations

import gzip
import json
from pathlib import Path

import pytest

from oracle import mjoracle as O
from paper_2605_20577_b200 import abi
from paritylib import diff, normalize, projection, record_from_dict

GOLD = Path(__file__).resolve().parent / "golden"


def _scenarios():
    return json.loads(gzip.open(GOLD / "scenarios.json.gz").read())


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


def test_scenarios_on_oracle():
    scs = _scenarios()
    assert len({s["test"] for s in scs}) >= 30
    for sc in scs:
        pre = record_from_dict(sc["pre"])
        env = O.OracleEnv(pre.cfg)
        env.load(pre)
        status = env.step(sc["action"])
        _check("oracle", status, env.record(), sc)


@pytest.mark.gpu
def test_scenarios_on_gpu():
    import torch

    from paper_2605_20577_b200.env import BatchEnv, EnvConfig

    scs = _scenarios()
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
