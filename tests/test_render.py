"""SVG rendering of device / oracle states (paper_2605_20577_b200.render)
against the reference renderer's documents (render/svg.py), byte for byte
(sha256 of reference renders in tests/golden/renders.json.gz)."""

from __future__ import annotations

import gzip
import hashlib
import json
from pathlib import Path

import pytest

from oracle import mjoracle as O
from paper_2605_20577_b200 import records, render

GOLD = Path(__file__).resolve().parent / "golden"


def _renders():
    return json.loads(gzip.open(GOLD / "renders.json.gz").read())


def _states():
    """(entry, record, last result) of every golden render, replayed on the oracle"""
    games = {}
    for g in _renders():
        games.setdefault((g["rule"], g["mode"], g["seed"], g["index"], g["policy"]), []).append(g)
    for (rule, mode, seed, idx, policy), entries in games.items():
        env = O.OracleEnv(O.make_config(rule=rule, mode=mode)).init(O.env_game_seed(seed, idx))
        kc = [O.env_policy_key(seed, idx), 0]
        t = 0
        for g in sorted(entries, key=lambda x: x["step"]):
            while t < g["step"]:
                a = env.random_policy(kc) if policy == "random" else env.heuristic_policy()
                env.step(a)
                t += 1
            rec = env.record()
            last = records.result_dict(rec.last_result) if rec.n_results else None
            yield g, rec, last


def test_render_matches_reference_documents():
    n = 0
    for g, rec, last in _states():
        svg = render.to_svg(rec, viewer=g["viewer"], locale=g["locale"], last_result=last)
        where = f"{g['rule']} {g['policy']} step {g['step']} viewer {g['viewer']} {g['locale']}"
        assert len(svg) == g["len"], where
        assert hashlib.sha256(svg.encode()).hexdigest() == g["sha256"], where
        n += 1
    assert n == len(_renders())


def test_render_rejects_unknown_locale():
    g, rec, last = next(_states())
    with pytest.raises(ValueError):
        render.to_svg(rec, locale="fr")


def test_action_table_rows():
    """actions.py:48-96 names and kinds"""
    from paper_2605_20577_b200 import sessions as S

    t = S.action_table()
    assert len(t) == 115 and [r["id"] for r in t] == list(range(115))
    assert t[0] == {"id": 0, "kind": "discard", "tile": "1m", "red": False, "name": "discard 1m"}
    assert t[35] == {"id": 35, "kind": "discard", "tile": "5p", "red": True, "name": "discard red 5p"}
    assert t[42] == {"id": 42, "kind": "chi", "name": "chi mid"}
    assert t[45 + 33] == {"id": 78, "kind": "kan_closed", "tile": "C", "name": "closed kan C"}
    assert t[79 + 27] == {"id": 106, "kind": "kan_added", "tile": "E", "name": "added kan E"}
    assert t[113]["kind"] == "pass" and t[114] == {"id": 114, "kind": "abort", "name": "nine terminals"}
