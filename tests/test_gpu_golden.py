"""The CUDA path against the REFERENCE's own outputs (golden fixtures made
by tests/golden/make_golden.py from the Python reference), through the
per-env Pgx facade `paper_2605_20577_b200.pgx` (same names as mjsim):
sha256 fingerprints of the full serialize_state at every step, observation
digests, legal ids, current player and rewards.  Needs a B200."""

from __future__ import annotations

import gzip
import hashlib
import json
from pathlib import Path

import pytest

from paper_2605_20577_b200 import pgx
from paper_2605_20577_b200.env import EnvConfig

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"


def _games():
    return json.loads(gzip.open(GOLD / "traces.json.gz").read())


def _obs_digest(o) -> str:
    return hashlib.sha256(json.dumps(o.to_dict(), sort_keys=True).encode()).hexdigest()[:16]


@pytest.mark.parametrize("chunk", range(4))
def test_reference_traces_through_pgx_facade(chunk):
    games = _games()[chunk::4]
    for g in games:
        cfg = EnvConfig(rule=g["rule"], mode=g["mode"])
        st = pgx.init(pgx.env_game_seed(g["seed"], g["index"]), cfg)
        pol = pgx.env_policy_state(g["seed"], g["index"])
        for t, row in enumerate(g["steps"]):
            fp, od, cp, legal, rewards, term, trunc = row[:7]
            where = f"{g['rule']} {g['mode']} {g['policy']} idx {g['index']} step {t}"
            assert st.fingerprint()[:16] == fp, where
            assert st.current_player == cp, where
            assert list(st.legal) == legal, where
            assert list(st.rewards) == list(rewards), where  # the reference's doubles exactly (pgx._reward)
            assert (st.terminated, st.truncated) == (bool(term), bool(trunc)), where
            assert _obs_digest(pgx.observe(st, cp)) == od, where
            if len(row) > 7:
                if g["policy"] == "random":
                    a, pol = pgx.random_policy(st.legal, pol)
                    assert a == row[7], where
                else:
                    a = row[7]  # the reference heuristic's choice
                    assert pgx.heuristic_policy(st) == a, where
                st = pgx.step(st, a)


def test_contract_and_illegal_semantics():
    """env/core.py:85-94: illegal id -> terminated with the penalty at the
    offender and no legal actions; stepping it again raises ContractError."""
    cfg = EnvConfig(rule="red", illegal_penalty=-0.5)
    st = pgx.init(1234, cfg)
    bad = next(a for a in range(115) if a not in st.legal)
    nxt = pgx.step(st, bad)
    assert nxt.terminated and not nxt.truncated and nxt.legal == ()
    want = [0.0] * 4
    want[st.current_player] = -0.5
    assert list(nxt.rewards) == want
    # the game itself is untouched (core.py:89-94)
    assert nxt.record.step_count == st.record.step_count
    with pytest.raises(pgx.ContractError):
        pgx.step(nxt, st.legal[0])
    for oob in (-1, 115, 10 ** 12):
        assert pgx.step(st, oob).terminated
    # the earlier state value is still usable (immutable semantics)
    ok = pgx.step(st, st.legal[0])
    assert not ok.terminated


def test_device_states_render_like_the_reference():
    """render.to_svg of pgx (device) states == the reference renderer's
    documents for the same games and steps (tests/golden/renders.json.gz)"""
    from paper_2605_20577_b200 import render

    renders = json.loads(gzip.open(GOLD / "renders.json.gz").read())
    games = {}
    for g in renders:
        games.setdefault((g["rule"], g["mode"], g["seed"], g["index"], g["policy"]), []).append(g)
    for (rule, mode, seed, idx, policy), entries in games.items():
        cfg = EnvConfig(rule=rule, mode=mode)
        st = pgx.init(pgx.env_game_seed(seed, idx), cfg)
        pol = pgx.env_policy_state(seed, idx)
        t = 0
        for g in sorted(entries, key=lambda x: x["step"]):
            while t < g["step"]:
                if policy == "random":
                    a, pol = pgx.random_policy(st.legal, pol)
                else:
                    a = pgx.heuristic_policy(st)
                st = pgx.step(st, a)
                t += 1
            svg = render.to_svg(st, viewer=g["viewer"], locale=g["locale"])
            assert hashlib.sha256(svg.encode()).hexdigest() == g["sha256"], (rule, policy, g["step"], g["viewer"])
