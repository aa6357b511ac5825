"""Game sessions over device states (`paper_2605_20577_b200.sessions`)
against the reference's session layer (service/sessions.py) and its view
documents (service/app.py `_view`): the golden fixtures
(tests/golden/make_golden.py make_sessions) hold, per game, the action list
a scripted human plus the agents produce, the final fingerprint, the
persisted store document and sha256 digests of the views.  Needs a B200."""

from __future__ import annotations

import gzip
import hashlib
import json
from pathlib import Path

import pytest

from paper_2605_20577_b200 import sessions as S
from paper_2605_20577_b200.env import EnvConfig

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"


def _cases():
    return json.loads(gzip.open(GOLD / "sessions.json.gz").read())


def _human_action(legal, n_actions):  # make_golden.session_human_action
    return legal[(7 * n_actions + 3) % len(legal)]


def _digest(view) -> str:
    v = dict(view)
    v.pop("game_id")
    return hashlib.sha256(json.dumps(v, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


@pytest.mark.parametrize("case", range(4))
def test_sessions_match_reference(case):
    g = _cases()[case]
    cfg = EnvConfig(rule=g["rule"], mode=g["mode"])
    agents = {int(k): v for k, v in g["agents"].items()}
    store = S.SessionStore(None)
    sess = store.create(cfg, g["seed"], g["human_seats"], agents)
    seat = g["human_seats"][0] if g["human_seats"] else 0
    want = {(n, loc): d for n, loc, d in g["views"]}
    got = {}

    def view(locale):
        got[(len(sess.actions), locale)] = _digest(S.session_view(sess, seat, locale))

    view("en")
    while sess.waiting_on() is not None:
        S.apply_session_action(sess, _human_action(sess.state.legal, len(sess.actions)))
        S.advance_agents(sess)
        if (len(sess.actions), "en") in want:
            view("en")
    view("ja")
    view("en")
    assert [list(a) for a in sess.actions] == g["actions"]
    assert sess.state.fingerprint() == g["fingerprint"]
    assert list(sess.state.rewards) == g["rewards"]
    for key, d in want.items():
        assert got.get(key) == d, key


def test_store_loads_reference_documents(tmp_path):
    """a store directory written by the reference loads here by action replay,
    and this store's documents carry the reference's fields and values"""
    cases = _cases()
    for i, g in enumerate(cases):
        (tmp_path / f"{i:016x}.json").write_text(json.dumps(dict(g["doc"], id=f"{i:016x}")))
    store = S.SessionStore(tmp_path)
    by_seed = {s.seed: s for s in store.sessions.values()}
    assert len(by_seed) == len(cases)
    for g in cases:
        sess = by_seed[g["seed"]]
        assert sess.state.fingerprint() == g["fingerprint"]
        assert sess.waiting_on() is None
        out = tmp_path / "out"
        S.SessionStore(out).persist(sess)
        doc = json.loads((out / f"{sess.id}.json").read_text())
        for k in ("seed", "config", "human_seats", "agents", "actions"):
            assert doc[k] == g["doc"][k], k


def test_session_persist_and_reload(tmp_path):
    """mid-game persistence: the reloaded session is at the same state and,
    with heuristic agents, continues identically (random agents restart
    their streams on reload, as in the reference: _load_file replays the
    actions without advancing agent_rng)"""
    store = S.SessionStore(tmp_path)
    sess = store.create(EnvConfig(rule="red"), 99, [0, 2], {1: "heuristic", 3: "heuristic"})
    for _ in range(10):
        if sess.waiting_on() is None:
            break
        S.apply_session_action(sess, _human_action(sess.state.legal, len(sess.actions)))
        S.advance_agents(sess)
        store.persist(sess)
    again = S.SessionStore(tmp_path).get(sess.id)
    assert again is not None and again.state.fingerprint() == sess.state.fingerprint()
    for s in (sess, again):
        while s.waiting_on() is not None:
            S.apply_session_action(s, _human_action(s.state.legal, len(s.actions)))
            S.advance_agents(s)
    assert again.actions == sess.actions and again.state.fingerprint() == sess.state.fingerprint()
    log = again.recorder.to_log(again.state)
    assert log["fingerprint"] == again.state.fingerprint()
