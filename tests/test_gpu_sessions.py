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


def _drive_batch(batch):
    """every waiting human decides (the scripted human of the golden games),
    all in one launch per tick"""
    while True:
        waiting = batch.waiting()
        if not waiting:
            return
        batch.apply_actions({i: _human_action(batch.sessions[i].state.legal, len(batch.sessions[i].actions))
                             for i in waiting})


@pytest.mark.parametrize("key", [("red", "single"), ("no-red", "single"), ("no-red", "east")])
def test_session_batch_matches_reference_and_single_sessions(key):
    """SessionBatch: the reference's golden games of this config, multiplexed
    with other sessions (different seeds, human seats and agent mixes) on one
    device batch, reproduce the reference's action lists, fingerprints and
    rewards; every other session equals the same game played alone through
    new_session / apply_session_action / advance_agents"""
    rule, mode = key
    cfg = EnvConfig(rule=rule, mode=mode)
    gold = [g for g in _cases() if (g["rule"], g["mode"]) == key]
    extra = [(1000 + k, hs, ag) for k, (hs, ag) in enumerate([
        ([0], {1: "random", 2: "heuristic", 3: "random"}),
        ([], {0: "heuristic", 1: "heuristic", 2: "random", 3: "heuristic"}),
        ([1, 2], {0: "heuristic", 3: "random"}),
        ([0, 1, 2, 3], {}),
        ([3], {0: "random", 1: "random", 2: "random"}),
    ])]
    if mode == "east":
        extra = extra[:2]
    spec = [(g["seed"], g["human_seats"], {int(k): v for k, v in g["agents"].items()}) for g in gold] + extra
    batch = S.SessionBatch(cfg, [s for s, _, _ in spec], [h for _, h, _ in spec], [a for _, _, a in spec])
    assert len(batch) == len(spec)
    _drive_batch(batch)
    for g, sess in zip(gold, batch.sessions):
        assert [list(a) for a in sess.actions] == g["actions"]
        assert sess.state.fingerprint() == g["fingerprint"]
        assert list(sess.state.rewards) == g["rewards"]
    for (seed, hs, ag), sess in list(zip(spec, batch.sessions))[len(gold):]:
        alone = S.new_session(cfg, seed, hs, ag)
        while alone.waiting_on() is not None:
            S.apply_session_action(alone, _human_action(alone.state.legal, len(alone.actions)))
            S.advance_agents(alone)
        assert sess.waiting_on() is None
        assert sess.actions == alone.actions
        assert sess.state.fingerprint() == alone.state.fingerprint()
        assert sess.state.rewards == alone.state.rewards and sess.state.results == alone.state.results
        assert sess.recorder.to_log(sess.state) == alone.recorder.to_log(alone.state)
        assert S.session_view(sess, 0)["final"] == S.session_view(alone, 0)["final"]


def test_session_batch_contract():
    """human decisions only for sessions waiting on a human; finished
    sessions refuse actions; the reserved SKIP id is an illegal action on
    the single-env facade, not a no-op"""
    from paper_2605_20577_b200 import abi, pgx
    cfg = EnvConfig()
    batch = S.SessionBatch(cfg, [5, 6], [[0, 1, 2, 3], []], [{}, {0: "heuristic", 1: "random",
                                                                  2: "heuristic", 3: "random"}])
    assert batch.sessions[1].waiting_on() is None and batch.waiting() == {0: batch.sessions[0].waiting_on()}
    with pytest.raises(pgx.ContractError):
        batch.apply_actions({1: 0})
    with pytest.raises(IndexError):
        batch.apply_actions({2: 0})
    st = pgx.init(5, cfg)
    bad = pgx.step(st, abi.ACTION_SKIP)
    assert bad.terminated and bad.record.status & abi.STATUS_ILLEGAL


def test_export_many_matches_export():
    """rs_export_envs: the records of a list of envs (any order, repeats)
    equal one rs_export_env per env"""
    import ctypes as C
    import torch
    from paper_2605_20577_b200.env import BatchEnv
    env = BatchEnv(37, EnvConfig(rule="red"))
    env.init(seed=3)
    for _ in range(25):
        env.step(env.random_actions(), autoreset=True)
    order = [36, 0, 5, 5, 17, 2]
    many = env.export_many(order)
    for i, rec in zip(order, many):
        assert bytes(rec) == bytes(env.export(i))
    assert env.export_many([]) == []
    with pytest.raises(Exception):
        env.export_many([37])
