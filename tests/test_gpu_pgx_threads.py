"""The per-env facade (paper_2605_20577_b200.pgx) shares one batch-of-1
device handle per config; callers on several threads (the reference's
service runs its sync handlers in a threadpool, service/sessions.py)
must each see their own game.  Four threads step four different games
concurrently, interleaving step / observe / heuristic_policy; every
trajectory must equal the same game played alone."""

from __future__ import annotations

import threading

import pytest

from paper_2605_20577_b200 import pgx
from paper_2605_20577_b200.env import EnvConfig

pytestmark = pytest.mark.gpu


def _play(seed: int, steps: int):
    cfg = EnvConfig(rule="red")
    st = pgx.init(seed, cfg)
    rng = pgx.env_policy_state(seed, 0)
    trace = []
    for _ in range(steps):
        if st.terminated or st.truncated:
            break
        obs = pgx.observe(st, st.current_player)
        h = pgx.heuristic_policy(st)
        a, rng = pgx.random_policy(st.legal, rng)
        st = pgx.step(st, a)
        trace.append((a, h, obs.hand_tokens, st.fingerprint()))
    return trace


def test_threads_stepping_different_games_do_not_interfere():
    seeds, steps = (11, 12, 13, 14), 60
    alone = {s: _play(s, steps) for s in seeds}
    got, errors = {}, []

    def run(s):
        try:
            got[s] = _play(s, steps)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    for _ in range(2):
        ts = [threading.Thread(target=run, args=(s,)) for s in seeds]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errors, errors
        assert got == alone
