"""The device engine source, compiled for the host (tests/hostcheck, test
only), against the CPU oracle.  Catches transition-logic bugs without a
GPU; the CUDA build itself is checked by tests/test_gpu_parity.py."""

from __future__ import annotations

import random
import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent / "hostcheck"))

import hc  # noqa: E402
from oracle import mjoracle as O  # noqa: E402
from paritylib import diff, projection  # noqa: E402


@pytest.mark.parametrize("rule", ("no-red", "red"))
@pytest.mark.parametrize("mode", ("single", "east", "half"))
def test_rollout_digests(rule, mode):
    cfg = O.make_config(rule=rule, mode=mode)
    n, steps = (128, 600) if mode == "single" else (48, 1200)
    games, ref = O.run_shard(cfg, 21, 0, n, steps, digests=True)
    hb = hc.HostBatch(n, cfg)
    hb.init_indexed(21, 0)
    g2, got, _ = hb.rollout(steps)
    assert got == ref
    assert g2 == games


@pytest.mark.parametrize("rule", ("no-red", "red"))
@pytest.mark.parametrize("mode", ("single", "half"))
def test_heuristic_rollout_digests(rule, mode):
    """the engine's heuristic_policy (env/policies.py:51-109, from the state)
    drives the same trajectories as the oracle's (from the observation)"""
    cfg = O.make_config(rule=rule, mode=mode)
    n, steps = (96, 500) if mode == "single" else (24, 1500)
    games, ref = O.run_shard(cfg, 7, 0, n, steps, policy="heuristic", digests=True)
    hb = hc.HostBatch(n, cfg)
    hb.init_indexed(7, 0)
    g2, got, _ = hb.rollout(steps, policy="heuristic")
    assert got == ref
    assert g2 == games


@pytest.mark.parametrize("rule", ("no-red", "red"))
@pytest.mark.parametrize("policy", ("random", "heuristic"))
def test_invariants_hold_during_play(rule, policy):
    """check_invariants (state.py:105-180, full) after every step of
    random and heuristic play: no violation"""
    cfg = O.make_config(rule=rule, mode="half")
    n = 16
    hb = hc.HostBatch(n, cfg)
    hb.init_indexed(31, 0)
    for t in range(400):
        hb.rollout(1, policy=policy)
        for e in range(n):
            assert hb.check(e) == 0, (t, e, hb.check(e))


def test_invariant_violations_are_detected():
    """crafted broken states trip the matching bits"""
    from paper_2605_20577_b200 import abi

    cfg = O.make_config(rule="red", mode="single")
    oe = O.OracleEnv(cfg).init(77)
    for _ in range(30):
        oe.step(oe.legal()[0])
    base = oe.record()
    hb = hc.HostBatch(1, cfg)

    def copy():
        return type(base).from_buffer_copy(base)

    hb.load(0, base)
    assert hb.check(0) == 0
    bad = copy()
    bad.scores[0] += 100
    hb.load(0, bad)
    assert hb.check(0) & abi.INV_SCORE_SUM
    bad = copy()
    h = bad.hands[0]
    h.concealed[0] = h.concealed[1]  # a duplicated tile, one missing
    hb.load(0, bad)
    assert hb.check(0, fast=True) & abi.INV_TILES
    bad = copy()
    s = next(i for i in range(4) if bad.hands[i].shanten > 0 and i != bad.actor)
    bad.hands[s].riichi = 1
    hb.load(0, bad)
    assert hb.check(0) & abi.INV_RIICHI_NOT_TENPAI


def _game(rule, mode, seed, policy):
    cfg = O.make_config(rule=rule, mode=mode)
    hb = hc.HostBatch(1, cfg)
    hb.init_seeds([seed])
    oe = O.OracleEnv(cfg).init(seed)
    rng = random.Random(seed)
    kc = [O.mix(seed ^ 0x5151), 0]
    t = 0
    kinds = []
    while True:
        a, b = projection(hb.record(0)), projection(oe.record())
        d = diff(a, b)
        assert not d, f"{rule} {mode} {policy} seed {seed} step {t}: {d[:5]}"
        r = oe.record()
        assert hb.observe(0, r.current_player) == oe.observe(r.current_player)
        if r.env_terminated or r.env_truncated:
            return [res["kind"] for res in oe.results()]
        legal = oe.legal()
        if policy == "heuristic":
            act = oe.heuristic_policy()
        elif policy == "random":
            act = oe.random_policy(kc)
        else:
            rare = [x for x in legal if x >= 37 and x != 113]
            if rare and rng.random() < 0.85:
                act = rng.choice(rare)
            elif rng.random() < 0.7:
                act = oe.heuristic_policy()
            else:
                act = rng.choice(legal)
            if rng.random() < 0.003:
                act = rng.randrange(-2, 120)  # illegal / out-of-range probe
        hb.step([act])
        oe.step(act)
        t += 1


@pytest.mark.parametrize("rule", ("no-red", "red"))
def test_lockstep_records_and_observations(rule):
    kinds = []
    for s in range(12):
        kinds += _game(rule, "single", 100 + s, "heuristic")
    for s in range(40):
        kinds += _game(rule, "single" if s % 4 else "east", 500 + s, "biased")
    kinds += _game(rule, "half", 7, "random")
    # the biased driver must reach the rare branches
    assert {"ron", "tsumo", "exhaustive"} <= set(kinds)


def test_crafted_import_roundtrip():
    cfg = O.make_config(rule="red")
    oe = O.OracleEnv(cfg).init(12345)
    for a in (oe.legal()[0],) * 5:
        oe.step(oe.legal()[0])
    rec = oe.record()
    hb = hc.HostBatch(2, cfg)
    hb.init_seeds([1, 2])
    hb.load(1, rec)
    o2 = O.OracleEnv(cfg)
    o2.load(rec)
    assert not diff(projection(hb.record(1)), projection(o2.record()))
