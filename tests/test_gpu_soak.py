"""North-star parity bar (BASELINE.json): bit-exact with the CPU oracle on
>= 10^5 randomly played hands per rule.  32,768 bench-seeded envs x 400
fused steps on the device; the oracle replays the same envs on all host
threads; every env's 64-bit trajectory digest must match.  The digest
folds, after every step: the action, player, flags, phase, round
counters, legal mask, scores, rewards, shanten of all seats, events
length and wall counters (digest_step); every state field in canonical
form -- the four concealed tile-id sets, HandState flags (riichi, riichi
index, ippatsu, temp / permanent furiten), waits, melds, river entries
with their flags, the call queue and ron list, both RNGs, the whole wall
with its dora / ura indicators, the newest events and the last kyoku
result with its win details (digest_state); and the current player's
observation exactly as encoded (digest_obs, env/observe.py:81-124).  The
random-policy soak also runs the fast invariant checker
(engine/state.py:105-178, the soak gate of bench/runner.py:226-284) after
every step of the whole run (RINSHAN_CHECK=1).  Needs a B200."""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import pytest
import torch

from oracle import mjoracle as O
from paper_2605_20577_b200.env import BatchEnv, EnvConfig

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rule", ("no-red", "red"))
def test_bit_exact_on_1e5_hands(rule, monkeypatch):
    from paper_2605_20577_b200 import abi

    monkeypatch.setenv("RINSHAN_CHECK", "1")  # invariants after every step (read at rs_create)
    n, steps, seed, chunk = 32768, 400, 2026, 1024
    env = BatchEnv(n, EnvConfig(rule=rule)).init(seed=seed, index_base=0)
    digests = torch.zeros(n, dtype=torch.int64, device="cuda")
    stats = torch.zeros(3, dtype=torch.int64, device="cuda")
    env.rollout(steps, digests=digests, stats=stats)
    torch.cuda.synchronize()
    # RS_STATUS_INVARIANT is sticky over the fused steps of a launch
    assert int((env.status.int() & abi.STATUS_INVARIANT).count_nonzero().item()) == 0
    got = [int(x) & ((1 << 64) - 1) for x in digests.cpu().tolist()]
    games = int(stats[1].item())
    env.close()
    cfg = O.make_config(rule=rule)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:  # ctypes releases the GIL
        parts = list(ex.map(lambda b: O.run_shard(cfg, seed, b, chunk, steps, digests=True), range(0, n, chunk)))
    ref = [d for _, ds in parts for d in ds]
    ref_games = sum(g for g, _ in parts)
    assert games == ref_games
    assert games >= 100_000, f"only {games} hands played"
    bad = [i for i in range(n) if got[i] != ref[i]]
    assert not bad, f"{len(bad)} of {n} envs diverge, first {bad[:8]}"


@pytest.mark.parametrize("rule", ("no-red", "red"))
def test_heuristic_soak_matches_oracle(rule, monkeypatch):
    """the heuristic policy (policies.py:51-109) reaches tenpai, riichi,
    calls and wins at rates random play never does: 65,536 envs x 500 fused
    heuristic steps (>= 10^5 hands), every trajectory digest equal to the
    oracle's, the fast invariants after every step and the full checker
    clean afterwards"""
    from paper_2605_20577_b200 import abi

    monkeypatch.setenv("RINSHAN_CHECK", "1")
    n, steps, seed, chunk = 65536, 500, 4242, 2048
    env = BatchEnv(n, EnvConfig(rule=rule)).init(seed=seed, index_base=0)
    digests = torch.zeros(n, dtype=torch.int64, device="cuda")
    stats = torch.zeros(3, dtype=torch.int64, device="cuda")
    env.rollout(steps, digests=digests, stats=stats, policy="heuristic")
    flags = env.check_invariants(fast=False)
    torch.cuda.synchronize()
    assert int((env.status.int() & abi.STATUS_INVARIANT).count_nonzero().item()) == 0
    got = [int(x) & ((1 << 64) - 1) for x in digests.cpu().tolist()]
    games = int(stats[1].item())
    assert int(flags.count_nonzero().item()) == 0
    env.close()
    cfg = O.make_config(rule=rule)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        parts = list(ex.map(lambda b: O.run_shard(cfg, seed, b, chunk, steps, policy="heuristic", digests=True),
                            range(0, n, chunk)))
    ref = [d for _, ds in parts for d in ds]
    assert games == sum(g for g, _ in parts) and games >= 100_000, games
    bad = [i for i in range(n) if got[i] != ref[i]]
    assert not bad, f"{len(bad)} of {n} envs diverge, first {bad[:8]}"


@pytest.mark.parametrize("n", (4096, 8192, 16384, 65536))
def test_lane_group_sizes_match_oracle(n):
    """every lane-group size the launch heuristic picks (16, 8, 4, 1 lanes
    per env at these batch sizes) gives the oracle's trajectories; 4096 is
    the bench configuration"""
    steps, seed, chunk = 250, 77, 1024
    rule = "red" if n % 8192 else "no-red"
    env = BatchEnv(n, EnvConfig(rule=rule)).init(seed=seed, index_base=0)
    digests = torch.zeros(n, dtype=torch.int64, device="cuda")
    env.rollout(steps, digests=digests)
    torch.cuda.synchronize()
    got = [int(x) & ((1 << 64) - 1) for x in digests.cpu().tolist()]
    env.close()
    cfg = O.make_config(rule=rule)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        parts = list(ex.map(lambda b: O.run_shard(cfg, seed, b, chunk, steps, digests=True), range(0, n, chunk)))
    ref = [d for _, ds in parts for d in ds]
    bad = [i for i in range(n) if got[i] != ref[i]]
    assert not bad, f"{len(bad)} of {n} envs diverge, first {bad[:8]}"


@pytest.mark.parametrize("n,force", ((2048, True), (131072, False)))
def test_env_ordering_matches_oracle(n, force, monkeypatch):
    """envs processed in next-step-kind order (CUB sort between launches,
    default at >= 131072 envs; forced below) keep every trajectory, one-step
    launches and fused launches alike"""
    if force:
        monkeypatch.setenv("RINSHAN_ORDER", "2")
    steps, seed, chunk = 120, 91, 1024
    env = BatchEnv(n, EnvConfig(rule="red")).init(seed=seed, index_base=0)
    digests = torch.zeros(n, dtype=torch.int64, device="cuda")
    for _ in range(steps // 2):
        env.rollout(1, digests=digests)
    env.rollout(steps - steps // 2, digests=digests)
    torch.cuda.synchronize()
    got = [int(x) & ((1 << 64) - 1) for x in digests.cpu().tolist()]
    env.close()
    cfg = O.make_config(rule="red")
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        parts = list(ex.map(lambda b: O.run_shard(cfg, seed, b, min(chunk, n - b), steps, digests=True),
                            range(0, n, chunk)))
    ref = [d for _, ds in parts for d in ds]
    bad = [i for i in range(n) if got[i] != ref[i]]
    assert not bad, f"{len(bad)} of {n} envs diverge, first {bad[:8]}"
