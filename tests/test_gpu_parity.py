"""CUDA path vs the CPU oracle (bit-exact).  Needs a B200: `pytest -m gpu`."""

from __future__ import annotations

import random

import pytest
import torch

from oracle import mjoracle as O
from paper_2605_20577_b200.env import BatchEnv, EnvConfig
from paritylib import diff, projection

pytestmark = pytest.mark.gpu

RULES = ("no-red", "red")


def _oracle_cfg(cfg: EnvConfig):
    return O.make_config(rule=cfg.rule, mode=cfg.mode, illegal_penalty=cfg.illegal_penalty,
                         reward_scheme=cfg.reward_scheme, max_steps=cfg.max_steps, kazoe=cfg.kazoe,
                         double_yakuman=cfg.double_yakuman, agari_yame=cfg.agari_yame,
                         renchan_cap=cfg.renchan_cap)


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("mode", ("single", "east", "half"))
def test_fused_rollout_digests_match_oracle(rule, mode):
    """fused rollout (auto-reset + random policy + step) == oracle run_shard,
    env by env, through the 64-bit trajectory digest."""
    n, steps = (2048, 300) if mode == "single" else (256, 900)
    cfg = EnvConfig(rule=rule, mode=mode)
    env = BatchEnv(n, cfg).init(seed=11, index_base=0)
    digests = torch.zeros(n, dtype=torch.int64, device="cuda")
    stats = torch.zeros(3, dtype=torch.int64, device="cuda")
    env.rollout(steps, digests=digests, stats=stats)
    torch.cuda.synchronize()
    games, ref = O.run_shard(_oracle_cfg(cfg), 11, 0, n, steps, digests=True)
    got = [int(x) & ((1 << 64) - 1) for x in digests.cpu().tolist()]
    bad = [i for i in range(n) if got[i] != ref[i]]
    assert not bad, f"{len(bad)} envs diverge, first {bad[:8]}"
    st = stats.cpu().tolist()
    assert st[0] == n * steps and st[1] == games


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("policy", ("random", "heuristic"))
def test_config_flags_rollouts_match_oracle(rule, policy):
    """GameConfig flags off their defaults (engine/types.py:49-57): kazoe and
    double yakuman on (the settlement values of 13+ han and of the
    double-yakuman waits), agari-yame off, a short renchan cap and the rank
    reward scheme, over hanchan games, fused rollouts vs the oracle"""
    n, steps = (1024, 900) if policy == "random" else (2048, 600)
    cfg = EnvConfig(rule=rule, mode="half", kazoe=True, double_yakuman=True, agari_yame=False,
                    renchan_cap=2, reward_scheme="rank")
    env = BatchEnv(n, cfg).init(seed=29, index_base=0)
    digests = torch.zeros(n, dtype=torch.int64, device="cuda")
    stats = torch.zeros(3, dtype=torch.int64, device="cuda")
    env.rollout(steps, digests=digests, stats=stats, policy=policy)
    torch.cuda.synchronize()
    games, ref = O.run_shard(_oracle_cfg(cfg), 29, 0, n, steps, policy=policy, digests=True)
    got = [int(x) & ((1 << 64) - 1) for x in digests.cpu().tolist()]
    bad = [i for i in range(n) if got[i] != ref[i]]
    assert not bad, f"{len(bad)} envs diverge, first {bad[:8]}"
    assert stats.cpu().tolist()[1] == games


@pytest.mark.parametrize("stage", ("1", "2"))
@pytest.mark.parametrize("rule", RULES)
def test_shared_memory_stage_matches_oracle(rule, stage, monkeypatch):
    """the stepping kernels on the shared-memory stage (RINSHAN_STAGE, read
    at rs_create) give the same trajectories, fused rollout and k_step alike"""
    monkeypatch.setenv("RINSHAN_STAGE", stage)
    n, steps = 1024, 240
    cfg = EnvConfig(rule=rule)
    env = BatchEnv(n, cfg).init(seed=13, index_base=0)
    digests = torch.zeros(n, dtype=torch.int64, device="cuda")
    env.rollout(steps, digests=digests)
    torch.cuda.synchronize()
    _, ref = O.run_shard(_oracle_cfg(cfg), 13, 0, n, steps, digests=True)
    got = [int(x) & ((1 << 64) - 1) for x in digests.cpu().tolist()]
    assert got == ref
    # k_step path on the stage: random actions through step() vs an unstaged env
    monkeypatch.setenv("RINSHAN_STAGE", "0")
    plain = BatchEnv(n, cfg).init(seed=13, index_base=0)
    plain.rollout(steps)
    for _ in range(40):
        acts = plain.random_actions()
        plain.step(acts, autoreset=True)
        env.step(acts, autoreset=True)
    torch.cuda.synchronize()
    assert torch.equal(env.legal_bits, plain.legal_bits)
    assert torch.equal(env.rewards, plain.rewards)


@pytest.mark.parametrize("cluster", ("2", "4"))
def test_cluster_multicast_tables_match_oracle(cluster, monkeypatch):
    """the stepping kernels launched as thread-block clusters with the table
    block multicast over the cluster (RINSHAN_CLUSTER, read at rs_create);
    1000 envs leave padding CTAs without envs in the last cluster"""
    monkeypatch.setenv("RINSHAN_CLUSTER", cluster)
    n, steps = 1000, 200
    cfg = EnvConfig(rule="red")
    env = BatchEnv(n, cfg).init(seed=21, index_base=0)
    digests = torch.zeros(n, dtype=torch.int64, device="cuda")
    env.rollout(steps, digests=digests)
    torch.cuda.synchronize()
    _, ref = O.run_shard(_oracle_cfg(cfg), 21, 0, n, steps, digests=True)
    assert [int(x) & ((1 << 64) - 1) for x in digests.cpu().tolist()] == ref
    monkeypatch.setenv("RINSHAN_CLUSTER", "1")
    plain = BatchEnv(n, cfg).init(seed=21, index_base=0)
    plain.rollout(steps)
    for _ in range(40):
        acts = plain.random_actions()
        plain.step(acts, autoreset=True)
        env.step(acts, autoreset=True)
    torch.cuda.synchronize()
    assert torch.equal(env.legal_bits, plain.legal_bits)
    assert torch.equal(env.rewards, plain.rewards)


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("mode", ("single", "half"))
def test_heuristic_rollout_digests_match_oracle(rule, mode):
    """fused rollout with heuristic_policy acting (policies.py:51-109) ==
    oracle run_shard(policy=heuristic): tenpai / riichi / win / call paths
    at a rate random play never reaches"""
    n, steps = (2048, 400) if mode == "single" else (256, 1500)
    cfg = EnvConfig(rule=rule, mode=mode)
    env = BatchEnv(n, cfg).init(seed=17, index_base=0)
    digests = torch.zeros(n, dtype=torch.int64, device="cuda")
    stats = torch.zeros(3, dtype=torch.int64, device="cuda")
    env.rollout(steps, digests=digests, stats=stats, policy="heuristic")
    torch.cuda.synchronize()
    games, ref = O.run_shard(_oracle_cfg(cfg), 17, 0, n, steps, policy="heuristic", digests=True)
    got = [int(x) & ((1 << 64) - 1) for x in digests.cpu().tolist()]
    bad = [i for i in range(n) if got[i] != ref[i]]
    assert not bad, f"{len(bad)} envs diverge, first {bad[:8]}"
    assert stats.cpu().tolist()[1] == games


@pytest.mark.parametrize("rule", RULES)
def test_heuristic_actions_and_next_actions(rule):
    """rs_policy_heuristic + step_ex(next_policy=heuristic, autoreset) act
    exactly like the heuristic rollout, step by step"""
    n, steps = 512, 150
    cfg = EnvConfig(rule=rule)
    a = BatchEnv(n, cfg).init(seed=23)
    b = BatchEnv(n, cfg).init(seed=23)
    log = torch.zeros(steps, n, dtype=torch.int16, device="cuda")
    b.rollout(steps, actions_log=log, policy="heuristic")
    nxt = torch.empty(n, dtype=torch.int32, device="cuda")
    acts = a.heuristic_actions()
    for t in range(steps):
        assert torch.equal(acts.to(torch.int16), log[t]), f"step {t}"
        a.step(acts, autoreset=True, next_actions=nxt, next_policy="heuristic")
        acts = nxt.clone()


@pytest.mark.parametrize("rule", RULES)
def test_rollout_chunks_equal_one_launch(rule):
    """K steps in one launch == K/3 steps in three launches (state fully in HBM between)."""
    n = 512
    cfg = EnvConfig(rule=rule)
    a = BatchEnv(n, cfg).init(seed=5)
    b = BatchEnv(n, cfg).init(seed=5)
    da = torch.zeros(n, dtype=torch.int64, device="cuda")
    db = torch.zeros(n, dtype=torch.int64, device="cuda")
    a.rollout(240, digests=da)
    for _ in range(3):
        b.rollout(80, digests=db)
    torch.cuda.synchronize()
    assert torch.equal(da, db)


def _lockstep(rule, mode, n, steps, policy, seed=3):
    cfg = EnvConfig(rule=rule, mode=mode)
    ocfg = _oracle_cfg(cfg)
    seeds = [O.env_game_seed(seed, i) for i in range(n)]
    env = BatchEnv(n, cfg).init(torch.tensor([s - (1 << 64) if s >= 1 << 63 else s for s in seeds]))
    oes = [O.OracleEnv(ocfg).init(s) for s in seeds]
    rng = random.Random(seed)
    for t in range(steps):
        for i in range(n):
            a, b = projection(env.export(i)), projection(oes[i].record())
            d = diff(a, b)
            assert not d, f"env {i} step {t}: {d[:6]}"
        acts = []
        for i in range(n):
            r = oes[i].record()
            if r.env_terminated or r.env_truncated:
                acts.append(0)
                continue
            legal = oes[i].legal()
            if policy == "heuristic":
                acts.append(oes[i].heuristic_policy())
            else:  # biased towards rare actions + occasional illegal probes
                rare = [x for x in legal if x >= 37 and x != 113]
                if rare and rng.random() < 0.8:
                    acts.append(rng.choice(rare))
                elif rng.random() < 0.01:
                    acts.append(rng.randrange(115))
                else:
                    acts.append(rng.choice(legal))
        env.step(torch.tensor(acts, dtype=torch.int32))
        for i in range(n):
            oes[i].step(acts[i])
        # observation of the current player, env by env
        if t % 7 == 0:
            obs = env.observe()
            torch.cuda.synchronize()
            for i in range(n):
                cp = oes[i].record().current_player
                o = oes[i].observe(cp)
                assert obs["hand_tokens"][i].tolist() == o["hand_tokens"]
                assert obs["event_tokens"][i].tolist() == o["event_tokens"]
                assert int(obs["shanten"][i]) == o["shanten"]
                assert obs["scores"][i].tolist() == o["scores"]
                assert obs["dora_indicator_tokens"][i].tolist() == o["dora_indicator_tokens"]
                assert obs["riichi_flags"][i].tolist() == o["riichi_flags"]
                assert [int(obs[k][i]) for k in ("round_wind", "seat_wind", "kyoku", "honba", "deposits", "live_wall")] == \
                    [o[k] for k in ("round_wind", "seat_wind", "kyoku", "honba", "deposits", "live_wall")]


@pytest.mark.parametrize("rule", RULES)
def test_lockstep_heuristic_records(rule):
    _lockstep(rule, "east", 16, 160, "heuristic")


@pytest.mark.parametrize("rule", RULES)
def test_lockstep_biased_records(rule):
    _lockstep(rule, "single", 16, 120, "biased")


def test_step_tensors_match_records():
    n = 64
    env = BatchEnv(n, EnvConfig(rule="red")).init(seed=1)
    for _ in range(50):
        env.step(env.random_actions())
    torch.cuda.synchronize()
    for i in range(0, n, 9):
        r = env.export(i)
        bits = [int(x) & 0xFFFFFFFF for x in env.legal_bits[i].tolist()]
        assert bits == [int(x) for x in r.legal_mask]
        mask = env.legal_action_mask[i].tolist()
        assert mask == [bool((bits[a >> 5] >> (a & 31)) & 1) for a in range(115)]
        assert int(env.current_player[i]) == r.current_player
        assert env.rewards[i].tolist() == [float(x) for x in r.rewards]
        assert bool(env.terminated[i]) == bool(r.env_terminated)


@pytest.mark.parametrize("zero_copy,order", ((True, "1"), (False, "1"), (True, "2")))
@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("autoreset", (True, "next"))
def test_host_stepper_equals_fused_rollout(rule, zero_copy, order, autoreset, monkeypatch):
    """HostStepper (CUDA graph: actions in, fused step+autoreset+observe+
    policy, result block out -- through mapped pinned memory or explicit
    copies) follows the same trajectories as k_rollout, with the reset in
    the finishing step (autoreset=True) or in the next one (autoreset="next",
    RS_STEP_RESET_FIRST: the runner's order, so finished envs match too)."""
    from paper_2605_20577_b200.env import HostStepper

    monkeypatch.setenv("RINSHAN_ORDER", order)  # "2": the env sort runs inside the captured graph
    n, steps = 300, 150
    cfg = EnvConfig(rule=rule)
    a = BatchEnv(n, cfg).init(seed=9)
    b = BatchEnv(n, cfg).init(seed=9)
    a.rollout(steps)
    hs = HostStepper(b, autoreset=autoreset, observe=True, policy=True, zero_copy=zero_copy)
    first = torch.empty(n, dtype=torch.int32, device="cuda")
    b.random_actions(out=first)
    hs.actions.copy_(first.cpu())
    # k_rollout resets before choosing; HostStepper resets after stepping:
    # identical sequence of (reset, policy draw, step)
    for _ in range(steps):
        hs.step()
        hs.actions.copy_(hs.next_actions)
    torch.cuda.synchronize()
    compared = finished = 0
    for i in range(0, n, 3):
        reca, recb = a.export(i), b.export(i)
        done = reca.env_terminated or reca.env_truncated
        if done and autoreset is True:
            continue  # b has already auto-reset this env
        if done:  # "next": both finished, no next action drawn
            finished += 1
            assert not diff(projection(reca), projection(recb)), (i, diff(projection(reca), projection(recb))[:5])
            assert recb.policy_counter == reca.policy_counter
            assert hs.next_actions[i] == -1
            continue
        assert recb.policy_counter == reca.policy_counter + 1
        compared += 1
        ra, rb = projection(reca), projection(recb)
        # b has already drawn (and consumed) the next policy action
        ra["internal"].pop("rewards"); rb["internal"].pop("rewards")
        ra["internal"].pop("legal_mask"); rb["internal"].pop("legal_mask")
        ra.pop("legal"); rb.pop("legal")
        for d in (ra, rb):
            d["internal"].pop("env_terminated"); d["internal"].pop("env_truncated")
        assert not diff(ra, rb), (i, diff(ra, rb)[:5])
    assert compared > 50
    if autoreset == "next":
        assert b.export(0).resets == a.export(0).resets


@pytest.mark.parametrize("rule", RULES)
@pytest.mark.parametrize("policy", ("random", "heuristic"))
def test_device_soak_invariants(rule, policy):
    """bench/runner.py:226-284 on the device: check_invariants (full) after
    every fused step of random / heuristic play over many envs"""
    env = BatchEnv(1024, EnvConfig(rule=rule, mode="half")).init(seed=41)
    flags = env.soak(300, policy=policy)
    torch.cuda.synchronize()
    bad = torch.nonzero(flags).flatten().tolist()
    assert not bad, f"{len(bad)} envs violate, first {bad[:4]} flags {flags[bad[0]].item() if bad else 0}"


def test_status_invariant_bit_when_checking_every_step(monkeypatch):
    """SURVEY 8(b) status bit 2 (debug): with RINSHAN_CHECK=1 every step runs
    the fast invariants; clean play never sets RS_STATUS_INVARIANT, a
    corrupted state does"""
    from paper_2605_20577_b200 import abi

    monkeypatch.setenv("RINSHAN_CHECK", "1")
    env = BatchEnv(256, EnvConfig(rule="red")).init(seed=31)
    for _ in range(60):
        env.rollout(1)
        torch.cuda.synchronize()
        assert int((env.status.int() & abi.STATUS_INVARIANT).sum().item()) == 0
    for _ in range(20):
        env.step(env.random_actions(), autoreset=True)
        torch.cuda.synchronize()
        assert int((env.status.int() & abi.STATUS_INVARIANT).sum().item()) == 0
    i = next(i for i in range(256) if not env.export(i).env_terminated)
    rec = env.export(i)
    rec.scores[0] += 100  # the score identity no longer holds
    env.load(i, rec)
    acts = env.random_actions()
    env.step(acts)
    torch.cuda.synchronize()
    assert int(env.status[i].item()) & abi.STATUS_INVARIANT


@pytest.mark.parametrize("rule", RULES)
def test_fused_trajectory_equals_single_steps(rule):
    """rs_rollout_policy traj: the per-step outputs of one K-step launch
    (mask, player, rewards, flags, and the observation with obs_slots = K)
    equal those of K one-step launches"""
    from paper_2605_20577_b200.env import alloc_observations, alloc_trajectory

    n, k = 512, 40
    cfg = EnvConfig(rule=rule)
    a = BatchEnv(n, cfg).init(seed=19)
    b = BatchEnv(n, cfg).init(seed=19)
    a.rollout(100)
    b.rollout(100)
    traj = alloc_trajectory(k, n, a.device)
    obs_a = alloc_observations(n, a.device, slots=k)
    a.rollout(k, obs=obs_a, obs_slots=k, traj=traj)
    obs_b = alloc_observations(n, b.device)
    for t in range(k):
        b.rollout(1, obs=obs_b, obs_slots=1)
        torch.cuda.synchronize()
        assert torch.equal(traj["legal_bits"][t], b.legal_bits), t
        assert torch.equal(traj["current_player"][t], b.current_player), t
        assert torch.equal(traj["rewards"][t], b.rewards), t
        assert torch.equal(traj["terminated"][t], b.terminated.to(torch.uint8)), t
        assert torch.equal(traj["status"][t], b.status), t
        for key in ("hand_tokens", "event_tokens", "scores", "dora_indicator_tokens"):
            assert torch.equal(obs_a[key][t], obs_b[key]), (t, key)


@pytest.mark.parametrize("zero_copy", (True, False))
def test_host_stepper_observations_to_host(zero_copy):
    """HostStepper(obs_to_host=True): after every step the host-side
    observations equal a device observe() of each env's current player, and
    the completion word (RS_STEP_SIGNAL / rs_signal_done) never lets the
    host read a step early (the result block and next actions agree with
    the env's own state)"""
    from paper_2605_20577_b200.env import HostStepper

    n = 257
    env = BatchEnv(n, EnvConfig(rule="red")).init(seed=21)
    hs = HostStepper(env, autoreset=True, observe=True, policy=True, zero_copy=zero_copy, obs_to_host=True)
    first = torch.empty(n, dtype=torch.int32, device="cuda")
    env.random_actions(out=first)
    hs.actions.copy_(first.cpu())
    acts, nxt = hs.actions.numpy(), hs.next_actions.numpy()
    for t in range(40):
        hs.step()
        host_obs = {k: v.clone() for k, v in hs.observations.items()}
        cp = hs.current_player.clone()
        acts[:] = nxt
        from paper_2605_20577_b200.env import alloc_observations

        dev_obs = env.observe(cp.to(torch.int8).cuda(), out=alloc_observations(n, "cuda"))
        torch.cuda.synchronize()
        for k, v in dev_obs.items():
            assert torch.equal(host_obs[k], v.cpu()), (t, k)
    hs.close()


@pytest.mark.parametrize("policy", ("random", "heuristic"))
def test_step_reset_first_equals_rollout(policy):
    """BatchEnv.step(autoreset="next") (RS_STEP_RESET_FIRST through rs_step_ex)
    with the next actions fed back equals the fused rollout of the same
    policy env for env, finished envs included (the runner's order)"""
    n, steps = 256, 160
    cfg = EnvConfig(rule="red")
    a = BatchEnv(n, cfg).init(seed=5)
    b = BatchEnv(n, cfg).init(seed=5)
    a.rollout(steps, policy=policy)
    acts = b.heuristic_actions() if policy == "heuristic" else b.random_actions()
    nxt = torch.empty(n, dtype=torch.int32, device="cuda")
    for _ in range(steps):
        b.step(acts, autoreset="next", next_actions=nxt, next_policy=policy)
        acts, nxt = nxt, acts
    torch.cuda.synchronize()
    for i in range(0, n, 5):
        ra, rb = a.export(i), b.export(i)
        pa, pb = projection(ra), projection(rb)
        if not (ra.env_terminated or ra.env_truncated) and policy == "random":
            # b has already drawn its next action from the policy stream
            assert rb.policy_counter == ra.policy_counter + 1
            for d in (pa, pb):
                d["internal"].pop("policy_counter", None)
        assert not diff(pa, pb), (i, diff(pa, pb)[:5])
