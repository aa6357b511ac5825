"""Edge sizes of the batched path: rejected sizes, ragged batches (one env,
partial warps / CTAs / lane groups) and the maximum batch (2^23 envs, the
32-bit index math at its limit) against the oracle.  Needs a B200."""

from __future__ import annotations

import os
import random
from concurrent.futures import ThreadPoolExecutor

import pytest
import torch

from oracle import mjoracle as O
from paper_2605_20577_b200.env import BatchEnv, EnvConfig

pytestmark = pytest.mark.gpu

MAX_ENVS = 1 << 23  # rs_create's bound (include/rinshan.h)


@pytest.mark.parametrize("n", (0, -1, MAX_ENVS + 1))
def test_create_rejects_bad_sizes(n):
    with pytest.raises(Exception):
        BatchEnv(n, EnvConfig())


@pytest.mark.parametrize("n", (1, 2, 33, 1000, 4097))
def test_ragged_batches_match_oracle(n):
    steps, seed = 160, 123
    rule = "red" if n % 2 else "no-red"
    env = BatchEnv(n, EnvConfig(rule=rule)).init(seed=seed, index_base=0)
    digests = torch.zeros(n, dtype=torch.int64, device="cuda")
    env.rollout(steps // 2, digests=digests)
    for _ in range(steps // 2):  # single-step launches too
        env.rollout(1, digests=digests)
    torch.cuda.synchronize()
    got = [int(x) & ((1 << 64) - 1) for x in digests.cpu().tolist()]
    env.close()
    _, ref = O.run_shard(O.make_config(rule=rule), seed, 0, n, steps, digests=True)
    assert got == ref


def test_max_batch_sampled_parity():
    """2^23 envs (~21 GB of state): fused and single-step launches, then 256
    sampled envs (the first and the last included) against the oracle run
    on those env indices alone"""
    n, seed = MAX_ENVS, 5
    env = BatchEnv(n, EnvConfig(rule="red")).init(seed=seed, index_base=0)
    digests = torch.zeros(n, dtype=torch.int64, device="cuda")
    stats = torch.zeros(3, dtype=torch.int64, device="cuda")
    env.rollout(40, digests=digests, stats=stats)
    for _ in range(4):
        env.rollout(1, digests=digests, stats=stats)
    torch.cuda.synchronize()
    assert int(stats[0].item()) == n * 44
    rnd = random.Random(7)
    picks = sorted({0, n - 1, n // 2, *rnd.sample(range(n), 253)})
    got = digests[torch.tensor(picks, device="cuda")].cpu().tolist()
    env.close()
    cfg = O.make_config(rule="red")
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        ref = list(ex.map(lambda i: O.run_shard(cfg, seed, i, 1, 44, digests=True)[1][0], picks))
    assert [int(x) & ((1 << 64) - 1) for x in got] == ref


@pytest.mark.parametrize("rule", ("no-red", "red"))
def test_skip_action_leaves_envs_untouched(rule):
    """RS_ACTION_SKIP: envs whose actor has not decided are not stepped.
    Each env's trajectory depends only on its own action sequence, so env A
    fed the same per-env action sequences as env B, with random SKIP ticks
    interleaved, ends every env in B's state; skipped ticks report the
    current mask / player, zero rewards and status 0"""
    from paper_2605_20577_b200 import abi

    n, T = 256, 120
    cfg = EnvConfig(rule=rule)
    b = BatchEnv(n, cfg).init(seed=31, index_base=0)
    seq = []
    for _ in range(T):
        a = b.random_actions()
        seq.append(a.clone())
        b.step(a, autoreset=True)
    seq = torch.stack(seq)  # [T][n]
    a_env = BatchEnv(n, cfg).init(seed=31, index_base=0)
    cnt = torch.zeros(n, dtype=torch.long, device="cuda")
    gen = torch.Generator(device="cuda").manual_seed(3)
    ar = torch.arange(n, device="cuda")
    while int(cnt.min().item()) < T:
        go = (torch.rand(n, device="cuda", generator=gen) < 0.6) & (cnt < T)
        acts = torch.where(go, seq[cnt.clamp(max=T - 1), ar], torch.full_like(seq[0], abi.ACTION_SKIP))
        before_bits, before_player = a_env.legal_bits.clone(), a_env.current_player.clone()
        a_env.step(acts, autoreset=True)
        skipped = ~go
        assert torch.equal(a_env.legal_bits[skipped], before_bits[skipped])
        assert torch.equal(a_env.current_player[skipped], before_player[skipped])
        assert int(a_env.rewards[skipped].abs().sum().item()) == 0
        assert int(a_env.status[skipped].sum().item()) == 0
        cnt += go.long()
    torch.cuda.synchronize()
    for i in range(0, n, 17):
        ra, rb = a_env.export(i), b.export(i)
        # B's random_actions() drew from each env's policy stream; A's did not
        assert ra.policy_counter == 0 and rb.policy_counter > 0
        ra.policy_counter = rb.policy_counter
        assert bytes(ra) == bytes(rb), i
    assert torch.equal(a_env.legal_bits, b.legal_bits)


def test_reset_first_flag_validation():
    """RS_STEP_RESET_FIRST needs a policy output and excludes
    RS_STEP_AUTORESET (include/rinshan.h); BatchEnv.step(autoreset="next")
    needs next_actions"""
    from paper_2605_20577_b200 import abi

    env = BatchEnv(8, EnvConfig()).init(seed=3)
    acts = env.random_actions()
    nxt = torch.empty(8, dtype=torch.int32, device="cuda")
    L, h, s = env._L, env._h, torch.cuda.current_stream().cuda_stream
    assert L.rs_step_ex(h, acts.data_ptr(), abi.STEP_RESET_FIRST | abi.STEP_AUTORESET, None, None, nxt.data_ptr(),
                        s) == abi.RS_E_ARG
    assert L.rs_step_ex(h, acts.data_ptr(), abi.STEP_RESET_FIRST, None, None, None, s) == abi.RS_E_ARG
    with pytest.raises(ValueError):
        env.step(acts, autoreset="next")
    env.step(acts, autoreset="next", next_actions=nxt)  # valid
    torch.cuda.synchronize()
    env.close()


@pytest.mark.parametrize("warm", ("0", "1"))
def test_warm_cta_leaves_trajectories_unchanged(warm, monkeypatch):
    """the win-path warm-up CTA (RINSHAN_WARM, small batches) writes nothing
    an env can see: digests with and without it equal the oracle's"""
    monkeypatch.setenv("RINSHAN_WARM", warm)
    n, steps, seed = 512, 200, 77
    env = BatchEnv(n, EnvConfig(rule="red")).init(seed=seed, index_base=0)
    digests = torch.zeros(n, dtype=torch.int64, device="cuda")
    for _ in range(steps):
        env.rollout(1, digests=digests)
    torch.cuda.synchronize()
    got = [int(x) & ((1 << 64) - 1) for x in digests.cpu().tolist()]
    env.close()
    _, ref = O.run_shard(O.make_config(rule="red"), seed, 0, n, steps, digests=True)
    assert got == ref
