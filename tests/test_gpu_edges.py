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
