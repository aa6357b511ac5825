"""examples/ppo_selfplay.py (BASELINE configs[4]) runs end to end on the
device env: observations and legal masks consumed on-device, masked
sampling never picks an illegal action, a PPO update with a finite loss."""

from __future__ import annotations

import argparse
import importlib.util
import math
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def _load():
    spec = importlib.util.spec_from_file_location("ppo_selfplay", ROOT / "examples" / "ppo_selfplay.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_ppo_selfplay_small():
    m = _load()
    args = argparse.Namespace(envs=256, horizon=24, iters=2, epochs=1, minibatch=2048, rule="no-red", seed=3)
    st = m.run(args)
    assert st["env_steps"] == 2 * 256 * 24
    assert math.isfinite(st["last_loss"])


def test_masked_sampling_is_always_legal():
    m = _load()
    from paper_2605_20577_b200.env import BatchEnv, EnvConfig

    env = BatchEnv(512, EnvConfig(rule="red")).init(seed=9)
    obs = env.observe()
    net = m.Policy().cuda()
    for _ in range(64):
        mask = m.legal_mask(env.legal_bits)
        with torch.no_grad():
            logits, _ = net(obs)
        a = torch.distributions.Categorical(logits=logits.masked_fill(~mask, -1e9)).sample()
        env.step(a.int(), autoreset=True, observe=True)
        torch.cuda.synchronize()
        assert int(env.status.sum().item()) == 0  # no illegal / contract status
