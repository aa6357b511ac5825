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


@pytest.mark.parametrize("graph", (False, True))
def test_ppo_selfplay_small(graph):
    """eager, and with the rollout horizon replayed as one CUDA graph"""
    m = _load()
    args = argparse.Namespace(envs=256, horizon=24, iters=3, epochs=1, minibatch=2048, rule="no-red", seed=3,
                              graph=graph)
    st = m.run(args)
    assert st["env_steps"] == 3 * 256 * 24 and st["graph"] == graph
    assert math.isfinite(st["last_loss"])
    assert st["env_steps_per_s_rollout"] > 0


def test_graph_rollout_steps_the_envs_like_eager():
    """the captured horizon replays real env steps: the same actions fed to
    a second env eagerly give the same rewards, masks and flags"""
    m = _load()
    from paper_2605_20577_b200.env import BatchEnv, EnvConfig

    n, T = 128, 16
    a_env = BatchEnv(n, EnvConfig(rule="red")).init(seed=5)
    b_env = BatchEnv(n, EnvConfig(rule="red")).init(seed=5)
    obs = a_env.observe()
    torch.manual_seed(0)
    net = m.Policy().cuda()
    acts = torch.empty(T, n, dtype=torch.int32, device="cuda")
    rews = torch.empty(T, n, 4, device="cuda")

    def body():
        with torch.no_grad():
            for t in range(T):
                logits, _ = net(obs)
                a, _ = m.sample_masked(logits, m.legal_mask(a_env.legal_bits))
                acts[t] = a.int()
                a_env.step(acts[t], autoreset=True, observe=True)
                rews[t] = a_env.rewards

    body()  # warm-up (eager)
    for t in range(T):
        b_env.step(acts[t], autoreset=True, observe=True)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body()
    for _ in range(2):
        g.replay()
        torch.cuda.synchronize()
        for t in range(T):
            b_env.step(acts[t], autoreset=True, observe=True)
            torch.cuda.synchronize()
        assert torch.equal(rews[T - 1], b_env.rewards)
        assert torch.equal(a_env.legal_bits, b_env.legal_bits)
        assert int(b_env.status.sum().item()) == 0


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


def test_ppo_two_ranks_on_one_gpu_gloo():
    """the DDP path (configs[4] across GPUs): two ranks sharing one B200
    over gloo, env shards by global index, gradients all-reduced by DDP,
    env steps and games summed over ranks by paper_2605_20577_b200.dist"""
    import json
    import os
    import socket
    import subprocess
    import sys

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), str(ROOT / "examples" / "ppo_selfplay.py"), "--envs", "128",
           "--horizon", "16", "--iters", "2", "--epochs", "1", "--minibatch", "1024", "--dist-backend", "gloo"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=dict(os.environ, OMP_NUM_THREADS="1"))
    assert r.returncode == 0, r.stderr[-3000:]
    dec, outs, i = json.JSONDecoder(), [], r.stdout.find("{")
    while i >= 0:  # every JSON object in the output, however the ranks' lines interleave
        obj, end = dec.raw_decode(r.stdout, i)
        outs.append(obj)
        i = r.stdout.find("{", end)
    assert len(outs) == 2 and {o["rank"] for o in outs} == {0, 1}
    for o in outs:
        assert o["world"] == 2 and o["env_steps_all_ranks"] == 2 * 2 * 128 * 16
        assert math.isfinite(o["last_loss"])
