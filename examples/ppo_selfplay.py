#!/usr/bin/env python
"""PPO self-play over the batched device env (BASELINE configs[4], SURVEY
8(d) C5): a random-init PyTorch policy consumes the observations and legal
masks where the env writes them (device tensors, no host round trip) and
acts for whichever seat is to move; one process per GPU, gradients averaged
by DDP over NCCL.

    python examples/ppo_selfplay.py --envs 1024 --horizon 256 --iters 2
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 examples/ppo_selfplay.py

Self-play reward: every env step is a sample of the seat that acted; its
reward is that seat's share of the transition's rewards (the env's
score-delta terminal rewards, env/core.py:74-78), so returns flow back only
through the same seat's decisions (per-seat GAE).  This is a consumer of the
env API, not a tuned agent.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import torch
import torch.nn as nn
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_20577_b200 import dist as D  # noqa: E402
from paper_2605_20577_b200.env import BatchEnv, EnvConfig  # noqa: E402

NUM_ACTIONS = 115


class Policy(nn.Module):
    """token embeddings (hand, 64-event window, dora) + scalars -> logits, value"""

    def __init__(self, d: int = 128):
        super().__init__()
        self.tok = nn.Embedding(38, d)
        self.ev_type = nn.Embedding(11, d)
        self.ev_actor = nn.Embedding(4, d)
        self.pos = nn.Parameter(torch.zeros(64, d))
        self.scal = nn.Linear(4 + 4 + 8, d)
        self.trunk = nn.Sequential(nn.Linear(4 * d, 2 * d), nn.GELU(), nn.Linear(2 * d, d), nn.GELU())
        self.pi = nn.Linear(d, NUM_ACTIONS)
        self.v = nn.Linear(d, 1)

    def forward(self, o: dict[str, torch.Tensor]):
        hand = self.tok(o["hand_tokens"].long()).mean(1)
        ev = o["event_tokens"].long()
        evh = (self.tok(ev[..., 2]) + self.ev_type(ev[..., 0]) + self.ev_actor(ev[..., 1]) + self.pos).mean(1)
        dora = self.tok(o["dora_indicator_tokens"].long()).mean(1)
        s = torch.cat([o["scores"].float() / 250.0, o["riichi_flags"].float(),
                       torch.stack([o["shanten"].float() / 8, o["round_wind"].float() - 27, o["seat_wind"].float() - 27,
                                    o["kyoku"].float() / 8, o["honba"].float() / 8, o["deposits"].float() / 4,
                                    o["live_wall"].float() / 70, torch.ones_like(o["live_wall"].float())], -1)], -1)
        h = self.trunk(torch.cat([hand, evh, dora, self.scal(s)], -1))
        return self.pi(h), self.v(h).squeeze(-1)


def sample_masked(logits: torch.Tensor, mask: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """masked categorical sample (Gumbel-max: no host sync, CUDA-graph safe)
    -> (action, log-probability)"""
    logits = logits.masked_fill(~mask, -1e9)
    u = torch.rand_like(logits).clamp_(1e-20, 1.0)
    a = (logits - torch.log(-torch.log(u))).argmax(-1)
    return a, F.log_softmax(logits, -1).gather(1, a[:, None]).squeeze(1)


def legal_mask(bits: torch.Tensor) -> torch.Tensor:
    """packed u32[n,4] env legal bits -> bool[n,115]"""
    shifts = torch.arange(32, device=bits.device, dtype=torch.int32)
    m = ((bits.unsqueeze(-1) >> shifts) & 1).bool().reshape(bits.shape[0], 128)
    return m[:, :NUM_ACTIONS]


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--envs", type=int, default=1024)
    p.add_argument("--horizon", type=int, default=256)
    p.add_argument("--iters", type=int, default=2)
    p.add_argument("--epochs", type=int, default=2)
    p.add_argument("--minibatch", type=int, default=8192)
    p.add_argument("--rule", default="no-red")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl")
    p.add_argument("--no-graph", dest="graph", action="store_false",
                   help="run the rollout eagerly instead of replaying it as one CUDA graph")
    args = p.parse_args()
    # one write per line: ranks share stdout under torchrun
    os.write(1, (json.dumps(run(args)) + "\n").encode())


def run(args) -> dict:
    rank, world, local = D.world()
    if world > 1:
        D.init(args.dist_backend, local)  # DDP gradient all-reduce + the stats reduction
    dev = D.device(local)
    torch.cuda.set_device(dev)
    torch.manual_seed(args.seed + rank)
    T = args.horizon
    # env shard of this rank: global indices [rank * n, (rank + 1) * n)
    base, n = D.shard(rank, world, args.envs)
    env = BatchEnv(n, EnvConfig(rule=args.rule, mode="single"), device=dev).init(seed=args.seed, index_base=base)
    obs = env.observe()
    net = Policy().to(dev)
    model = nn.parallel.DistributedDataParallel(net, device_ids=[dev.index]) if world > 1 else net
    opt = torch.optim.Adam(model.parameters(), lr=3e-4)
    keys = list(obs.keys())
    buf = {k: torch.empty((T,) + tuple(obs[k].shape), dtype=obs[k].dtype, device=dev) for k in keys}
    b_mask = torch.empty(T, n, NUM_ACTIONS, dtype=torch.bool, device=dev)
    b_act = torch.empty(T, n, dtype=torch.long, device=dev)
    b_logp = torch.empty(T, n, device=dev)
    b_val = torch.empty(T, n, device=dev)
    b_seat = torch.empty(T, n, dtype=torch.long, device=dev)
    b_rew = torch.empty(T, n, 4, device=dev)
    b_done = torch.empty(T, n, device=dev)
    stats = {"env_steps": 0, "rollout_s": 0.0, "update_s": 0.0, "games": 0, "graph": bool(getattr(args, "graph", True))}

    def collect():
        """T steps: policy on the device observation and mask, masked sample,
        env step with auto-reset + observation; everything stays on the GPU
        (no host sync), so the whole horizon can be one CUDA graph"""
        with torch.no_grad():
            for t in range(T):
                for k in keys:
                    buf[k][t].copy_(obs[k])
                mask = legal_mask(env.legal_bits)
                logits, v = net(obs)
                a, logp = sample_masked(logits, mask)
                b_mask[t], b_act[t], b_val[t], b_logp[t] = mask, a, v, logp
                b_seat[t] = env.current_player.long()
                env.step(a.int(), autoreset=True, observe=True)  # obs / mask now the next state's
                b_rew[t] = env.rewards
                b_done[t] = (env.terminated | env.truncated).float()

    graph = None
    for it in range(args.iters):
        t0 = time.perf_counter()
        if graph is not None:
            graph.replay()
        else:
            collect()
            if stats["graph"]:
                # the eager horizon above warmed up every kernel; capture the
                # next one (the weights are read in place, so updates apply)
                torch.cuda.synchronize(dev)
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    collect()
        torch.cuda.synchronize(dev)
        if it > 0 or not stats["graph"]:  # the capture iteration's time is not a rollout
            stats["rollout_s"] += time.perf_counter() - t0
            stats["timed_steps"] = stats.get("timed_steps", 0) + n * T
        stats["env_steps"] += n * T
        stats["games"] += int(b_done.sum().item())
        t1 = time.perf_counter()
        # per-seat GAE: a sample's return continues at that seat's next turn
        with torch.no_grad():
            r = b_rew.gather(2, b_seat[..., None]).squeeze(-1)
            adv = torch.zeros(T, n, device=dev)
            nxt_adv = torch.zeros(n, 4, device=dev)
            nxt_val = torch.zeros(n, 4, device=dev)
            ar = torch.arange(n, device=dev)
            gamma, lam = 0.997, 0.95
            for t in reversed(range(T)):
                s = b_seat[t]
                # a finished game pays every seat at once: seats that did not
                # act this step still bank their terminal reward
                done = b_done[t]
                nxt_adv = nxt_adv * (1 - done)[:, None]
                nxt_val = nxt_val * (1 - done)[:, None]
                delta = r[t] + gamma * nxt_val[ar, s] - b_val[t]
                adv[t] = delta + gamma * lam * nxt_adv[ar, s]
                nxt_adv[ar, s] = adv[t]
                nxt_val[ar, s] = b_val[t]
            ret = adv + b_val
        flat = {k: buf[k].reshape((T * n,) + tuple(buf[k].shape[2:])) for k in keys}
        f_mask, f_act, f_logp = b_mask.reshape(T * n, -1), b_act.reshape(-1), b_logp.reshape(-1)
        f_adv, f_ret = adv.reshape(-1), ret.reshape(-1)
        f_adv = (f_adv - f_adv.mean()) / (f_adv.std() + 1e-8)
        for _ in range(args.epochs):
            perm = torch.randperm(T * n, device=dev)
            for i in range(0, T * n, args.minibatch):
                idx = perm[i:i + args.minibatch]
                logits, v = model({k: flat[k][idx] for k in keys})
                logits = logits.masked_fill(~f_mask[idx], -1e9)
                logp = F.log_softmax(logits, -1)
                lp = logp.gather(1, f_act[idx, None]).squeeze(1)
                ratio = (lp - f_logp[idx]).exp()
                pg = -torch.min(ratio * f_adv[idx], ratio.clamp(0.8, 1.2) * f_adv[idx]).mean()
                vl = F.mse_loss(v, f_ret[idx])
                ent = -(logp.exp() * logp).sum(-1).mean()
                loss = pg + 0.5 * vl - 0.01 * ent
                opt.zero_grad(set_to_none=True)
                loss.backward()
                nn.utils.clip_grad_norm_(model.parameters(), 0.5)
                opt.step()
        torch.cuda.synchronize(dev)
        stats["update_s"] += time.perf_counter() - t1
        stats["last_loss"] = float(loss.item())
    stats["env_steps_per_s_rollout"] = stats.get("timed_steps", 0) / max(stats["rollout_s"], 1e-9)
    if world > 1:
        t = D.reduce_stats(torch.tensor([stats["env_steps"], stats["games"]], dtype=torch.int64, device=dev))
        stats["env_steps_all_ranks"], stats["games_all_ranks"] = int(t[0]), int(t[1])
        D.finish()
    env.close()
    stats["rank"], stats["world"] = rank, world
    return stats


if __name__ == "__main__":
    main()
