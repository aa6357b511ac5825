"""Batched sessions (sessions.SessionBatch) against one batch-of-1 handle per
session (new_session / apply_session_action / advance_agents): decisions
per second over whole games, one scripted human seat per session plus three
agents (random / heuristic mixed).  Usage: python tools/session_batch_bench.py [n ...]"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_20577_b200 import sessions as S  # noqa: E402
from paper_2605_20577_b200.env import EnvConfig  # noqa: E402

AGENTS = {1: "heuristic", 2: "random", 3: "heuristic"}


def human(legal, n):
    return legal[(7 * n + 3) % len(legal)]


def batched(cfg, n):
    torch.cuda.synchronize()
    t = time.perf_counter()
    b = S.SessionBatch(cfg, range(n), [0], AGENTS)
    ticks = 0
    while True:
        w = b.waiting()
        if not w:
            break
        b.apply_actions({i: human(b.sessions[i].state.legal, len(b.sessions[i].actions)) for i in w})
        ticks += 1
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    return sum(len(s.actions) for s in b.sessions), dt, ticks


def singles(cfg, n):
    torch.cuda.synchronize()
    t = time.perf_counter()
    total = 0
    for seed in range(n):
        s = S.new_session(cfg, seed, [0], AGENTS)
        while s.waiting_on() is not None:
            S.apply_session_action(s, human(s.state.legal, len(s.actions)))
            S.advance_agents(s)
        total += len(s.actions)
    torch.cuda.synchronize()
    return total, time.perf_counter() - t


def main():
    cfg = EnvConfig()
    batched(cfg, 4)  # warm-up (handles, tables)
    singles(cfg, 2)
    ns = [int(x) for x in sys.argv[1:]] or [1, 16, 64, 256, 1024]
    a, dt = singles(cfg, 8)
    print(json.dumps({"mode": "singles", "sessions": 8, "decisions": a, "s": round(dt, 3),
                      "decisions_per_s": round(a / dt)}))
    for n in ns:
        a, dt, ticks = batched(cfg, n)
        print(json.dumps({"mode": "batch", "sessions": n, "decisions": a, "ticks": ticks, "s": round(dt, 3),
                          "decisions_per_s": round(a / dt)}))


if __name__ == "__main__":
    main()
