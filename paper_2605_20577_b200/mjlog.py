"""Replayable game logs, "mjlog-lite v1" (reference engine/log.py:1-89,
pkg/docs/formats.md:9-30), produced from device games.

A log carries the game seed, the config and the applied [seat, action]
pairs -- enough to re-simulate -- plus the full event stream, per-kyoku
results, final scores / ranks and the sha256 fingerprint of the terminal
state, in the reference's canonical JSON form, so a log of the same game is
byte-identical to the reference's.

Two producers:
  * `GameRecorder` mirrors the reference class over `pgx` states;
  * `logs_from_rollout` turns one fused device rollout (actions + acting
    seats of every env and step, rs_rollout_policy) into the logs of every
    finished game; events / results / fingerprints come from replaying the
    actions through the device engine (`replay_log`).
"""

from __future__ import annotations

import json

import torch

from . import pgx
from .env import BatchEnv, EnvConfig

LOG_VERSION = "mjlog-lite-v1"

# engine/types.py:26-39 EV_NAMES
EV_NAMES = ("draw", "discard", "chi", "pon", "kan_open", "kan_closed", "kan_added", "riichi", "ron", "tsumo",
            "draw_end", "new_dora")


def config_to_dict(config: EnvConfig) -> dict:
    """engine/log.py:22-31"""
    return {
        "rule": config.rule,
        "mode": config.mode,
        "kazoe": bool(config.kazoe),
        "double_yakuman": bool(config.double_yakuman),
        "agari_yame": bool(config.agari_yame),
        "max_steps": int(config.max_steps),
        "renchan_cap": int(config.renchan_cap),
    }


def config_from_dict(d: dict, **env_kwargs) -> EnvConfig:
    """engine/log.py:34-43 (the env-level fields, e.g. illegal_penalty, are
    not part of a log and come from `env_kwargs`)"""
    return EnvConfig(rule=d["rule"], mode=d["mode"], kazoe=bool(d.get("kazoe", False)),
                     double_yakuman=bool(d.get("double_yakuman", False)),
                     agari_yame=bool(d.get("agari_yame", True)), max_steps=int(d.get("max_steps", 10_000)),
                     renchan_cap=int(d.get("renchan_cap", 32)), **env_kwargs)


def final_ranks(scores) -> list[int]:
    """engine/engine.py:885-891: ranks[seat], ties to the earlier seat"""
    order = sorted(range(4), key=lambda s: (-scores[s], s))
    ranks = [0, 0, 0, 0]
    for pos, seat in enumerate(order):
        ranks[seat] = pos
    return ranks


def _log(config: EnvConfig, seed: int, actions, final: pgx.EnvState) -> dict:
    rec = final.record
    scores = [int(x) for x in rec.scores]
    return {
        "version": LOG_VERSION,
        "seed": int(seed),
        "config": config_to_dict(config),
        "actions": [[int(s), int(a)] for s, a in actions],
        "events": [{"type": EV_NAMES[t], "actor": a, "tile": tile} for t, a, tile in final.events],
        "results": [dict(r) for r in final.results],
        "final_scores": scores,
        "ranks": final_ranks(scores),
        "terminated": bool(rec.terminated),
        "truncated": bool(rec.truncated),
        "fingerprint": final.fingerprint(),
    }


class GameRecorder:
    """engine/log.py:46-71: collects (actor, action) while a game is stepped"""

    def __init__(self, config: EnvConfig, seed: int):
        self.config = config
        self.seed = seed
        self.actions: list[tuple[int, int]] = []

    def record(self, state: pgx.EnvState, action: int) -> None:
        self.actions.append((int(state.record.actor), int(action)))

    def to_log(self, final_state: pgx.EnvState) -> dict:
        return _log(self.config, self.seed, self.actions, final_state)


def log_to_json(log: dict) -> str:
    """engine/log.py:74-75 canonical form"""
    return json.dumps(log, sort_keys=True, separators=(",", ":"))


def replay_log(log: dict, upto: int | None = None, **env_kwargs) -> pgx.EnvState:
    """engine/log.py:78-89: re-simulate the actions on the device engine;
    `upto` stops after that many actions.  Raises ValueError on an actor
    mismatch (log desync)."""
    config = config_from_dict(log["config"], **env_kwargs)
    st = pgx.init(int(log["seed"]), config)
    actions = log["actions"] if upto is None else log["actions"][:upto]
    for seat, action in actions:
        if int(st.record.actor) != seat:
            raise ValueError(f"log desync: expected actor {int(st.record.actor)}, log says {seat}")
        st = pgx.step(st, int(action))
    return st


def logs_from_rollout(seed: int, index_base: int, n: int, steps: int, config: EnvConfig = EnvConfig(),
                      policy: str = "random", include_unfinished: bool = False) -> list[dict]:
    """Run the fused device rollout of the bench envs [index_base,
    index_base + n) from their first game for `steps` steps and return the
    mjlog-lite log of every game played (finished ones; the game still in
    progress at the end too with `include_unfinished`), env by env.  Game r
    of env i uses seed pgx.env_game_seed(seed, i, r) (bench/runner.py:25-33)."""
    env = BatchEnv(n, config).init(seed=seed, index_base=index_base)
    acts = torch.zeros(steps, n, dtype=torch.int16, device=env.device)
    seats = torch.zeros(steps, n, dtype=torch.int8, device=env.device)
    env.rollout(steps, actions_log=acts, actors_log=seats, policy=policy)
    done = env.terminated.cpu().tolist()
    trunc = env.truncated.cpu().tolist()
    acts = acts.cpu().t().tolist()
    seats = seats.cpu().t().tolist()
    env.close()
    logs = []
    for i in range(n):
        games: list[list[tuple[int, int]]] = [[]]
        for t in range(steps):
            s = seats[i][t]
            if s & 4:  # auto-reset before this step: a new game
                games.append([])
            games[-1].append((s & 3, acts[i][t]))
        finished_last = bool(done[i] or trunc[i])
        for r, actions in enumerate(games):
            last = r == len(games) - 1
            if last and not finished_last and not include_unfinished:
                continue
            gseed = pgx.env_game_seed(seed, index_base + i, r)
            final = replay_log({"seed": gseed, "config": config_to_dict(config), "actions": actions},
                               illegal_penalty=config.illegal_penalty, reward_scheme=config.reward_scheme)
            logs.append(_log(config, gseed, actions, final))
    return logs
