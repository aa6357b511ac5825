"""Per-env Pgx-style facade with the reference's names and semantics.

Drop-in for `mjsim.init / mjsim.step / mjsim.observe` (reference
pkg/src/mjsim/__init__.py:8-12, env/core.py:81-94, env/observe.py:81-124)
and `random_policy` (env/policies.py:17-22): immutable `EnvState` values,
`ContractError` when stepping a finished episode, illegal actions ending
the episode with the penalty at the offender.  Every transition runs on
the GPU through the C ABI (a batch-of-1 handle per config); the state value
carries the exported projection record plus the event / result history,
so `serialize()` / `fingerprint()` reproduce the reference's
`serialize_state` / `state_fingerprint` (engine/state.py:191-278).

This path exists for parity and interactive use; throughput work goes
through `BatchEnv`.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

import torch

from . import abi, records
from ._lib import check
from .env import BatchEnv, EnvConfig, alloc_observations, obs_struct

RANK_REWARDS = (1.0, 0.333, -0.333, -1.0)
NUM_ACTIONS = abi.NUM_ACTIONS
_MASK64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


class ContractError(ValueError):
    """Raised when a caller violates an operation precondition (tiles.py:41-42)."""


@dataclass(frozen=True)
class Observation:
    """env/observe.py:50-78"""

    hand_tokens: tuple
    event_tokens: tuple
    shanten: int
    scores: tuple
    round_wind: int
    seat_wind: int
    kyoku: int
    honba: int
    deposits: int
    dora_indicator_tokens: tuple
    live_wall: int
    riichi_flags: tuple

    def to_dict(self) -> dict:
        return {
            "hand_tokens": list(self.hand_tokens),
            "event_tokens": [list(e) for e in self.event_tokens],
            "shanten": self.shanten,
            "scores": list(self.scores),
            "round_wind": self.round_wind,
            "seat_wind": self.seat_wind,
            "kyoku": self.kyoku,
            "honba": self.honba,
            "deposits": self.deposits,
            "dora_indicator_tokens": list(self.dora_indicator_tokens),
            "live_wall": self.live_wall,
            "riichi_flags": list(self.riichi_flags),
        }


@dataclass(frozen=True, eq=False)
class EnvState:
    """env/core.py:49-62, plus the device projection of the game"""

    config: EnvConfig
    current_player: int
    legal: tuple
    legal_mask_int: int
    rewards: tuple
    terminated: bool
    truncated: bool
    record: abi.rs_env_rec = field(repr=False)
    events: tuple = field(repr=False, default=())
    results: tuple = field(repr=False, default=())
    game_legal: tuple = field(repr=False, default=())

    @property
    def legal_action_mask(self) -> tuple:
        m = self.legal_mask_int
        return tuple(bool((m >> a) & 1) for a in range(NUM_ACTIONS))

    def serialize(self) -> dict:
        return records.serialize_state(self.record, self.events, self.results, list(self.game_legal))

    def fingerprint(self) -> str:
        return records.fingerprint(self.serialize())


class _Runner:
    """one batch-of-1 device handle per (config, device), shared by every
    caller of the facade; `lock` is held from loading a state through
    reading the result, so threads stepping different games (the
    reference's service runs sync handlers in a threadpool) never see each
    other's state"""

    _cache: dict = {}
    _cache_lock = threading.Lock()

    def __init__(self, config: EnvConfig, device):
        self.env = BatchEnv(1, config, device=device)
        self.obs = alloc_observations(1, self.env.device)
        self.current: EnvState | None = None  # the state the handle holds
        self.lock = threading.RLock()

    @classmethod
    def get(cls, config: EnvConfig, device=None) -> "_Runner":
        dev = torch.device(device if device is not None else "cuda")
        key = (config, str(dev))
        with cls._cache_lock:
            if key not in cls._cache:
                cls._cache[key] = cls(config, dev)
            return cls._cache[key]

    def load(self, state: EnvState):
        if self.current is not state:
            self.env.load(0, state.record)
            self.current = state


def _mask_int(words) -> int:
    v = 0
    for i, w in enumerate(words):
        v |= (int(w) & 0xFFFFFFFF) << (32 * i)
    return v


def _reward(config: EnvConfig, x: float, illegal: bool) -> float:
    """The reference's Python double for a device float32 reward
    (core.py:74-78, 89-94).  Terminal rewards are (s - 25000) / 25000 with s a
    multiple of 100, the rank values 1 / .333 / -.333 / -1, or the illegal
    penalty: decimals of at most 6 significant digits, which the shortest
    float32 representation recovers exactly; the penalty comes from the
    config itself.  The device value must be that double rounded to float32."""
    f32 = np.float32(x)
    if illegal and f32 != 0 and f32 == np.float32(config.illegal_penalty):
        d = float(config.illegal_penalty)
    else:
        d = float(str(f32))
    if np.float32(d) != f32:
        raise RuntimeError(f"device reward {x!r} is not a reference reward")
    return d


def _wrap(config: EnvConfig, rec: abi.rs_env_rec, events, results, game_legal=None) -> EnvState:
    """game_legal None: the record's own legal ids"""
    m = _mask_int(rec.legal_mask)
    illegal = bool(rec.status & abi.STATUS_ILLEGAL)
    legal = abi.mask_to_ids(rec.legal_mask)
    if game_legal is None:
        game_legal = legal
    return EnvState(config=config, current_player=int(rec.current_player),
                    legal=legal, legal_mask_int=m,
                    rewards=tuple(_reward(config, float(x), illegal) for x in rec.rewards),
                    terminated=bool(rec.env_terminated), truncated=bool(rec.env_truncated),
                    record=rec, events=tuple(events), results=tuple(results), game_legal=tuple(game_legal))


def init(seed: int, config: EnvConfig = EnvConfig(), device=None) -> EnvState:
    """env/core.py:81-82"""
    r = _Runner.get(config, device)
    with r.lock:
        r.env.init(torch.tensor([_signed64(seed)], dtype=torch.int64))
        st = _initial(config, r.env.export(0))
        r.current = st
    return st


def _signed64(seed: int) -> int:
    s = seed & _MASK64
    return s - (1 << 64) if s >= (1 << 63) else s


def _initial(config: EnvConfig, rec: abi.rs_env_rec) -> EnvState:
    """the EnvState of a freshly dealt env's exported record"""
    return _wrap(config, rec, records.window_events(rec), ())


def step(state: EnvState, action: int) -> EnvState:
    """env/core.py:85-94"""
    if state.terminated or state.truncated:
        raise ContractError("cannot step a finished episode")
    r = _Runner.get(state.config, None)
    acts = torch.tensor([_action32(action)], dtype=torch.int32)
    with r.lock:
        r.load(state)
        r.env.step(acts)
        rec = r.env.export(0)
        st = _advance(state, rec)
        r.current = st
    return st


def _action32(action) -> int:
    """an action id as the step kernel's int32; ids outside int32, and the
    one int32 value the ABI reserves (RS_ACTION_SKIP, "not stepped"), become
    -1 so they are illegal like any other unknown id (core.py:89-94)"""
    a = int(action)
    return a if -(1 << 31) < a < (1 << 31) else -1


def _advance(state: EnvState, rec: abi.rs_env_rec) -> EnvState:
    """the EnvState after one step of `state`, from the stepped env's
    exported record (the event history and results extend `state`'s)"""
    old_len = int(state.record.events_len)
    added = int(rec.events_len) - old_len
    if added > abi.EVENT_WINDOW:
        raise RuntimeError("more than 64 events in one step")
    events = state.events + tuple(records.window_events(rec, added)) if added > 0 else state.events
    results = state.results
    if rec.n_results > state.record.n_results:
        results = results + (records.result_dict(rec.last_result),)
    illegal = bool(rec.status & abi.STATUS_ILLEGAL)
    game_legal = state.game_legal if illegal else None
    return _wrap(state.config, rec, events, results, game_legal)


def observe(state: EnvState, seat: int) -> Observation:
    """env/observe.py:81-124"""
    if not 0 <= seat <= 3:
        raise ValueError(f"bad seat {seat}")
    r = _Runner.get(state.config, None)
    with r.lock:
        r.load(state)
        seats = torch.tensor([seat], dtype=torch.int8, device=r.env.device)
        o = r.env.observe(seats, out=r.obs)
        torch.cuda.synchronize(r.env.device)
        o = {k: v.cpu() for k, v in o.items()}
    ev = o["event_tokens"][0].tolist()
    return Observation(
        hand_tokens=tuple(o["hand_tokens"][0].tolist()), event_tokens=tuple(tuple(e) for e in ev),
        shanten=int(o["shanten"][0]), scores=tuple(o["scores"][0].tolist()),
        round_wind=int(o["round_wind"][0]), seat_wind=int(o["seat_wind"][0]), kyoku=int(o["kyoku"][0]),
        honba=int(o["honba"][0]), deposits=int(o["deposits"][0]),
        dora_indicator_tokens=tuple(o["dora_indicator_tokens"][0].tolist()), live_wall=int(o["live_wall"][0]),
        riichi_flags=tuple(o["riichi_flags"][0].tolist()))


def heuristic_policy(state: EnvState, legal: tuple | None = None) -> int:
    """policies.py:51-109 heuristic_policy, evaluated on the device from
    `state` (the reference takes observe(state, current_player) and the
    legal ids; the hand and the called tile it reconstructs from them are
    read from the state here).  `legal`, when given, must be state.legal."""
    if legal is not None and tuple(legal) != tuple(state.legal):
        raise ValueError("legal must be the state's legal ids")
    if not state.legal:
        raise ValueError("no legal actions")
    r = _Runner.get(state.config, None)
    with r.lock:
        r.load(state)
        a = r.env.heuristic_actions()
        return int(a[0].item())


# --- rng.py:18-65 and policies.py:17-22 on the host (pure functions) ---

class RngState(tuple):
    """(key, counter), rng.py:28-30"""

    def __new__(cls, key: int, counter: int):
        return super().__new__(cls, (key, counter))

    @property
    def key(self):
        return self[0]

    @property
    def counter(self):
        return self[1]


def _mix(x: int) -> int:
    x &= _MASK64
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & _MASK64
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & _MASK64
    x ^= x >> 31
    return x


def derive_key(key: int, stream: int) -> int:
    return _mix((key ^ _GOLDEN) + _mix(stream & _MASK64))


def env_game_seed(seed: int, index: int, reset: int = 0) -> int:
    """bench/runner.py:25-28"""
    return derive_key(derive_key(_mix(seed & _MASK64), index), 2 + reset)


def env_policy_state(seed: int, index: int) -> RngState:
    """bench/runner.py:31-33"""
    return RngState(derive_key(derive_key(_mix(seed & _MASK64), index), 1), 0)


def random_policy(legal: tuple, rng: RngState) -> tuple:
    """policies.py:17-22: uniform over the ascending legal ids"""
    if not legal:
        raise ValueError("no legal actions to sample")
    c = rng.counter + 1
    x = _mix((rng.key + c * _GOLDEN) & _MASK64)
    return legal[(x * len(legal)) >> 64], RngState(rng.key, c)
