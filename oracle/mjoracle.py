"""ctypes wrapper of the CPU ORACLE (test infrastructure only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg import this module; the product package never does.
It exposes the oracle with the reference's env-facing names
(init / step / observe / random_policy / heuristic_policy) plus the
projection helpers used by the parity tests.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from pathlib import Path

from paper_2605_20577_b200 import abi, records

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libmjoracle.so"
_lib = None
_lock = threading.Lock()


def build(force: bool = False) -> Path:
    srcs = [_HERE / "mjoracle.c", _HERE / "mjoracle.h", _HERE.parent / "include" / "rinshan.h"]
    if force or not _LIB_PATH.exists() or any(s.stat().st_mtime > _LIB_PATH.stat().st_mtime for s in srcs):
        subprocess.check_call(["make", "-s", "-C", str(_HERE)])
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(str(_LIB_PATH))
            u64, i32, vp = C.c_uint64, C.c_int32, C.c_void_p
            L.orc_mix.restype = u64; L.orc_mix.argtypes = [u64]
            L.orc_derive_key.restype = u64; L.orc_derive_key.argtypes = [u64, u64]
            L.orc_seed_key.restype = u64; L.orc_seed_key.argtypes = [u64]
            L.orc_env_game_seed.restype = u64; L.orc_env_game_seed.argtypes = [u64, u64, u64]
            L.orc_env_policy_key.restype = u64; L.orc_env_policy_key.argtypes = [u64, u64]
            L.orc_shuffle136.argtypes = [u64, u64, vp, vp]
            L.orc_tables_build.restype = C.c_int
            L.orc_tables_crc.restype = C.c_uint32
            L.orc_tables_blob.restype = C.c_int64; L.orc_tables_blob.argtypes = [vp, C.c_int64]
            L.orc_suit_vals.restype = vp
            L.orc_honor_vals.restype = vp
            L.orc_shanten.argtypes = [vp, C.c_int]
            L.orc_shanten_standard.argtypes = [vp, C.c_int]
            L.orc_waits.restype = u64; L.orc_waits.argtypes = [vp, C.c_int]
            L.orc_decompose.argtypes = [vp, C.c_int, vp, C.c_int]
            L.orc_score_win.argtypes = [vp, vp, vp, vp]
            L.orc_base_points.argtypes = [C.c_int] * 4
            L.orc_settle.argtypes = [C.c_int] * 7 + [vp, vp]
            L.orc_env_new.restype = vp
            L.orc_env_free.argtypes = [vp]
            L.orc_env_copy.argtypes = [vp, vp]
            L.orc_env_init.argtypes = [vp, vp, u64]
            L.orc_env_step.argtypes = [vp, C.c_int]
            L.orc_env_export.argtypes = [vp, vp]
            L.orc_env_import.argtypes = [vp, vp]
            L.orc_env_num_events.argtypes = [vp]
            L.orc_env_events.argtypes = [vp, vp]
            L.orc_env_num_results.argtypes = [vp]
            L.orc_env_result.argtypes = [vp, C.c_int, vp, vp, vp]
            L.orc_env_legal.argtypes = [vp, vp]
            L.orc_env_game_legal.argtypes = [vp, vp]
            L.orc_env_observe.argtypes = [vp, C.c_int, vp]
            L.orc_random_policy.argtypes = [vp, vp]
            L.orc_heuristic_policy.argtypes = [vp]
            L.orc_run_shard.restype = C.c_int64
            L.orc_run_shard.argtypes = [vp, u64, C.c_int64, C.c_int64, i32, i32, vp]
            L.orc_digest_step.restype = u64; L.orc_digest_step.argtypes = [u64, C.c_int, vp]
            L.orc_batch_new.restype = vp; L.orc_batch_new.argtypes = [vp, u64, C.c_int64, C.c_int64]
            L.orc_batch_free.argtypes = [vp]
            L.orc_batch_step.restype = C.c_int64; L.orc_batch_step.argtypes = [vp, i32, i32]
            _lib = L
    return _lib


class orc_obs(C.Structure):
    _fields_ = [
        ("hand_tokens", C.c_uint8 * 14),
        ("event_tokens", (C.c_uint8 * 3) * 64),
        ("shanten", C.c_int32),
        ("scores", C.c_int32 * 4),
        ("round_wind", C.c_int32),
        ("seat_wind", C.c_int32),
        ("kyoku", C.c_int32),
        ("honba", C.c_int32),
        ("deposits", C.c_int32),
        ("dora_tokens", C.c_uint8 * 5),
        ("live_wall", C.c_int32),
        ("riichi_flags", C.c_uint8 * 4),
    ]


# the oracle's orc_winctx (mjoracle.h) has rs_winctx's layout (include/rinshan.h)
orc_winctx = abi.rs_winctx


def make_config(rule="red", mode="single", illegal_penalty=-1.0, reward_scheme="score_delta",
                max_steps=10_000, kazoe=False, double_yakuman=False, agari_yame=True,
                renchan_cap=32) -> abi.rs_config:
    return abi.rs_config(
        rule=abi.RULE_RED if rule == "red" else abi.RULE_NO_RED,
        mode={"single": 0, "east": 1, "half": 2}[mode],
        reward_scheme=0 if reward_scheme == "score_delta" else 1,
        illegal_penalty=illegal_penalty, max_steps=max_steps, kazoe=int(kazoe),
        double_yakuman=int(double_yakuman), agari_yame=int(agari_yame), renchan_cap=renchan_cap)


def obs_to_dict(o: orc_obs) -> dict:
    """reference env/observe.py:64-78 (Observation.to_dict)"""
    return {
        "hand_tokens": list(o.hand_tokens),
        "event_tokens": [list(o.event_tokens[i]) for i in range(64)],
        "shanten": o.shanten,
        "scores": list(o.scores),
        "round_wind": o.round_wind,
        "seat_wind": o.seat_wind,
        "kyoku": o.kyoku,
        "honba": o.honba,
        "deposits": o.deposits,
        "dora_indicator_tokens": list(o.dora_tokens),
        "live_wall": o.live_wall,
        "riichi_flags": list(o.riichi_flags),
    }


class OracleEnv:
    """One mutable oracle env (the reference's EnvState is immutable; the
    oracle steps in place and `clone()` gives value semantics)."""

    def __init__(self, config: abi.rs_config | None = None):
        self._L = lib()
        self._p = self._L.orc_env_new()
        self.config = config if config is not None else make_config()

    def __del__(self):
        try:
            self._L.orc_env_free(self._p)
        except Exception:
            pass

    def clone(self) -> "OracleEnv":
        o = OracleEnv(self.config)
        self._L.orc_env_copy(o._p, self._p)
        return o

    # --- env API (reference env/core.py:81-94, observe.py:81) ---
    def init(self, seed: int) -> "OracleEnv":
        self._L.orc_env_init(self._p, C.byref(self.config), seed & ((1 << 64) - 1))
        return self

    def step(self, action: int) -> int:
        return self._L.orc_env_step(self._p, int(action))

    def observe(self, seat: int) -> dict:
        o = orc_obs()
        self._L.orc_env_observe(self._p, seat, C.byref(o))
        return obs_to_dict(o)

    def legal(self) -> tuple[int, ...]:
        buf = (C.c_int32 * 115)()
        n = self._L.orc_env_legal(self._p, buf)
        return tuple(buf[:n])

    def game_legal(self) -> list[int]:
        buf = (C.c_int32 * 115)()
        n = self._L.orc_env_game_legal(self._p, buf)
        return list(buf[:n])

    def record(self) -> abi.rs_env_rec:
        r = abi.rs_env_rec()
        self._L.orc_env_export(self._p, C.byref(r))
        return r

    def load(self, rec: abi.rs_env_rec) -> None:
        self._L.orc_env_import(self._p, C.byref(rec))

    def events(self) -> list[tuple[int, int, int]]:
        n = self._L.orc_env_num_events(self._p)
        buf = (C.c_int16 * (3 * max(n, 1)))()
        self._L.orc_env_events(self._p, buf)
        return [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n)]

    def results(self) -> list[dict]:
        out = []
        for i in range(self._L.orc_env_num_results(self._p)):
            r = abi.rs_result_rec()
            orders = (C.c_int8 * (3 * 48))()
            norders = (C.c_int32 * 3)()
            self._L.orc_env_result(self._p, i, C.byref(r), orders, norders)
            d = records.result_dict(r)
            # the oracle also reports the explicit entry order: check the
            # host-side reconstruction (records.yaku_entries) against it
            for w in range(r.n_winners):
                explicit = [int(orders[48 * w + j]) for j in range(norders[w])]
                rebuilt = [y for y, _ in d["win_details"][w]["yaku"]]
                assert explicit == rebuilt, (explicit, rebuilt)
            out.append(d)
        return out

    def serialize(self) -> dict:
        return records.serialize_state(self.record(), self.events(), self.results(), self.game_legal())

    def fingerprint(self) -> str:
        return records.fingerprint(self.serialize())

    def random_policy(self, key_counter: list[int]) -> int:
        kc = (C.c_uint64 * 2)(*key_counter)
        a = self._L.orc_random_policy(self._p, kc)
        key_counter[1] = kc[1]
        return a

    def heuristic_policy(self) -> int:
        return self._L.orc_heuristic_policy(self._p)

    def digest_step(self, d: int, action: int) -> int:
        return self._L.orc_digest_step(d, action, self._p)


# --- free functions with reference names ---

def mix(x: int) -> int:
    return lib().orc_mix(x & ((1 << 64) - 1))


def derive_key(key: int, stream: int) -> int:
    return lib().orc_derive_key(key & ((1 << 64) - 1), stream & ((1 << 64) - 1))


def env_game_seed(seed: int, index: int, reset: int = 0) -> int:
    return lib().orc_env_game_seed(seed & ((1 << 64) - 1), index, reset)


def env_policy_key(seed: int, index: int) -> int:
    return lib().orc_env_policy_key(seed & ((1 << 64) - 1), index)


def shuffle136(key: int, counter: int = 0) -> tuple[list[int], int]:
    out = (C.c_uint8 * 136)()
    c = C.c_uint64()
    lib().orc_shuffle136(key, counter, out, C.byref(c))
    return list(out), c.value


def tables_crc() -> int:
    return lib().orc_tables_crc()


def tables_blob() -> bytes:
    L = lib()
    n = L.orc_tables_blob(None, 0)
    buf = (C.c_uint8 * n)()
    L.orc_tables_blob(buf, n)
    return bytes(buf)


def _counts_buf(counts):
    return (C.c_uint8 * 34)(*[int(c) for c in counts])


def shanten(counts, melds: int = 0) -> int:
    return lib().orc_shanten(_counts_buf(counts), melds)


def waits(counts, melds: int = 0) -> tuple[int, ...]:
    m = lib().orc_waits(_counts_buf(counts), melds)
    return tuple(k for k in range(34) if (m >> k) & 1)


def decompose(counts, melds: int = 0) -> list[tuple[int, tuple[tuple[str, int], ...]]]:
    out = (C.c_int32 * 1024)()
    n = lib().orc_decompose(_counts_buf(counts), melds, out, 1024)
    res, p, need = [], 0, 4 - melds
    for _ in range(n):
        pair = out[p]
        sets = tuple(("triplet" if k >= 64 else "run", k & 63) for k in out[p + 1:p + 1 + need])
        res.append((pair, sets))
        p += 1 + need
    return res


def run_shard(config: abi.rs_config, seed: int, idx0: int, n: int, steps: int,
              policy: str = "random", digests: bool = False):
    d = (C.c_uint64 * n)() if digests else None
    games = lib().orc_run_shard(C.byref(config), seed, idx0, n, steps,
                                0 if policy == "random" else 1, d)
    return games, (list(d) if digests else None)


def score(ctx: orc_winctx):
    w = abi.rs_win_rec()
    order = (C.c_int8 * 48)()
    norder = C.c_int32()
    ok = lib().orc_score_win(C.byref(ctx), C.byref(w), order, C.byref(norder))
    if not ok:
        return None
    return w, [int(order[i]) for i in range(norder.value)]


class OracleBatch:
    """Persistent shard [idx0, idx0+n) of bench-seeded envs (CPU baseline)."""

    def __init__(self, config: abi.rs_config, seed: int, idx0: int, n: int):
        self._L = lib()
        self.config = config
        self._p = self._L.orc_batch_new(C.byref(config), seed, idx0, n)

    def step(self, steps: int = 1, observe: bool = True) -> int:
        return self._L.orc_batch_step(self._p, steps, 1 if observe else 0)

    def __del__(self):
        try:
            self._L.orc_batch_free(self._p)
        except Exception:
            pass
