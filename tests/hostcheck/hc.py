"""ctypes wrapper of the TEST-ONLY host build of the engine (hostcheck.cpp)."""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

from paper_2605_20577_b200 import abi

_HERE = Path(__file__).resolve().parent
_lib = None


def lib():
    global _lib
    if _lib is None:
        # HOSTCHECK_LIB: another build of the same source (the sanitized one,
        # tests/test_hostcheck_sanitized.py)
        name = os.environ.get("HOSTCHECK_LIB", "libhostcheck.so")
        subprocess.check_call(["make", "-s", "-C", str(_HERE), name])
        L = C.CDLL(str(_HERE / name))
        vp = C.c_void_p
        L.hc_create.restype = vp
        L.hc_create.argtypes = [C.c_int, vp]
        L.hc_free.argtypes = [vp]
        L.hc_init_indexed.argtypes = [vp, C.c_uint64, C.c_int64, vp]
        L.hc_init_seeds.argtypes = [vp, vp, vp]
        L.hc_step.argtypes = [vp, vp, vp, vp]
        L.hc_random_actions.argtypes = [vp, vp]
        L.hc_export.argtypes = [vp, C.c_int, vp]
        L.hc_import.argtypes = [vp, C.c_int, vp]
        L.hc_observe.argtypes = [vp, C.c_int, C.c_int] + [vp] * 8
        L.hc_rollout.restype = C.c_int64
        L.hc_rollout.argtypes = [vp, C.c_int, vp, vp, C.c_int]
        L.hc_check.restype = C.c_uint32
        L.hc_check.argtypes = [vp, C.c_int, C.c_int]
        _lib = L
    return _lib


class HostBatch:
    def __init__(self, n: int, cfg: abi.rs_config):
        self.L = lib()
        self.n = n
        self.cfg = cfg
        self.p = self.L.hc_create(n, C.byref(cfg))
        self.rewards = (C.c_float * (4 * n))()

    def __del__(self):
        try:
            self.L.hc_free(self.p)
        except Exception:
            pass

    def init_indexed(self, seed: int, base: int = 0):
        self.L.hc_init_indexed(self.p, seed, base, self.rewards)

    def init_seeds(self, seeds):
        arr = (C.c_uint64 * self.n)(*seeds)
        self.L.hc_init_seeds(self.p, arr, self.rewards)

    def step(self, actions):
        a = (C.c_int32 * self.n)(*actions)
        st = (C.c_uint8 * self.n)()
        self.L.hc_step(self.p, a, st, self.rewards)
        return list(st)

    def random_actions(self):
        a = (C.c_int32 * self.n)()
        self.L.hc_random_actions(self.p, a)
        return list(a)

    def record(self, e: int) -> abi.rs_env_rec:
        r = abi.rs_env_rec()
        self.L.hc_export(self.p, e, C.byref(r))
        return r

    def load(self, e: int, rec: abi.rs_env_rec):
        self.L.hc_import(self.p, e, C.byref(rec))

    def observe(self, e: int, seat: int) -> dict:
        hand = (C.c_uint8 * 14)(); ev = (C.c_uint8 * 192)(); sh = (C.c_int8 * 1)()
        sc = (C.c_int16 * 4)(); misc = (C.c_uint8 * 4)(); hd = (C.c_int16 * 2)()
        dora = (C.c_uint8 * 5)(); ri = (C.c_uint8 * 4)()
        self.L.hc_observe(self.p, e, seat, hand, ev, sh, sc, misc, hd, dora, ri)
        return {
            "hand_tokens": list(hand),
            "event_tokens": [list(ev[3 * i:3 * i + 3]) for i in range(64)],
            "shanten": sh[0],
            "scores": list(sc),
            "round_wind": misc[0],
            "seat_wind": misc[1],
            "kyoku": misc[2],
            "honba": hd[0],
            "deposits": hd[1],
            "dora_indicator_tokens": list(dora),
            "live_wall": misc[3],
            "riichi_flags": list(ri),
        }

    def check(self, e: int, fast: bool = False) -> int:
        return int(self.L.hc_check(self.p, e, 1 if fast else 0))

    def rollout(self, steps: int, digests=None, policy: str = "random"):
        d = (C.c_uint64 * self.n)(*(digests or [0] * self.n))
        log = (C.c_int16 * (steps * self.n))()
        games = self.L.hc_rollout(self.p, steps, d, log, 0 if policy == "random" else 1)
        return games, list(d), [list(log[t * self.n:(t + 1) * self.n]) for t in range(steps)]
