"""Loader of the in-tree sm_100a library `_rinshan.so` (C ABI: include/rinshan.h).

There is no fallback: if the library is missing or cannot be loaded the
import of the batched API fails loudly.  `build()` compiles it with nvcc
(cross-compiles without a GPU).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from pathlib import Path

from . import abi

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("RINSHAN_LIB", PKG_DIR / "_rinshan.so"))  # override: build experiments
CSRC = PKG_DIR / "csrc"
INCLUDE = PKG_DIR.parent / "include" / "rinshan.h"

# every entry point declared in include/rinshan.h (tests/test_abi.py checks
# this list against the header and the shared object)
SYMBOLS = (
    "rs_last_error", "rs_abi_version", "rs_tables_build", "rs_tables_load", "rs_tables_blob",
    "rs_tables_crc", "rs_tables_info", "rs_tables_shanten_std", "rs_create", "rs_destroy",
    "rs_num_envs", "rs_state_bytes", "rs_init", "rs_init_indexed", "rs_step", "rs_step_ex", "rs_step_rec_out",
    "rs_observe",
    "rs_policy_random", "rs_policy_heuristic", "rs_rollout", "rs_rollout_policy", "rs_autoreset", "rs_check_invariants", "rs_export_env", "rs_export_envs", "rs_import_env", "rs_record_sizes", "rs_debug_rollout_cycles",
    "rs_debug_score", "rs_set_done_flag", "rs_signal_done",
)

_lib = None
_lock = threading.Lock()


class RinshanError(RuntimeError):
    pass


def _stale() -> bool:
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    srcs = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.cpp")) + \
        list(CSRC.glob("*.h")) + [INCLUDE]
    return any(s.stat().st_mtime > t for s in srcs)


def build(force: bool = False) -> Path:
    """nvcc -gencode arch=compute_100a,code=sm_100a ... -> _rinshan.so"""
    if force or _stale():
        subprocess.check_call(["make", "-s", "-C", str(CSRC)])
    return LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            if os.environ.get("RINSHAN_NO_BUILD"):
                raise RinshanError(f"{LIB_PATH} missing (set up with paper_2605_20577_b200._lib.build())")
            build()
        L = C.CDLL(str(LIB_PATH))
        vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
        L.rs_last_error.restype = C.c_char_p
        L.rs_abi_version.restype = C.c_int
        L.rs_tables_build.restype = C.c_int
        L.rs_tables_load.argtypes = [vp, i64]
        L.rs_tables_blob.argtypes = [vp, i64, vp]
        L.rs_tables_crc.argtypes = [vp]
        L.rs_tables_info.argtypes = [vp, vp, vp, vp]
        L.rs_tables_shanten_std.argtypes = [C.c_uint32] * 4 + [i32, vp]
        L.rs_create.argtypes = [vp, i64, vp, i32]
        L.rs_destroy.argtypes = [vp]
        L.rs_num_envs.restype = i64
        L.rs_num_envs.argtypes = [vp]
        L.rs_state_bytes.restype = i64
        L.rs_state_bytes.argtypes = [vp]
        L.rs_init.argtypes = [vp, vp, vp, vp]
        L.rs_init_indexed.argtypes = [vp, u64, i64, vp, vp]
        L.rs_step.argtypes = [vp, vp, vp, vp]
        L.rs_step_ex.argtypes = [vp, vp, i32, vp, vp, vp, vp]
        L.rs_step_rec_out.argtypes = [vp, vp, i32, vp, vp, vp, vp]
        L.rs_observe.argtypes = [vp, vp, vp, vp]
        L.rs_policy_random.argtypes = [vp, vp, vp]
        L.rs_rollout.argtypes = [vp, i32, vp, i32, vp, vp, vp, vp, vp]
        L.rs_rollout_policy.argtypes = [vp, i32, i32, vp, i32, vp, vp, vp, vp, vp, vp, vp]
        L.rs_policy_heuristic.argtypes = [vp, vp, vp]
        L.rs_autoreset.argtypes = [vp, vp, vp]
        L.rs_check_invariants.argtypes = [vp, i32, vp, vp]
        L.rs_export_env.argtypes = [vp, i64, vp]
        L.rs_export_envs.argtypes = [vp, vp, i64, vp]
        L.rs_import_env.argtypes = [vp, i64, vp]
        L.rs_record_sizes.argtypes = [vp]
        L.rs_debug_rollout_cycles.argtypes = [vp, i32, vp, vp, vp]
        if hasattr(L, "rs_set_done_flag"):
            L.rs_set_done_flag.argtypes = [vp, vp]
            L.rs_signal_done.argtypes = [vp, vp]
        if hasattr(L, "rs_debug_score"):  # (A/B builds of older sources lack it)
            L.rs_debug_score.argtypes = [vp, i64, vp, vp, i32]
        if L.rs_abi_version() != 1:
            raise RinshanError("ABI version mismatch between _rinshan.so and the Python layer")
        _lib = L
        return L


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = _lib.rs_last_error().decode() if _lib is not None else ""
        raise RinshanError(f"{what} failed ({rc}): {msg}")


def record_sizes() -> list[int]:
    out = (C.c_int32 * 7)()
    check(lib().rs_record_sizes(out), "rs_record_sizes")
    return list(out)


def ctypes_record_sizes() -> list[int]:
    return [C.sizeof(t) for t in (abi.rs_config, abi.rs_meld_rec, abi.rs_hand_rec,
                                  abi.rs_win_rec, abi.rs_result_rec, abi.rs_env_rec, abi.rs_step_rec)]


def debug_score(ctxs, device: int = 0) -> list:
    """score_win (scoring/score.py:45-82) of abi.rs_winctx contexts on the
    device (rs_debug_score): a list of abi.rs_win_rec, None where the
    reference raises NoYakuError."""
    n = len(ctxs)
    arr = (abi.rs_winctx * max(n, 1))(*ctxs)
    out = (abi.rs_win_rec * max(n, 1))()
    ok = (C.c_int32 * max(n, 1))()
    check(lib().rs_debug_score(arr, n, out, ok, device), "rs_debug_score")
    return [out[i] if ok[i] else None for i in range(n)]
