"""ctypes mirrors of the C ABI records in include/rinshan.h.

The layouts here must match the header byte for byte; tests/test_abi.py
checks the sizes against the compiled library (rs_record_sizes).
"""

from __future__ import annotations

import ctypes as C

NUM_TILES = 136
NUM_KINDS = 34
NUM_ACTIONS = 115
EVENT_WINDOW = 64
MAX_RIVER = 40
MAX_QUEUE = 8

RULE_RED = 0
RULE_NO_RED = 1
MODE_SINGLE = 0
MODE_EAST = 1
MODE_HALF = 2
REWARD_SCORE_DELTA = 0
REWARD_RANK = 1

STATUS_ILLEGAL = 1
STATUS_CONTRACT = 2
# river flags (include/rinshan.h RS_RIVER_*)
RIVER_TSUMOGIRI = 1
RIVER_RIICHI = 2
RIVER_CALLED = 4
STATUS_INVARIANT = 4
ACTION_SKIP = -(1 << 31)  # RS_ACTION_SKIP: the env is not stepped
# rs_step_ex / rs_step_rec_out flags
STEP_AUTORESET = 1
STEP_OBSERVE = 2
STEP_HEURISTIC = 4
STEP_SIGNAL = 8
STEP_RESET_FIRST = 16

# status returns (include/rinshan.h; positive values are cudaError_t)
RS_E_ARG = -1
RS_E_TABLES = -2
RS_E_STATE = -3
RS_E_CORRUPT = -4
# rs_check_invariants bits (include/rinshan.h RS_INV_*)
INV_SCORE_SUM = 1
INV_TILES = 2
INV_EMPTY_LEGAL = 4
INV_TERMINAL_LEGAL = 8
INV_FURITEN_RON = 16
INV_HAND_SYNC = 32
INV_HAND_SIZE = 64
INV_RIICHI_NOT_TENPAI = 128

RES_KINDS = ("tsumo", "ron", "exhaustive", "abort_nine_terminals",
             "abort_triple_ron", "abort_four_riichi", "abort_four_kan")
FORMS = ("standard", "seven_pairs", "kokushi")


class rs_config(C.Structure):
    _fields_ = [
        ("rule", C.c_int32),
        ("mode", C.c_int32),
        ("reward_scheme", C.c_int32),
        ("illegal_penalty", C.c_float),
        ("max_steps", C.c_int32),
        ("kazoe", C.c_int32),
        ("double_yakuman", C.c_int32),
        ("agari_yame", C.c_int32),
        ("renchan_cap", C.c_int32),
    ]


class rs_meld_rec(C.Structure):
    _fields_ = [
        ("type", C.c_int8),
        ("n_tiles", C.c_int8),
        ("from_seat", C.c_int8),
        ("pad0", C.c_int8),
        ("tiles", C.c_uint8 * 4),
        ("called_tile", C.c_int16),
        ("pad1", C.c_int16),
    ]


class rs_hand_rec(C.Structure):
    _fields_ = [
        ("concealed", C.c_uint8 * 14),
        ("n_concealed", C.c_uint8),
        ("n_melds", C.c_uint8),
        ("melds", rs_meld_rec * 4),
        ("river_tile", C.c_uint8 * MAX_RIVER),
        ("river_flags", C.c_uint8 * MAX_RIVER),
        ("n_river", C.c_int32),
        ("riichi", C.c_int8),
        ("riichi_index", C.c_int8),
        ("ippatsu", C.c_int8),
        ("temp_furiten", C.c_int8),
        ("perm_furiten", C.c_int8),
        ("shanten", C.c_int8),
        ("pad", C.c_int16),
        ("waits", C.c_uint64),
    ]


class rs_win_rec(C.Structure):
    _fields_ = [
        ("yaku_han", C.c_int8 * 40),
        ("yakuman", C.c_int32),
        ("han", C.c_int32),
        ("fu", C.c_int32),
        ("base", C.c_int32),
        ("dora", C.c_int32),
        ("ura", C.c_int32),
        ("reds", C.c_int32),
        ("form", C.c_int32),
    ]


class rs_winctx(C.Structure):
    """include/rinshan.h rs_winctx: WinContext (scoring/context.py:19-57)"""
    _fields_ = [
        ("concealed", C.c_uint8 * 34),
        ("n_melds", C.c_int32),
        ("melds", rs_meld_rec * 4),
        ("win_tile", C.c_int32),
        ("tsumo", C.c_int32),
        ("seat_wind", C.c_int32),
        ("round_wind", C.c_int32),
        ("n_ids", C.c_int32),
        ("ids", C.c_uint8 * 18),
        ("riichi", C.c_int32),
        ("ippatsu", C.c_int32),
        ("last_tile", C.c_int32),
        ("rinshan", C.c_int32),
        ("chankan", C.c_int32),
        ("first_draw", C.c_int32),
        ("n_dora", C.c_int32),
        ("dora", C.c_uint8 * 5),
        ("n_ura", C.c_int32),
        ("ura", C.c_uint8 * 5),
        ("rule", C.c_int32),
        ("kazoe", C.c_int32),
        ("double_yakuman", C.c_int32),
    ]


class rs_result_rec(C.Structure):
    _fields_ = [
        ("kyoku", C.c_int32),
        ("honba", C.c_int32),
        ("kind", C.c_int32),
        ("n_winners", C.c_int32),
        ("winners", C.c_int8 * 4),
        ("loser", C.c_int32),
        ("n_settlements", C.c_int32),
        ("deltas", (C.c_int32 * 4) * 3),
        ("honba_component", C.c_int32 * 3),
        ("deposits_claimed", C.c_int32 * 3),
        ("wins", rs_win_rec * 3),
        ("tenpai_mask", C.c_int32),
        ("scores_after", C.c_int32 * 4),
    ]


class rs_step_rec(C.Structure):
    """include/rinshan.h rs_step_rec (40 bytes)"""
    _fields_ = [
        ("rewards", C.c_float * 4),
        ("legal_bits", C.c_uint32 * 4),
        ("next_action", C.c_int32),
        ("current_player", C.c_int8),
        ("terminated", C.c_uint8),
        ("truncated", C.c_uint8),
        ("status", C.c_uint8),
    ]


class rs_env_rec(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int32),
        ("cfg", rs_config),
        ("wall", C.c_uint8 * NUM_TILES),
        ("cursor", C.c_int32),
        ("kan_draws", C.c_int32),
        ("dora_count", C.c_int32),
        ("hands", rs_hand_rec * 4),
        ("scores", C.c_int32 * 4),
        ("kyoku", C.c_int32),
        ("honba", C.c_int32),
        ("deposits", C.c_int32),
        ("repeats", C.c_int32),
        ("phase", C.c_int32),
        ("actor", C.c_int32),
        ("drawn", C.c_int32),
        ("riichi_pending", C.c_int32),
        ("rinshan_pending", C.c_int32),
        ("call_tile", C.c_int32),
        ("call_from", C.c_int32),
        ("n_queue", C.c_int32),
        ("queue_seat", C.c_int8 * MAX_QUEUE),
        ("queue_stage", C.c_int8 * MAX_QUEUE),
        ("n_rons", C.c_int32),
        ("rons", C.c_int8 * 4),
        ("call_chankan", C.c_int32),
        ("kakan_kind", C.c_int32),
        ("pending_dora", C.c_int32),
        ("four_kan_pending", C.c_int32),
        ("any_call_made", C.c_int32),
        ("rng_key", C.c_uint64),
        ("rng_counter", C.c_uint64),
        ("step_count", C.c_int32),
        ("terminated", C.c_int32),
        ("truncated", C.c_int32),
        ("events_len", C.c_int32),
        ("events", (C.c_int16 * 3) * EVENT_WINDOW),
        ("n_results", C.c_int32),
        ("last_result", rs_result_rec),
        ("legal_mask", C.c_uint32 * 4),
        ("current_player", C.c_int32),
        ("env_terminated", C.c_int32),
        ("env_truncated", C.c_int32),
        ("status", C.c_int32),
        ("rewards", C.c_float * 4),
        ("env_key", C.c_uint64),
        ("policy_key", C.c_uint64),
        ("policy_counter", C.c_uint64),
        ("resets", C.c_int32),
        ("pad", C.c_int32),
    ]


class rs_step_out(C.Structure):
    _fields_ = [
        ("legal_mask", C.c_void_p),
        ("legal_bits", C.c_void_p),
        ("current_player", C.c_void_p),
        ("rewards", C.c_void_p),
        ("terminated", C.c_void_p),
        ("truncated", C.c_void_p),
        ("status", C.c_void_p),
    ]


class rs_obs_out(C.Structure):
    _fields_ = [
        ("hand_tokens", C.c_void_p),
        ("event_tokens", C.c_void_p),
        ("shanten", C.c_void_p),
        ("scores", C.c_void_p),
        ("round_wind", C.c_void_p),
        ("seat_wind", C.c_void_p),
        ("kyoku", C.c_void_p),
        ("honba", C.c_void_p),
        ("deposits", C.c_void_p),
        ("dora_tokens", C.c_void_p),
        ("live_wall", C.c_void_p),
        ("riichi_flags", C.c_void_p),
    ]


class rs_rollout_stats(C.Structure):
    _fields_ = [
        ("steps", C.c_uint64),
        ("games_completed", C.c_uint64),
        ("illegal", C.c_uint64),
    ]


def mask_to_ids(words) -> tuple[int, ...]:
    m = 0
    for i, w in enumerate(words):
        m |= (int(w) & 0xFFFFFFFF) << (32 * i)
    m &= (1 << NUM_ACTIONS) - 1
    out = []
    while m:
        low = m & -m
        out.append(low.bit_length() - 1)
        m ^= low
    return tuple(out)
