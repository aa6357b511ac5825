"""Host-side decoding of exported env records.

Turns an `rs_env_rec` (include/rinshan.h) plus the event/result history
collected while stepping into the reference's canonical JSON projection
(`serialize_state`, reference pkg/src/mjsim/engine/state.py:191-242 and
`_result_dict` :245-274) and its sha256 fingerprint (:276-278), so parity
can be asserted field by field against the reference.
"""

from __future__ import annotations

import hashlib
import json

from . import abi

EV_NAMES = ("draw", "discard", "chi", "pon", "kan_open", "kan_closed",
            "kan_added", "riichi", "ron", "tsumo", "draw_end", "new_dora")
MODE_NAMES = {0: "single", 1: "east", 2: "half"}
MELD_NAMES = {0: "chi", 1: "pon", 2: "kan_open", 3: "kan_closed", 4: "kan_added"}
_HONOR_LETTERS = "ESWNPFC"
RED_FIVE_TILES = (16, 52, 88)

# yaku entry order of the reference detectors (scoring/yaku.py):
# detect_standard appends regular yaku in ascending id order (yaku.py:239-300)
_STD_YAKUMAN_ORDER = (38, 39, 29, 30, 32, 31, 33, 34, 35, 37, 36)  # yaku.py:207-230
_SEVEN_PAIRS_ORDER = (0, 1, 2, 3, 19, 5, 20, 22, 23, 24, 25, 26, 27)  # yaku.py:353-369
_SEVEN_PAIRS_YAKUMAN_ORDER = (38, 39, 33)  # yaku.py:341-344
_KOKUSHI_ORDER = (38, 39, 28)  # yaku.py:376-379


def kind_name(kind: int) -> str:
    if kind < 27:
        return f"{kind % 9 + 1}{'mps'[kind // 9]}"
    return _HONOR_LETTERS[kind - 27]


def tile_name(tile: int, rule: int) -> str:
    """reference tiles.py:75-80"""
    k = tile >> 2
    if rule == abi.RULE_RED and tile in RED_FIVE_TILES:
        return f"0{'mps'[k // 9]}"
    return kind_name(k)


def yaku_entries(win) -> list[list[int]]:
    """(id, han) entries in the reference's detection order, rebuilt from a
    per-id han vector and the winning form."""
    han = [int(win.yaku_han[i]) for i in range(40)]
    form = int(win.form)
    if form == 2:
        order = _KOKUSHI_ORDER
    elif form == 1:
        order = _SEVEN_PAIRS_YAKUMAN_ORDER if win.yakuman else _SEVEN_PAIRS_ORDER
    else:
        order = _STD_YAKUMAN_ORDER if win.yakuman else tuple(range(28))
    return [[y, han[y]] for y in order if han[y]]


def result_dict(r) -> dict:
    """reference engine/state.py:245-274 (_result_dict)"""
    winners = [int(r.winners[i]) for i in range(r.n_winners)]
    tenpai = [s for s in range(4) if (r.tenpai_mask >> s) & 1]
    return {
        "kyoku": int(r.kyoku),
        "honba": int(r.honba),
        "kind": abi.RES_KINDS[r.kind],
        "winners": winners,
        "loser": int(r.loser),
        "tenpai": tenpai,
        "settlements": [
            {"deltas": [int(r.deltas[i][s]) for s in range(4)],
             "honba": int(r.honba_component[i]),
             "deposits": int(r.deposits_claimed[i])}
            for i in range(r.n_settlements)
        ],
        "win_details": [
            {
                "yaku": yaku_entries(w),
                "yakuman": int(w.yakuman),
                "han": int(w.han),
                "fu": int(w.fu),
                "base": int(w.base),
                "dora": int(w.dora),
                "ura": int(w.ura),
                "reds": int(w.reds),
                "form": abi.FORMS[w.form],
            }
            for w in (r.wins[i] for i in range(r.n_winners))
        ],
        "scores_after": [int(x) for x in r.scores_after],
    }


def _meld_dict(m, rule: int) -> dict:
    tiles = [int(m.tiles[i]) for i in range(m.n_tiles)]
    return {
        "type": MELD_NAMES[m.type],
        "tiles": [tile_name(t, rule) for t in tiles],
        "tile_ids": tiles,
        "called_tile": int(m.called_tile),
        "from_seat": int(m.from_seat),
    }


def game_legal(rec) -> list[int]:
    return list(abi.mask_to_ids(rec.legal_mask))


def serialize_state(rec, events, results, legal=None) -> dict:
    """reference engine/state.py:191-242.  `events` is the full
    chronological (type, actor, tile) list, `results` the full list of
    result dicts; `legal` overrides the record's env-view mask (the game
    keeps its cached list after an illegal env step)."""
    cfg = rec.cfg
    rule = cfg.rule
    dora = [tile_name(rec.wall[122 + 2 * i], rule) for i in range(rec.dora_count)]
    hands = []
    for s in range(4):
        h = rec.hands[s]
        conc = [int(h.concealed[i]) for i in range(h.n_concealed)]
        hands.append({
            "concealed": [tile_name(t, rule) for t in conc],
            "concealed_ids": conc,
            "melds": [_meld_dict(h.melds[i], rule) for i in range(h.n_melds)],
            "river": [
                {"tile": tile_name(h.river_tile[i], rule), "id": int(h.river_tile[i]),
                 "tsumogiri": bool(h.river_flags[i] & 1),
                 "riichi": bool(h.river_flags[i] & 2),
                 "called": bool(h.river_flags[i] & 4)}
                for i in range(h.n_river)
            ],
            "riichi": int(h.riichi),
            "ippatsu": bool(h.ippatsu),
            "shanten": int(h.shanten),
        })
    return {
        "config": {
            "rule": "no-red" if rule == abi.RULE_NO_RED else "red",
            "mode": MODE_NAMES[cfg.mode],
            "kazoe": bool(cfg.kazoe),
            "double_yakuman": bool(cfg.double_yakuman),
            "agari_yame": bool(cfg.agari_yame),
            "max_steps": int(cfg.max_steps),
        },
        "kyoku": int(rec.kyoku),
        "honba": int(rec.honba),
        "deposits": int(rec.deposits),
        "scores": [int(x) for x in rec.scores],
        "phase": int(rec.phase),
        "actor": int(rec.actor),
        "drawn": int(rec.drawn),
        "terminated": bool(rec.terminated),
        "truncated": bool(rec.truncated),
        "step_count": int(rec.step_count),
        "wall": {
            "tiles": [int(x) for x in rec.wall],
            "cursor": int(rec.cursor),
            "kan_draws": int(rec.kan_draws),
            "dora_count": int(rec.dora_count),
        },
        "dora_indicators": dora,
        "hands": hands,
        "events": [{"type": EV_NAMES[t], "actor": int(a), "tile": int(tile)} for t, a, tile in events],
        "results": list(results),
        "legal": list(legal) if legal is not None else game_legal(rec),
    }


def fingerprint(state_dict: dict) -> str:
    """reference engine/state.py:276-278"""
    blob = json.dumps(state_dict, sort_keys=True, separators=(",", ":"))
    return hashlib.sha256(blob.encode()).hexdigest()


def internal_fields(rec) -> dict:
    """Fields outside serialize_state that still define the transition
    (engine/types.py:124-158 + HandState flags): compared in parity too."""
    return {
        "repeats": int(rec.repeats),
        "riichi_pending": int(rec.riichi_pending),
        "rinshan_pending": int(rec.rinshan_pending),
        "call_tile": int(rec.call_tile),
        "call_from": int(rec.call_from),
        "queue": [(int(rec.queue_seat[i]), int(rec.queue_stage[i])) for i in range(rec.n_queue)],
        "rons": [int(rec.rons[i]) for i in range(rec.n_rons)],
        "call_chankan": int(rec.call_chankan),
        "kakan_kind": int(rec.kakan_kind),
        "pending_dora": int(rec.pending_dora),
        "four_kan_pending": int(rec.four_kan_pending),
        "any_call_made": int(rec.any_call_made),
        "rng": (int(rec.rng_key), int(rec.rng_counter)),
        "events_len": int(rec.events_len),
        "n_results": int(rec.n_results),
        "hands": [
            {
                "riichi_index": int(rec.hands[s].riichi_index),
                "temp_furiten": int(rec.hands[s].temp_furiten),
                "perm_furiten": int(rec.hands[s].perm_furiten),
                "waits": int(rec.hands[s].waits),
            }
            for s in range(4)
        ],
        "legal_mask": [int(x) for x in rec.legal_mask],
        "current_player": int(rec.current_player),
        "env_terminated": int(rec.env_terminated),
        "env_truncated": int(rec.env_truncated),
        "rewards": [float(x) for x in rec.rewards],
    }


def window_events(rec, last: int | None = None) -> list[tuple[int, int, int]]:
    """the events in the record's window (the `last` ones only, if given)"""
    n = min(int(rec.events_len), abi.EVENT_WINDOW)
    ev = rec.events
    return [(int(e[0]), int(e[1]), int(e[2])) for e in
            (ev[i] for i in range(n - min(n, last) if last is not None else 0, n))]
