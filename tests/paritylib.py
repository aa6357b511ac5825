"""Shared helpers of the parity tests: projections of records compared
field by field between the CUDA path and the CPU oracle."""

from __future__ import annotations

from paper_2605_20577_b200 import records


def projection(rec) -> dict:
    """Everything a record says about the state, excluding the full event /
    result history (compared through the 64-event window and the last
    result; full histories are compared by the fingerprint tests)."""
    d = records.serialize_state(rec, [], [], None)
    d.pop("events")
    d.pop("results")
    d["internal"] = records.internal_fields(rec)
    d["window"] = records.window_events(rec)
    d["last_result"] = records.result_dict(rec.last_result) if rec.n_results else None
    return d


def diff(a: dict, b: dict, path: str = "") -> list[str]:
    out = []
    for k in sorted(set(a) | set(b)):
        va, vb = a.get(k), b.get(k)
        if isinstance(va, dict) and isinstance(vb, dict):
            out += diff(va, vb, f"{path}{k}.")
        elif va != vb:
            out.append(f"{path}{k}: {str(va)[:200]} != {str(vb)[:200]}")
    return out


def record_from_dict(d: dict):
    """rs_env_rec from the JSON dict of tests/golden/make_golden.state_record"""
    from paper_2605_20577_b200 import abi

    r = abi.rs_env_rec()
    r.abi_version = 1
    for k, v in d["cfg"].items():
        setattr(r.cfg, k, v)
    for i, t in enumerate(d["wall"]):
        r.wall[i] = t
    for s, h in enumerate(d["hands"]):
        hr = r.hands[s]
        for i, t in enumerate(h["concealed"]):
            hr.concealed[i] = t
        hr.n_concealed, hr.n_melds = h["n_concealed"], h["n_melds"]
        for i, m in enumerate(h["melds"]):
            mr = hr.melds[i]
            mr.type, mr.n_tiles, mr.from_seat, mr.called_tile = m["type"], m["n_tiles"], m["from_seat"], m["called_tile"]
            for j, t in enumerate(m["tiles"]):
                mr.tiles[j] = t
        for i, (t, f) in enumerate(zip(h["river_tile"], h["river_flags"])):
            hr.river_tile[i], hr.river_flags[i] = t, f
        hr.n_river = h["n_river"]
        for k in ("riichi", "riichi_index", "ippatsu", "temp_furiten", "perm_furiten", "shanten", "waits"):
            setattr(hr, k, h[k])
    for k in ("cursor", "kan_draws", "dora_count", "kyoku", "honba", "deposits", "repeats", "phase", "actor",
              "drawn", "riichi_pending", "rinshan_pending", "call_tile", "call_from", "n_queue", "n_rons",
              "call_chankan", "kakan_kind", "pending_dora", "four_kan_pending", "any_call_made", "rng_key",
              "rng_counter", "step_count", "terminated", "truncated", "events_len", "n_results", "current_player",
              "env_terminated", "env_truncated"):
        setattr(r, k, d[k])
    for i, v in enumerate(d["scores"]):
        r.scores[i] = v
    for i, (s, t) in enumerate(zip(d["queue_seat"], d["queue_stage"])):
        r.queue_seat[i], r.queue_stage[i] = s, t
    for i, s in enumerate(d["rons"]):
        r.rons[i] = s
    for i, ev in enumerate(d["events"]):
        for j in range(3):
            r.events[i][j] = ev[j]
    for i, w in enumerate(d["legal_mask"]):
        r.legal_mask[i] = w
    return r


def normalize(d: dict) -> dict:
    """JSON round trip (tuples -> lists) and rewards as float32 values"""
    import json
    import struct

    d = json.loads(json.dumps(d))
    if d and "internal" in d:
        d["internal"]["rewards"] = [struct.unpack("f", struct.pack("f", x))[0] for x in d["internal"]["rewards"]]
    return d


def ctx_from_json(c, kazoe, dy):
    """abi.rs_winctx (= the oracle's orc_winctx) from a scoring fixture's
    context (tests/golden/make_golden.ctx_to_json)"""
    from paper_2605_20577_b200 import abi

    x = abi.rs_winctx()
    for k in range(34):
        x.concealed[k] = c["concealed"][k]
    x.n_melds = len(c["melds"])
    for i, (typ, tiles, called, frm) in enumerate(c["melds"]):
        m = x.melds[i]
        m.type, m.n_tiles, m.from_seat = typ, len(tiles), frm
        for j, t in enumerate(tiles):
            m.tiles[j] = t
        m.called_tile = called
    x.win_tile = c["win_tile"]
    x.tsumo = int(c["tsumo"])
    x.seat_wind, x.round_wind = c["seat_wind"], c["round_wind"]
    x.n_ids = len(c["ids"])
    for i, t in enumerate(c["ids"]):
        x.ids[i] = t
    x.riichi, x.ippatsu = c["riichi"], int(c["ippatsu"])
    x.last_tile, x.rinshan, x.chankan, x.first_draw = (int(c[k]) for k in ("last_tile", "rinshan", "chankan", "first_draw"))
    x.n_dora = len(c["dora"])
    for i, t in enumerate(c["dora"]):
        x.dora[i] = t
    x.n_ura = len(c["ura"])
    for i, t in enumerate(c["ura"]):
        x.ura[i] = t
    x.rule = c["rule"]
    x.kazoe, x.double_yakuman = int(kazoe), int(dy)
    return x
