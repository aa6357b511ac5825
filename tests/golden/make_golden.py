#!/usr/bin/env python
"""Generate golden fixtures from the Python reference (`mjsim`).

Run in the build container, where the reference is importable from
/root/reference (it is NOT on the GPU box):

    python tests/golden/make_golden.py

Writes small, deterministic JSON(.gz) files next to this script:
  rng.json          SplitMix64 mixer, key derivation, bench seeding, walls
  tables.json       suit-table blob CRC / sha256 and sampled value rows
  shanten.json.gz   random hands (with melds) -> shanten, waits
  scoring.json.gz   the reference's 38 GOLDEN_CASES + random wins -> score_win
  traces.json.gz    full games (random / heuristic policies, both rules, all
                    modes): per step the action, legal ids, current player,
                    rewards and the sha256 state fingerprint prefix
                    (engine/state.py:276-278) and observation digest
"""

from __future__ import annotations

import gzip
import hashlib
import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import refbridge  # noqa: E402

mjsim = refbridge.load()
sys.path.insert(0, str(refbridge.REF_SRC.parent / "tests"))

from mjsim import rng as R  # noqa: E402
from mjsim import tiles  # noqa: E402
from mjsim.bench.runner import env_game_seed, env_policy_state  # noqa: E402
from mjsim.engine import state_fingerprint  # noqa: E402
from mjsim.env import EnvConfig, heuristic_policy, init, observe, random_policy, step  # noqa: E402
from mjsim.hand import shanten as hshanten  # noqa: E402
from mjsim.hand import waits as hwaits  # noqa: E402
from mjsim.hand.tables import get_tables, save_tables  # noqa: E402
from mjsim.melds import CHI, KAN_CLOSED, KAN_OPEN, PON, Meld  # noqa: E402
from mjsim.scoring import NoYakuError, WinContext, score_win  # noqa: E402


def dump(name, obj):
    data = json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()
    path = HERE / name
    if name.endswith(".gz"):
        with gzip.GzipFile(path, "wb", mtime=0) as f:
            f.write(data)
    else:
        path.write_bytes(data)
    print(f"{name}: {len(data)} bytes")


def make_rng():
    xs = [0, 1, 2, 3, 12345, (1 << 63) + 7, (1 << 64) - 1] + [random.Random(1).getrandbits(64) for _ in range(8)]
    out = {
        "mix": [[x, R._mix(x)] for x in xs],
        "derive_key": [[a, b, R.derive_key(a, b)] for a in xs[:6] for b in (0, 1, 2, 99)],
        "env_game_seed": [[s, i, r, env_game_seed(s, i, r)] for s in (0, 7, 12345) for i in (0, 1, 4095)
                          for r in (0, 1, 5)],
        "env_policy_key": [[s, i, env_policy_state(s, i).key] for s in (0, 7, 12345) for i in (0, 1, 4095)],
        "walls": [],
    }
    for seed in (0, 1, 42, 999):
        wall, st = tiles.new_wall(R.seed_state(seed))
        out["walls"].append([seed, list(wall.tiles), st.counter])
    dump("rng.json", out)


def make_tables():
    t = get_tables()
    tmp = Path("/tmp/_golden_tables.bin")
    save_tables(t, tmp)
    blob = tmp.read_bytes()
    rnd = random.Random(3)
    rows = []
    for _ in range(300):
        code = rnd.randrange(5 ** 9)
        rows.append(["suit", code, [int(v) for v in t.suit_vals[code]]])
    for _ in range(100):
        code = rnd.randrange(5 ** 7)
        rows.append(["honor", code, [int(v) for v in t.honor_vals[code]]])
    dump("tables.json", {"crc32": int.from_bytes(blob[16:20], "little"), "size": len(blob),
                         "sha256": hashlib.sha256(blob).hexdigest(), "rows": rows})


def random_hand(rnd, size):
    counts = [0] * 34
    n = 0
    while n < size:
        k = rnd.randrange(34)
        if rnd.random() < 0.5 and n + 3 <= size and k < 27 and k % 9 <= 6:
            ks = [k, k + 1, k + 2]
        elif rnd.random() < 0.3 and n + 2 <= size:
            ks = [k, k]
        else:
            ks = [k]
        if all(counts[x] + ks.count(x) <= 4 for x in ks):
            for x in ks:
                counts[x] += 1
            n += len(ks)
    return counts


def make_shanten():
    rnd = random.Random(11)
    cases = []
    for i in range(3000):
        melds = rnd.choice([0, 0, 0, 1, 2, 3, 4])
        size = (14 if i % 2 else 13) - 3 * melds
        c = random_hand(rnd, size)
        w = list(hwaits(c, melds)) if size + 3 * melds == 13 else None
        cases.append([c, melds, hshanten(c, melds), w])
    dump("shanten.json.gz", cases)


def meld_obj(kind, typ, rnd):
    if typ == CHI:
        tiles_ = tuple(4 * (kind + i) + rnd.randrange(4) for i in range(3))
        return Meld(CHI, tuple(sorted(tiles_)), tiles_[rnd.randrange(3)], rnd.randrange(4))
    n = 3 if typ == PON else 4
    copies = sorted(rnd.sample(range(4), n))
    ts = tuple(4 * kind + c for c in copies)
    if typ == KAN_CLOSED:
        return Meld(KAN_CLOSED, ts)
    return Meld(typ, ts, ts[0], rnd.randrange(4))


def ctx_to_json(ctx):
    return {
        "concealed": list(ctx.concealed),
        "melds": [[m.type, list(m.tiles), m.called_tile, m.from_seat] for m in ctx.melds],
        "win_tile": ctx.win_tile, "tsumo": ctx.win_type == "tsumo", "seat_wind": ctx.seat_wind,
        "round_wind": ctx.round_wind, "ids": list(ctx.all_tile_ids), "riichi": ctx.riichi,
        "ippatsu": ctx.ippatsu, "last_tile": ctx.is_last_tile, "rinshan": ctx.is_rinshan,
        "chankan": ctx.is_chankan, "first_draw": ctx.is_first_uninterrupted_draw,
        "dora": list(ctx.dora_indicators), "ura": list(ctx.ura_indicators), "rule": ctx.rule,
    }


def score_json(ctx, kazoe=False, dy=False):
    try:
        ws = score_win(ctx, kazoe, dy)
    except NoYakuError:
        return None
    return {"yaku": [list(e) for e in ws.yaku.entries], "yakuman": ws.yaku.yakuman_count, "han": ws.han,
            "fu": ws.fu, "base": ws.base, "dora": ws.dora, "ura": ws.ura, "reds": ws.reds, "form": ws.form}


def make_scoring():
    import test_scoring as TS  # the reference's own golden cases

    cases = []
    for hand, win, wtype, melds, kw, _ in TS.GOLDEN_CASES:
        ctx = TS.make_ctx(hand, win, wtype, melds=melds, **kw)
        cases.append({"ctx": ctx_to_json(ctx), "kazoe": False, "dy": False, "want": score_json(ctx)})
    rnd = random.Random(0xFEED)
    made = 0
    while made < 600:
        m = TS._random_win(rnd)
        if m is None:
            continue
        ctx, _ = m
        kz, dy = rnd.random() < 0.2, rnd.random() < 0.3
        cases.append({"ctx": ctx_to_json(ctx), "kazoe": kz, "dy": dy, "want": score_json(ctx, kz, dy)})
        made += 1
    # closed kans / open kans / reds in melds, seven pairs, kokushi shapes
    while made < 900:
        counts = [0] * 34
        melds = []
        for _ in range(rnd.randint(0, 2)):
            k = rnd.randrange(34)
            typ = rnd.choice([PON, KAN_OPEN, KAN_CLOSED, CHI])
            if typ == CHI:
                if k >= 27 or k % 9 > 6:
                    continue
            melds.append(meld_obj(k, typ, rnd))
        used = [t for mm in melds for t in mm.tiles]
        if len(set(used)) != len(used):
            continue
        need = 14 - 3 * len(melds)
        c = random_hand(rnd, need)
        if any(c[t >> 2] + sum(1 for u in used if u >> 2 == t >> 2) > 4 for t in used):
            continue
        if hshanten(c, len(melds)) != -1:
            continue
        ids = []
        avail = {k: [4 * k + j for j in range(4) if 4 * k + j not in used] for k in range(34)}
        ok = True
        for k in range(34):
            if c[k] > len(avail[k]):
                ok = False
                break
            rnd.shuffle(avail[k])
            ids += avail[k][:c[k]]
        if not ok:
            continue
        win = rnd.choice(ids)
        riichi = rnd.choice([0, 1, 2]) if all(mm.type == KAN_CLOSED for mm in melds) else 0
        ctx = WinContext(
            concealed=bytes(c), melds=tuple(melds), win_tile=win, win_type=rnd.choice(["tsumo", "ron"]),
            seat_wind=27 + rnd.randrange(4), round_wind=rnd.choice([27, 28]), all_tile_ids=tuple(ids + used),
            riichi=riichi, ippatsu=bool(riichi and rnd.random() < 0.5), is_last_tile=rnd.random() < 0.1,
            is_rinshan=False, is_chankan=False, is_first_uninterrupted_draw=rnd.random() < 0.05,
            dora_indicators=tuple(rnd.randrange(136) for _ in range(rnd.randint(1, 5))),
            ura_indicators=tuple(rnd.randrange(136) for _ in range(rnd.randint(1, 5))) if riichi else (),
            rule=rnd.choice([0, 1]))
        kz, dy = rnd.random() < 0.2, rnd.random() < 0.3
        cases.append({"ctx": ctx_to_json(ctx), "kazoe": kz, "dy": dy, "want": score_json(ctx, kz, dy)})
        made += 1
    dump("scoring.json.gz", cases)


def obs_digest(o) -> str:
    return hashlib.sha256(json.dumps(o.to_dict(), sort_keys=True).encode()).hexdigest()[:16]


def play(rule, mode, seed, index, policy):
    cfg = EnvConfig(rule=rule, mode=mode)
    st = init(env_game_seed(seed, index), cfg)
    pol = env_policy_state(seed, index)
    rows = []
    while True:
        rows.append([state_fingerprint(st.game)[:16], obs_digest(observe(st, st.current_player)),
                     st.current_player, list(st.legal), [round(x, 9) for x in st.rewards],
                     int(st.terminated), int(st.truncated)])
        if st.terminated or st.truncated:
            break
        if policy == "random":
            a, pol = random_policy(st.legal, pol)
        else:
            a = heuristic_policy(observe(st, st.current_player), st.legal)
        rows[-1].append(a)
        st = step(st, a)
    return {"rule": rule, "mode": mode, "seed": seed, "index": index, "policy": policy, "steps": rows}


def make_traces():
    games = []
    for rule in ("no-red", "red"):
        for i in range(24):
            games.append(play(rule, "single", 0, i, "random"))
        for i in range(24):
            games.append(play(rule, "single", 1, i, "heuristic"))
        for i in range(2):
            games.append(play(rule, "east", 2, i, "heuristic"))
            games.append(play(rule, "half", 3, i, "random"))
    dump("traces.json.gz", games)


if __name__ == "__main__":
    make_rng()
    make_tables()
    make_shanten()
    make_scoring()
    make_traces()
