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
  scoring_rare.json.gz  yakuman / double-yakuman waits / kazoe hands under
                    every (kazoe, double_yakuman) flag pair -> score_win
  traces.json.gz    full games (random / heuristic policies, both rules, all
                    modes): per step the action, legal ids, current player,
                    rewards and the sha256 state fingerprint prefix
                    (engine/state.py:276-278) and observation digest
  wins.json.gz      tsumo / ron transitions of states crafted around the
                    scoring fixtures' hands (settlement + result record)
  logs.json.gz      mjlog-lite-v1 logs (engine/log.py) of the bench loop's
                    games, canonical JSON
  renders.json.gz   render/svg.py documents (sha256) of reference states
  cli.json.gz       cli.py selfplay logs and render SVGs (sha256), bench
                    rows' games_completed (bench/runner.py rollout)
  sessions.json.gz  service/sessions.py games (agents + a scripted human):
                    action lists, persisted documents, final fingerprints
                    and the service/app.py view documents (sha256)
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


# rare scoring branches the reference's fixtures above barely reach:
# counted yakuman (kazoe) and the double-yakuman waits, each under every
# (kazoe, double_yakuman) combination (engine/types.py:53-54)
RARE_HANDS = [
    # (concealed-13, win, type, melds, ctx kwargs)
    ("19m19p19s1234567z", "9m", "tsumo", (), {}),                      # kokushi 13-sided
    ("19m19p19s1234567z", "1z", "ron", (), {}),                        # kokushi 13-sided, ron
    ("119m19p19s123456z", "7z", "ron", (), {}),                        # kokushi single wait
    ("19m19p19s1234567z", "7z", "tsumo", (), {"seat_wind": 27, "is_first_uninterrupted_draw": True}),
    ("19m19p19s1234567z", "1m", "tsumo", (), {"seat_wind": 28, "is_first_uninterrupted_draw": True}),
    ("1112345678999m", "5m", "tsumo", (), {}),                          # chuuren 9-sided
    ("1112345678999p", "9p", "ron", (), {}),                            # chuuren 9-sided on a terminal
    ("1112345678999s", "1s", "tsumo", (), {"seat_wind": 27, "is_first_uninterrupted_draw": True}),
    ("1112345678899m", "9m", "ron", (), {}),                            # chuuren, not 9-sided
    ("111m999m111s999s1p", "1p", "tsumo", (), {}),                      # suuankou tanki
    ("111m999m111s999s1p", "1p", "ron", (), {}),                        # suuankou tanki, ron
    ("111m999m111s99s11p", "1p", "tsumo", (), {}),                      # suuankou shanpon
    ("111m999m111s99s11p", "9s", "ron", (), {}),                        # sanankou only (ron)
    ("111z222z333z444z5m", "5m", "ron", (), {}),                        # daisuushii + suuankou tanki
    ("111z222z333z44z55m", "5m", "tsumo", (), {}),                      # shousuushi + suuankou
    ("111z222z333z44z55m", "4z", "ron", (), {}),                        # daisuushii shanpon (ron)
    ("222z333z44z55m", "4z", "ron", ("pon", 27), {}),                   # daisuushii with a pon
    ("555z666z77z123m99p", "7z", "ron", (), {}),                        # daisangen
    ("111z222z555z66z77z", "7z", "tsumo", (), {}),                      # tsuuiisou + suuankou
    ("1122z3344z5566z7z", "7z", "ron", (), {}),                         # tsuuiisou seven pairs
    ("111m999m111p99p11s", "1s", "ron", (), {}),                        # chinroutou
    ("223344s666s888s6z", "6z", "tsumo", (), {}),                       # ryuuiisou
    ("2m", "2m", "tsumo", ("kans",), {}),                               # suukantsu
    ("123m456m789m11m23m", "4m", "tsumo", (),                           # kazoe: 13+ han
     {"riichi": 1, "ippatsu": True, "dora_indicators": (32, 33), "ura_indicators": (34,)}),
    ("123m456m789m11m23m", "4m", "ron", (),                             # 11-12 han
     {"riichi": 1, "dora_indicators": (32,)}),
    ("11223355577799p", "", "tsumo", (),                                # chinitsu seven pairs
     {"riichi": 2, "ippatsu": True, "dora_indicators": (4 * 9 + 3,)}),
    ("234m456p888s44m67p", "8p", "tsumo", (), {"seat_wind": 27, "is_first_uninterrupted_draw": True}),
    ("234m456p888s44m67p", "5p", "tsumo", (), {"seat_wind": 29, "is_first_uninterrupted_draw": True}),
    ("1122m4455p88s33z5z", "5z", "tsumo", (), {"seat_wind": 30, "is_first_uninterrupted_draw": True}),
    ("234m456p888s44m67p", "8p", "tsumo", (), {"is_rinshan": True, "dora_indicators": (0, 4, 8, 12, 16)}),
    ("234m456p888s44m67p", "8p", "ron", (), {"is_chankan": True, "is_last_tile": False}),
    ("234m456p888s44m67p", "8p", "ron", (), {"is_last_tile": True, "riichi": 2, "ippatsu": True}),
    ("123456789m1234p", "1p", "ron", (), {"rule": 1}),                # no-red rule
    ("234m406p888s44m67p", "8p", "tsumo", (), {"reds": (13,)}),       # red five held
    ("234m456p44m67p", "8p", "tsumo", ("ckan", 26), {"is_rinshan": True}),  # rinshan after a kan
    ("234m456p44m67p", "5p", "tsumo", ("ckan", 31), {"is_rinshan": True, "riichi": 1}),
]


def rare_ctx(hand, win, wtype, melds, kw):
    import test_scoring as TS
    from mjsim.melds import KAN_CLOSED as KC

    kw = dict(kw)
    reds = kw.pop("reds", ())
    ml = ()
    if melds and melds[0] == "pon":
        ml = (TS.pon(melds[1]),)
    elif melds and melds[0] == "ckan":
        ml = (TS.kan(melds[1], KC),)
    elif melds and melds[0] == "kans":
        ml = (TS.kan(4, KC), TS.kan(13, KC), TS.kan(22), TS.kan(31))
    if not win:  # 14-tile text: the last tile wins
        counts, _ = __import__("oracle").parse_hand(hand)
        win_kind = max(k for k in range(34) if counts[k])
        hand = hand  # keep the text; make_ctx adds the win kind, so drop it here
        digits = {"m": 0, "p": 9, "s": 18, "z": 27}
        suit = next(s for s, b in digits.items() if b <= win_kind < b + 9)
        win = f"{win_kind - digits[suit] + 1}{suit}"
        body, sfx = hand[:-1], hand[-1]
        i = body.rindex(win[0])
        hand = body[:i] + body[i + 1:] + sfx
    return TS.make_ctx(hand, win, wtype, melds=ml, reds=reds, **kw)


def make_scoring_rare():
    cases = []
    for hand, win, wtype, melds, kw in RARE_HANDS:
        ctx = rare_ctx(hand, win, wtype, melds, kw)
        for kz in (False, True):
            for dy in (False, True):
                cases.append({"ctx": ctx_to_json(ctx), "kazoe": kz, "dy": dy, "want": score_json(ctx, kz, dy)})
    dump("scoring_rare.json.gz", cases)


# wins through the engine: states crafted around the scoring fixtures'
# hands (winner, seat / round wind, melds, riichi / ippatsu, dora and ura
# indicators in the dead wall, haitei / houtei, rinshan, chankan, first
# draw, honba, deposits, kazoe / double-yakuman configs), then TSUMO on the
# winner's draw or RON on an opponent's discard / added kan, recorded like
# the scenarios above: (pre-state record, action, post-state projection |
# exception).  The post state carries the settled scores and the result
# record with the win details; in half mode the next kyoku is dealt.

def craft_win(c, kazoe, dy, rnd):
    """GameState for a fixture context (ctx_to_json form) or None"""
    from mjsim.engine.engine import _B, _finish
    from mjsim.engine.state import make_hand
    from mjsim.engine.types import MODE_HALF, PH_ACT, GameConfig, GameState, RiverTile
    from mjsim.melds import KAN_CLOSED as KC
    from mjsim.melds import PON as PN
    from mjsim.rng import seed_state
    from mjsim.tiles import Wall

    melds = [Meld(t, tuple(ts), cal, frm) for t, ts, cal, frm in c["melds"]]
    meld_ids = [t for m in melds for t in m.tiles]
    conc = [t for t in c["ids"] if t not in meld_ids]
    win = c["win_tile"]
    if win not in conc:
        same = [t for t in conc if t >> 2 == win >> 2]
        if not same or win in meld_ids:
            return None
        conc[conc.index(same[0])] = win
    tsumo = c["tsumo"]
    chankan, rinshan, last, first = c["chankan"], c["rinshan"], c["last_tile"], c["first_draw"]
    riichi = c["riichi"]
    kans = sum(1 for m in melds if m.type in (2, 3, 4))
    if rinshan and not kans:
        return None
    if first and (riichi or melds or not tsumo):
        return None
    if len(set(conc + meld_ids)) != len(conc) + len(meld_ids):
        return None
    kyoku = (c["round_wind"] - 27) * 4 + rnd.randrange(4)
    dealer = kyoku % 4
    winner = (dealer + c["seat_wind"] - 27) % 4
    # open melds were called from someone: chi from the left, others anyone
    melds = [m if m.type == KC else Meld(m.type, m.tiles, m.tiles[0] if m.called_tile < 0 else m.called_tile,
                                         (winner + 3) % 4 if m.type == 0 else (winner + 1 + rnd.randrange(3)) % 4)
             for m in melds]
    used = set(conc) | set(meld_ids)
    hands = [None] * 4
    discarder = None
    disc_pon = None
    if not tsumo:
        discarder = (winner + 1 + rnd.randrange(3)) % 4
        conc.remove(win)
        if chankan:
            others = [4 * (win >> 2) + j for j in range(4) if 4 * (win >> 2) + j != win]
            if any(t in used for t in others):
                return None
            used |= set(others)
            disc_pon = Meld(PN, tuple(sorted(others)), others[0], (discarder + 2) % 4)
    free = [t for t in range(136) if t not in used]
    rnd.shuffle(free)

    def take(pred=lambda t: True):
        for i, t in enumerate(free):
            if pred(t):
                return free.pop(i)
        return None

    # dead wall: dora indicators (slot 122 + 2i) and ura (123 + 2i)
    n_dora = min(5, max(len(c["dora"]), 1 + kans))
    dora, ura = [], []
    for i in range(n_dora):
        d = take(lambda t: t >> 2 == c["dora"][i] >> 2) if i < len(c["dora"]) else take()
        u = take(lambda t: t >> 2 == c["ura"][i] >> 2) if i < len(c["ura"]) else None
        u = u if u is not None else take()
        if d is None or u is None:
            return None
        dora.append(d)
        ura.append(u)
    # hands: winner's from the context, opponents' random
    wh = make_hand(conc, melds=tuple(melds))
    wait_kinds = set(wh.waits) | {win >> 2}
    for s in range(4):
        if s == winner:
            continue
        n = 13
        if s == discarder and disc_pon is not None:
            n = 10
        hs = [take(lambda t: t >> 2 not in wait_kinds or s != discarder) for _ in range(n)]
        if None in hs:
            return None
        hands[s] = hs
    drawn = win if tsumo else -1
    actor = winner if tsumo else discarder
    if not tsumo:
        hands[discarder] = hands[discarder] + [win]
        drawn = win
    # rivers: the winner's avoids its waits (furiten); riichi needs a
    # declaration discard; haitei / houtei fill the rivers up to the last tile
    rivers = [[] for _ in range(4)]
    wr = 0 if first else (rnd.randint(1, 3) if (riichi or not melds or rnd.random() < 0.5) else 0)
    if riichi and wr == 0:
        wr = 1
    for _ in range(wr):
        t = take(lambda t: t >> 2 not in wait_kinds)
        if t is None:
            return None
        rivers[winner].append(t)
    in_play = sum(len(h) for h in hands if h) + len(conc) + len(meld_ids) + \
        (len(disc_pon.tiles) if disc_pon else 0) + wr
    target = (122 - kans if last else in_play + rnd.randint(0, 30)) + kans
    if first:
        target = in_play
    seat_cycle = [s for s in range(4) if s != winner]
    k = 0
    while in_play < target:
        s = seat_cycle[k % 3]
        k += 1
        if len(rivers[s]) >= 30:
            if all(len(rivers[x]) >= 30 for x in seat_cycle):
                return None
            continue
        t = take()
        if t is None:
            return None
        rivers[s].append(t)
        in_play += 1
    cursor = in_play - kans
    if cursor > 122 - kans:
        return None
    front = [t for h in hands if h for t in h] + conc + meld_ids + (list(disc_pon.tiles) if disc_pon else []) + \
        [t for r in rivers for t in r]
    assert len(front) == in_play
    rnd.shuffle(front)
    tail = front[cursor:]
    front = front[:cursor]
    live = free[:]  # whatever is left goes to the live wall and dead wall rest
    wall = front + live[: 122 - cursor]  # [122 - kans, 122) are never drawn
    live = live[122 - cursor:]
    dead = [None] * 14
    for i in range(n_dora):
        dead[2 * i], dead[2 * i + 1] = dora[i], ura[i]
    rest = [x for x in live]
    for i in range(14 - kans):
        if dead[i] is None:
            dead[i] = rest.pop()
    for i in range(kans):
        dead[13 - i] = tail[i]
    wall += dead
    assert sorted(wall) == list(range(136)), (len(wall), len(set(wall)))
    hs = []
    for s in range(4):
        riv = tuple(RiverTile(t, False, riichi and s == winner and i == 0, False) for i, t in enumerate(rivers[s]))
        if s == winner:
            hs.append(make_hand(conc + ([] if tsumo else []), melds=tuple(melds), river=riv, riichi=riichi,
                                riichi_index=0 if riichi else -1, ippatsu=bool(c["ippatsu"] and riichi)))
        else:
            hs.append(make_hand(hands[s], melds=(disc_pon,) if (s == discarder and disc_pon) else (), river=riv))
    deposits = rnd.randint(0, 2) + (1 if riichi else 0)
    scores = [25000] * 4
    if riichi:
        scores[winner] -= 1000
    for _ in range(deposits - (1 if riichi else 0)):
        scores[rnd.randrange(4)] -= 1000
    cfg = GameConfig(rule=c["rule"], mode=MODE_HALF, kazoe=kazoe, double_yakuman=dy)
    template = GameState(
        config=cfg, wall=Wall(tiles=tuple(wall), cursor=cursor, kan_draws=kans, dora_count=n_dora),
        hands=tuple(hs), scores=tuple(scores), kyoku=kyoku, honba=rnd.randint(0, 3), deposits=deposits,
        phase=PH_ACT, actor=actor, drawn=drawn, rinshan_pending=bool(rinshan), rng=seed_state(rnd.randrange(1 << 30)),
        any_call_made=bool(melds and any(m.type != KC for m in melds)) or disc_pon is not None)
    return _finish(_B(template)), winner, discarder, disc_pon


def make_wins():
    import test_scoring as TS
    from mjsim import actions as A
    from mjsim.engine.engine import apply_action

    srcs = []
    for hand, win, wtype, melds, kw, _ in TS.GOLDEN_CASES:
        srcs.append(("golden", ctx_to_json(TS.make_ctx(hand, win, wtype, melds=melds, **kw)), False, False))
    for hand, win, wtype, melds, kw in RARE_HANDS:
        cj = ctx_to_json(rare_ctx(hand, win, wtype, melds, kw))
        for kz in (False, True):
            for dy in (False, True):
                srcs.append(("rare", cj, kz, dy))
    for case in json.loads(gzip.open(HERE / "scoring.json.gz").read())[38::2]:
        srcs.append(("random", case["ctx"], case["kazoe"], case["dy"]))
    rnd = random.Random(0x5EED)
    out = []
    stats = {}

    def record(tag, pre, action):
        try:
            post, err = state_projection(apply_action(pre, action)), None
        except Exception as e:  # IllegalActionError
            post, err = None, type(e).__name__
        out.append({"test": tag, "pre": state_record(pre), "action": int(action), "post": post, "error": err})
        stats[(tag, err)] = stats.get((tag, err), 0) + 1

    for tag, cj, kz, dy in srcs:
        made = None
        for _ in range(4):
            made = craft_win(cj, kz, dy, rnd)
            if made is not None:
                break
        if made is None:
            stats[(tag, "skipped")] = stats.get((tag, "skipped"), 0) + 1
            continue
        st, winner, discarder, disc_pon = made
        if cj["tsumo"]:
            record(tag, st, A.TSUMO)
            continue
        kind = cj["win_tile"] >> 2
        if disc_pon is not None:
            act = A.KAN_ADDED_BASE + kind
        elif cj["rule"] == 0 and cj["win_tile"] in (16, 52, 88):
            act = A.RED_ACTION_BY_KIND[kind]
        else:
            act = kind
        if not (st.legal_mask >> act) & 1:
            stats[(tag, "no-discard")] = stats.get((tag, "no-discard"), 0) + 1
            continue
        st = apply_action(st, act)
        while st.phase == 1 and st.actor != winner and (st.legal_mask >> A.PASS) & 1:
            st = apply_action(st, A.PASS)
        if st.phase == 1 and st.actor == winner:
            record(tag, st, A.RON)  # legal or not: a NoYaku / furiten ron is an IllegalActionError
        else:
            stats[(tag, "no-call")] = stats.get((tag, "no-call"), 0) + 1
    print("wins:", sorted(stats.items(), key=str))
    dump("wins.json.gz", out)


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


# ---------------------------------------------------------------------------
# crafted engine scenarios: every apply_action made by the reference's own
# engine tests (tests/test_engine.py, tests/test_engine_rounds.py), recorded
# as (pre-state record, action, post-state projection | exception)

def state_record(gs) -> dict:
    """GameState -> the fields of rs_env_rec (include/rinshan.h)"""
    cfg = gs.config
    hands = []
    for h in gs.hands:
        hands.append({
            "concealed": list(h.concealed), "n_concealed": len(h.concealed), "n_melds": len(h.melds),
            "melds": [{"type": m.type, "n_tiles": len(m.tiles), "from_seat": m.from_seat, "tiles": list(m.tiles),
                       "called_tile": m.called_tile} for m in h.melds],
            "river_tile": [rt.tile for rt in h.river],
            "river_flags": [int(rt.tsumogiri) | (2 * int(rt.riichi)) | (4 * int(rt.called)) for rt in h.river],
            "n_river": len(h.river), "riichi": h.riichi, "riichi_index": h.riichi_index, "ippatsu": int(h.ippatsu),
            "temp_furiten": int(h.temp_furiten), "perm_furiten": int(h.perm_furiten), "shanten": h.shanten,
            "waits": sum(1 << k for k in h.waits),
        })
    ev = gs.events()
    win = ev[-64:]
    mask = gs.legal_mask if not (gs.terminated or gs.truncated) else 0
    return {
        "cfg": {"rule": cfg.rule, "mode": cfg.mode, "reward_scheme": 0, "illegal_penalty": -1.0,
                "max_steps": cfg.max_steps, "kazoe": int(cfg.kazoe), "double_yakuman": int(cfg.double_yakuman),
                "agari_yame": int(cfg.agari_yame), "renchan_cap": cfg.renchan_cap},
        "wall": list(gs.wall.tiles), "cursor": gs.wall.cursor, "kan_draws": gs.wall.kan_draws,
        "dora_count": gs.wall.dora_count, "hands": hands, "scores": list(gs.scores), "kyoku": gs.kyoku,
        "honba": gs.honba, "deposits": gs.deposits, "repeats": gs.repeats, "phase": gs.phase, "actor": gs.actor,
        "drawn": gs.drawn, "riichi_pending": int(gs.riichi_pending), "rinshan_pending": int(gs.rinshan_pending),
        "call_tile": gs.call_tile, "call_from": gs.call_from, "n_queue": len(gs.call_queue),
        "queue_seat": [s for s, _ in gs.call_queue], "queue_stage": [t for _, t in gs.call_queue],
        "n_rons": len(gs.call_rons), "rons": list(gs.call_rons), "call_chankan": int(gs.call_chankan),
        "kakan_kind": gs.kakan_kind, "pending_dora": gs.pending_dora, "four_kan_pending": int(gs.four_kan_pending),
        "any_call_made": int(gs.any_call_made), "rng_key": gs.rng.key, "rng_counter": gs.rng.counter,
        "step_count": gs.step_count, "terminated": int(gs.terminated), "truncated": int(gs.truncated),
        "events_len": len(ev), "events": [list(e) for e in win], "n_results": len(gs.results),
        "legal_mask": [(mask >> (32 * i)) & 0xFFFFFFFF for i in range(4)],
        "current_player": gs.actor, "env_terminated": int(gs.terminated), "env_truncated": int(gs.truncated),
    }


def state_projection(gs) -> dict:
    """the same projection tests/paritylib.projection computes from records"""
    from mjsim.engine.state import _result_dict, serialize_state
    d = serialize_state(gs)
    d.pop("events")
    d.pop("results")
    d["legal"] = list(gs.legal) if not (gs.terminated or gs.truncated) else []
    if gs.terminated or gs.truncated:
        rewards = [(s - 25000) / 25000 for s in gs.scores]
    else:
        rewards = [0.0] * 4
    mask = gs.legal_mask if not (gs.terminated or gs.truncated) else 0
    d["internal"] = {
        "repeats": gs.repeats, "riichi_pending": int(gs.riichi_pending),
        "rinshan_pending": int(gs.rinshan_pending), "call_tile": gs.call_tile, "call_from": gs.call_from,
        "queue": [list(q) for q in gs.call_queue], "rons": list(gs.call_rons),
        "call_chankan": int(gs.call_chankan), "kakan_kind": gs.kakan_kind, "pending_dora": gs.pending_dora,
        "four_kan_pending": int(gs.four_kan_pending), "any_call_made": int(gs.any_call_made),
        "rng": [gs.rng.key, gs.rng.counter], "events_len": len(gs.events()), "n_results": len(gs.results),
        "hands": [{"riichi_index": h.riichi_index, "temp_furiten": int(h.temp_furiten),
                   "perm_furiten": int(h.perm_furiten), "waits": sum(1 << k for k in h.waits)} for h in gs.hands],
        "legal_mask": [(mask >> (32 * i)) & 0xFFFFFFFF for i in range(4)],
        "current_player": gs.actor, "env_terminated": int(gs.terminated), "env_truncated": int(gs.truncated),
        "rewards": [float(round(r, 9)) for r in rewards],
    }
    d["window"] = [list(e) for e in gs.events()[-64:]]
    d["last_result"] = _result_dict(gs.results[-1]) if gs.results else None
    return d


def make_scenarios():
    import engine_helpers
    import test_engine
    import test_engine_rounds
    from mjsim.engine import engine as eng
    from mjsim.engine.state import state_fingerprint as fp

    seen = {}
    per_test = {}
    out = []
    real_apply = eng.apply_action
    current = {"test": None}

    def recording_apply(state, action):
        key = (fp(state), int(action))
        exc = None
        try:
            nxt = real_apply(state, action)
            post, err = state_projection(nxt), None
        except Exception as e:  # IllegalActionError / ContractError
            nxt, post, err, exc = None, None, type(e).__name__, e
        per_test[current["test"]] = per_test.get(current["test"], 0) + 1
        # keep every transition of the crafted scenarios, cap the long random
        # plays some tests run (the traces fixture covers those)
        if key not in seen and per_test[current["test"]] <= 80:
            seen[key] = True
            out.append({"test": current["test"], "pre": state_record(state), "action": int(action),
                        "post": post, "error": err})
        if exc is not None:
            raise exc
        return nxt

    test_engine.apply_action = recording_apply
    test_engine_rounds.apply_action = recording_apply
    tables = get_tables()
    import inspect
    for mod in (test_engine, test_engine_rounds):
        for cname, cls in inspect.getmembers(mod, inspect.isclass):
            if not cname.startswith("Test"):
                continue
            for mname, meth in inspect.getmembers(cls, inspect.isfunction):
                if not mname.startswith("test_"):
                    continue
                current["test"] = f"{mod.__name__}::{cname}::{mname}"
                obj = cls()
                args = ["tables"] if "tables" in inspect.signature(meth).parameters else []
                try:
                    meth(obj, *[tables for _ in args])
                except Exception as e:  # a reference test that fails here is simply not harvested
                    print("  (skipped)", current["test"], type(e).__name__, e)
    by_test = {}
    for s in out:
        by_test[s["test"]] = by_test.get(s["test"], 0) + 1
    print(f"scenarios: {len(out)} transitions from {len(by_test)} tests")
    dump("scenarios.json.gz", out)


def make_logs():
    """mjlog-lite-v1 logs (engine/log.py) of the games the bench loop plays
    (bench/runner.py:97-121: env_game_seed per reset, one continuing
    env_policy_state per env), recorded with the reference GameRecorder;
    a steps budget per env like a fused device rollout"""
    from mjsim.engine.log import GameRecorder, log_to_json

    out = []
    for rule, mode, seed, n, steps in (("no-red", "single", 3, 4, 260), ("red", "single", 4, 4, 260),
                                       ("red", "east", 5, 1, 700)):
        cfg = EnvConfig(rule=rule, mode=mode)
        for idx in range(n):
            pol = env_policy_state(seed, idx)
            r = 0
            gseed = env_game_seed(seed, idx, r)
            st = init(gseed, cfg)
            rec = GameRecorder(st.game.config, gseed)
            for _ in range(steps):
                if st.terminated or st.truncated:
                    r += 1
                    gseed = env_game_seed(seed, idx, r)
                    st = init(gseed, cfg)
                    rec = GameRecorder(st.game.config, gseed)
                a, pol = random_policy(st.legal, pol)
                rec.record(st.game, a)
                st = step(st, a)
                if st.terminated or st.truncated:
                    out.append({"rule": rule, "mode": mode, "seed": seed, "index": idx, "game": r,
                                "steps": steps, "log": log_to_json(rec.to_log(st.game))})
    print(f"logs: {len(out)} games")
    dump("logs.json.gz", out)


def make_renders():
    """render/svg.py to_svg of reference states: a few steps of random and
    heuristic games (mid-game and the final state with its result panel),
    every viewer (None / seat) and both locales -> sha256 of the document"""
    from mjsim.render.svg import to_svg

    out = []
    for rule, mode, seed, idx, policy in (("red", "single", 1, 0, "random"), ("no-red", "single", 2, 3, "heuristic"),
                                         ("red", "east", 3, 1, "heuristic"), ("red", "single", 4, 5, "heuristic")):
        cfg = EnvConfig(rule=rule, mode=mode)
        st = init(env_game_seed(seed, idx), cfg)
        pol = env_policy_state(seed, idx)
        t = 0
        picks = {7, 40, 90}
        while True:
            game = st.game
            if t in picks or st.terminated or st.truncated:
                for viewer in (None, 0, 2):
                    for locale in ("en", "ja"):
                        svg = to_svg(game, viewer=viewer, locale=locale)
                        out.append({"rule": rule, "mode": mode, "seed": seed, "index": idx, "policy": policy,
                                    "step": t, "viewer": viewer, "locale": locale,
                                    "sha256": hashlib.sha256(svg.encode()).hexdigest(), "len": len(svg)})
            if st.terminated or st.truncated:
                break
            if policy == "random":
                a, pol = random_policy(st.legal, pol)
            else:
                a = heuristic_policy(observe(st, st.current_player), st.legal)
            st = step(st, a)
            t += 1
    print(f"renders: {len(out)}")
    dump("renders.json.gz", out)


# (rule, mode, seed, human seats, agents): every agent kind, several humans,
# no human at all (the whole game runs inside new_session)
SESSION_CASES = (("red", "single", 11, [0], {1: "heuristic", 2: "random", 3: "heuristic"}),
                 ("no-red", "east", 12, [1, 3], {0: "random", 2: "heuristic"}),
                 ("red", "single", 13, [], {0: "heuristic", 1: "random", 2: "heuristic", 3: "random"}),
                 ("no-red", "single", 14, [2], {0: "random", 1: "random", 3: "random"}))


def session_human_action(legal, n_actions):
    """the scripted human: a deterministic pick from the ascending legal ids"""
    return legal[(7 * n_actions + 3) % len(legal)]


def view_digest(view) -> str:
    v = dict(view)
    v.pop("game_id")
    return hashlib.sha256(json.dumps(v, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


def make_sessions():
    """service/sessions.py new_session / apply_session_action / advance_agents
    with a scripted human, the service/app.py `_view` of the human seat after
    creation, every 25 actions and at the end, and the SessionStore document"""
    from mjsim.service.app import _view
    from mjsim.service.sessions import SessionStore, advance_agents, apply_session_action

    out = []
    for rule, mode, seed, humans, agents in SESSION_CASES:
        cfg = EnvConfig(rule=rule, mode=mode)
        store = SessionStore(None)
        sess = store.create(cfg, seed, humans, agents)
        seat = humans[0] if humans else 0
        views = [(len(sess.actions), "en", view_digest(_view(sess, seat, "en")))]
        while sess.waiting_on() is not None:
            apply_session_action(sess, session_human_action(sess.state.legal, len(sess.actions)))
            advance_agents(sess)
            if len(views) < 40 and len(sess.actions) % 25 < 4:
                views.append((len(sess.actions), "en", view_digest(_view(sess, seat, "en"))))
        views.append((len(sess.actions), "ja", view_digest(_view(sess, seat, "ja"))))
        views.append((len(sess.actions), "en", view_digest(_view(sess, seat, "en"))))
        doc = {"id": "0123456789abcdef", "seed": seed,
               "config": {"rule": rule, "mode": mode, "reward_scheme": cfg.reward_scheme, "max_steps": cfg.max_steps},
               "human_seats": humans, "agents": {str(k): v for k, v in agents.items()},
               "actions": [list(a) for a in sess.actions], "created_at": 0.0, "updated_at": 0.0}
        out.append({"rule": rule, "mode": mode, "seed": seed, "human_seats": humans,
                    "agents": {str(k): v for k, v in agents.items()}, "actions": [list(a) for a in sess.actions],
                    "fingerprint": state_fingerprint(sess.state.game), "views": views, "doc": doc,
                    "rewards": list(sess.state.rewards)})
        print(f"session {rule} {mode} {seed}: {len(sess.actions)} actions, {len(views)} views")
    dump("sessions.json.gz", out)


def make_cli():
    """cli.py _cmd_selfplay / _cmd_render outputs and bench/runner.py
    rollout rows (games completed in the first pass)"""
    import argparse
    import tempfile

    from mjsim import cli
    from mjsim.bench import BenchConfig
    from mjsim.bench.runner import rollout

    out = {"selfplay": [], "render": [], "bench": []}
    tmp = Path(tempfile.mkdtemp())
    logs = []
    for rule, mode, seed, policy in (("red", "single", 5, "random"), ("no-red", "single", 6, "heuristic"),
                                     ("red", "east", 7, "random"), ("no-red", "single", 8, "random")):
        path = tmp / f"log{seed}.json"
        cli._cmd_selfplay(argparse.Namespace(rule=rule, mode=mode, seed=seed, policy=policy, out=str(path)))
        text = path.read_text()
        logs.append(path)
        out["selfplay"].append({"rule": rule, "mode": mode, "seed": seed, "policy": policy,
                                "sha256": hashlib.sha256(text.encode()).hexdigest(), "len": len(text)})
    for li, step, viewer, locale in ((0, None, None, "en"), (0, 30, 1, "ja"), (1, 60, -1, "en"), (2, None, 3, "en"),
                                     (2, 250, 0, "ja")):
        path = tmp / "r.svg"
        cli._cmd_render(argparse.Namespace(log=str(logs[li]), step=step, viewer=viewer, locale=locale,
                                           out=str(path)))
        svg = path.read_text()
        out["render"].append({"log": li, "step": step, "viewer": viewer, "locale": locale,
                              "sha256": hashlib.sha256(svg.encode()).hexdigest(), "len": len(svg)})
    for rule, mode, seed, batch, steps in (("no-red", "single", 0, 64, 100), ("red", "single", 1, 48, 150),
                                           ("red", "east", 2, 16, 300), ("no-red", "single", 3, 32, 400)):
        row, _ = rollout(BenchConfig(rule=rule, mode=mode, batch=batch, steps=steps, seed=seed, threads=4),
                         warmup=False)
        out["bench"].append({"rule": rule, "mode": mode, "seed": seed, "batch": batch, "steps": steps,
                             "games_completed": row.games_completed})
    print(f"cli: {len(out['selfplay'])} logs, {len(out['render'])} renders, {len(out['bench'])} bench rows")
    dump("cli.json.gz", out)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[f"make_{name}"]()
        sys.exit(0)
    make_rng()
    make_tables()
    make_shanten()
    make_scoring()
    make_scoring_rare()
    make_traces()
    make_scenarios()
    make_wins()
    make_logs()
    make_renders()
    make_sessions()
    make_cli()
