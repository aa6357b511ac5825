// rs_score.cuh — win evaluation on the device (rare path).
//
// Reference: scoring/score.py:45-82 (score_win: maximise (base, yakuman,
// han, fu) over every reading, first maximum wins), hand/decompose.py:24-68
// (decompositions, ordered by pair then sorted set list), scoring/yaku.py
// :146-380 (wait placements, standard / seven-pairs / kokushi yaku),
// scoring/fu.py:11-54, scoring/dora.py:9-26, scoring/points.py:16-86.
//
// Counts are 34 nibbles packed in five words; yaku lists are 40-bit id
// masks (+ a mask of ids counted twice), so a reading needs no arrays.
#pragma once

#include <cstddef>

#include "../../include/rinshan.h"
#include "rs_common.cuh"

namespace rs {

enum : int {
  Y_RIICHI = 0, Y_DOUBLE_RIICHI, Y_IPPATSU, Y_MENZEN_TSUMO, Y_PINFU, Y_TANYAO,
  Y_WHITE, Y_GREEN, Y_RED, Y_SEAT, Y_ROUND, Y_SANSHOKU_DOUJUN, Y_SANSHOKU_DOUKOU,
  Y_ITTSU, Y_CHANTA, Y_JUNCHAN, Y_TOITOI, Y_SANANKOU, Y_SANKANTSU, Y_CHIITOITSU,
  Y_HONROUTOU, Y_SHOUSANGEN, Y_HONITSU, Y_CHINITSU, Y_HAITEI, Y_HOUTEI, Y_RINSHAN,
  Y_CHANKAN, Y_KOKUSHI, Y_SUUANKOU, Y_DAISANGEN, Y_SHOUSUUSHI, Y_DAISUUSHI,
  Y_TSUUIISOU, Y_CHINROUTOU, Y_RYUUIISOU, Y_CHUUREN, Y_SUUKANTSU, Y_TENHOU, Y_CHIIHOU
};
enum : int { W_RYANMEN = 0, W_KANCHAN, W_PENCHAN, W_SHANPON, W_TANKI };

// han of a regular yaku id (yaku.py:239-310 / :353-369); closed-hand value
// when `closed`
RS_HD int yaku_han_of(int id, bool closed) {
  switch (id) {
    case Y_DOUBLE_RIICHI: return 2;
    case Y_SANSHOKU_DOUJUN: case Y_ITTSU: case Y_CHANTA: return closed ? 2 : 1;
    case Y_JUNCHAN: case Y_HONITSU: return closed ? 3 : 2;
    case Y_CHINITSU: return closed ? 6 : 5;
    case Y_SANSHOKU_DOUKOU: case Y_TOITOI: case Y_SANANKOU: case Y_SANKANTSU:
    case Y_CHIITOITSU: case Y_HONROUTOU: case Y_SHOUSANGEN: return 2;
    default: return 1;
  }
}
RS_HD int mask_han(uint64_t m, bool closed) {
  int t = 0;
  while (m) {
    const int id = ctz64(m);
    m &= m - 1;
    t += yaku_han_of(id, closed);
  }
  return t;
}

// five words of per-kind nibble counts
struct Counts {
  uint32_t c[5];
  RS_HD int get(int k) const { return (c[k >> 3] >> ((k & 7) * 4)) & 15; }
  RS_HD void add(int k, int v) { c[k >> 3] += (uint32_t)v << ((k & 7) * 4); }
  RS_HD void sub(int k, int v) { c[k >> 3] -= (uint32_t)v << ((k & 7) * 4); }
  RS_HD bool empty() const { return !(c[0] | c[1] | c[2] | c[3] | c[4]); }
  RS_HD int lowest() const {
    for (int i = 0; i < 5; i++)
      if (c[i]) return 8 * i + ctz32(c[i]) / 4;
    return 34;
  }
  RS_HD uint64_t ge(int t) const {
    return (uint64_t)nib_ge(c[0], t) | ((uint64_t)nib_ge(c[1], t) << 8) | ((uint64_t)nib_ge(c[2], t) << 16) |
           ((uint64_t)nib_ge(c[3], t) << 24) | ((uint64_t)(nib_ge(c[4], t) & 3u) << 32);
  }
  RS_HD uint64_t eq(int t) const {
    return (uint64_t)nib_eq(c[0], t) | ((uint64_t)nib_eq(c[1], t) << 8) | ((uint64_t)nib_eq(c[2], t) << 16) |
           ((uint64_t)nib_eq(c[3], t) << 24) | ((uint64_t)(nib_eq(c[4], t) & 3u) << 32);
  }
};

// scoring/context.py:19-57 (WinContext)
struct WinIn {
  Counts conc;              // concealed counts incl. the winning tile
  int nmelds;
  int mtype[4], mbase[4];   // meld type / lowest kind
  int win_kind;
  bool tsumo;
  int seat_wind, round_wind;
  int riichi;
  bool ippatsu, last_tile, rinshan, chankan, first_draw;
  bool closed;              // every meld is a closed kan
  int dora, ura, reds;      // dora.py:9-26, precomputed by the caller
  bool double_yakuman, kazoe;
};

struct Reading {
  uint64_t mask;  // yaku ids present
  uint64_t x2;    // ids counted twice (double yakuman)
  int yakuman;    // yakuman count (0: regular hand)
  int han;        // han of the reading incl. dora (0 for yakuman)
  int fu, base, form;
};

// scoring/points.py:16-37
RS_HD int base_points(int fu, int han, int yakuman, bool kazoe) {
  if (yakuman) return 8000 * yakuman;
  if (han >= 13) return kazoe ? 8000 : 6000;
  if (han >= 11) return 6000;
  if (han >= 8) return 4000;
  if (han >= 6) return 3000;
  if (han >= 5) return 2000;
  const int v = fu * (1 << (2 + han));
  return v < 2000 ? v : 2000;
}
RS_HD int ceil100(int x) { return (x + 99) / 100 * 100; }

RS_HD uint64_t situational(const WinIn& w) {  // yaku.py:304-310
  uint64_t m = 0;
  if (w.last_tile) m |= 1ull << (w.tsumo ? Y_HAITEI : Y_HOUTEI);
  if (w.rinshan) m |= 1ull << Y_RINSHAN;
  if (w.chankan) m |= 1ull << Y_CHANKAN;
  return m;
}

// yaku.py:313-334 (_is_chuuren): 0 no, 1 nine gates, 2 pure nine-sided
RS_HD int chuuren(const WinIn& w) {
  if (w.nmelds) return 0;
  const uint64_t present = w.conc.ge(1);
  if (present & HONOR_MASK) return 0;
  int suit = -1;
  #pragma unroll 1
  for (int s = 0; s < 3; s++)
    if ((present >> (9 * s)) & 0x1FF) {
      if (suit >= 0) return 0;
      suit = s;
    }
  if (suit < 0) return 0;
  int extra = -1;
  #pragma unroll 1
  for (int i = 0; i < 9; i++) {
    const int d = w.conc.get(9 * suit + i) - ((i == 0 || i == 8) ? 3 : 1);
    if (d == 0) continue;
    if (d == 1 && extra < 0) extra = i;
    else return 0;
  }
  if (extra < 0) return 0;
  return 9 * suit + extra == w.win_kind ? 2 : 1;
}

// blocks: concealed sets (sorted keys) then melds (yaku.py:146-155)
struct Blocks {
  int n;
  int start[8];
  bool run[8], open[8], kan[8], ronfill[8];
};
RS_HD void make_blocks(const WinIn& w, const int* keys, int nsets, int wait_block, Blocks& b) {
  b.n = 0;
  #pragma unroll 1
  for (int i = 0; i < nsets; i++) {
    const bool run = keys[i] < 64;
    b.start[b.n] = keys[i] & 63;
    b.run[b.n] = run;
    b.open[b.n] = false;
    b.kan[b.n] = false;
    b.ronfill[b.n] = !w.tsumo && i == wait_block && !run;
    b.n++;
  }
  #pragma unroll 1
  for (int i = 0; i < w.nmelds; i++) {
    b.start[b.n] = w.mbase[i];
    b.run[b.n] = w.mtype[i] == 0;
    b.open[b.n] = w.mtype[i] != 3;
    b.kan[b.n] = w.mtype[i] >= 2;
    b.ronfill[b.n] = false;
    b.n++;
  }
}

// detect_standard (yaku.py:188-301) + fu_for_placement (fu.py:35-54)
RS_HD void standard_reading(const WinIn& w, int pair, const int* keys, int nsets, int wait_block, int wait,
                            Reading& r) {
  Blocks b;
  make_blocks(w, keys, nsets, wait_block, b);
  uint64_t present = 1ull << pair, trip = 0, run_starts = 0;
  int concealed_trips = 0, kans = 0;
  bool all_trip = true, has_run = false, outside = is_orphan(pair);
  int fu_blocks = 0;
  #pragma unroll 1
  for (int i = 0; i < b.n; i++) {
    const int s = b.start[i];
    if (b.run[i]) {
      present |= 7ull << s;
      run_starts |= 1ull << s;
      all_trip = false;
      has_run = true;
      if (!(is_orphan(s) || is_orphan(s + 1) || is_orphan(s + 2))) outside = false;
    } else {
      present |= 1ull << s;
      trip |= 1ull << s;
      if (!b.open[i] && !b.ronfill[i]) concealed_trips++;
      if (!is_orphan(s)) outside = false;
      int f = 2;  // fu.py:11-20
      if (!b.open[i] && !b.ronfill[i]) f *= 2;
      if (b.kan[i]) f *= 4;
      if (is_orphan(s)) f *= 2;
      fu_blocks += f;
    }
    if (b.kan[i]) kans++;
  }
  uint64_t m = 0, x2 = 0;
  int yakuman = 0;
  // yakuman (yaku.py:206-232)
  if (w.first_draw && w.tsumo && w.nmelds == 0) { m |= 1ull << (w.seat_wind == 27 ? Y_TENHOU : Y_CHIIHOU); yakuman++; }
  if (concealed_trips == 4) {
    m |= 1ull << Y_SUUANKOU;
    const bool d = w.double_yakuman && wait == W_TANKI;
    if (d) x2 |= 1ull << Y_SUUANKOU;
    yakuman += d ? 2 : 1;
  }
  if ((trip & (7ull << 31)) == (7ull << 31)) { m |= 1ull << Y_DAISANGEN; yakuman++; }
  const int wind_trips = popc64(trip & (15ull << 27));
  if (wind_trips == 4) {
    m |= 1ull << Y_DAISUUSHI;
    if (w.double_yakuman) x2 |= 1ull << Y_DAISUUSHI;
    yakuman += w.double_yakuman ? 2 : 1;
  } else if (wind_trips == 3 && pair >= 27 && pair <= 30) { m |= 1ull << Y_SHOUSUUSHI; yakuman++; }
  if (!(present & ~HONOR_MASK)) { m |= 1ull << Y_TSUUIISOU; yakuman++; }
  if (!(present & ~TERMINAL_MASK)) { m |= 1ull << Y_CHINROUTOU; yakuman++; }
  if (!(present & ~GREEN_MASK)) { m |= 1ull << Y_RYUUIISOU; yakuman++; }
  if (kans == 4) { m |= 1ull << Y_SUUKANTSU; yakuman++; }
  const int ch = chuuren(w);
  if (ch) {
    m |= 1ull << Y_CHUUREN;
    const bool d = w.double_yakuman && ch == 2;
    if (d) x2 |= 1ull << Y_CHUUREN;
    yakuman += d ? 2 : 1;
  }
  if (!yakuman) {
    const bool closed = w.closed;
    if (w.riichi == 2) m |= 1ull << Y_DOUBLE_RIICHI;
    else if (w.riichi == 1) m |= 1ull << Y_RIICHI;
    if (w.ippatsu) m |= 1ull << Y_IPPATSU;
    if (closed && w.tsumo) m |= 1ull << Y_MENZEN_TSUMO;
    if (closed && all_trip == false && !trip && pair < 31 && pair != w.seat_wind && pair != w.round_wind &&
        wait == W_RYANMEN)
      m |= 1ull << Y_PINFU;
    if (!(present & ORPHAN_MASK)) m |= 1ull << Y_TANYAO;
    if ((trip >> 31) & 1) m |= 1ull << Y_WHITE;
    if ((trip >> 32) & 1) m |= 1ull << Y_GREEN;
    if ((trip >> 33) & 1) m |= 1ull << Y_RED;
    if ((trip >> w.seat_wind) & 1) m |= 1ull << Y_SEAT;
    if ((trip >> w.round_wind) & 1) m |= 1ull << Y_ROUND;
    if (run_starts & (run_starts >> 9) & (run_starts >> 18) & 0x7Full) m |= 1ull << Y_SANSHOKU_DOUJUN;
    if (trip & (trip >> 9) & (trip >> 18) & 0x1FFull) m |= 1ull << Y_SANSHOKU_DOUKOU;
    #pragma unroll 1
    for (int s = 0; s < 3; s++)
      if (((run_starts >> (9 * s)) & 0x49ull) == 0x49ull) { m |= 1ull << Y_ITTSU; break; }
    const bool has_honor = (present & HONOR_MASK) != 0;
    if (outside && has_run) m |= 1ull << (has_honor ? Y_CHANTA : Y_JUNCHAN);
    if (all_trip) m |= 1ull << Y_TOITOI;
    if (concealed_trips == 3) m |= 1ull << Y_SANANKOU;
    if (kans == 3) m |= 1ull << Y_SANKANTSU;
    if (outside && !has_run && has_honor) m |= 1ull << Y_HONROUTOU;
    if (popc64(trip & (7ull << 31)) == 2 && pair >= 31) m |= 1ull << Y_SHOUSANGEN;
    const int nsuits = ((present & 0x1FFull) != 0) + ((present & (0x1FFull << 9)) != 0) +
                       ((present & (0x1FFull << 18)) != 0);
    if (nsuits == 1) m |= 1ull << (has_honor ? Y_HONITSU : Y_CHINITSU);
    m |= situational(w);
  }
  r.mask = m;
  r.x2 = x2;
  r.yakuman = yakuman;
  r.form = 0;
  // fu (fu.py:35-54): chiitoitsu cannot occur in a standard reading
  if ((m >> Y_PINFU) & 1) {
    r.fu = w.tsumo ? 20 : 30;
  } else {
    int fu = 20 + fu_blocks;
    if (pair >= 31) fu += 2;
    if (pair == w.seat_wind) fu += 2;
    if (pair == w.round_wind) fu += 2;
    if (wait == W_KANCHAN || wait == W_PENCHAN || wait == W_TANKI) fu += 2;
    if (!w.tsumo && w.closed) fu += 10;
    if (w.tsumo) fu += 2;
    r.fu = (fu + 9) / 10 * 10;
  }
}

// detect_seven_pairs (yaku.py:337-370)
RS_HD void seven_pairs_reading(const WinIn& w, Reading& r) {
  const uint64_t present = w.conc.ge(1);
  uint64_t m = 0;
  int yakuman = 0;
  if (w.first_draw && w.tsumo) { m |= 1ull << (w.seat_wind == 27 ? Y_TENHOU : Y_CHIIHOU); yakuman++; }
  if (!(present & ~HONOR_MASK)) { m |= 1ull << Y_TSUUIISOU; yakuman++; }
  if (!yakuman) {
    if (w.riichi == 2) m |= 1ull << Y_DOUBLE_RIICHI;
    else if (w.riichi == 1) m |= 1ull << Y_RIICHI;
    if (w.ippatsu) m |= 1ull << Y_IPPATSU;
    if (w.tsumo) m |= 1ull << Y_MENZEN_TSUMO;
    m |= 1ull << Y_CHIITOITSU;
    if (!(present & ORPHAN_MASK)) m |= 1ull << Y_TANYAO;
    if (!(present & ~ORPHAN_MASK)) m |= 1ull << Y_HONROUTOU;
    const int nsuits = ((present & 0x1FFull) != 0) + ((present & (0x1FFull << 9)) != 0) +
                       ((present & (0x1FFull << 18)) != 0);
    if (nsuits == 1) m |= 1ull << ((present & HONOR_MASK) ? Y_HONITSU : Y_CHINITSU);
    m |= situational(w);
  }
  r.mask = m;
  r.x2 = 0;
  r.yakuman = yakuman;
  r.fu = 25;
  r.form = 1;
}

// detect_kokushi (yaku.py:373-380)
RS_HD void kokushi_reading(const WinIn& w, Reading& r) {
  uint64_t m = 1ull << Y_KOKUSHI, x2 = 0;
  int yakuman = 1;
  if (w.double_yakuman && w.conc.get(w.win_kind) == 2) { x2 = m; yakuman = 2; }
  if (w.first_draw && w.tsumo) { m |= 1ull << (w.seat_wind == 27 ? Y_TENHOU : Y_CHIIHOU); yakuman++; }
  r.mask = m;
  r.x2 = x2;
  r.yakuman = yakuman;
  r.fu = 0;
  r.form = 2;
}

// consider() of score.py:55-67: returns true when `r` is a valid reading
// and fills han/base; `key` orders (base, yakuman, han, fu)
RS_HD bool finalize_reading(const WinIn& w, Reading& r, uint64_t& key) {
  if (r.yakuman) {
    r.han = 0;
  } else {
    // seven pairs values equal the closed values (yaku.py:353-369)
    const int yh = mask_han(r.mask, r.form == 1 ? true : w.closed);
    if (yh == 0) return false;
    r.han = yh + w.dora + w.ura + w.reds;
  }
  r.base = base_points(r.fu, r.han, r.yakuman, w.kazoe);
  key = ((uint64_t)r.base << 32) | ((uint64_t)r.yakuman << 24) | ((uint64_t)r.han << 12) | (uint64_t)r.fu;
  return true;
}

// score_win (score.py:45-82).  Returns false on NoYakuError.  With
// `first_only` it stops at the first valid reading (the legality checks
// _can_tsumo / _can_ron only need existence).
RS_COLD bool score_win(const WinIn& w, Reading& best, bool first_only) {
  RS_ACC(1);
  bool found = false;
  uint64_t best_key = 0;
  Reading r;
  uint64_t key;
  if (w.nmelds == 0) {
    const uint64_t present = w.conc.ge(1);
    // _is_kokushi (score.py:37-42)
    if (!(present & ~ORPHAN_MASK) && popc64(present) == 13 && popc64(w.conc.eq(2) & ORPHAN_MASK) == 1) {
      kokushi_reading(w, r);
      if (finalize_reading(w, r, key) && (!found || key > best_key)) {
        best = r; best_key = key; found = true;
        if (first_only) return true;
      }
    }
    // _is_seven_pairs (score.py:33-34)
    if (popc64(w.conc.eq(2)) == 7) {
      seven_pairs_reading(w, r);
      if (finalize_reading(w, r, key) && (!found || key > best_key)) {
        best = r; best_key = key; found = true;
        if (first_only) return true;
      }
    }
  }
  const int needed = 4 - w.nmelds;
  uint64_t pairs = w.conc.ge(2);
  while (pairs) {
    const int p = ctz64(pairs);
    pairs &= pairs - 1;
    Counts base = w.conc;
    base.sub(p, 2);
    // enumerate set extractions (decompose.py:24-47): at each level take the
    // lowest kind as a triplet (bit clear) or a run (bit set); level d reads
    // choice bit needed-1-d, so the choices sharing a prefix are contiguous
    // and a level that fails skips all of them
    uint32_t decs[16];
    int nd = 0;
#pragma unroll 1
    for (int choice = 0; choice < (1 << needed); choice++) {
      Counts c = base;
      int keys[4];
      int fail = -1;
#pragma unroll 1
      for (int d = 0; d < needed; d++) {
        const int i = c.lowest();
        bool ok = i < 34;
        if (ok && !((choice >> (needed - 1 - d)) & 1)) {
          ok = c.get(i) >= 3;
          if (ok) { c.sub(i, 3); keys[d] = 64 + i; }
        } else if (ok) {
          ok = i < 27 && i % 9 <= 6 && c.get(i + 1) && c.get(i + 2);
          if (ok) {
            c.sub(i, 1); c.sub(i + 1, 1); c.sub(i + 2, 1);
            keys[d] = i;
          }
        }
        if (!ok) { fail = d; break; }
      }
      if (fail >= 0) {
        choice |= (1 << (needed - 1 - fail)) - 1;
        continue;
      }
      if (!c.empty()) continue;
      // sorted(sets): insertion sort of <= 4 keys, packed 7 bits each
      #pragma unroll 1
      for (int a = 1; a < needed; a++)
        for (int q = a; q > 0 && keys[q - 1] > keys[q]; q--) { int t = keys[q]; keys[q] = keys[q - 1]; keys[q - 1] = t; }
      uint32_t packed = 0;
      #pragma unroll 1
      for (int d = 0; d < needed; d++) packed = (packed << 7) | (uint32_t)keys[d];
      // keep decs sorted ascending (results sorted by set tuple)
      int q = nd++;
      while (q > 0 && decs[q - 1] > packed) { decs[q] = decs[q - 1]; q--; }
      decs[q] = packed;
    }
    #pragma unroll 1
    for (int di = 0; di < nd; di++) {
      int keys[4];
      #pragma unroll 1
      for (int d = 0; d < needed; d++) keys[d] = (decs[di] >> (7 * (needed - 1 - d))) & 127;
      // wait_placements (yaku.py:158-174)
      const int k = w.win_kind;
      #pragma unroll 1
      for (int i = 0; i <= needed; i++) {
        int blk, wait;
        if (i < needed) {
          const int start = keys[i] & 63;
          if (keys[i] < 64) {
            if (start == k) wait = k % 9 <= 5 ? W_RYANMEN : W_PENCHAN;
            else if (start + 1 == k) wait = W_KANCHAN;
            else if (start + 2 == k) wait = k % 9 >= 3 ? W_RYANMEN : W_PENCHAN;
            else continue;
          } else if (start == k) wait = W_SHANPON;
          else continue;
          blk = i;
        } else {
          if (p != k) continue;
          blk = -1;
          wait = W_TANKI;
        }
        standard_reading(w, p, keys, needed, blk, wait, r);
        if (finalize_reading(w, r, key) && (!found || key > best_key)) {
          best = r; best_key = key; found = true;
          if (first_only) return true;
        }
      }
    }
  }
  return found;
}

// WinScore (score.py:23-32) as the result record's per-win entry: han per
// yaku id (yakuman multiplicity for yakuman hands), the reading's totals and
// the dora parts of the win context
RS_HD void fill_win_rec(rs_win_rec& x, const Reading& rd, const WinIn& w) {
  // ten zero words, then the han of the (few) yaku present
  static_assert(offsetof(rs_win_rec, yaku_han) == 0 && alignof(rs_win_rec) >= 4 && sizeof(x.yaku_han) == 40,
                "yaku_han: ten aligned words");
  uint32_t* yh = reinterpret_cast<uint32_t*>(x.yaku_han);
#pragma unroll 1
  for (int i = 0; i < 10; i++) yh[i] = 0u;
  uint64_t ym = rd.mask;
  while (ym) {
    const int id = ctz64(ym);
    ym &= ym - 1;
    RS_CHECK(id < 40);
    x.yaku_han[id] = (int8_t)(rd.yakuman ? (((rd.x2 >> id) & 1) ? 2 : 1)
                                         : yaku_han_of(id, rd.form == 1 ? true : w.closed));
  }
  x.yakuman = rd.yakuman;
  x.han = rd.han;
  x.fu = rd.fu;
  x.base = rd.base;
  x.dora = w.dora;
  x.ura = w.ura;
  x.reds = w.reds;
  x.form = rd.form;
}

// settle (points.py:56-86)
RS_HD void settle(bool tsumo, int base, int dealer, int winner, int loser, int honba, int deposits,
                  int* deltas, int* honba_comp) {
  #pragma unroll 1
  for (int s = 0; s < 4; s++) deltas[s] = 0;
  const bool dealer_win = winner == dealer;
  if (!tsumo) {
    const int pay = ceil100(base * (dealer_win ? 6 : 4)) + 300 * honba;
    deltas[loser] -= pay;
    deltas[winner] += pay;
    *honba_comp = 300 * honba;
  } else {
    *honba_comp = 0;
    #pragma unroll 1
    for (int s = 0; s < 4; s++) {
      if (s == winner) continue;
      const int share = (dealer_win || s == dealer) ? 2 * base : base;
      const int pay = ceil100(share) + 100 * honba;
      deltas[s] -= pay;
      deltas[winner] += pay;
      *honba_comp += 100 * honba;
    }
  }
  deltas[winner] += 1000 * deposits;
}

}  // namespace rs
