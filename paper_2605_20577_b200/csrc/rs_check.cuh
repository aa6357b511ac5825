// rs_check.cuh — on-device invariant checker (debug / soak path).
//
// Reference: engine/state.py:105-178 (check_invariants: score identity,
// tile conservation, mask sanity, then the per-hand coherence sweeps) and
// bench/runner.py:226-284 (play_games soak gates: furiten ron offered).
// The device state also keeps derived caches the reference recomputes
// (suit codes, table classes, observation tokens, shanten, waits, river
// kinds); the full check verifies those against the tile sets too.
#pragma once

#include "rs_engine.cuh"

namespace rs {

// tile ids of one set of 136 bits, marking duplicates
struct TileMarks {
  uint32_t w[5] = {0, 0, 0, 0, 0};
  int count = 0;
  bool dup = false;
  RS_HD void mark(int t) {
    if (t < 0 || t >= 136) { dup = true; return; }
    const uint32_t b = 1u << (t & 31);
    if (w[t >> 5] & b) dup = true;
    w[t >> 5] |= b;
    count++;
  }
  RS_HD bool complete() const {
    return !dup && count == 136 && w[0] == ~0u && w[1] == ~0u && w[2] == ~0u && w[3] == ~0u && w[4] == 0xFFu;
  }
};

RS_COLD uint32_t check_invariants(const Engine& E, bool fast) {
  const Soa& S = E.S;
  const Game& g = E.g;
  uint32_t bad = 0;
  // score identity (state.py:111-113)
  const int total = g.scores[0] + g.scores[1] + g.scores[2] + g.scores[3] + 1000 * g.deposits;
  if (total != 100000) bad |= RS_INV_SCORE_SUM;
  // tile conservation (state.py:115-143): wall from the cursor to the end
  // of the shifted dead wall, concealed sets, meld tiles, uncalled river
  TileMarks tm;
  for (int pos = g.cursor; pos < 136 - g.kan_draws; pos++) tm.mark(E.wall(pos));
  for (int s = 0; s < 4; s++) {
    const Hand h = load_hand(E.bp, s);
    for (int i = 0; i < 5; i++) {
      uint32_t x = h.word(i);
      while (x) {
        tm.mark(32 * i + ctz32(x));
        x &= x - 1;
      }
    }
    const int nm = hi::nmelds(h.info);
    for (int i = 0; i < nm; i++) {
      const uint32_t mt = E.meld_tiles(s, i);
      const int nt = mi::ntiles(E.meld_info(s, i));
      for (int j = 0; j < nt; j++) tm.mark((int)((mt >> (8 * j)) & 255u));
    }
    const int nr = hi::nriver(h.info);
    for (int i = 0; i < nr; i++) {
      const uint16_t rt = S.river[E.at(s * RS_MAX_RIVER + i)];
      if (!((rt >> 8) & RS_RIVER_CALLED)) tm.mark(rt & 255);
    }
  }
  if (!tm.complete()) bad |= RS_INV_TILES;
  // mask sanity (state.py:145-150), on the game's legal list
  const Mask115 m = E.load_legal();
  const bool empty = !(m.m[0] | m.m[1] | m.m[2] | m.m[3]);
  if ((g.phase == PH_ACT || g.phase == PH_CALL) && !g.terminated && !g.truncated && empty) bad |= RS_INV_EMPTY_LEGAL;
  if ((g.terminated || g.truncated) && !empty) bad |= RS_INV_TERMINAL_LEGAL;
  // furiten ron offered (runner.py:257-259)
  if (g.phase == PH_CALL && m.test(A_RON)) {
    const uint32_t inf = E.info(g.actor);
    if (hi::temp(inf) || hi::perm(inf) || (E.waits(g.actor) & sdword(E.bp, W_HRKIND + 2 * g.actor)))
      bad |= RS_INV_FURITEN_RON;
  }
  if (fast) return bad;
  for (int s = 0; s < 4; s++) {
    const Hand h = load_hand(E.bp, s);
    // the caches against the tile set (state.py:157-162 and the device-only ones)
    Hand x;
    x.w0 = h.w0; x.w1 = h.w1; x.w2 = h.w2; x.w3 = h.w3; x.w4 = h.w4;
    x.cm = x.cp = x.cs = x.cz = 0;
    for (int k = 0; k < 34; k++) {
      const uint32_t c = (uint32_t)h.count(k);
      x.set_code(kind_suit(k), x.code(kind_suit(k)) + c * kind_pow_calc(k));
    }
    x.cls = class_of(E.T, 0, x.cm) | (class_of(E.T, 1, x.cp) << 8) | (class_of(E.T, 2, x.cs) << 16) |
            (class_of(E.T, 3, x.cz) << 24);
    x.info = h.info;
    tokens_from_set(x, E.C.rule == RS_RULE_RED);
    const int nm = hi::nmelds(h.info), nconc = h.ntiles();
    if (x.cm != h.cm || x.cp != h.cp || x.cs != h.cs || x.cz != h.cz || x.cls != h.cls || x.tlo != h.tlo ||
        x.thi != h.thi || hi::nconc(h.info) != nconc)
      bad |= RS_INV_HAND_SYNC;
    const int size = nconc + 3 * nm;
    // shanten of the concealed part (13-form or 14-form alike) and, when
    // tenpai in the 13-form, the wait mask
    if (size == 13 || size == 14) {
      const int sh = full_shanten(E.T, x, nm);
      if (sh != hi::shanten(h.info)) bad |= RS_INV_HAND_SYNC;
      if (size == 13 && sh == 0 && compute_waits(E.T, x, nm) != h.waits) bad |= RS_INV_HAND_SYNC;
    }
    uint64_t rk = 0;
    const int nr = hi::nriver(h.info);
    for (int i = 0; i < nr; i++) rk |= 1ull << ((S.river[E.at(s * RS_MAX_RIVER + i)] & 255) >> 2);
    if (rk != sdword(E.bp, W_HRKIND + 2 * s)) bad |= RS_INV_HAND_SYNC;
    // tile-equivalents held (state.py:163-176)
    int expected = 13;
    if (g.phase == PH_ACT && g.actor == s) expected = 14;
    else if (g.phase == PH_CALL && g.call_chankan && s == g.call_from) expected = 14;
    if (g.phase == PH_GAME_END) {
      if (size != 13 && size != 14) bad |= RS_INV_HAND_SIZE;
    } else if (size != expected) {
      bad |= RS_INV_HAND_SIZE;
    }
    // riichi implies tenpai (state.py:178-180)
    if (hi::riichi(h.info) && hi::shanten(h.info) > 0 && size == 13) bad |= RS_INV_RIICHI_NOT_TENPAI;
  }
  return bad;
}

}  // namespace rs
