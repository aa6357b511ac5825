// rs_hand.cuh — per-seat hand state and shanten / waits on the device.
//
// Reference: engine/state.py:31-98 (incremental hand rebuild),
// hand/shanten.py:98-244 (standard form via suit tables, seven pairs,
// thirteen orphans, waits).  The standard-form value is one lookup of the
// pre-merged tables (rs_tables.h) instead of the reference's budget-split
// merge loop.
#pragma once

#include "rs_state.cuh"
#include "rs_tables.h"

namespace rs {

// One seat's hand held in registers.
struct Hand {
  uint32_t w0, w1, w2, w3, w4;  // 136-bit concealed tile-id set
  uint32_t cm, cp, cs, cz;      // base-5 codes
  uint32_t cls;                 // class byte per suit
  uint32_t info;                // hi:: flags
  uint64_t waits;
  uint64_t tlo, thi;            // sorted observation tokens, 16 bytes, pad 37

  // dynamic word / code index as selects (no branches: the 32 envs of a
  // warp index different words at large batches)
  RS_HD uint32_t word(int i) const {
    uint32_t x = w4;
    x = i == 3 ? w3 : x;
    x = i == 2 ? w2 : x;
    x = i == 1 ? w1 : x;
    return i == 0 ? w0 : x;
  }
  RS_HD void set_word(int i, uint32_t v) {
    w0 = i == 0 ? v : w0;
    w1 = i == 1 ? v : w1;
    w2 = i == 2 ? v : w2;
    w3 = i == 3 ? v : w3;
    w4 = i >= 4 ? v : w4;
  }
  RS_HD bool has(int t) const { return (word(t >> 5) >> (t & 31)) & 1u; }
  RS_HD uint32_t nibble(int k) const { return (word(k >> 3) >> ((k & 7) * 4)) & 0xFu; }
  RS_HD int count(int k) const { return popc32(nibble(k)); }
  RS_HD int lowest_of_kind(int k) const { return 4 * k + ctz32(nibble(k)); }
  RS_HD uint32_t code(int s) const {
    uint32_t x = cz;
    x = s == 2 ? cs : x;
    x = s == 1 ? cp : x;
    return s == 0 ? cm : x;
  }
  RS_HD void set_code(int s, uint32_t v) {
    cm = s == 0 ? v : cm;
    cp = s == 1 ? v : cp;
    cs = s == 2 ? v : cs;
    cz = s >= 3 ? v : cz;
  }

  // 34-bit mask of kinds with count >= t
  RS_HD uint64_t kinds_ge(int t) const {
    return (uint64_t)nib_ge(nib_counts(w0), t) | ((uint64_t)nib_ge(nib_counts(w1), t) << 8) |
           ((uint64_t)nib_ge(nib_counts(w2), t) << 16) | ((uint64_t)nib_ge(nib_counts(w3), t) << 24) |
           ((uint64_t)(nib_ge(nib_counts(w4), t) & 3u) << 32);
  }
  RS_HD uint64_t kinds_eq(int t) const {
    return (uint64_t)nib_eq(nib_counts(w0), t) | ((uint64_t)nib_eq(nib_counts(w1), t) << 8) |
           ((uint64_t)nib_eq(nib_counts(w2), t) << 16) | ((uint64_t)nib_eq(nib_counts(w3), t) << 24) |
           ((uint64_t)(nib_eq(nib_counts(w4), t) & 3u) << 32);
  }
  RS_HD int ntiles() const { return popc32(w0) + popc32(w1) + popc32(w2) + popc32(w3) + popc32(w4); }
};

RS_HD Hand load_hand(const uint8_t* bp, int seat) {
  Hand h;
  const uint32_t m = W_HMASK + 5 * (uint32_t)seat, c = W_HCODE + 4 * (uint32_t)seat;
  h.w0 = sword(bp, m); h.w1 = sword(bp, m + 1); h.w2 = sword(bp, m + 2); h.w3 = sword(bp, m + 3);
  h.w4 = sword(bp, m + 4);
  h.cm = sword(bp, c); h.cp = sword(bp, c + 1); h.cs = sword(bp, c + 2); h.cz = sword(bp, c + 3);
  h.cls = sword(bp, W_HCLS + seat);
  h.info = sword(bp, W_HINFO + seat);
  h.waits = sdword(bp, W_HWAITS + 2 * seat);
  const uint4 t = squad(bp, W_HTOK + 4 * seat);
  h.tlo = (uint64_t)t.x | ((uint64_t)t.y << 32);
  h.thi = (uint64_t)t.z | ((uint64_t)t.w << 32);
  return h;
}
RS_HD void store_hand(uint8_t* bp, int seat, const Hand& h) {
  const uint32_t m = W_HMASK + 5 * (uint32_t)seat, c = W_HCODE + 4 * (uint32_t)seat;
  sword(bp, m) = h.w0; sword(bp, m + 1) = h.w1; sword(bp, m + 2) = h.w2; sword(bp, m + 3) = h.w3;
  sword(bp, m + 4) = h.w4;
  sword(bp, c) = h.cm; sword(bp, c + 1) = h.cp; sword(bp, c + 2) = h.cs; sword(bp, c + 3) = h.cz;
  sword(bp, W_HCLS + seat) = h.cls;
  sword(bp, W_HINFO + seat) = h.info;
  sdword(bp, W_HWAITS + 2 * seat) = h.waits;
  squad(bp, W_HTOK + 4 * seat) = make_uint4((uint32_t)h.tlo, (uint32_t)(h.tlo >> 32), (uint32_t)h.thi, (uint32_t)(h.thi >> 32));
}

// ---- sorted observation tokens (observe.py:89-90) kept incrementally ----
// Tokens are < 128, so bytewise compares need no carries: (b | 0x80) - v
// keeps the high bit exactly where b >= v.
constexpr uint64_t TOK_PAD8 = 0x2525252525252525ull;  // 37 in every byte
RS_HD int tok_rank(uint64_t lo, uint64_t hi, uint32_t v) {  // bytes < v
  const uint64_t H = 0x8080808080808080ull, vv = 0x0101010101010101ull * v;
  return 16 - popc64(((lo | H) - vv) & H) - popc64(((hi | H) - vv) & H);
}
// the low p bytes (0 <= p <= 8) of a 64-bit word
RS_HD uint64_t low_bytes(int p) { return p >= 8 ? ~0ull : ((1ull << (8 * (p & 7))) - 1ull); }
// insert / remove token v in the sorted 16-byte register (lo | hi << 64):
// both halves' results are computed and selected, no branch (the envs of a
// warp insert at different positions)
RS_HD void tok_insert(uint64_t& lo, uint64_t& hi, uint32_t v) {
  const int p = tok_rank(lo, hi, v);
  const bool low = p < 8;
  const int q = low ? p : p - 8;
  const uint64_t m = low_bytes(q), x = low ? lo : hi;
  const uint64_t ins = (x & m) | ((uint64_t)v << (8 * q)) | ((x & ~m) << 8);
  hi = low ? (hi << 8) | (lo >> 56) : ins;
  lo = low ? ins : lo;
}
RS_HD void tok_remove(uint64_t& lo, uint64_t& hi, uint32_t v) {  // v present
  const int p = tok_rank(lo, hi, v);
  const bool low = p < 8;
  const int q = low ? p : p - 8;
  const uint64_t m = low_bytes(q), x = low ? lo : hi;
  const uint64_t rem = (x & m) | ((x >> 8) & ~m);
  lo = low ? rem | (hi << 56) : lo;
  hi = low ? (hi >> 8) | (0x25ull << 56) : rem | (0x25ull << 56);
}
RS_HD uint32_t token_of(int t, bool red) {
  return (red && is_red_tile(t)) ? (uint32_t)(34 + red_index_of_kind(t >> 2)) : (uint32_t)(t >> 2);
}
// from scratch (deal, import): walk the set from the highest id down and
// shift each token in at the bottom, held red fives first (they sort last);
// the 16-byte register ends sorted with the pads on top
RS_HD void tokens_from_set(Hand& h, bool red) {
  uint64_t lo = TOK_PAD8, hi = TOK_PAD8;
  auto push = [&](uint32_t v) {
    hi = (hi << 8) | (lo >> 56);
    lo = (lo << 8) | v;
  };
  uint32_t w[5] = {h.w0, h.w1, h.w2, h.w3, h.w4};
  if (red) {
    if ((w[2] >> 24) & 1u) { push(36); w[2] &= ~(1u << 24); }  // tile 88
    if ((w[1] >> 20) & 1u) { push(35); w[1] &= ~(1u << 20); }  // tile 52
    if ((w[0] >> 16) & 1u) { push(34); w[0] &= ~(1u << 16); }  // tile 16
  }
#pragma unroll 1
  for (int i = 4; i >= 0; i--) {
    uint32_t x = w[i];
    while (x) {
      const int b = 31 - clz32(x);
      x &= ~(1u << b);
      push((uint32_t)((32 * i + b) >> 2));
    }
  }
  h.tlo = lo;
  h.thi = hi;
}

RS_HD uint32_t kind_pow_table(int k);  // below (table on the device)

// branchless accumulation of one dealt tile into the set and the suit codes
RS_HD void deal_tile(Hand& h, int t) {
  const uint32_t bit = 1u << (t & 31);
  const int wi = t >> 5;
  h.w0 |= wi == 0 ? bit : 0u;
  h.w1 |= wi == 1 ? bit : 0u;
  h.w2 |= wi == 2 ? bit : 0u;
  h.w3 |= wi == 3 ? bit : 0u;
  h.w4 |= wi == 4 ? bit : 0u;
  const int k = t >> 2, s = kind_suit(k);
  const uint32_t p = kind_pow_table(k);
  h.cm += s == 0 ? p : 0u;
  h.cp += s == 1 ? p : 0u;
  h.cs += s == 2 ? p : 0u;
  h.cz += s == 3 ? p : 0u;
}

#if defined(__CUDACC__)
// device copies of the class maps (per-device, set once) and the staged
// t3 | t1 | t2 block at the start of dynamic shared memory
__constant__ const uint8_t* c_suit_cls;
__constant__ const uint8_t* c_honor_cls;
__constant__ const uint8_t* c_tblock;  // the t3 | t1 | t2 | pow block in global memory
#endif
// the factored tables through the read-only cache (default) or from the
// shared-memory stage (-DRS_TABLES_SMEM, rs_tables.h)
#if !defined(RS_TABLES_SMEM) && defined(__CUDA_ARCH__)
#define RS_TBL(off) (c_tblock + (off))
#elif defined(__CUDA_ARCH__)
#define RS_TBL(off) (g_smem + (off))
#endif

RS_HD uint32_t class_of(const Tabs& T, int suit, uint32_t code) {
#if defined(__CUDA_ARCH__)
  return suit < 3 ? __ldg(c_suit_cls + code) : __ldg(c_honor_cls + code);
#else
  return suit < 3 ? T.suit_cls[code] : T.honor_cls[code];
#endif
}
RS_HD int t1_at(const Tabs& T, int i) {
#if defined(__CUDA_ARCH__)
  return RS_TBL(T1_OFF)[i];
#else
  return T.t1[i];
#endif
}
RS_HD int t2_at(const Tabs& T, int i) {
#if defined(__CUDA_ARCH__)
  return RS_TBL(T2_OFF)[i];
#else
  return T.t2[i];
#endif
}
RS_HD uint32_t t3_at(const Tabs& T, int i) {
#if defined(__CUDA_ARCH__)
  return reinterpret_cast<const uint32_t*>(RS_TBL(0))[i];
#else
  return T.t3[i];
#endif
}
RS_HD int cls_byte(uint32_t cls, int s) { return (cls >> (8 * s)) & 255; }
// base-5 code delta of one tile of kind k: computed in the hand updates of
// the step (no dependent load); the deal's 13 independent lookups read the
// table (fewer instructions in cold code: DESIGN §4 item 48)
RS_HD uint32_t kind_pow(int k) {
#if defined(__CUDA_ARCH__) && defined(RS_POW_TABLE)
  return reinterpret_cast<const uint32_t*>(RS_TBL(POW_OFF))[k];
#elif defined(__CUDA_ARCH__)
  return pow5_bits(k < 27 ? 8 - (k - 9 * (k / 9)) : 33 - k);
#else
  return kind_pow_calc(k);
#endif
}
RS_HD uint32_t kind_pow_table(int k) {
#if defined(__CUDA_ARCH__)
  return reinterpret_cast<const uint32_t*>(RS_TBL(POW_OFF))[k];
#else
  return kind_pow_calc(k);
#endif
}

// best value (2*sets + partials + head) at block budget `budget` (shanten.py:30-63)
RS_HD int std_best(const Tabs& T, int cm, int cp, int cs, int cz, int budget) {
  const int a = t1_at(T, cm * NS + cp);
  const int b = t2_at(T, cs * NH + cz);
  return (t3_at(T, a * NB + b) >> (4 * budget)) & 15;
}
RS_HD int std_shanten_cls(const Tabs& T, uint32_t cls, int melds) {
  const int budget = 4 - melds;
  return 2 * budget - std_best(T, cls_byte(cls, 0), cls_byte(cls, 1), cls_byte(cls, 2), cls_byte(cls, 3), budget);
}

// seven pairs (shanten.py:142-150) and thirteen orphans (:152-161) from the set
RS_HD int seven_pairs_shanten(const Hand& h) {
  const uint64_t present = h.kinds_ge(1), pairs = h.kinds_ge(2);
  const int kinds = popc64(present), np = popc64(pairs);
  return 6 - np + (7 - kinds > 0 ? 7 - kinds : 0);
}
RS_HD int kokushi_shanten(const Hand& h) {
  const int kinds = popc64(h.kinds_ge(1) & ORPHAN_MASK);
  const int has_pair = (h.kinds_ge(2) & ORPHAN_MASK) ? 1 : 0;
  return 13 - kinds - has_pair;
}
// seven pairs and thirteen orphans in one pass over the nibble counts,
// without gathering kind masks: a nibble count c >= 1 (>= 2) sets bit 3 of
// c + 7 (c + 6); orphan kinds select those bits per word
RS_HD void special_shanten(const Hand& h, int& seven, int& kokushi) {
  constexpr uint32_t OM[5] = {0x8u, 0x88u, 0x880u, 0x88888800u, 0x88u};
  int kinds = 0, pairs = 0, okinds = 0;
  uint32_t opair = 0;
#pragma unroll
  for (int w = 0; w < 5; w++) {
    const uint32_t c = nib_counts(h.word(w));
    const uint32_t pf = (c + 0x77777777u) & 0x88888888u, qf = (c + 0x66666666u) & 0x88888888u;
    kinds += popc32(pf);
    pairs += popc32(qf);
    okinds += popc32(pf & OM[w]);
    opair |= qf & OM[w];
  }
  seven = 6 - pairs + (7 - kinds > 0 ? 7 - kinds : 0);
  kokushi = 13 - okinds - (opair ? 1 : 0);
}
// shanten_codes (shanten.py:172-182)
RS_HD int full_shanten_impl(const Tabs& T, const Hand& h, int melds) {
  const int s = std_shanten_cls(T, h.cls, melds);
  // seven pairs / thirteen orphans count only for closed hands that are not
  // complete (shanten.py:172-182); evaluated unconditionally and selected
  // (the envs of a warp differ in melds, and most need it)
  int sp, kk;
  special_shanten(h, sp, kk);
  const int a = sp < s ? sp : s;
  const int b = (a > -1 && kk < a) ? kk : a;
  return (melds == 0 && s > -1) ? b : s;
}
// one out-of-line copy shared by every call site: the engine inlines its
// hand updates in many places, and eight inlined copies of the shanten
// evaluation made the executed code outgrow the instruction caches
// (DESIGN §4 item 24: +3 % at 4,096 envs); the hand crosses the call as
// scalars, so the caller's Hand stays in registers
RS_COLD int full_shanten_s(const Tabs& T, uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t w4,
                           uint32_t cls, int melds) {
  Hand h;
  h.w0 = w0; h.w1 = w1; h.w2 = w2; h.w3 = w3; h.w4 = w4;
  h.cls = cls;
  return full_shanten_impl(T, h, melds);
}
RS_HD int full_shanten(const Tabs& T, const Hand& h, int melds) {
  return full_shanten_s(T, h.w0, h.w1, h.w2, h.w3, h.w4, h.cls, melds);
}

// waits_from_codes (shanten.py:198-244) for a 13-form hand
RS_HD uint64_t compute_waits_impl(const Tabs& T, const Hand& h, int melds);
// the hand crosses the call as scalars (registers), so the caller's Hand is
// never materialised in local memory
RS_COLD uint64_t compute_waits_s(const Tabs& T, uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t w4,
                                 uint32_t cm, uint32_t cp, uint32_t cs, uint32_t cz, uint32_t cls, int melds) {
  Hand h;
  h.w0 = w0; h.w1 = w1; h.w2 = w2; h.w3 = w3; h.w4 = w4;
  h.cm = cm; h.cp = cp; h.cs = cs; h.cz = cz; h.cls = cls;
  return compute_waits_impl(T, h, melds);
}
RS_HD uint64_t compute_waits(const Tabs& T, const Hand& h, int melds) {
  return compute_waits_s(T, h.w0, h.w1, h.w2, h.w3, h.w4, h.cm, h.cp, h.cs, h.cz, h.cls, melds);
}
RS_HD uint64_t compute_waits_impl(const Tabs& T, const Hand& h, int melds) {
  RS_ACC(2);
  const int budget = 4 - melds, target = 2 * budget + 1;
  const int c0 = cls_byte(h.cls, 0), c1 = cls_byte(h.cls, 1), c2 = cls_byte(h.cls, 2), c3 = cls_byte(h.cls, 3);
  const int a_cur = t1_at(T, c0 * NS + c1), b_cur = t2_at(T, c2 * NH + c3);
  const uint64_t full = h.kinds_ge(4);
  uint64_t mask = 0;
  const int G = grp_size();
  if (G > 1) {
    // the lanes of the env's group split the 34 kinds
    for (int k = grp_sub(); k < 34; k += G) {
      if ((full >> k) & 1) continue;
      const int s = kind_suit(k);
      const int nc = (int)class_of(T, s, h.code(s) + kind_pow(k));
      int a = a_cur, b = b_cur;
      if (s == 0) a = t1_at(T, nc * NS + c1);
      else if (s == 1) a = t1_at(T, c0 * NS + nc);
      else if (s == 2) b = t2_at(T, nc * NH + c3);
      else b = t2_at(T, c2 * NH + nc);
      if ((int)((t3_at(T, a * NB + b) >> (4 * budget)) & 15) >= target) mask |= 1ull << k;
    }
    mask = grp_or64(mask);
  } else {
  // issue the 34 class loads independently: the suit codes are known
#pragma unroll
  for (int s = 0; s < 4; s++) {
    const int nd = s < 3 ? 9 : 7;
    const uint32_t code = h.code(s);
    uint32_t p = s < 3 ? 390625u : 15625u;
#pragma unroll
    for (int i = 0; i < 9; i++) {
      if (i < nd) {
        const int k = (s < 3 ? 9 * s : 27) + i;
        if (!((full >> k) & 1)) {
          const int nc = (int)class_of(T, s, code + p);
          int a = a_cur, b = b_cur;
          if (s == 0) a = t1_at(T, nc * NS + c1);
          else if (s == 1) a = t1_at(T, c0 * NS + nc);
          else if (s == 2) b = t2_at(T, nc * NH + c3);
          else b = t2_at(T, c2 * NH + nc);
          if ((int)((t3_at(T, a * NB + b) >> (4 * budget)) & 15) >= target) mask |= 1ull << k;
        }
        p /= 5u;
      }
    }
  }
  }
  if (melds == 0) {
    const uint64_t one = h.kinds_eq(1), two = h.kinds_eq(2), three_up = h.kinds_ge(3);
    if (!three_up && popc64(two) == 6 && popc64(one) == 1) mask |= one;
    const uint64_t present = h.kinds_ge(1);
    if (!(present & ~ORPHAN_MASK)) {
      const int np = popc64(present);
      if (np == 13) mask |= ORPHAN_MASK & ~full;
      else if (np == 12 && (h.kinds_ge(2) & ORPHAN_MASK)) mask |= ORPHAN_MASK & ~present;
    }
  }
  return mask;
}

// _finish_hand (state.py:31-39): shanten always, waits for 13-form tenpai
RS_HD void finish_hand(const Tabs& T, Hand& h) {
  RS_ACC(7);
  const int melds = hi::nmelds(h.info);
  const int sh = full_shanten(T, h, melds);
  h.info = hi::set_shanten(h.info, sh);
  h.waits = (sh == 0 && hi::nconc(h.info) + 3 * melds == 13) ? compute_waits(T, h, melds) : 0ull;
}

// add / remove one tile without the rebuild (hand_add / hand_remove parts);
// -DRS_OL_HANDOPS puts them out of line (A/B)
#if defined(RS_OL_HANDOPS)
#define RS_OL_HANDOP RS_COLD
#else
#define RS_OL_HANDOP RS_HD
#endif
// tok: 0 no-red tokens, 1 red-rule tokens, -1 scratch copy (tokens unused)
RS_OL_HANDOP void hand_put(const Tabs& T, Hand& h, int t, int tok) {
  RS_CHECK((unsigned)t < (unsigned)RS_NUM_TILES && !h.has(t) && hi::nconc(h.info) < 14);
  const int k = t >> 2, s = kind_suit(k);
  h.set_word(t >> 5, h.word(t >> 5) | (1u << (t & 31)));
  const uint32_t nc = h.code(s) + kind_pow(k);
  h.set_code(s, nc);
  h.cls = (h.cls & ~(255u << (8 * s))) | (class_of(T, s, nc) << (8 * s));
  h.info = hi::set_nconc(h.info, hi::nconc(h.info) + 1);
  if (tok >= 0) tok_insert(h.tlo, h.thi, token_of(t, tok == 1));
}
RS_OL_HANDOP void hand_take(const Tabs& T, Hand& h, int t, int tok) {
  RS_CHECK((unsigned)t < (unsigned)RS_NUM_TILES && h.has(t) && hi::nconc(h.info) > 0);
  const int k = t >> 2, s = kind_suit(k);
  h.set_word(t >> 5, h.word(t >> 5) & ~(1u << (t & 31)));
  const uint32_t nc = h.code(s) - kind_pow(k);
  h.set_code(s, nc);
  h.cls = (h.cls & ~(255u << (8 * s))) | (class_of(T, s, nc) << (8 * s));
  h.info = hi::set_nconc(h.info, hi::nconc(h.info) - 1);
  if (tok >= 0) tok_remove(h.tlo, h.thi, token_of(t, tok == 1));
}

// _shanten_minus_kind (engine.py:214-227)
RS_HD int shanten_minus_kind(const Tabs& T, const Hand& h, int k) {
  RS_ACC(3);
  Hand x = h;
  hand_take(T, x, x.lowest_of_kind(k), -1);
  return full_shanten(T, x, hi::nmelds(h.info));
}

// waits of an arbitrary count change, used by _kan_keeps_waits (engine.py:331-339)
RS_HD uint64_t waits_of(const Tabs& T, const Hand& h, int melds) {
  return compute_waits(T, h, melds);
}

}  // namespace rs
