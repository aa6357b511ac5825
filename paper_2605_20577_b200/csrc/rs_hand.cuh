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

  RS_HD uint32_t word(int i) const {
    return i == 0 ? w0 : i == 1 ? w1 : i == 2 ? w2 : i == 3 ? w3 : w4;
  }
  RS_HD void set_word(int i, uint32_t v) {
    if (i == 0) w0 = v;
    else if (i == 1) w1 = v;
    else if (i == 2) w2 = v;
    else if (i == 3) w3 = v;
    else w4 = v;
  }
  RS_HD bool has(int t) const { return (word(t >> 5) >> (t & 31)) & 1u; }
  RS_HD uint32_t nibble(int k) const { return (word(k >> 3) >> ((k & 7) * 4)) & 0xFu; }
  RS_HD int count(int k) const { return popc32(nibble(k)); }
  RS_HD int lowest_of_kind(int k) const { return 4 * k + ctz32(nibble(k)); }
  RS_HD uint32_t code(int s) const { return s == 0 ? cm : s == 1 ? cp : s == 2 ? cs : cz; }
  RS_HD void set_code(int s, uint32_t v) {
    if (s == 0) cm = v;
    else if (s == 1) cp = v;
    else if (s == 2) cs = v;
    else cz = v;
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

RS_HD Hand load_hand(const Soa& S, int e, int seat) {
  const uint32_t n = (uint32_t)S.n, s = (uint32_t)seat, x = (uint32_t)e;
  Hand h;
  const uint32_t* m = S.hmask + (s * 5u * n + x);
  h.w0 = m[0]; h.w1 = m[n]; h.w2 = m[2 * n]; h.w3 = m[3 * n]; h.w4 = m[4 * n];
  const uint32_t* c = S.hcode + (s * 4u * n + x);
  h.cm = c[0]; h.cp = c[n]; h.cs = c[2 * n]; h.cz = c[3 * n];
  h.cls = S.hcls[s * n + x];
  h.info = S.hinfo[s * n + x];
  h.waits = S.hwaits[s * n + x];
  return h;
}
RS_HD void store_hand(const Soa& S, int e, int seat, const Hand& h) {
  const uint32_t n = (uint32_t)S.n, s = (uint32_t)seat, x = (uint32_t)e;
  uint32_t* m = S.hmask + (s * 5u * n + x);
  m[0] = h.w0; m[n] = h.w1; m[2 * n] = h.w2; m[3 * n] = h.w3; m[4 * n] = h.w4;
  uint32_t* c = S.hcode + (s * 4u * n + x);
  c[0] = h.cm; c[n] = h.cp; c[2 * n] = h.cs; c[3 * n] = h.cz;
  S.hcls[s * n + x] = h.cls;
  S.hinfo[s * n + x] = h.info;
  S.hwaits[s * n + x] = h.waits;
}

#if defined(__CUDACC__)
// device copies of the class maps (per-device, set once) and the staged
// t3 | t1 | t2 block at the start of dynamic shared memory
__constant__ const uint8_t* c_suit_cls;
__constant__ const uint8_t* c_honor_cls;
extern __shared__ __align__(16) uint8_t g_smem[];
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
  return g_smem[T1_OFF + i];
#else
  return T.t1[i];
#endif
}
RS_HD int t2_at(const Tabs& T, int i) {
#if defined(__CUDA_ARCH__)
  return g_smem[T2_OFF + i];
#else
  return T.t2[i];
#endif
}
RS_HD uint32_t t3_at(const Tabs& T, int i) {
#if defined(__CUDA_ARCH__)
  return reinterpret_cast<const uint32_t*>(g_smem)[i];
#else
  return T.t3[i];
#endif
}
RS_HD int cls_byte(uint32_t cls, int s) { return (cls >> (8 * s)) & 255; }
// base-5 code delta of one tile of kind k (staged table on the device)
RS_HD uint32_t kind_pow(int k) {
#if defined(__CUDA_ARCH__)
  return reinterpret_cast<const uint32_t*>(g_smem + POW_OFF)[k];
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
// shanten_codes (shanten.py:172-182)
RS_HD int full_shanten(const Tabs& T, const Hand& h, int melds) {
  int s = std_shanten_cls(T, h.cls, melds);
  if (melds == 0 && s > -1) {
    const int sp = seven_pairs_shanten(h);
    if (sp < s) s = sp;
    if (s > -1) {
      const int kk = kokushi_shanten(h);
      if (kk < s) s = kk;
    }
  }
  return s;
}

// waits_from_codes (shanten.py:198-244) for a 13-form hand
RS_COLD uint64_t compute_waits(const Tabs& T, const Hand& h, int melds) {
  const int budget = 4 - melds, target = 2 * budget + 1;
  const int c0 = cls_byte(h.cls, 0), c1 = cls_byte(h.cls, 1), c2 = cls_byte(h.cls, 2), c3 = cls_byte(h.cls, 3);
  const int a_cur = t1_at(T, c0 * NS + c1), b_cur = t2_at(T, c2 * NH + c3);
  const uint64_t full = h.kinds_ge(4);
  uint64_t mask = 0;
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
  const int melds = hi::nmelds(h.info);
  const int sh = full_shanten(T, h, melds);
  h.info = hi::set_shanten(h.info, sh);
  h.waits = (sh == 0 && hi::nconc(h.info) + 3 * melds == 13) ? compute_waits(T, h, melds) : 0ull;
}

// add / remove one tile without the rebuild (hand_add / hand_remove parts)
RS_HD void hand_put(const Tabs& T, Hand& h, int t) {
  const int k = t >> 2, s = kind_suit(k);
  h.set_word(t >> 5, h.word(t >> 5) | (1u << (t & 31)));
  const uint32_t nc = h.code(s) + kind_pow(k);
  h.set_code(s, nc);
  h.cls = (h.cls & ~(255u << (8 * s))) | (class_of(T, s, nc) << (8 * s));
  h.info = hi::set_nconc(h.info, hi::nconc(h.info) + 1);
}
RS_HD void hand_take(const Tabs& T, Hand& h, int t) {
  const int k = t >> 2, s = kind_suit(k);
  h.set_word(t >> 5, h.word(t >> 5) & ~(1u << (t & 31)));
  const uint32_t nc = h.code(s) - kind_pow(k);
  h.set_code(s, nc);
  h.cls = (h.cls & ~(255u << (8 * s))) | (class_of(T, s, nc) << (8 * s));
  h.info = hi::set_nconc(h.info, hi::nconc(h.info) - 1);
}

// _shanten_minus_kind (engine.py:214-227)
RS_COLD int shanten_minus_kind(const Tabs& T, const Hand& h, int k) {
  Hand x = h;
  hand_take(T, x, x.lowest_of_kind(k));
  return full_shanten(T, x, hi::nmelds(h.info));
}

// waits of an arbitrary count change, used by _kan_keeps_waits (engine.py:331-339)
RS_HD uint64_t waits_of(const Tabs& T, const Hand& h, int melds) {
  return compute_waits(T, h, melds);
}

}  // namespace rs
