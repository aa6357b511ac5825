/*
 * mjoracle.c — CPU ORACLE (test infrastructure only; see mjoracle.h).
 *
 * Scalar C restatement of the reference `mjsim` engine.  Mutable state,
 * sorted-id hands, full event/result history — deliberately the simplest
 * faithful restatement, not a fast design.  Paths in citations are relative
 * to the reference's pkg/src/mjsim/.
 */
#include "mjoracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ull
#define NEG (-99)

/* ------------------------------------------------------------------ rng */

/* rng.py:18-25 */
uint64_t orc_mix(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
/* rng.py:38-41 */
uint64_t orc_derive_key(uint64_t key, uint64_t stream) {
  return orc_mix((key ^ GOLDEN) + orc_mix(stream));
}
/* rng.py:33-35 */
uint64_t orc_seed_key(uint64_t seed) { return orc_mix(seed); }
/* bench/runner.py:25-28 */
uint64_t orc_env_game_seed(uint64_t seed, uint64_t index, uint64_t reset) {
  uint64_t env_key = orc_derive_key(orc_seed_key(seed), index);
  return orc_derive_key(env_key, 2 + reset);
}
/* bench/runner.py:31-33 */
uint64_t orc_env_policy_key(uint64_t seed, uint64_t index) {
  uint64_t env_key = orc_derive_key(orc_seed_key(seed), index);
  return orc_derive_key(env_key, 1);
}

typedef struct { uint64_t key, counter; } ORng;

/* rng.py:48-50 */
static uint64_t o_next_u64(ORng* r) {
  r->counter += 1;
  return orc_mix(r->key + r->counter * GOLDEN);
}
/* rng.py:53-56 */
static uint64_t o_randbelow(ORng* r, uint64_t n) {
  uint64_t x = o_next_u64(r);
  return (uint64_t)(((unsigned __int128)x * n) >> 64);
}
uint64_t orc_randbelow(uint64_t* kc, uint64_t n) {
  ORng r = {kc[0], kc[1]};
  uint64_t v = o_randbelow(&r, n);
  kc[1] = r.counter;
  return v;
}
/* rng.py:59-65 + tiles.py:142-144 */
static void o_shuffle136(ORng* r, uint8_t* out) {
  for (int i = 0; i < 136; i++) out[i] = (uint8_t)i;
  for (int i = 135; i > 0; i--) {
    int j = (int)o_randbelow(r, (uint64_t)(i + 1));
    uint8_t t = out[i];
    out[i] = out[j];
    out[j] = t;
  }
}
void orc_shuffle136(uint64_t key, uint64_t counter, uint8_t* out, uint64_t* counter_out) {
  ORng r = {key, counter};
  o_shuffle136(&r, out);
  if (counter_out) *counter_out = r.counter;
}

/* --------------------------------------------------------------- tables */

#define SUIT_CODES 1953125
#define HONOR_CODES 78125
static int8_t* g_suit_vals;
static int8_t* g_honor_vals;
static uint32_t g_crc;
static uint64_t* g_suit_words; /* legal codes only, ascending */
static uint64_t* g_honor_words;
static int64_t g_n_suit_words, g_n_honor_words;

/* hand/tables.py:51-120 (_fill_stats) */
static void o_fill_stats(int n_digits, int allow_runs, int8_t* dp, int64_t ncodes) {
  int64_t pow5[9];
  int64_t p = 1;
  for (int i = n_digits - 1; i >= 0; i--) { pow5[i] = p; p *= 5; }
  for (int j = 0; j < 10; j++) dp[j] = -1;
  dp[0] = 0;
  for (int64_t code = 1; code < ncodes; code++) {
    int i = 0;
    while ((code / pow5[i]) % 5 == 0) i++;
    int d = (int)((code / pow5[i]) % 5);
    int8_t* row = dp + code * 10;
    for (int j = 0; j < 10; j++) row[j] = -1;
    const int8_t* child = dp + (code - pow5[i]) * 10;
    for (int j = 0; j < 10; j++) if (child[j] > row[j]) row[j] = child[j];
    if (d >= 2) {
      child = dp + (code - 2 * pow5[i]) * 10;
      for (int h = 0; h < 2; h++)
        for (int s = 0; s < 5; s++) {
          int q = child[h * 5 + s];
          if (q < 0) continue;
          if (h == 0 && q > row[5 + s]) row[5 + s] = (int8_t)q;
          int q2 = q < 4 ? q + 1 : 4;
          if (q2 > row[h * 5 + s]) row[h * 5 + s] = (int8_t)q2;
        }
    }
    if (d >= 3) {
      child = dp + (code - 3 * pow5[i]) * 10;
      for (int h = 0; h < 2; h++)
        for (int s = 0; s < 4; s++) {
          int q = child[h * 5 + s];
          if (q >= 0 && q > row[h * 5 + s + 1]) row[h * 5 + s + 1] = (int8_t)q;
        }
    }
    if (allow_runs) {
      if (i + 2 < n_digits && (code / pow5[i + 1]) % 5 > 0 && (code / pow5[i + 2]) % 5 > 0) {
        child = dp + (code - pow5[i] - pow5[i + 1] - pow5[i + 2]) * 10;
        for (int h = 0; h < 2; h++)
          for (int s = 0; s < 4; s++) {
            int q = child[h * 5 + s];
            if (q >= 0 && q > row[h * 5 + s + 1]) row[h * 5 + s + 1] = (int8_t)q;
          }
      }
      if (i + 1 < n_digits && (code / pow5[i + 1]) % 5 > 0) {
        child = dp + (code - pow5[i] - pow5[i + 1]) * 10;
        for (int h = 0; h < 2; h++)
          for (int s = 0; s < 5; s++) {
            int q = child[h * 5 + s];
            if (q >= 0) {
              int q2 = q < 4 ? q + 1 : 4;
              if (q2 > row[h * 5 + s]) row[h * 5 + s] = (int8_t)q2;
            }
          }
      }
      if (i + 2 < n_digits && (code / pow5[i + 2]) % 5 > 0) {
        child = dp + (code - pow5[i] - pow5[i + 2]) * 10;
        for (int h = 0; h < 2; h++)
          for (int s = 0; s < 5; s++) {
            int q = child[h * 5 + s];
            if (q >= 0) {
              int q2 = q < 4 ? q + 1 : 4;
              if (q2 > row[h * 5 + s]) row[h * 5 + s] = (int8_t)q2;
            }
          }
      }
    }
  }
}

/* hand/tables.py:123-147 (_pack_words) */
static uint64_t o_pack_word(const int8_t* row) {
  uint64_t word = 0;
  for (int m = 0; m < 5; m++)
    for (int h = 0; h < 2; h++) {
      int best_v = -1, best_s = 0, best_p = 0;
      for (int s = 0; s <= m; s++) {
        int q = row[h * 5 + s];
        if (q < 0) continue;
        int pe = q < m - s ? q : m - s;
        int v = 2 * s + pe;
        if (v > best_v || (v == best_v && s > best_s)) { best_v = v; best_s = s; best_p = pe; }
      }
      uint64_t sub = best_v < 0 ? 0x3F : (uint64_t)(best_s | (best_p << 3));
      word |= sub << (6 * (m * 2 + h));
    }
  return word;
}

static int o_digit_sum(int64_t code, int n_digits) {
  int t = 0;
  for (int i = 0; i < n_digits; i++) { t += (int)(code % 5); code /= 5; }
  return t;
}

/* hand/tables.py:169-178 (_values_from_words) */
static void o_values_from_word(uint64_t w, int8_t* vals) {
  for (int idx = 0; idx < 10; idx++) {
    uint64_t sub = (w >> (6 * idx)) & 0x3F;
    int s = (int)(sub & 7), p = (int)(sub >> 3);
    vals[idx] = sub == 0x3F ? (int8_t)NEG : (int8_t)(2 * s + p);
  }
}

static uint32_t o_crc32(const uint8_t* data, int64_t n, uint32_t crc) {
  static uint32_t table[256];
  static int init = 0;
  if (!init) {
    for (uint32_t i = 0; i < 256; i++) {
      uint32_t c = i;
      for (int k = 0; k < 8; k++) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[i] = c;
    }
    init = 1;
  }
  crc = ~crc;
  for (int64_t i = 0; i < n; i++) crc = table[(crc ^ data[i]) & 0xFF] ^ (crc >> 8);
  return ~crc;
}

static void o_build_one(int n_digits, int allow_runs, int64_t ncodes, int8_t** vals_out,
                        uint64_t** words_out, int64_t* nwords) {
  int8_t* dp = (int8_t*)malloc((size_t)ncodes * 10);
  o_fill_stats(n_digits, allow_runs, dp, ncodes);
  int8_t* vals = (int8_t*)malloc((size_t)ncodes * 10);
  uint64_t* words = (uint64_t*)malloc((size_t)ncodes * 8);
  int64_t nw = 0;
  /* tables.py:191-209: illegal codes (digit sum > 14) are zeroed */
  for (int64_t c = 0; c < ncodes; c++) {
    uint64_t w = 0;
    if (o_digit_sum(c, n_digits) <= 14) {
      w = o_pack_word(dp + c * 10);
      words[nw++] = w;
    }
    o_values_from_word(w, vals + c * 10);
  }
  free(dp);
  *vals_out = vals;
  *words_out = words;
  *nwords = nw;
}

/* hand/tables.py:212-224 (build_tables) + 227-240 (blob crc) */
int orc_tables_build(void) {
  if (g_suit_vals) return 0;
  o_build_one(9, 1, SUIT_CODES, &g_suit_vals, &g_suit_words, &g_n_suit_words);
  o_build_one(7, 0, HONOR_CODES, &g_honor_vals, &g_honor_words, &g_n_honor_words);
  uint8_t buf[8];
  uint32_t crc = 0;
  for (int64_t i = 0; i < g_n_suit_words; i++) {
    for (int b = 0; b < 8; b++) buf[b] = (uint8_t)(g_suit_words[i] >> (8 * b));
    crc = o_crc32(buf, 8, crc);
  }
  for (int64_t i = 0; i < g_n_honor_words; i++) {
    for (int b = 0; b < 8; b++) buf[b] = (uint8_t)(g_honor_words[i] >> (8 * b));
    crc = o_crc32(buf, 8, crc);
  }
  g_crc = crc;
  return 0;
}
uint32_t orc_tables_crc(void) { orc_tables_build(); return g_crc; }
const int8_t* orc_suit_vals(void) { orc_tables_build(); return g_suit_vals; }
const int8_t* orc_honor_vals(void) { orc_tables_build(); return g_honor_vals; }

/* docs/formats.md:54-74 blob layout */
int64_t orc_tables_blob(uint8_t* out, int64_t cap) {
  orc_tables_build();
  int64_t size = 24 + 8 * (g_n_suit_words + g_n_honor_words);
  if (!out || cap < size) return size;
  memcpy(out, "MJSUIT1\0", 8);
  uint32_t hdr[4] = {(uint32_t)g_n_suit_words, (uint32_t)g_n_honor_words, g_crc, 0};
  for (int i = 0; i < 4; i++)
    for (int b = 0; b < 4; b++) out[8 + 4 * i + b] = (uint8_t)(hdr[i] >> (8 * b));
  uint8_t* p = out + 24;
  for (int64_t i = 0; i < g_n_suit_words; i++)
    for (int b = 0; b < 8; b++) *p++ = (uint8_t)(g_suit_words[i] >> (8 * b));
  for (int64_t i = 0; i < g_n_honor_words; i++)
    for (int b = 0; b < 8; b++) *p++ = (uint8_t)(g_honor_words[i] >> (8 * b));
  return size;
}

/* -------------------------------------------------------------- shanten */

static const int POW5_SUIT[9] = {390625, 78125, 15625, 3125, 625, 125, 25, 5, 1};
static const int POW5_HONOR[7] = {15625, 3125, 625, 125, 25, 5, 1};
static const int ORPHANS[13] = {0, 8, 9, 17, 18, 26, 27, 28, 29, 30, 31, 32, 33};

static int o_is_orphan(int k) { return k >= 27 || k % 9 == 0 || k % 9 == 8; }
static int o_is_terminal(int k) { return k < 27 && (k % 9 == 0 || k % 9 == 8); }

/* hand/shanten.py:30-63 (_std_best) */
static int o_std_best(int cm, int cp, int cs, int cz, int budget) {
  int a0[5], a1[5], n0[5], n1[5];
  const int8_t* row = g_suit_vals + (int64_t)cm * 10;
  for (int b = 0; b <= budget; b++) { a0[b] = row[b * 2]; a1[b] = row[b * 2 + 1]; }
  for (int g = 0; g < 3; g++) {
    if (g == 0) row = g_suit_vals + (int64_t)cp * 10;
    else if (g == 1) row = g_suit_vals + (int64_t)cs * 10;
    else row = g_honor_vals + (int64_t)cz * 10;
    for (int b = 0; b <= budget; b++) { n0[b] = NEG; n1[b] = NEG; }
    for (int b = 0; b <= budget; b++)
      for (int k = 0; k <= b; k++) {
        int v0 = row[k * 2], v1 = row[k * 2 + 1];
        if (v0 > NEG) {
          if (a0[b - k] > NEG && a0[b - k] + v0 > n0[b]) n0[b] = a0[b - k] + v0;
          if (a1[b - k] > NEG && a1[b - k] + v0 > n1[b]) n1[b] = a1[b - k] + v0;
        }
        if (v1 > NEG && a0[b - k] > NEG && a0[b - k] + v1 > n1[b]) n1[b] = a0[b - k] + v1;
      }
    for (int b = 0; b <= budget; b++) { a0[b] = n0[b]; a1[b] = n1[b]; }
  }
  int best = a0[budget];
  if (a1[budget] > NEG && a1[budget] + 1 > best) best = a1[budget] + 1;
  return best;
}

/* hand/shanten.py:98-106 (codes_from_counts) */
static void o_codes(const uint8_t* c, int* codes) {
  int cm = 0, cp = 0, cs = 0, cz = 0;
  for (int i = 0; i < 9; i++) {
    cm = cm * 5 + c[i];
    cp = cp * 5 + c[9 + i];
    cs = cs * 5 + c[18 + i];
  }
  for (int i = 0; i < 7; i++) cz = cz * 5 + c[27 + i];
  codes[0] = cm; codes[1] = cp; codes[2] = cs; codes[3] = cz;
}

/* hand/shanten.py:129-133 */
static int o_std_codes(const int* codes, int melds) {
  int budget = 4 - melds;
  return 2 * budget - o_std_best(codes[0], codes[1], codes[2], codes[3], budget);
}
/* hand/shanten.py:142-150 */
static int o_seven_pairs(const uint8_t* c) {
  int pairs = 0, kinds = 0;
  for (int k = 0; k < 34; k++)
    if (c[k]) { kinds++; if (c[k] >= 2) pairs++; }
  return 6 - pairs + (7 - kinds > 0 ? 7 - kinds : 0);
}
/* hand/shanten.py:153-161 */
static int o_kokushi(const uint8_t* c) {
  int kinds = 0, has_pair = 0;
  for (int i = 0; i < 13; i++)
    if (c[ORPHANS[i]]) { kinds++; if (c[ORPHANS[i]] >= 2) has_pair = 1; }
  return 13 - kinds - has_pair;
}
/* hand/shanten.py:172-182 (shanten_codes) */
static int o_shanten_codes(const int* codes, const uint8_t* c, int melds) {
  int s = o_std_codes(codes, melds);
  if (melds == 0 && s > -1) {
    int sp = o_seven_pairs(c);
    if (sp < s) s = sp;
    if (s > -1) {
      int kk = o_kokushi(c);
      if (kk < s) s = kk;
    }
  }
  return s;
}
int orc_shanten(const uint8_t* c, int melds) {
  orc_tables_build();
  int codes[4];
  o_codes(c, codes);
  return o_shanten_codes(codes, c, melds);
}
int orc_shanten_standard(const uint8_t* c, int melds) {
  orc_tables_build();
  int codes[4];
  o_codes(c, codes);
  return o_std_codes(codes, melds);
}

/* hand/shanten.py:69-89 + 198-244 (waits_from_codes) */
static uint64_t o_waits_codes(const int* codes, const uint8_t* c, int melds) {
  int budget = 4 - melds, target = 2 * budget + 1;
  uint64_t mask = 0;
  for (int k = 0; k < 34; k++) {
    if (c[k] >= 4) continue;
    int cc[4] = {codes[0], codes[1], codes[2], codes[3]};
    if (k < 9) cc[0] += POW5_SUIT[k];
    else if (k < 18) cc[1] += POW5_SUIT[k - 9];
    else if (k < 27) cc[2] += POW5_SUIT[k - 18];
    else cc[3] += POW5_HONOR[k - 27];
    if (o_std_best(cc[0], cc[1], cc[2], cc[3], budget) >= target) mask |= 1ull << k;
  }
  if (melds == 0) {
    int pairs = 0, single = -1, ok = 1;
    for (int k = 0; k < 34; k++) {
      if (c[k] == 2) pairs++;
      else if (c[k] == 1) single = k;
      else if (c[k] != 0) ok = 0;
    }
    if (ok && pairs == 6 && single >= 0) mask |= 1ull << single;
    int present = 0, has_pair = 0, clean = 1;
    for (int k = 0; k < 34; k++) {
      if (!c[k]) continue;
      if (o_is_orphan(k)) { present++; if (c[k] >= 2) has_pair = 1; }
      else clean = 0;
    }
    if (clean) {
      if (present == 13) {
        for (int i = 0; i < 13; i++) if (c[ORPHANS[i]] < 4) mask |= 1ull << ORPHANS[i];
      } else if (present == 12 && has_pair) {
        for (int i = 0; i < 13; i++) if (c[ORPHANS[i]] == 0) mask |= 1ull << ORPHANS[i];
      }
    }
  }
  return mask;
}
uint64_t orc_waits(const uint8_t* c, int melds) {
  orc_tables_build();
  int codes[4];
  o_codes(c, codes);
  return o_waits_codes(codes, c, melds);
}

/* ------------------------------------------------------------ decompose */

/* hand/decompose.py:24-68.  A set key is is_triplet*64 + start, so that
 * ascending keys reproduce Python's tuple order ("run" < "triplet"). */
typedef struct { int pair; int n; int keys[4]; } ODec;

static void o_sets_rec(uint8_t* c, int needed, int* cur, int depth, ODec* out, int* nout,
                       int cap, int pair) {
  if (needed == 0) {
    for (int k = 0; k < 34; k++) if (c[k]) return;
    if (*nout >= cap) return;
    ODec d;
    d.pair = pair;
    d.n = depth;
    for (int i = 0; i < depth; i++) d.keys[i] = cur[i];
    /* sorted(sets) */
    for (int i = 1; i < d.n; i++)
      for (int j = i; j > 0 && d.keys[j - 1] > d.keys[j]; j--) {
        int t = d.keys[j]; d.keys[j] = d.keys[j - 1]; d.keys[j - 1] = t;
      }
    /* de-duplicate (results is a set in the reference) */
    for (int i = 0; i < *nout; i++) {
      if (out[i].pair != d.pair || out[i].n != d.n) continue;
      int same = 1;
      for (int j = 0; j < d.n; j++) if (out[i].keys[j] != d.keys[j]) { same = 0; break; }
      if (same) return;
    }
    out[(*nout)++] = d;
    return;
  }
  int i = 0;
  while (i < 34 && c[i] == 0) i++;
  if (i == 34) return;
  if (c[i] >= 3) {
    c[i] -= 3;
    cur[depth] = 64 + i;
    o_sets_rec(c, needed - 1, cur, depth + 1, out, nout, cap, pair);
    c[i] += 3;
  }
  if (i < 27 && i % 9 <= 6 && c[i + 1] && c[i + 2]) {
    c[i]--; c[i + 1]--; c[i + 2]--;
    cur[depth] = i;
    o_sets_rec(c, needed - 1, cur, depth + 1, out, nout, cap, pair);
    c[i]++; c[i + 1]++; c[i + 2]++;
  }
}

static int o_dec_cmp(const void* a, const void* b) {
  const ODec* x = (const ODec*)a;
  const ODec* y = (const ODec*)b;
  if (x->pair != y->pair) return x->pair - y->pair;
  for (int i = 0; i < x->n && i < y->n; i++)
    if (x->keys[i] != y->keys[i]) return x->keys[i] - y->keys[i];
  return x->n - y->n;
}

static int o_decompose(const uint8_t* counts, int melds, ODec* out, int cap) {
  uint8_t w[34];
  memcpy(w, counts, 34);
  int needed = 4 - melds, n = 0, cur[4];
  for (int pair = 0; pair < 34; pair++) {
    if (w[pair] < 2) continue;
    w[pair] -= 2;
    o_sets_rec(w, needed, cur, 0, out, &n, cap, pair);
    w[pair] += 2;
  }
  qsort(out, (size_t)n, sizeof(ODec), o_dec_cmp);
  return n;
}
int orc_decompose(const uint8_t* counts, int melds, int32_t* out, int cap) {
  ODec d[64];
  int n = o_decompose(counts, melds, d, 64);
  int w = 0;
  for (int i = 0; i < n; i++) {
    if (w + 1 + d[i].n > cap) break;
    out[w++] = d[i].pair;
    for (int j = 0; j < d[i].n; j++) out[w++] = d[i].keys[j];
  }
  return n;
}

/* -------------------------------------------------------------- scoring */

enum {
  Y_RIICHI = 0, Y_DOUBLE_RIICHI, Y_IPPATSU, Y_MENZEN_TSUMO, Y_PINFU, Y_TANYAO,
  Y_WHITE, Y_GREEN, Y_RED, Y_SEAT, Y_ROUND, Y_SANSHOKU_DOUJUN, Y_SANSHOKU_DOUKOU,
  Y_ITTSU, Y_CHANTA, Y_JUNCHAN, Y_TOITOI, Y_SANANKOU, Y_SANKANTSU, Y_CHIITOITSU,
  Y_HONROUTOU, Y_SHOUSANGEN, Y_HONITSU, Y_CHINITSU, Y_HAITEI, Y_HOUTEI, Y_RINSHAN,
  Y_CHANKAN, Y_KOKUSHI, Y_SUUANKOU, Y_DAISANGEN, Y_SHOUSUUSHI, Y_DAISUUSHI,
  Y_TSUUIISOU, Y_CHINROUTOU, Y_RYUUIISOU, Y_CHUUREN, Y_SUUKANTSU, Y_TENHOU, Y_CHIIHOU
};

enum { W_RYANMEN = 0, W_KANCHAN, W_PENCHAN, W_SHANPON, W_TANKI };

/* scoring/context.py:60-73 (YakuList) in entry order */
typedef struct { int n; int id[24]; int han[24]; int yakuman; } OYaku;
static void oy_add(OYaku* y, int id, int han) { y->id[y->n] = id; y->han[y->n] = han; y->n++; }
static int oy_han(const OYaku* y) { int t = 0; for (int i = 0; i < y->n; i++) t += y->han[i]; return t; }
static int oy_has(const OYaku* y, int id) { for (int i = 0; i < y->n; i++) if (y->id[i] == id) return 1; return 0; }

static int o_ctx_closed(const orc_winctx* c) {
  for (int i = 0; i < c->n_melds; i++) if (c->melds[i].type != 3) return 0;
  return 1;
}
static int o_meld_base_kind(const rs_meld_rec* m) { return m->tiles[0] >> 2; }
static int o_meld_is_kan(const rs_meld_rec* m) { return m->type >= 2; }

/* tiles.py:108-115 */
static int o_dora_kind(int ind) {
  if (ind < 27) return ind - ind % 9 + (ind % 9 + 1) % 9;
  if (ind < 31) return 27 + (ind - 27 + 1) % 4;
  return 31 + (ind - 31 + 1) % 3;
}

/* scoring/dora.py:9-26 */
static void o_dora_parts(const orc_winctx* c, int* dora, int* ura, int* reds) {
  int kc[34] = {0};
  *reds = 0;
  for (int i = 0; i < c->n_ids; i++) {
    int t = c->ids[i];
    kc[t >> 2]++;
    if (c->rule == RS_RULE_RED && (t == 16 || t == 52 || t == 88)) (*reds)++;
  }
  *dora = 0;
  for (int i = 0; i < c->n_dora; i++) *dora += kc[o_dora_kind(c->dora[i] >> 2)];
  *ura = 0;
  if (c->riichi)
    for (int i = 0; i < c->n_ura; i++) *ura += kc[o_dora_kind(c->ura[i] >> 2)];
}

/* scoring/yaku.py:130-155 (_Block, blocks_of) */
typedef struct { int run, start, open, kan, ron_completed; } OBlock;
static int o_blocks(const ODec* d, const orc_winctx* c, int wait_block, OBlock* b) {
  int n = 0;
  for (int i = 0; i < d->n; i++) {
    int run = d->keys[i] < 64;
    int start = d->keys[i] & 63;
    OBlock x = {run, start, 0, 0, (!c->tsumo && i == wait_block && !run)};
    b[n++] = x;
  }
  for (int i = 0; i < c->n_melds; i++) {
    const rs_meld_rec* m = &c->melds[i];
    OBlock x = {m->type == 0, o_meld_base_kind(m), m->type != 3, o_meld_is_kan(m), 0};
    b[n++] = x;
  }
  return n;
}

/* scoring/yaku.py:158-174 */
static int o_wait_placements(const ODec* d, int k, int* blk, int* shape) {
  int n = 0;
  for (int i = 0; i < d->n; i++) {
    int run = d->keys[i] < 64, start = d->keys[i] & 63;
    if (run) {
      if (start == k) { blk[n] = i; shape[n++] = k % 9 <= 5 ? W_RYANMEN : W_PENCHAN; }
      else if (start + 1 == k) { blk[n] = i; shape[n++] = W_KANCHAN; }
      else if (start + 2 == k) { blk[n] = i; shape[n++] = k % 9 >= 3 ? W_RYANMEN : W_PENCHAN; }
    } else if (start == k) { blk[n] = i; shape[n++] = W_SHANPON; }
  }
  if (d->pair == k) { blk[n] = -1; shape[n++] = W_TANKI; }
  return n;
}

/* scoring/yaku.py:313-334 */
static int o_chuuren(const orc_winctx* c) {
  if (c->n_melds || !o_ctx_closed(c)) return 0;
  const uint8_t* cnt = c->concealed;
  int suit = -1;
  for (int k = 0; k < 27; k++)
    if (cnt[k]) {
      if (suit < 0) suit = k / 9;
      else if (suit != k / 9) return 0;
    }
  if (suit < 0) return 0;
  for (int k = 27; k < 34; k++) if (cnt[k]) return 0;
  static const int base[9] = {3, 1, 1, 1, 1, 1, 1, 1, 3};
  int s = suit * 9, extra = -1;
  for (int i = 0; i < 9; i++) {
    int d = cnt[s + i] - base[i];
    if (d == 0) continue;
    if (d == 1 && extra < 0) extra = i;
    else return 0;
  }
  if (extra < 0) return 0;
  return s + extra == (c->win_tile >> 2) ? 2 : 1;
}

static void o_situational(const orc_winctx* c, OYaku* y) {
  if (c->last_tile) oy_add(y, c->tsumo ? Y_HAITEI : Y_HOUTEI, 1);
  if (c->rinshan) oy_add(y, Y_RINSHAN, 1);
  if (c->chankan) oy_add(y, Y_CHANKAN, 1);
}

static int o_green(int k) { return k == 19 || k == 20 || k == 21 || k == 23 || k == 25 || k == 32; }

/* scoring/yaku.py:188-301 (detect_standard) */
static void o_detect_standard(const orc_winctx* c, const ODec* d, int wait_block, int wait, OYaku* y) {
  OBlock b[8];
  int nb = o_blocks(d, c, wait_block, b);
  int closed = o_ctx_closed(c), tsumo = c->tsumo, pair = d->pair;
  int present[34] = {0}, trip[34] = {0};
  int concealed_trips = 0, kans = 0, all_trip = 1, run_start[34] = {0}, has_run = 0;
  for (int i = 0; i < nb; i++) {
    if (b[i].run) {
      present[b[i].start] = present[b[i].start + 1] = present[b[i].start + 2] = 1;
      run_start[b[i].start] = 1;
      all_trip = 0;
      has_run = 1;
    } else {
      present[b[i].start] = 1;
      trip[b[i].start] = 1;
      if (!b[i].open && !b[i].ron_completed) concealed_trips++;
    }
    if (b[i].kan) kans++;
  }
  present[pair] = 1;
  memset(y, 0, sizeof(*y));
  /* yakuman, reference order yaku.py:206-232 */
  if (c->first_draw && tsumo && c->n_melds == 0)
    oy_add(y, c->seat_wind == 27 ? Y_TENHOU : Y_CHIIHOU, 1);
  if (concealed_trips == 4) oy_add(y, Y_SUUANKOU, (c->double_yakuman && wait == W_TANKI) ? 2 : 1);
  if (trip[31] && trip[32] && trip[33]) oy_add(y, Y_DAISANGEN, 1);
  int wind_trips = trip[27] + trip[28] + trip[29] + trip[30];
  if (wind_trips == 4) oy_add(y, Y_DAISUUSHI, c->double_yakuman ? 2 : 1);
  else if (wind_trips == 3 && pair >= 27 && pair <= 30) oy_add(y, Y_SHOUSUUSHI, 1);
  int all_honor = 1, all_term = 1, all_green = 1, all_simple = 1, outside_any_honor = 0;
  for (int k = 0; k < 34; k++)
    if (present[k]) {
      if (k < 27) all_honor = 0;
      if (!o_is_terminal(k)) all_term = 0;
      if (!o_green(k)) all_green = 0;
      if (o_is_orphan(k)) all_simple = 0;
      if (k >= 27) outside_any_honor = 1;
    }
  if (all_honor) oy_add(y, Y_TSUUIISOU, 1);
  if (all_term) oy_add(y, Y_CHINROUTOU, 1);
  if (all_green) oy_add(y, Y_RYUUIISOU, 1);
  if (kans == 4) oy_add(y, Y_SUUKANTSU, 1);
  int ch = o_chuuren(c);
  if (ch) oy_add(y, Y_CHUUREN, (c->double_yakuman && ch == 2) ? 2 : 1);
  if (y->n) {
    int t = 0;
    for (int i = 0; i < y->n; i++) t += y->han[i];
    y->yakuman = t;
    return;
  }
  if (c->riichi == 2) oy_add(y, Y_DOUBLE_RIICHI, 2);
  else if (c->riichi == 1) oy_add(y, Y_RIICHI, 1);
  if (c->ippatsu) oy_add(y, Y_IPPATSU, 1);
  if (closed && tsumo) oy_add(y, Y_MENZEN_TSUMO, 1);
  int all_run = 1;
  for (int i = 0; i < nb; i++) if (!b[i].run) all_run = 0;
  if (closed && all_run && !(pair >= 31) && pair != c->seat_wind && pair != c->round_wind &&
      wait == W_RYANMEN)
    oy_add(y, Y_PINFU, 1);
  if (all_simple) oy_add(y, Y_TANYAO, 1);
  if (trip[31]) oy_add(y, Y_WHITE, 1);
  if (trip[32]) oy_add(y, Y_GREEN, 1);
  if (trip[33]) oy_add(y, Y_RED, 1);
  if (trip[c->seat_wind]) oy_add(y, Y_SEAT, 1);
  if (trip[c->round_wind]) oy_add(y, Y_ROUND, 1);
  for (int n = 0; n < 7; n++)
    if (run_start[n] && run_start[n + 9] && run_start[n + 18]) {
      oy_add(y, Y_SANSHOKU_DOUJUN, closed ? 2 : 1);
      break;
    }
  for (int n = 0; n < 9; n++)
    if (trip[n] && trip[n + 9] && trip[n + 18]) { oy_add(y, Y_SANSHOKU_DOUKOU, 2); break; }
  for (int s = 0; s < 3; s++)
    if (run_start[9 * s] && run_start[9 * s + 3] && run_start[9 * s + 6]) {
      oy_add(y, Y_ITTSU, closed ? 2 : 1);
      break;
    }
  int outside = o_is_orphan(pair);
  for (int i = 0; i < nb && outside; i++) {
    int any = 0;
    if (b[i].run) any = o_is_orphan(b[i].start) || o_is_orphan(b[i].start + 2) || o_is_orphan(b[i].start + 1);
    else any = o_is_orphan(b[i].start);
    if (!any) outside = 0;
  }
  int has_honor = outside_any_honor;
  if (outside && has_run) {
    if (has_honor) oy_add(y, Y_CHANTA, closed ? 2 : 1);
    else oy_add(y, Y_JUNCHAN, closed ? 3 : 2);
  }
  if (all_trip) oy_add(y, Y_TOITOI, 2);
  if (concealed_trips == 3) oy_add(y, Y_SANANKOU, 2);
  if (kans == 3) oy_add(y, Y_SANKANTSU, 2);
  if (outside && !has_run && has_honor) oy_add(y, Y_HONROUTOU, 2);
  if (trip[31] + trip[32] + trip[33] == 2 && pair >= 31) oy_add(y, Y_SHOUSANGEN, 2);
  int suits[3] = {0, 0, 0}, nsuits = 0;
  for (int k = 0; k < 27; k++) if (present[k]) suits[k / 9] = 1;
  nsuits = suits[0] + suits[1] + suits[2];
  if (nsuits == 1) {
    if (has_honor) oy_add(y, Y_HONITSU, closed ? 3 : 2);
    else oy_add(y, Y_CHINITSU, closed ? 6 : 5);
  }
  o_situational(c, y);
  y->yakuman = 0;
}

/* scoring/yaku.py:337-370 */
static void o_detect_seven_pairs(const orc_winctx* c, OYaku* y) {
  memset(y, 0, sizeof(*y));
  const uint8_t* cnt = c->concealed;
  if (c->first_draw && c->tsumo) oy_add(y, c->seat_wind == 27 ? Y_TENHOU : Y_CHIIHOU, 1);
  int all_honor = 1, all_simple = 1, all_orphan = 1, suits[3] = {0, 0, 0}, honors = 0;
  for (int k = 0; k < 34; k++)
    if (cnt[k]) {
      if (k < 27) { all_honor = 0; suits[k / 9] = 1; } else honors = 1;
      if (o_is_orphan(k)) all_simple = 0; else all_orphan = 0;
    }
  if (all_honor) oy_add(y, Y_TSUUIISOU, 1);
  if (y->n) { y->yakuman = oy_han(y); return; }
  if (c->riichi == 2) oy_add(y, Y_DOUBLE_RIICHI, 2);
  else if (c->riichi == 1) oy_add(y, Y_RIICHI, 1);
  if (c->ippatsu) oy_add(y, Y_IPPATSU, 1);
  if (c->tsumo) oy_add(y, Y_MENZEN_TSUMO, 1);
  oy_add(y, Y_CHIITOITSU, 2);
  if (all_simple) oy_add(y, Y_TANYAO, 1);
  if (all_orphan) oy_add(y, Y_HONROUTOU, 2);
  if (suits[0] + suits[1] + suits[2] == 1) oy_add(y, honors ? Y_HONITSU : Y_CHINITSU, honors ? 3 : 6);
  o_situational(c, y);
  y->yakuman = 0;
}

/* scoring/yaku.py:373-380 */
static void o_detect_kokushi(const orc_winctx* c, OYaku* y) {
  memset(y, 0, sizeof(*y));
  int pure = c->concealed[c->win_tile >> 2] == 2;
  if (c->first_draw && c->tsumo) oy_add(y, c->seat_wind == 27 ? Y_TENHOU : Y_CHIIHOU, 1);
  oy_add(y, Y_KOKUSHI, (c->double_yakuman && pure) ? 2 : 1);
  y->yakuman = oy_han(y);
}

/* scoring/fu.py:11-54 */
static int o_block_fu(const OBlock* b) {
  if (b->run) return 0;
  int base = 2;
  if (!b->open && !b->ron_completed) base *= 2;
  if (b->kan) base *= 4;
  if (o_is_orphan(b->start)) base *= 2;
  return base;
}
static int o_fu(const orc_winctx* c, const ODec* d, int wait_block, int wait, const OYaku* y) {
  if (oy_has(y, Y_CHIITOITSU)) return 25;
  int ron = !c->tsumo;
  if (oy_has(y, Y_PINFU)) return ron ? 30 : 20;
  int fu = 20;
  OBlock b[8];
  int nb = o_blocks(d, c, wait_block, b);
  for (int i = 0; i < nb; i++) fu += o_block_fu(&b[i]);
  if (d->pair >= 31) fu += 2;
  if (d->pair == c->seat_wind) fu += 2;
  if (d->pair == c->round_wind) fu += 2;
  if (wait == W_KANCHAN || wait == W_PENCHAN || wait == W_TANKI) fu += 2;
  if (ron && o_ctx_closed(c)) fu += 10;
  if (!ron) fu += 2;
  return (fu + 9) / 10 * 10;
}

/* scoring/points.py:16-37 */
int orc_base_points(int fu, int han, int yakuman, int kazoe) {
  if (yakuman) return 8000 * yakuman;
  if (han >= 13) return kazoe ? 8000 : 6000;
  if (han >= 11) return 6000;
  if (han >= 8) return 4000;
  if (han >= 6) return 3000;
  if (han >= 5) return 2000;
  int v = fu * (1 << (2 + han));
  return v < 2000 ? v : 2000;
}
static int o_ceil100(int x) { return (x + 99) / 100 * 100; }

/* scoring/points.py:56-86 */
void orc_settle(int tsumo, int base, int dealer, int winner, int loser, int honba, int deposits,
                int32_t* deltas, int32_t* honba_comp) {
  for (int s = 0; s < 4; s++) deltas[s] = 0;
  int dealer_win = winner == dealer;
  if (!tsumo) {
    int pay = o_ceil100(base * (dealer_win ? 6 : 4)) + 300 * honba;
    deltas[loser] -= pay;
    deltas[winner] += pay;
    *honba_comp = 300 * honba;
  } else {
    *honba_comp = 0;
    for (int s = 0; s < 4; s++) {
      if (s == winner) continue;
      int share = (dealer_win || s == dealer) ? 2 * base : base;
      int pay = o_ceil100(share) + 100 * honba;
      deltas[s] -= pay;
      deltas[winner] += pay;
      *honba_comp += 100 * honba;
    }
  }
  deltas[winner] += 1000 * deposits;
}

typedef struct {
  int valid;
  int base, yakuman, han, fu;
  OYaku yaku;
  int form;
} OCand;

/* scoring/score.py:45-82 (score_win) */
static int o_score_win(const orc_winctx* c, rs_win_rec* out, int8_t* order, int32_t* n_order) {
  int dora, ura, reds;
  o_dora_parts(c, &dora, &ura, &reds);
  int bonus = dora + ura + reds;
  OCand best;
  memset(&best, 0, sizeof(best));
#define CONSIDER(YK, FU, FORM)                                                         \
  do {                                                                                 \
    OCand cd;                                                                          \
    cd.valid = 1;                                                                      \
    cd.yaku = (YK);                                                                    \
    cd.fu = (FU);                                                                      \
    cd.form = (FORM);                                                                  \
    cd.yakuman = (YK).yakuman;                                                         \
    int ok = 1;                                                                        \
    if (cd.yakuman) {                                                                  \
      cd.han = 0;                                                                      \
      cd.base = orc_base_points(cd.fu, 0, cd.yakuman, c->kazoe);                       \
    } else {                                                                           \
      int yh = oy_han(&cd.yaku);                                                       \
      if (yh == 0) ok = 0;                                                             \
      cd.han = yh + bonus;                                                             \
      if (ok) cd.base = orc_base_points(cd.fu, cd.han, 0, c->kazoe);                  \
    }                                                                                  \
    if (ok) {                                                                          \
      int better = !best.valid;                                                        \
      if (!better) {                                                                   \
        if (cd.base != best.base) better = cd.base > best.base;                        \
        else if (cd.yakuman != best.yakuman) better = cd.yakuman > best.yakuman;       \
        else if (cd.han != best.han) better = cd.han > best.han;                       \
        else better = cd.fu > best.fu;                                                 \
      }                                                                                \
      if (better) best = cd;                                                           \
    }                                                                                  \
  } while (0)

  int concealed_only = c->n_melds == 0;
  if (concealed_only) {
    /* score.py:33-42 (_is_kokushi, _is_seven_pairs) */
    int other = 0, kinds = 0, pairs13 = 0;
    for (int k = 0; k < 34; k++) if (c->concealed[k] && !o_is_orphan(k)) other = 1;
    for (int i = 0; i < 13; i++) {
      if (c->concealed[ORPHANS[i]]) kinds++;
      if (c->concealed[ORPHANS[i]] == 2) pairs13++;
    }
    if (!other && kinds == 13 && pairs13 == 1) {
      OYaku y;
      o_detect_kokushi(c, &y);
      CONSIDER(y, 0, RS_FORM_KOKUSHI);
    }
    int np = 0;
    for (int k = 0; k < 34; k++) if (c->concealed[k] == 2) np++;
    if (np == 7) {
      OYaku y;
      o_detect_seven_pairs(c, &y);
      CONSIDER(y, 25, RS_FORM_SEVEN_PAIRS);
    }
  }
  ODec decs[64];
  int nd = o_decompose(c->concealed, c->n_melds, decs, 64);
  int wk = c->win_tile >> 2;
  for (int i = 0; i < nd; i++) {
    int blk[8], shp[8];
    int np = o_wait_placements(&decs[i], wk, blk, shp);
    for (int j = 0; j < np; j++) {
      OYaku y;
      o_detect_standard(c, &decs[i], blk[j], shp[j], &y);
      int fu = o_fu(c, &decs[i], blk[j], shp[j], &y);
      CONSIDER(y, fu, RS_FORM_STANDARD);
    }
  }
#undef CONSIDER
  if (!best.valid) return 0;
  if (out) {
    memset(out, 0, sizeof(*out));
    for (int i = 0; i < best.yaku.n; i++) out->yaku_han[best.yaku.id[i]] = (int8_t)best.yaku.han[i];
    out->yakuman = best.yakuman;
    out->han = best.han;
    out->fu = best.fu;
    out->base = best.base;
    out->dora = dora;
    out->ura = ura;
    out->reds = reds;
    out->form = best.form;
  }
  if (order) {
    for (int i = 0; i < best.yaku.n; i++) order[i] = (int8_t)best.yaku.id[i];
  }
  if (n_order) *n_order = best.yaku.n;
  return 1;
}
int orc_score_win(const orc_winctx* ctx, rs_win_rec* out, int8_t* order, int32_t* n_order) {
  orc_tables_build();
  return o_score_win(ctx, out, order, n_order);
}

/* ---------------------------------------------------------------- engine */

#define PH_ACT 0
#define PH_CALL 1
#define PH_GAME_END 2
#define ST_RON 0
#define ST_PONKAN 1
#define ST_CHI 2
#define EV_DRAW 0
#define EV_DISCARD 1
#define EV_CHI 2
#define EV_PON 3
#define EV_KAN_OPEN 4
#define EV_KAN_CLOSED 5
#define EV_KAN_ADDED 6
#define EV_RIICHI 7
#define EV_RON 8
#define EV_TSUMO 9
#define EV_DRAW_END 10
#define EV_NEW_DORA 11
#define A_RIICHI 37
#define A_TSUMO 38
#define A_RON 39
#define A_PON 40
#define A_CHI_LOW 41
#define A_CHI_MID 42
#define A_CHI_HIGH 43
#define A_KAN_OPEN 44
#define A_KAN_CLOSED 45
#define A_KAN_ADDED 79
#define A_PASS 113
#define A_NINE 114
#define MELD_CHI 0
#define MELD_PON 1
#define MELD_KAN_OPEN 2
#define MELD_KAN_CLOSED 3
#define MELD_KAN_ADDED 4
#define MAX_RESULTS 96

/* engine/types.py:72-106 (HandState) */
typedef struct {
  int conc[15]; /* sorted ids */
  int nconc;
  uint8_t counts[34];
  int codes[4];
  rs_meld_rec melds[4];
  int nmelds;
  int river_tile[RS_MAX_RIVER];
  int river_flags[RS_MAX_RIVER];
  int nriver;
  int riichi, riichi_index, ippatsu, temp_furiten, perm_furiten, shanten;
  uint64_t waits;
} OHand;

typedef struct {
  rs_result_rec rec;
  int8_t order[3][48];
  int32_t norder[3];
} OResult;

/* engine/types.py:124-179 (GameState) + env/core.py:49-62 (EnvState) */
struct orc_env {
  rs_config cfg;
  uint8_t wall[136];
  int cursor, kan_draws, dora_count;
  OHand hands[4];
  int scores[4];
  int kyoku, honba, deposits, repeats, phase, actor, drawn;
  int riichi_pending, rinshan_pending, call_tile, call_from;
  int qseat[RS_MAX_QUEUE], qstage[RS_MAX_QUEUE], nq;
  int rons[4], nrons;
  int call_chankan, kakan_kind, pending_dora, four_kan_pending, any_call_made;
  ORng rng;
  int step_count, terminated, truncated;
  int16_t* events;
  int nevents, evcap;
  int ev_base; /* events emitted before an imported window */
  OResult results[MAX_RESULTS];
  int nresults;
  uint32_t mask[4];
  int legal[RS_NUM_ACTIONS];
  int nlegal;
  /* env wrapper */
  int current_player, env_terminated, env_truncated, status;
  float rewards[4];
  uint64_t env_key, policy_key, policy_counter;
  int resets;
};

orc_env* orc_env_new(void) {
  orc_env* e = (orc_env*)calloc(1, sizeof(orc_env));
  e->evcap = 1024;
  e->events = (int16_t*)malloc(sizeof(int16_t) * 3 * (size_t)e->evcap);
  return e;
}
void orc_env_free(orc_env* e) {
  if (!e) return;
  free(e->events);
  free(e);
}
void orc_env_copy(orc_env* dst, const orc_env* src) {
  int16_t* ev = dst->events;
  int cap = dst->evcap;
  memcpy(dst, src, sizeof(orc_env));
  if (cap < src->evcap) {
    ev = (int16_t*)realloc(ev, sizeof(int16_t) * 3 * (size_t)src->evcap);
    cap = src->evcap;
  }
  dst->events = ev;
  dst->evcap = cap;
  memcpy(dst->events, src->events, sizeof(int16_t) * 3 * (size_t)src->nevents);
}

/* engine/engine.py:100-102 */
static void o_emit(orc_env* g, int type, int actor, int tile) {
  if (g->nevents == g->evcap) {
    g->evcap *= 2;
    g->events = (int16_t*)realloc(g->events, sizeof(int16_t) * 3 * (size_t)g->evcap);
  }
  int16_t* p = g->events + 3 * g->nevents;
  p[0] = (int16_t)type;
  p[1] = (int16_t)actor;
  p[2] = (int16_t)tile;
  g->nevents++;
}

static int o_dealer(const orc_env* g) { return g->kyoku % 4; }
static int o_round_wind(const orc_env* g) { return g->kyoku >= 4 ? 28 : 27; }
static int o_seat_wind(const orc_env* g, int s) { return 27 + ((s - o_dealer(g)) % 4 + 4) % 4; }
static int o_live(const orc_env* g) { return 122 - g->kan_draws - g->cursor; }
static int o_is_red(int t, int rule) { return rule == RS_RULE_RED && (t == 16 || t == 52 || t == 88); }
static int o_hand_closed(const OHand* h) {
  for (int i = 0; i < h->nmelds; i++) if (h->melds[i].type != MELD_KAN_CLOSED) return 0;
  return 1;
}
static int o_kan_count(const OHand* h) {
  int n = 0;
  for (int i = 0; i < h->nmelds; i++) if (h->melds[i].type >= MELD_KAN_OPEN) n++;
  return n;
}

/* engine/state.py:31-39 (_finish_hand) */
static void o_finish_hand(OHand* h) {
  h->shanten = o_shanten_codes(h->codes, h->counts, h->nmelds);
  h->waits = 0;
  if (h->shanten == 0 && h->nconc + 3 * h->nmelds == 13)
    h->waits = o_waits_codes(h->codes, h->counts, h->nmelds);
}
/* engine/state.py:56-66 (_code_shift) */
static void o_code_shift(int* codes, int kind, int delta) {
  if (kind < 9) codes[0] += delta * POW5_SUIT[kind];
  else if (kind < 18) codes[1] += delta * POW5_SUIT[kind - 9];
  else if (kind < 27) codes[2] += delta * POW5_SUIT[kind - 18];
  else codes[3] += delta * POW5_HONOR[kind - 27];
}
/* engine/state.py:42-53 (make_hand) for a fresh deal */
static void o_make_hand(OHand* h, const int* ids, int n) {
  memset(h, 0, sizeof(*h));
  for (int i = 0; i < n; i++) h->conc[i] = ids[i];
  h->nconc = n;
  for (int i = 1; i < n; i++)
    for (int j = i; j > 0 && h->conc[j - 1] > h->conc[j]; j--) {
      int t = h->conc[j]; h->conc[j] = h->conc[j - 1]; h->conc[j - 1] = t;
    }
  for (int i = 0; i < n; i++) h->counts[h->conc[i] >> 2]++;
  o_codes(h->counts, h->codes);
  h->riichi_index = -1;
  o_finish_hand(h);
}
/* engine/state.py:69-76 (hand_add) */
static void o_hand_add(OHand* h, int tile) {
  int i = h->nconc;
  while (i > 0 && h->conc[i - 1] > tile) { h->conc[i] = h->conc[i - 1]; i--; }
  h->conc[i] = tile;
  h->nconc++;
  h->counts[tile >> 2]++;
  o_code_shift(h->codes, tile >> 2, 1);
  o_finish_hand(h);
}
/* engine/state.py:79-90 (hand_remove) without the rebuild */
static void o_hand_remove_nofinish(OHand* h, int tile) {
  int i = 0;
  while (i < h->nconc && h->conc[i] != tile) i++;
  if (i == h->nconc) { fprintf(stderr, "oracle: removing absent tile %d\n", tile); abort(); }
  for (; i + 1 < h->nconc; i++) h->conc[i] = h->conc[i + 1];
  h->nconc--;
  h->counts[tile >> 2]--;
  o_code_shift(h->codes, tile >> 2, -1);
}

/* engine/types.py:93-100 */
static int o_furiten(const OHand* h) {
  if (h->temp_furiten || h->perm_furiten) return 1;
  if (h->waits) {
    for (int i = 0; i < h->nriver; i++)
      if ((h->waits >> (h->river_tile[i] >> 2)) & 1) return 1;
  }
  return 0;
}

/* engine/engine.py:345-375 (_win_context) */
static void o_win_context(const orc_env* g, int seat, int win_tile, int tsumo, int chankan,
                          orc_winctx* c) {
  const OHand* h = &g->hands[seat];
  memset(c, 0, sizeof(*c));
  memcpy(c->concealed, h->counts, 34);
  int n = 0;
  for (int i = 0; i < h->nconc; i++) c->ids[n++] = (uint8_t)h->conc[i];
  if (tsumo) {
    c->last_tile = o_live(g) == 0 && !g->rinshan_pending;
    c->rinshan = g->rinshan_pending;
    c->first_draw = h->nriver == 0 && !g->any_call_made && h->nmelds == 0 && !c->rinshan;
  } else {
    c->concealed[win_tile >> 2]++;
    c->ids[n++] = (uint8_t)win_tile;
    c->last_tile = o_live(g) == 0 && !chankan;
  }
  for (int i = 0; i < h->nmelds; i++)
    for (int j = 0; j < h->melds[i].n_tiles; j++) c->ids[n++] = h->melds[i].tiles[j];
  c->n_ids = n;
  c->n_melds = h->nmelds;
  for (int i = 0; i < h->nmelds; i++) c->melds[i] = h->melds[i];
  c->win_tile = win_tile;
  c->tsumo = tsumo;
  c->seat_wind = o_seat_wind(g, seat);
  c->round_wind = o_round_wind(g);
  c->riichi = h->riichi;
  c->ippatsu = h->ippatsu;
  c->chankan = chankan;
  c->n_dora = g->dora_count;
  for (int i = 0; i < g->dora_count; i++) c->dora[i] = g->wall[122 + 2 * i];
  if (h->riichi) {
    c->n_ura = g->dora_count;
    for (int i = 0; i < g->dora_count; i++) c->ura[i] = g->wall[123 + 2 * i];
  }
  c->rule = g->cfg.rule;
  c->kazoe = g->cfg.kazoe;
  c->double_yakuman = g->cfg.double_yakuman;
}

/* engine/engine.py:378-383 */
static int o_try_score(const orc_env* g, int seat, int tile, int tsumo, int chankan, rs_win_rec* out,
                       int8_t* order, int32_t* norder) {
  orc_winctx c;
  o_win_context(g, seat, tile, tsumo, chankan, &c);
  return o_score_win(&c, out, order, norder);
}
/* engine/engine.py:386-390 */
static int o_can_tsumo(const orc_env* g, int seat) {
  if (g->hands[seat].shanten != -1) return 0;
  return o_try_score(g, seat, g->drawn, 1, 0, NULL, NULL, NULL);
}
/* engine/engine.py:393-399 */
static int o_can_ron(const orc_env* g, int seat, int tile, int chankan) {
  const OHand* h = &g->hands[seat];
  if (h->shanten != 0 || !((h->waits >> (tile >> 2)) & 1)) return 0;
  if (o_furiten(h)) return 0;
  return o_try_score(g, seat, tile, 0, chankan, NULL, NULL, NULL);
}

/* engine/engine.py:214-227 */
static int o_shanten_minus_kind(const OHand* h, int kind) {
  uint8_t c[34];
  memcpy(c, h->counts, 34);
  c[kind]--;
  int codes[4] = {h->codes[0], h->codes[1], h->codes[2], h->codes[3]};
  o_code_shift(codes, kind, -1);
  return o_shanten_codes(codes, c, h->nmelds);
}

static void o_set(uint32_t* m, int a) { m[a >> 5] |= 1u << (a & 31); }

/* engine/engine.py:230-246 */
static void o_discard_bits(const OHand* h, int rule, int only_tenpai, uint32_t* m) {
  for (int kind = 0; kind < 34; kind++) {
    int c = h->counts[kind];
    if (!c) continue;
    if (only_tenpai && o_shanten_minus_kind(h, kind) != 0) continue;
    int has_red = 0;
    if (rule == RS_RULE_RED && (kind == 4 || kind == 13 || kind == 22)) {
      int red_id = kind * 4;
      for (int i = 0; i < h->nconc; i++) if (h->conc[i] == red_id) has_red = 1;
      if (has_red) o_set(m, 34 + (kind == 4 ? 0 : kind == 13 ? 1 : 2));
    }
    if (c > (has_red ? 1 : 0)) o_set(m, kind);
  }
}

static int o_kan_draw_ok(const orc_env* g) { return o_live(g) >= 1 && g->kan_draws < 4; }

/* engine/engine.py:331-339 */
static int o_kan_keeps_waits(const OHand* h, int kind) {
  uint8_t before[34], after[34];
  memcpy(before, h->counts, 34);
  before[kind]--;
  uint64_t old = orc_waits(before, h->nmelds);
  memcpy(after, h->counts, 34);
  after[kind] -= 4;
  uint64_t nw = orc_waits(after, h->nmelds + 1);
  return old == nw && !((old >> kind) & 1);
}

/* engine/engine.py:265-306 */
static void o_legal_act(const orc_env* g, uint32_t* m) {
  int seat = g->actor, rule = g->cfg.rule;
  const OHand* h = &g->hands[seat];
  if (g->riichi_pending) { o_discard_bits(h, rule, 1, m); return; }
  if (h->riichi) {
    if (o_can_tsumo(g, seat)) o_set(m, A_TSUMO);
    int kind = g->drawn >> 2;
    if (o_is_red(g->drawn, rule)) o_set(m, 34 + (kind == 4 ? 0 : kind == 13 ? 1 : 2));
    else o_set(m, kind);
    if (h->counts[kind] == 4 && o_kan_draw_ok(g) && o_kan_keeps_waits(h, kind)) o_set(m, A_KAN_CLOSED + kind);
    return;
  }
  o_discard_bits(h, rule, 0, m);
  if (g->drawn < 0) return;
  if (h->riichi == 0 && o_hand_closed(h) && g->scores[seat] >= 1000 && o_live(g) >= 4 && h->shanten <= 0)
    o_set(m, A_RIICHI);
  if (o_can_tsumo(g, seat)) o_set(m, A_TSUMO);
  if (o_kan_draw_ok(g)) {
    for (int k = 0; k < 34; k++) if (h->counts[k] == 4) o_set(m, A_KAN_CLOSED + k);
    for (int i = 0; i < h->nmelds; i++)
      if (h->melds[i].type == MELD_PON) {
        int k = o_meld_base_kind(&h->melds[i]);
        if (h->counts[k] >= 1) o_set(m, A_KAN_ADDED + k);
      }
  }
  if (rule == RS_RULE_RED && !g->any_call_made && h->nriver == 0 && h->nmelds == 0) {
    int n = 0;
    for (int i = 0; i < 13; i++) if (h->counts[ORPHANS[i]]) n++;
    if (n >= 9) o_set(m, A_NINE);
  }
}

/* engine/engine.py:309-328 */
static void o_legal_call(const orc_env* g, uint32_t* m) {
  int seat = g->qseat[0], stage = g->qstage[0];
  const OHand* h = &g->hands[seat];
  int kind = g->call_tile >> 2;
  o_set(m, A_PASS);
  if (stage == ST_RON) o_set(m, A_RON);
  else if (stage == ST_PONKAN) {
    o_set(m, A_PON);
    if (h->counts[kind] >= 3 && o_kan_draw_ok(g)) o_set(m, A_KAN_OPEN);
  } else {
    int n = kind % 9;
    if (n <= 6 && h->counts[kind + 1] && h->counts[kind + 2]) o_set(m, A_CHI_LOW);
    if (n >= 1 && n <= 7 && h->counts[kind - 1] && h->counts[kind + 1]) o_set(m, A_CHI_MID);
    if (n >= 2 && h->counts[kind - 2] && h->counts[kind - 1]) o_set(m, A_CHI_HIGH);
  }
}

/* engine/engine.py:105-122 (_finish) + 253-262 (_compute_legal) */
static void o_finish(orc_env* g) {
  memset(g->mask, 0, sizeof(g->mask));
  g->nlegal = 0;
  if (g->terminated || g->truncated) return;
  if (g->phase == PH_CALL) o_legal_call(g, g->mask);
  else o_legal_act(g, g->mask);
  for (int a = 0; a < RS_NUM_ACTIONS; a++)
    if ((g->mask[a >> 5] >> (a & 31)) & 1) g->legal[g->nlegal++] = a;
}

/* engine/engine.py:167-178 */
static void o_draw(orc_env* g, int seat) {
  OHand* h = &g->hands[seat];
  h->temp_furiten = 0;
  int tile = g->wall[g->cursor];
  g->cursor++;
  o_hand_add(h, tile);
  g->drawn = tile;
  g->rinshan_pending = 0;
  g->phase = PH_ACT;
  g->actor = seat;
  o_emit(g, EV_DRAW, seat, tile);
}
/* engine/engine.py:181-189 */
static void o_rinshan_draw(orc_env* g, int seat) {
  int tile = g->wall[135 - g->kan_draws];
  g->kan_draws++;
  o_hand_add(&g->hands[seat], tile);
  g->drawn = tile;
  g->rinshan_pending = 1;
  g->phase = PH_ACT;
  g->actor = seat;
  o_emit(g, EV_DRAW, seat, tile);
}

/* engine/engine.py:139-164 */
static void o_start_kyoku(orc_env* g) {
  o_shuffle136(&g->rng, g->wall);
  int dealer = o_dealer(g);
  int dealt[4][14], nd[4] = {0, 0, 0, 0}, pos = 0;
  for (int r = 0; r < 3; r++)
    for (int i = 0; i < 4; i++) {
      int s = (dealer + i) % 4;
      for (int j = 0; j < 4; j++) dealt[s][nd[s]++] = g->wall[pos++];
    }
  for (int i = 0; i < 4; i++) {
    int s = (dealer + i) % 4;
    dealt[s][nd[s]++] = g->wall[pos++];
  }
  for (int s = 0; s < 4; s++) o_make_hand(&g->hands[s], dealt[s], nd[s]);
  g->cursor = pos;
  g->kan_draws = 0;
  g->dora_count = 1;
  g->riichi_pending = 0;
  g->rinshan_pending = 0;
  g->call_tile = g->call_from = -1;
  g->nq = 0;
  g->nrons = 0;
  g->call_chankan = 0;
  g->kakan_kind = -1;
  g->pending_dora = 0;
  g->four_kan_pending = 0;
  g->any_call_made = 0;
  o_draw(g, dealer);
}

static int o_leader(const int* sc) {
  int best = 0;
  for (int s = 1; s < 4; s++) if (sc[s] > sc[best]) best = s;
  return best;
}
static void o_end_game(orc_env* g) {
  g->phase = PH_GAME_END;
  g->terminated = 1;
  g->nq = 0;
}
static int o_final_kyoku(const orc_env* g) {
  return g->cfg.mode == RS_MODE_SINGLE ? 0 : (g->cfg.mode == RS_MODE_EAST ? 3 : 7);
}

static OResult* o_new_result(orc_env* g, int kind) {
  if (g->nresults >= MAX_RESULTS) { fprintf(stderr, "oracle: result overflow\n"); abort(); }
  OResult* r = &g->results[g->nresults];
  memset(r, 0, sizeof(*r));
  r->rec.kyoku = g->kyoku;
  r->rec.honba = g->honba;
  r->rec.kind = kind;
  r->rec.loser = -1;
  return r;
}

/* engine/engine.py:842-872 */
static void o_advance_round(orc_env* g, int dealer_repeat, int reset_honba) {
  g->nresults++;
  g->drawn = -1;
  if (dealer_repeat && g->repeats >= g->cfg.renchan_cap) dealer_repeat = 0;
  if (dealer_repeat) g->repeats++;
  int bankrupt = 0;
  for (int s = 0; s < 4; s++) if (g->scores[s] < 0) bankrupt = 1;
  int next_honba = reset_honba ? 0 : g->honba + 1;
  if (g->cfg.mode == RS_MODE_SINGLE || bankrupt) { o_end_game(g); return; }
  if (dealer_repeat) {
    if (g->kyoku == o_final_kyoku(g) && g->cfg.agari_yame && o_leader(g->scores) == o_dealer(g)) {
      o_end_game(g);
      return;
    }
    g->honba = next_honba;
    o_start_kyoku(g);
    return;
  }
  if (g->kyoku + 1 > o_final_kyoku(g)) { o_end_game(g); return; }
  g->kyoku++;
  g->honba = next_honba;
  o_start_kyoku(g);
}

static void o_clear_call(orc_env* g) {
  g->call_tile = g->call_from = -1;
  g->nq = 0;
  g->nrons = 0;
  g->call_chankan = 0;
  g->kakan_kind = -1;
}

/* engine/engine.py:829-839 */
static void o_abort(orc_env* g, int kind) {
  for (int s = 0; s < 4; s++)
    if (g->hands[s].riichi) { g->scores[s] += 1000; g->deposits -= 1; }
  OResult* r = o_new_result(g, kind);
  for (int s = 0; s < 4; s++) r->rec.scores_after[s] = g->scores[s];
  o_clear_call(g);
  o_advance_round(g, 1, 0);
}

/* engine/engine.py:810-826 */
static void o_exhaustive(orc_env* g) {
  o_emit(g, EV_DRAW_END, -1, -1);
  int tmask = 0, n = 0;
  for (int s = 0; s < 4; s++) if (g->hands[s].shanten == 0) { tmask |= 1 << s; n++; }
  int d[4] = {0, 0, 0, 0};
  if (n > 0 && n < 4) {
    int gain = 3000 / n, loss = 3000 / (4 - n);
    for (int s = 0; s < 4; s++) d[s] = ((tmask >> s) & 1) ? gain : -loss;
  }
  for (int s = 0; s < 4; s++) g->scores[s] += d[s];
  OResult* r = o_new_result(g, RS_RES_EXHAUSTIVE);
  r->rec.tenpai_mask = tmask;
  r->rec.n_settlements = 1;
  for (int s = 0; s < 4; s++) { r->rec.deltas[0][s] = d[s]; r->rec.scores_after[s] = g->scores[s]; }
  o_advance_round(g, (tmask >> o_dealer(g)) & 1, 0);
}

/* engine/engine.py:764-779 */
static void o_apply_tsumo(orc_env* g, int seat) {
  OResult* r = o_new_result(g, RS_RES_TSUMO);
  if (!o_try_score(g, seat, g->drawn, 1, 0, &r->rec.wins[0], r->order[0], &r->norder[0])) {
    fprintf(stderr, "oracle: tsumo without yaku\n");
    abort();
  }
  orc_settle(1, r->rec.wins[0].base, o_dealer(g), seat, -1, g->honba, g->deposits, r->rec.deltas[0],
             &r->rec.honba_component[0]);
  r->rec.deposits_claimed[0] = g->deposits;
  for (int s = 0; s < 4; s++) g->scores[s] += r->rec.deltas[0][s];
  g->deposits = 0;
  o_emit(g, EV_TSUMO, seat, g->drawn);
  r->rec.n_winners = 1;
  r->rec.winners[0] = (int8_t)seat;
  r->rec.n_settlements = 1;
  for (int s = 0; s < 4; s++) r->rec.scores_after[s] = g->scores[s];
  int dealer = o_dealer(g);
  o_advance_round(g, seat == dealer, seat != dealer);
}

/* engine/engine.py:782-807 */
static void o_apply_ron_wins(orc_env* g) {
  int loser = g->call_from;
  int w[4], nw = g->nrons;
  for (int i = 0; i < nw; i++) w[i] = g->rons[i];
  for (int i = 1; i < nw; i++)
    for (int j = i; j > 0 && ((w[j - 1] - loser + 4) % 4) > ((w[j] - loser + 4) % 4); j--) {
      int t = w[j]; w[j] = w[j - 1]; w[j - 1] = t;
    }
  OResult* r = o_new_result(g, RS_RES_RON);
  r->rec.loser = loser;
  r->rec.n_winners = nw;
  r->rec.n_settlements = nw;
  int dealer = o_dealer(g), dealer_won = 0;
  for (int i = 0; i < nw; i++) {
    int seat = w[i];
    r->rec.winners[i] = (int8_t)seat;
    if (!o_try_score(g, seat, g->call_tile, 0, g->call_chankan, &r->rec.wins[i], r->order[i], &r->norder[i])) {
      fprintf(stderr, "oracle: ron without yaku\n");
      abort();
    }
    int honba = i == 0 ? g->honba : 0, dep = i == 0 ? g->deposits : 0;
    orc_settle(0, r->rec.wins[i].base, dealer, seat, loser, honba, dep, r->rec.deltas[i],
               &r->rec.honba_component[i]);
    r->rec.deposits_claimed[i] = dep;
    for (int s = 0; s < 4; s++) g->scores[s] += r->rec.deltas[i][s];
    o_emit(g, EV_RON, seat, g->call_tile);
    if (seat == dealer) dealer_won = 1;
  }
  g->deposits = 0;
  for (int s = 0; s < 4; s++) r->rec.scores_after[s] = g->scores[s];
  o_clear_call(g);
  o_advance_round(g, dealer_won, !dealer_won);
}

/* engine/engine.py:580-591 */
static void o_mark_passed_furiten(orc_env* g, int kind, int discarder) {
  for (int s = 0; s < 4; s++) {
    if (s == discarder) continue;
    OHand* h = &g->hands[s];
    if (h->shanten == 0 && ((h->waits >> kind) & 1)) {
      if (h->riichi) h->perm_furiten = 1;
      else h->temp_furiten = 1;
    }
  }
}

static void o_draw_or_exhaust(orc_env* g, int discarder);

/* engine/engine.py:594-615 */
static void o_discard_stands(orc_env* g) {
  int discarder = g->phase == PH_CALL ? g->call_from : g->actor;
  g->phase = PH_ACT;
  OHand* h = &g->hands[discarder];
  if (h->riichi && h->riichi_index == h->nriver - 1 && !h->ippatsu) {
    h->ippatsu = 1;
    if (g->cfg.rule == RS_RULE_RED && g->hands[0].riichi && g->hands[1].riichi && g->hands[2].riichi &&
        g->hands[3].riichi) {
      o_emit(g, EV_DRAW_END, discarder, -1);
      o_abort(g, RS_RES_ABORT_FOUR_RIICHI);
      return;
    }
  }
  if (g->four_kan_pending && g->cfg.rule == RS_RULE_RED) {
    o_emit(g, EV_DRAW_END, discarder, -1);
    o_abort(g, RS_RES_ABORT_FOUR_KAN);
    return;
  }
  g->call_tile = g->call_from = -1;
  g->nq = 0;
  g->nrons = 0;
  o_draw_or_exhaust(g, discarder);
}
static void o_draw_or_exhaust(orc_env* g, int discarder) {
  if (o_live(g) == 0) { o_exhaustive(g); return; }
  o_draw(g, (discarder + 1) % 4);
}

/* engine/engine.py:489-495 */
static void o_reveal_pending_dora(orc_env* g) {
  while (g->pending_dora > 0 && g->dora_count < 5) {
    g->dora_count++;
    g->pending_dora--;
    o_emit(g, EV_NEW_DORA, -1, g->wall[122 + 2 * (g->dora_count - 1)]);
  }
  g->pending_dora = 0;
}

static int o_can_chi(const OHand* h, int kind) {
  int n = kind % 9;
  return (n <= 6 && h->counts[kind + 1] && h->counts[kind + 2]) ||
         (n >= 1 && n <= 7 && h->counts[kind - 1] && h->counts[kind + 1]) ||
         (n >= 2 && h->counts[kind - 2] && h->counts[kind - 1]);
}

/* engine/engine.py:498-531 */
static int o_begin_call_phase(orc_env* g, int tile, int discarder, int chankan) {
  int kind = tile >> 2, n = 0;
  int qs[RS_MAX_QUEUE], qt[RS_MAX_QUEUE];
  for (int off = 1; off <= 3; off++) {
    int s = (discarder + off) % 4;
    if (o_can_ron(g, s, tile, chankan)) { qs[n] = s; qt[n++] = ST_RON; }
  }
  if (!chankan && o_live(g) >= 1) {
    for (int off = 1; off <= 3; off++) {
      int s = (discarder + off) % 4;
      const OHand* h = &g->hands[s];
      if (h->riichi) continue;
      if (h->counts[kind] >= 2) { qs[n] = s; qt[n++] = ST_PONKAN; }
    }
    int s = (discarder + 1) % 4;
    const OHand* h = &g->hands[s];
    if (kind < 27 && !h->riichi && o_can_chi(h, kind)) { qs[n] = s; qt[n++] = ST_CHI; }
  }
  if (!n) return 0;
  g->phase = PH_CALL;
  g->call_tile = tile;
  g->call_from = discarder;
  for (int i = 0; i < n; i++) { g->qseat[i] = qs[i]; g->qstage[i] = qt[i]; }
  g->nq = n;
  g->nrons = 0;
  g->call_chankan = chankan;
  g->actor = qs[0];
  return 1;
}

/* engine/engine.py:447-455 */
static int o_pick_discard(const orc_env* g, const OHand* h, int action) {
  int kind = action < 34 ? action : (action == 34 ? 4 : action == 35 ? 13 : 22);
  int want_red = action >= 34, rule = g->cfg.rule;
  if (g->drawn >= 0 && (g->drawn >> 2) == kind && o_is_red(g->drawn, rule) == want_red) return g->drawn;
  for (int i = 0; i < h->nconc; i++)
    if ((h->conc[i] >> 2) == kind && o_is_red(h->conc[i], rule) == want_red) return h->conc[i];
  fprintf(stderr, "oracle: no discard tile\n");
  abort();
}

/* engine/engine.py:458-486 */
static void o_apply_discard(orc_env* g, int seat, int action) {
  OHand* h = &g->hands[seat];
  int tile = o_pick_discard(g, h, action);
  int tsumogiri = tile == g->drawn;
  int declaring = g->riichi_pending;
  int riichi_val = h->riichi, riichi_index = h->riichi_index;
  if (declaring) {
    riichi_val = (h->nriver == 0 && !g->any_call_made) ? 2 : 1;
    riichi_index = h->nriver;
    g->riichi_pending = 0;
  }
  int ippatsu = h->ippatsu;
  if (h->riichi && !declaring && ippatsu) ippatsu = 0;
  if (h->nriver >= RS_MAX_RIVER) { fprintf(stderr, "oracle: river overflow\n"); abort(); }
  h->river_tile[h->nriver] = tile;
  h->river_flags[h->nriver] = (tsumogiri ? RS_RIVER_TSUMOGIRI : 0) | (declaring ? RS_RIVER_RIICHI : 0);
  h->nriver++;
  o_hand_remove_nofinish(h, tile);
  h->riichi = riichi_val;
  h->riichi_index = riichi_index;
  h->ippatsu = ippatsu;
  o_finish_hand(h);
  g->drawn = -1;
  g->rinshan_pending = 0;
  o_emit(g, EV_DISCARD, seat, tile);
  o_reveal_pending_dora(g);
  if (!o_begin_call_phase(g, tile, seat, 0)) {
    o_mark_passed_furiten(g, tile >> 2, seat);
    o_discard_stands(g);
  }
}

static void o_clear_all_ippatsu(orc_env* g) {
  for (int s = 0; s < 4; s++) g->hands[s].ippatsu = 0;
}
/* engine/engine.py:624-628: lowest ids of the kind */
static int o_consume_lowest(const OHand* h, int kind, int n, int* out) {
  int k = 0;
  for (int i = 0; i < h->nconc && k < n; i++) if ((h->conc[i] >> 2) == kind) out[k++] = h->conc[i];
  if (k != n) { fprintf(stderr, "oracle: not enough copies\n"); abort(); }
  return k;
}
/* engine/engine.py:631-636 */
static void o_mark_called_tile(orc_env* g) {
  OHand* h = &g->hands[g->call_from];
  h->river_flags[h->nriver - 1] |= RS_RIVER_CALLED;
}
/* engine/engine.py:639-644 */
static void o_check_four_kans(orc_env* g) {
  if (g->cfg.rule != RS_RULE_RED) return;
  int total = 0, seats = 0;
  for (int s = 0; s < 4; s++) {
    int c = o_kan_count(&g->hands[s]);
    total += c;
    if (c) seats++;
  }
  if (total == 4 && seats >= 2) g->four_kan_pending = 1;
}

static void o_sort_ids(uint8_t* t, int n) {
  for (int i = 1; i < n; i++)
    for (int j = i; j > 0 && t[j - 1] > t[j]; j--) { uint8_t x = t[j]; t[j] = t[j - 1]; t[j - 1] = x; }
}
static void o_add_meld(OHand* h, int type, const int* used, int nused, int called, int from) {
  rs_meld_rec* m = &h->melds[h->nmelds++];
  memset(m, 0, sizeof(*m));
  m->type = (int8_t)type;
  int n = 0;
  for (int i = 0; i < nused; i++) m->tiles[n++] = (uint8_t)used[i];
  if (called >= 0) m->tiles[n++] = (uint8_t)called;
  m->n_tiles = (int8_t)n;
  o_sort_ids(m->tiles, n);
  m->called_tile = (int16_t)called;
  m->from_seat = (int8_t)from;
}
/* engine/engine.py:696-702 */
static void o_finish_meld_call(orc_env* g, int seat) {
  g->any_call_made = 1;
  o_clear_all_ippatsu(g);
  g->phase = PH_ACT;
  g->actor = seat;
  g->drawn = -1;
  g->rinshan_pending = 0;
}
/* engine/engine.py:647-657 */
static void o_apply_pon(orc_env* g, int seat) {
  int kind = g->call_tile >> 2, used[2];
  o_mark_passed_furiten(g, kind, g->call_from);
  o_mark_called_tile(g);
  OHand* h = &g->hands[seat];
  o_consume_lowest(h, kind, 2, used);
  o_add_meld(h, MELD_PON, used, 2, g->call_tile, g->call_from);
  for (int i = 0; i < 2; i++) o_hand_remove_nofinish(h, used[i]);
  o_finish_hand(h);
  o_finish_meld_call(g, seat);
  o_emit(g, EV_PON, seat, g->call_tile);
  o_clear_call(g);
}
/* engine/engine.py:660-676 */
static void o_apply_chi(orc_env* g, int seat, int action) {
  int kind = g->call_tile >> 2, need[2];
  if (action == A_CHI_LOW) { need[0] = kind + 1; need[1] = kind + 2; }
  else if (action == A_CHI_MID) { need[0] = kind - 1; need[1] = kind + 1; }
  else { need[0] = kind - 2; need[1] = kind - 1; }
  o_mark_passed_furiten(g, kind, g->call_from);
  o_mark_called_tile(g);
  OHand* h = &g->hands[seat];
  int used[2];
  for (int i = 0; i < 2; i++) o_consume_lowest(h, need[i], 1, &used[i]);
  o_add_meld(h, MELD_CHI, used, 2, g->call_tile, g->call_from);
  for (int i = 0; i < 2; i++) o_hand_remove_nofinish(h, used[i]);
  o_finish_hand(h);
  o_finish_meld_call(g, seat);
  o_emit(g, EV_CHI, seat, g->call_tile);
  o_clear_call(g);
}
/* engine/engine.py:679-693 */
static void o_apply_open_kan(orc_env* g, int seat) {
  int kind = g->call_tile >> 2, used[3];
  o_mark_passed_furiten(g, kind, g->call_from);
  o_mark_called_tile(g);
  OHand* h = &g->hands[seat];
  o_consume_lowest(h, kind, 3, used);
  o_add_meld(h, MELD_KAN_OPEN, used, 3, g->call_tile, g->call_from);
  for (int i = 0; i < 3; i++) o_hand_remove_nofinish(h, used[i]);
  o_finish_hand(h);
  g->any_call_made = 1;
  o_clear_all_ippatsu(g);
  g->pending_dora++;
  o_emit(g, EV_KAN_OPEN, seat, g->call_tile);
  o_clear_call(g);
  o_check_four_kans(g);
  o_rinshan_draw(g, seat);
}
/* engine/engine.py:714-727 */
static void o_apply_closed_kan(orc_env* g, int seat, int kind) {
  OHand* h = &g->hands[seat];
  int used[4];
  o_consume_lowest(h, kind, 4, used);
  o_add_meld(h, MELD_KAN_CLOSED, used, 4, -1, -1);
  for (int i = 0; i < 4; i++) o_hand_remove_nofinish(h, used[i]);
  o_finish_hand(h);
  g->any_call_made = 1;
  o_clear_all_ippatsu(g);
  g->dora_count = g->dora_count + 1 < 5 ? g->dora_count + 1 : 5;
  o_emit(g, EV_KAN_CLOSED, seat, used[0]);
  o_emit(g, EV_NEW_DORA, -1, g->wall[122 + 2 * (g->dora_count - 1)]);
  o_check_four_kans(g);
  o_rinshan_draw(g, seat);
}
/* engine/engine.py:742-758 */
static void o_complete_added_kan(orc_env* g, int seat, int kind) {
  OHand* h = &g->hands[seat];
  int tile;
  o_consume_lowest(h, kind, 1, &tile);
  for (int i = 0; i < h->nmelds; i++) {
    rs_meld_rec* m = &h->melds[i];
    if (m->type == MELD_PON && o_meld_base_kind(m) == kind) {
      m->type = MELD_KAN_ADDED;
      m->tiles[m->n_tiles++] = (uint8_t)tile;
      o_sort_ids(m->tiles, m->n_tiles);
    }
  }
  o_hand_remove_nofinish(h, tile);
  o_finish_hand(h);
  g->any_call_made = 1;
  o_clear_all_ippatsu(g);
  g->pending_dora++;
  o_clear_call(g);
  o_check_four_kans(g);
  o_rinshan_draw(g, seat);
}
/* engine/engine.py:730-739 */
static void o_apply_added_kan(orc_env* g, int seat, int kind) {
  int tile;
  o_consume_lowest(&g->hands[seat], kind, 1, &tile);
  o_emit(g, EV_KAN_ADDED, seat, tile);
  if (o_begin_call_phase(g, tile, seat, 1)) { g->kakan_kind = kind; return; }
  o_mark_passed_furiten(g, kind, seat);
  o_complete_added_kan(g, seat, kind);
}

/* engine/engine.py:561-577 */
static void o_resolve_call_end(orc_env* g) {
  if (g->nrons) {
    if (g->nrons >= 3 && g->cfg.rule == RS_RULE_RED) {
      o_emit(g, EV_DRAW_END, g->call_from, -1);
      o_abort(g, RS_RES_ABORT_TRIPLE_RON);
      return;
    }
    o_apply_ron_wins(g);
    return;
  }
  o_mark_passed_furiten(g, g->call_tile >> 2, g->call_from);
  if (g->call_chankan) {
    int seat = g->call_from;
    g->call_chankan = 0;
    g->phase = PH_ACT;
    g->actor = seat;
    o_complete_added_kan(g, seat, g->kakan_kind);
    return;
  }
  o_discard_stands(g);
}
/* engine/engine.py:552-558 */
static void o_advance_call_queue(orc_env* g) {
  if (g->nrons) {
    int n = 0;
    for (int i = 0; i < g->nq; i++)
      if (g->qstage[i] == ST_RON) { g->qseat[n] = g->qseat[i]; g->qstage[n] = g->qstage[i]; n++; }
    g->nq = n;
  }
  if (g->nq) { g->actor = g->qseat[0]; return; }
  o_resolve_call_end(g);
}
/* engine/engine.py:534-549 */
static void o_apply_call_action(orc_env* g, int action) {
  int seat = g->qseat[0];
  for (int i = 1; i < g->nq; i++) { g->qseat[i - 1] = g->qseat[i]; g->qstage[i - 1] = g->qstage[i]; }
  g->nq--;
  if (action == A_RON) { g->rons[g->nrons++] = seat; o_advance_call_queue(g); }
  else if (action == A_PASS) o_advance_call_queue(g);
  else if (action == A_PON) o_apply_pon(g, seat);
  else if (action == A_KAN_OPEN) o_apply_open_kan(g, seat);
  else o_apply_chi(g, seat, action);
}
/* engine/engine.py:425-444 */
static void o_apply_turn_action(orc_env* g, int action) {
  int seat = g->actor;
  if (action <= 36) o_apply_discard(g, seat, action);
  else if (action == A_RIICHI) {
    g->scores[seat] -= 1000;
    g->deposits += 1;
    g->riichi_pending = 1;
    o_emit(g, EV_RIICHI, seat, -1);
  } else if (action == A_TSUMO) o_apply_tsumo(g, seat);
  else if (action >= A_KAN_CLOSED && action < A_KAN_ADDED) o_apply_closed_kan(g, seat, action - A_KAN_CLOSED);
  else if (action >= A_KAN_ADDED && action < A_PASS) o_apply_added_kan(g, seat, action - A_KAN_ADDED);
  else if (action == A_NINE) {
    o_emit(g, EV_DRAW_END, seat, -1);
    o_abort(g, RS_RES_ABORT_NINE);
  }
}

/* env/core.py:74-78 + engine.py:885-891 */
static void o_terminal_rewards(orc_env* e) {
  if (e->cfg.reward_scheme == RS_REWARD_RANK) {
    static const double RR[4] = {1.0, 0.333, -0.333, -1.0};
    for (int s = 0; s < 4; s++) {
      int rank = 0;
      for (int t = 0; t < 4; t++)
        if (e->scores[t] > e->scores[s] || (e->scores[t] == e->scores[s] && t < s)) rank++;
      e->rewards[s] = (float)RR[rank];
    }
  } else {
    for (int s = 0; s < 4; s++) e->rewards[s] = (float)((double)(e->scores[s] - 25000) / 25000.0);
  }
}
/* env/core.py:65-71 (_wrap) */
static void o_wrap(orc_env* e) {
  e->current_player = e->actor;
  e->env_terminated = e->terminated;
  e->env_truncated = e->truncated;
  if (e->terminated || e->truncated) o_terminal_rewards(e);
  else for (int s = 0; s < 4; s++) e->rewards[s] = 0.0f;
}

/* engine/engine.py:128-136 + env/core.py:81-82 */
void orc_env_init(orc_env* e, const rs_config* cfg, uint64_t seed) {
  orc_tables_build();
  int16_t* ev = e->events;
  int cap = e->evcap;
  uint64_t ek = e->env_key, pk = e->policy_key, pc = e->policy_counter;
  int resets = e->resets;
  memset(e, 0, sizeof(*e));
  e->events = ev;
  e->evcap = cap;
  e->env_key = ek; e->policy_key = pk; e->policy_counter = pc; e->resets = resets;
  e->cfg = *cfg;
  for (int s = 0; s < 4; s++) e->scores[s] = 25000;
  e->drawn = -1;
  e->call_tile = e->call_from = -1;
  e->kakan_kind = -1;
  e->rng.key = orc_seed_key(seed);
  e->rng.counter = 0;
  o_start_kyoku(e);
  o_finish(e);
  o_wrap(e);
}

/* env/core.py:85-94 + engine/engine.py:405-422 */
int orc_env_step(orc_env* e, int action) {
  if (e->env_terminated || e->env_truncated) { e->status = RS_STATUS_CONTRACT; return e->status; }
  e->status = 0;
  if (action < 0 || action >= RS_NUM_ACTIONS || !((e->mask[action >> 5] >> (action & 31)) & 1)) {
    for (int s = 0; s < 4; s++) e->rewards[s] = 0.0f;
    e->rewards[e->current_player] = e->cfg.illegal_penalty;
    e->env_terminated = 1;
    e->env_truncated = 0;
    e->status = RS_STATUS_ILLEGAL; /* the game (and its cached legal list) is untouched */
    return e->status;
  }
  e->step_count++;
  if (e->phase == PH_CALL) o_apply_call_action(e, action);
  else o_apply_turn_action(e, action);
  if (!e->terminated && e->step_count >= e->cfg.max_steps) e->truncated = 1;
  o_finish(e);
  o_wrap(e);
  return 0;
}

int orc_env_legal(const orc_env* e, int32_t* out) {
  if (e->env_terminated || e->env_truncated) return 0;
  for (int i = 0; i < e->nlegal; i++) out[i] = e->legal[i];
  return e->nlegal;
}
/* the game's cached legal list (engine/types.py:157-158), kept after an illegal env step */
int orc_env_game_legal(const orc_env* e, int32_t* out) {
  for (int i = 0; i < e->nlegal; i++) out[i] = e->legal[i];
  return e->nlegal;
}

/* env/observe.py:43-46 */
static int o_token(int tile, int rule) {
  if (rule == RS_RULE_RED && (tile == 16 || tile == 52 || tile == 88)) return 34 + (tile == 16 ? 0 : tile == 52 ? 1 : 2);
  return tile >> 2;
}
static const int EV_TOKEN[12] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 8, 9, 10};

/* env/observe.py:81-124 */
void orc_env_observe(const orc_env* e, int seat, orc_obs* o) {
  int rule = e->cfg.rule;
  const OHand* h = &e->hands[seat];
  int toks[14], n = h->nconc;
  for (int i = 0; i < n; i++) toks[i] = o_token(h->conc[i], rule);
  for (int i = 1; i < n; i++)
    for (int j = i; j > 0 && toks[j - 1] > toks[j]; j--) { int t = toks[j]; toks[j] = toks[j - 1]; toks[j - 1] = t; }
  for (int i = 0; i < 14; i++) o->hand_tokens[i] = (uint8_t)(i < n ? toks[i] : 37);
  int cnt = e->nevents < 64 ? e->nevents : 64;
  int pad = 64 - cnt;
  for (int i = 0; i < pad; i++) { o->event_tokens[i][0] = 0; o->event_tokens[i][1] = 0; o->event_tokens[i][2] = 37; }
  for (int i = 0; i < cnt; i++) {
    const int16_t* ev = e->events + 3 * (e->nevents - cnt + i);
    int type = ev[0], actor = ev[1], tile = ev[2];
    int rel = actor >= 0 ? ((actor - seat) % 4 + 4) % 4 : 0;
    int tok;
    if (type == EV_DRAW && actor != seat) tok = 37;
    else if (tile >= 0) tok = o_token(tile, rule);
    else tok = 37;
    o->event_tokens[pad + i][0] = (uint8_t)EV_TOKEN[type];
    o->event_tokens[pad + i][1] = (uint8_t)rel;
    o->event_tokens[pad + i][2] = (uint8_t)tok;
  }
  o->shanten = h->shanten;
  for (int i = 0; i < 4; i++) {
    int s = e->scores[(seat + i) % 4];
    o->scores[i] = s >= 0 ? s / 100 : -((-s + 99) / 100); /* floor division */
  }
  o->round_wind = o_round_wind(e);
  o->seat_wind = o_seat_wind(e, seat);
  o->kyoku = e->kyoku;
  o->honba = e->honba;
  o->deposits = e->deposits;
  for (int i = 0; i < 5; i++) o->dora_tokens[i] = (uint8_t)(i < e->dora_count ? o_token(e->wall[122 + 2 * i], rule) : 37);
  o->live_wall = o_live(e);
  for (int i = 0; i < 4; i++) o->riichi_flags[i] = (uint8_t)(e->hands[(seat + i) % 4].riichi ? 1 : 0);
}

/* env/policies.py:17-22 */
int orc_random_policy(const orc_env* e, uint64_t* kc) {
  ORng r = {kc[0], kc[1]};
  int i = (int)o_randbelow(&r, (uint64_t)e->nlegal);
  kc[1] = r.counter;
  return e->legal[i];
}

/* hand/shanten.py:164-169 on a raw count vector (used by the heuristic) */
static int o_shanten_counts(const int* counts, int melds) {
  uint8_t c[34];
  for (int k = 0; k < 34; k++) c[k] = (uint8_t)counts[k];
  int codes[4];
  o_codes(c, codes);
  return o_shanten_codes(codes, c, melds);
}

/* env/policies.py:51-109 */
int orc_heuristic_policy(const orc_env* e) {
  orc_obs obs;
  int seat = e->current_player;
  orc_env_observe(e, seat, &obs);
  const uint32_t* m = e->mask;
#define LEGAL(a) ((m[(a) >> 5] >> ((a) & 31)) & 1)
  if (LEGAL(A_TSUMO)) return A_TSUMO;
  if (LEGAL(A_RON)) return A_RON;
  if (LEGAL(A_RIICHI)) return A_RIICHI;
  int counts[34] = {0}, n = 0;
  for (int i = 0; i < 14; i++) {
    int t = obs.hand_tokens[i];
    if (t == 37) continue;
    n++;
    counts[t < 34 ? t : (t == 34 ? 4 : t == 35 ? 13 : 22)]++;
  }
  int melds = n % 3 == 2 ? (14 - n) / 3 : (13 - n) / 3;
  int best_a = -1, bk[4] = {0, 0, 0, 0};
  for (int a = 0; a <= 36; a++) {
    if (!LEGAL(a)) continue;
    int kind = a < 34 ? a : (a == 34 ? 4 : a == 35 ? 13 : 22);
    counts[kind]--;
    int sh = o_shanten_counts(counts, melds);
    counts[kind]++;
    int cls = kind >= 27 ? 0 : (o_is_terminal(kind) ? 1 : 2);
    int key[4] = {sh, cls, kind, a >= 34 ? 1 : 0};
    int better = best_a < 0;
    for (int i = 0; i < 4 && !better; i++) {
      if (key[i] < bk[i]) { better = 1; break; }
      if (key[i] > bk[i]) break;
    }
    if (better) { best_a = a; for (int i = 0; i < 4; i++) bk[i] = key[i]; }
  }
  if (best_a >= 0) return best_a;
  if (LEGAL(A_PASS)) {
    int current = o_shanten_counts(counts, melds);
    int call_kind = -1;
    for (int i = 63; i >= 0; i--) {
      int t = obs.event_tokens[i][0], tok = obs.event_tokens[i][2];
      if ((t == 1 || t == 6) && tok != 37) { call_kind = tok < 34 ? tok : (tok == 34 ? 4 : tok == 35 ? 13 : 22); break; }
    }
    int best_sh = 0, best_call = -1;
    for (int ai = 0; ai < e->nlegal; ai++) {
      int a = e->legal[ai];
      if (a == A_PASS || a == A_RON) continue;
      int after[34];
      memcpy(after, counts, sizeof(after));
      if (a == A_PON) after[call_kind] -= 2;
      else if (a == A_KAN_OPEN) after[call_kind] -= 3;
      else if (a == A_CHI_LOW) { after[call_kind + 1]--; after[call_kind + 2]--; }
      else if (a == A_CHI_MID) { after[call_kind - 1]--; after[call_kind + 1]--; }
      else if (a == A_CHI_HIGH) { after[call_kind - 2]--; after[call_kind - 1]--; }
      else continue;
      int sh = o_shanten_counts(after, melds + 1);
      if (sh < current && (best_call < 0 || sh < best_sh)) { best_sh = sh; best_call = a; }
    }
    if (best_call >= 0) return best_call;
    return A_PASS;
  }
  return e->legal[0];
#undef LEGAL
}

/* ------------------------------------------------------- export / import */

static void o_hand_to_rec(const OHand* h, rs_hand_rec* r) {
  memset(r, 0, sizeof(*r));
  for (int i = 0; i < h->nconc; i++) r->concealed[i] = (uint8_t)h->conc[i];
  r->n_concealed = (uint8_t)h->nconc;
  r->n_melds = (uint8_t)h->nmelds;
  for (int i = 0; i < h->nmelds; i++) r->melds[i] = h->melds[i];
  for (int i = 0; i < h->nriver; i++) {
    r->river_tile[i] = (uint8_t)h->river_tile[i];
    r->river_flags[i] = (uint8_t)h->river_flags[i];
  }
  r->n_river = h->nriver;
  r->riichi = (int8_t)h->riichi;
  r->riichi_index = (int8_t)h->riichi_index;
  r->ippatsu = (int8_t)h->ippatsu;
  r->temp_furiten = (int8_t)h->temp_furiten;
  r->perm_furiten = (int8_t)h->perm_furiten;
  r->shanten = (int8_t)h->shanten;
  r->waits = h->waits;
}

void orc_env_export(const orc_env* e, rs_env_rec* r) {
  memset(r, 0, sizeof(*r));
  r->abi_version = RS_ABI_VERSION;
  r->cfg = e->cfg;
  memcpy(r->wall, e->wall, 136);
  r->cursor = e->cursor;
  r->kan_draws = e->kan_draws;
  r->dora_count = e->dora_count;
  for (int s = 0; s < 4; s++) o_hand_to_rec(&e->hands[s], &r->hands[s]);
  for (int s = 0; s < 4; s++) r->scores[s] = e->scores[s];
  r->kyoku = e->kyoku; r->honba = e->honba; r->deposits = e->deposits; r->repeats = e->repeats;
  r->phase = e->phase; r->actor = e->actor; r->drawn = e->drawn;
  r->riichi_pending = e->riichi_pending; r->rinshan_pending = e->rinshan_pending;
  r->call_tile = e->call_tile; r->call_from = e->call_from;
  r->n_queue = e->nq;
  for (int i = 0; i < e->nq; i++) { r->queue_seat[i] = (int8_t)e->qseat[i]; r->queue_stage[i] = (int8_t)e->qstage[i]; }
  r->n_rons = e->nrons;
  for (int i = 0; i < e->nrons; i++) r->rons[i] = (int8_t)e->rons[i];
  r->call_chankan = e->call_chankan; r->kakan_kind = e->kakan_kind; r->pending_dora = e->pending_dora;
  r->four_kan_pending = e->four_kan_pending; r->any_call_made = e->any_call_made;
  r->rng_key = e->rng.key; r->rng_counter = e->rng.counter;
  r->step_count = e->step_count; r->terminated = e->terminated; r->truncated = e->truncated;
  r->events_len = e->ev_base + e->nevents;
  int cnt = e->nevents < 64 ? e->nevents : 64;
  for (int i = 0; i < cnt; i++)
    for (int j = 0; j < 3; j++) r->events[i][j] = e->events[3 * (e->nevents - cnt + i) + j];
  r->n_results = e->nresults;
  if (e->nresults) r->last_result = e->results[e->nresults - 1].rec;
  /* env view: a finished episode exposes no legal actions (env/core.py:65-71,106-109) */
  for (int i = 0; i < 4; i++) r->legal_mask[i] = (e->env_terminated || e->env_truncated) ? 0u : e->mask[i];
  r->current_player = e->current_player;
  r->env_terminated = e->env_terminated;
  r->env_truncated = e->env_truncated;
  r->status = e->status;
  for (int s = 0; s < 4; s++) r->rewards[s] = e->rewards[s];
  r->env_key = e->env_key; r->policy_key = e->policy_key; r->policy_counter = e->policy_counter;
  r->resets = e->resets;
}

int orc_env_import(orc_env* e, const rs_env_rec* r) {
  orc_tables_build();
  int16_t* ev = e->events;
  int cap = e->evcap;
  memset(e, 0, sizeof(*e));
  e->events = ev;
  e->evcap = cap;
  e->cfg = r->cfg;
  memcpy(e->wall, r->wall, 136);
  e->cursor = r->cursor; e->kan_draws = r->kan_draws; e->dora_count = r->dora_count;
  for (int s = 0; s < 4; s++) {
    OHand* h = &e->hands[s];
    const rs_hand_rec* hr = &r->hands[s];
    h->nconc = hr->n_concealed;
    for (int i = 0; i < h->nconc; i++) h->conc[i] = hr->concealed[i];
    for (int i = 0; i < h->nconc; i++) h->counts[h->conc[i] >> 2]++;
    o_codes(h->counts, h->codes);
    h->nmelds = hr->n_melds;
    for (int i = 0; i < h->nmelds; i++) h->melds[i] = hr->melds[i];
    h->nriver = hr->n_river;
    for (int i = 0; i < h->nriver; i++) { h->river_tile[i] = hr->river_tile[i]; h->river_flags[i] = hr->river_flags[i]; }
    h->riichi = hr->riichi; h->riichi_index = hr->riichi_index; h->ippatsu = hr->ippatsu;
    h->temp_furiten = hr->temp_furiten; h->perm_furiten = hr->perm_furiten;
    o_finish_hand(h); /* shanten / waits are derived (state.py:31-39) */
  }
  for (int s = 0; s < 4; s++) e->scores[s] = r->scores[s];
  e->kyoku = r->kyoku; e->honba = r->honba; e->deposits = r->deposits; e->repeats = r->repeats;
  e->phase = r->phase; e->actor = r->actor; e->drawn = r->drawn;
  e->riichi_pending = r->riichi_pending; e->rinshan_pending = r->rinshan_pending;
  e->call_tile = r->call_tile; e->call_from = r->call_from;
  e->nq = r->n_queue;
  for (int i = 0; i < e->nq; i++) { e->qseat[i] = r->queue_seat[i]; e->qstage[i] = r->queue_stage[i]; }
  e->nrons = r->n_rons;
  for (int i = 0; i < e->nrons; i++) e->rons[i] = r->rons[i];
  e->call_chankan = r->call_chankan; e->kakan_kind = r->kakan_kind; e->pending_dora = r->pending_dora;
  e->four_kan_pending = r->four_kan_pending; e->any_call_made = r->any_call_made;
  e->rng.key = r->rng_key; e->rng.counter = r->rng_counter;
  e->step_count = r->step_count; e->terminated = r->terminated; e->truncated = r->truncated;
  int cnt = r->events_len < 64 ? r->events_len : 64;
  for (int i = 0; i < cnt; i++) o_emit(e, r->events[i][0], r->events[i][1], r->events[i][2]);
  e->nevents = cnt; /* history before the window is not importable */
  e->ev_base = r->events_len - cnt;
  e->nresults = 0;
  e->env_key = r->env_key; e->policy_key = r->policy_key; e->policy_counter = r->policy_counter;
  e->resets = r->resets;
  o_finish(e);
  o_wrap(e);
  return 0;
}

int orc_env_num_events(const orc_env* e) { return e->nevents; }
void orc_env_events(const orc_env* e, int16_t* out) {
  memcpy(out, e->events, sizeof(int16_t) * 3 * (size_t)e->nevents);
}
int orc_env_num_results(const orc_env* e) { return e->nresults; }
void orc_env_result(const orc_env* e, int i, rs_result_rec* out, int8_t* orders, int32_t* n_orders) {
  *out = e->results[i].rec;
  if (orders) memcpy(orders, e->results[i].order, sizeof(e->results[i].order));
  if (n_orders) memcpy(n_orders, e->results[i].norder, sizeof(e->results[i].norder));
}

/* ------------------------------------------------------------- digests */

static uint64_t o_fold(uint64_t d, uint64_t w) { return orc_mix((d ^ w) + GOLDEN); }
static uint64_t o_digest_summary(uint64_t d, int action, const orc_env* e);

static uint64_t o_pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t x) {
  return (uint64_t)(a & 0xFFFFu) | ((uint64_t)(b & 0xFFFFu) << 16) | ((uint64_t)(c & 0xFFFFu) << 32) |
         ((uint64_t)(x & 0xFFFFu) << 48);
}

/* The wide part of the digest (device: rs_io.cuh digest_state): every
 * field of the state in a canonical form -- hands (concealed tile-id set,
 * HandState flags and waits, melds, river), call state, both RNGs, the
 * wall, the newest 8 events and the last kyoku result
 * (engine/types.py:72-179, engine/state.py:191-242). */
static uint64_t o_digest_state(uint64_t d, const orc_env* e) {
  for (int s = 0; s < 4; s++) {
    const OHand* h = &e->hands[s];
    uint64_t set[3] = {0, 0, 0};
    for (int i = 0; i < h->nconc; i++) set[h->conc[i] >> 6] |= 1ull << (h->conc[i] & 63);
    d = o_fold(d, set[0]);
    d = o_fold(d, set[1]);
    d = o_fold(d, set[2]);
    d = o_fold(d, (uint64_t)h->riichi | ((uint64_t)(h->riichi_index + 1) << 2) | ((uint64_t)h->ippatsu << 8) |
                      ((uint64_t)h->temp_furiten << 9) | ((uint64_t)h->perm_furiten << 10) |
                      ((uint64_t)h->nmelds << 12) | ((uint64_t)h->nriver << 16) | ((uint64_t)h->nconc << 24) |
                      (h->waits << 30));
    for (int i = 0; i < h->nmelds; i++) {
      const rs_meld_rec* m = &h->melds[i];
      uint32_t tiles = 0;
      for (int j = 0; j < m->n_tiles; j++) tiles |= (uint32_t)m->tiles[j] << (8 * j);
      d = o_fold(d, (uint64_t)tiles | ((uint64_t)m->type << 32) | ((uint64_t)m->n_tiles << 36) |
                        ((uint64_t)(m->from_seat + 1) << 40) | ((uint64_t)(m->called_tile + 1) << 48));
    }
    for (int i = 0; i < h->nriver; i += 4) {
      uint32_t v[4];
      for (int j = 0; j < 4; j++)
        v[j] = i + j < h->nriver ? (uint32_t)h->river_tile[i + j] | ((uint32_t)h->river_flags[i + j] << 8) : 0u;
      d = o_fold(d, o_pack4(v[0], v[1], v[2], v[3]));
    }
  }
  d = o_fold(d, (uint64_t)(uint32_t)(e->drawn + 1) | ((uint64_t)(uint32_t)(e->call_tile + 1) << 8) |
                    ((uint64_t)(uint32_t)(e->kakan_kind + 1) << 16) | ((uint64_t)(uint32_t)(e->call_from + 1) << 24) |
                    ((uint64_t)e->actor << 28) | ((uint64_t)e->riichi_pending << 32) |
                    ((uint64_t)e->rinshan_pending << 33) | ((uint64_t)e->call_chankan << 34) |
                    ((uint64_t)e->four_kan_pending << 35) | ((uint64_t)e->any_call_made << 36) |
                    ((uint64_t)e->terminated << 37) | ((uint64_t)e->truncated << 38) |
                    ((uint64_t)e->pending_dora << 40) | ((uint64_t)e->repeats << 48) |
                    ((uint64_t)e->nresults << 56));
  uint64_t q = (uint64_t)e->nq;
  for (int i = 0; i < e->nq; i++) q |= (uint64_t)(e->qseat[i] | (e->qstage[i] << 2)) << (4 + 4 * i);
  q |= (uint64_t)e->nrons << 40;
  for (int i = 0; i < e->nrons; i++) q |= (uint64_t)e->rons[i] << (44 + 2 * i);
  d = o_fold(d, q);
  d = o_fold(d, e->rng.key);
  d = o_fold(d, e->rng.counter);
  d = o_fold(d, e->policy_key);
  d = o_fold(d, e->policy_counter);
  for (int i = 0; i < 136; i += 8) {
    uint64_t w = 0;
    for (int j = 0; j < 8; j++) w |= (uint64_t)e->wall[i + j] << (8 * j);
    d = o_fold(d, w);
  }
  for (int j = 0; j < 8; j += 4) {
    uint32_t v[4];
    for (int k = 0; k < 4; k++) {
      int idx = e->nevents - 1 - (j + k);
      v[k] = 0;
      if (idx >= 0) {
        const int16_t* ev = e->events + 3 * idx;
        v[k] = (uint32_t)ev[0] | ((uint32_t)(ev[1] + 1) << 4) | ((uint32_t)(ev[2] + 1) << 7);
      }
    }
    d = o_fold(d, o_pack4(v[0], v[1], v[2], v[3]));
  }
  if (e->nresults > 0) {
    const rs_result_rec* r = &e->results[e->nresults - 1].rec;
    uint64_t wn = 0;
    for (int i = 0; i < r->n_winners; i++) wn |= (uint64_t)(uint8_t)r->winners[i] << (2 * i);
    d = o_fold(d, (uint64_t)(uint32_t)r->kyoku | ((uint64_t)(uint32_t)r->honba << 8) |
                      ((uint64_t)(uint32_t)r->kind << 16) | ((uint64_t)(uint32_t)r->n_winners << 24) |
                      ((uint64_t)(uint32_t)r->n_settlements << 28) | ((uint64_t)(uint32_t)(r->loser + 1) << 32) |
                      ((uint64_t)(uint32_t)r->tenpai_mask << 40) | (wn << 48));
    for (int i = 0; i < r->n_settlements; i++) {
      d = o_fold(d, (uint64_t)(uint32_t)r->deltas[i][0] | ((uint64_t)(uint32_t)r->deltas[i][1] << 32));
      d = o_fold(d, (uint64_t)(uint32_t)r->deltas[i][2] | ((uint64_t)(uint32_t)r->deltas[i][3] << 32));
      d = o_fold(d, (uint64_t)(uint32_t)r->honba_component[i] | ((uint64_t)(uint32_t)r->deposits_claimed[i] << 32));
    }
    for (int i = 0; i < r->n_winners; i++) {
      const rs_win_rec* w = &r->wins[i];
      for (int k = 0; k < 40; k += 8) {
        uint64_t y = 0;
        for (int j = 0; j < 8; j++) y |= (uint64_t)(uint8_t)w->yaku_han[k + j] << (8 * j);
        d = o_fold(d, y);
      }
      d = o_fold(d, (uint64_t)(uint32_t)w->yakuman | ((uint64_t)(uint32_t)w->han << 8) |
                        ((uint64_t)(uint32_t)w->fu << 16) | ((uint64_t)(uint32_t)w->base << 32));
      d = o_fold(d, (uint64_t)(uint32_t)w->dora | ((uint64_t)(uint32_t)w->ura << 8) |
                        ((uint64_t)(uint32_t)w->reds << 16) | ((uint64_t)(uint32_t)w->form << 24));
    }
    d = o_fold(d, (uint64_t)(uint32_t)r->scores_after[0] | ((uint64_t)(uint32_t)r->scores_after[1] << 32));
    d = o_fold(d, (uint64_t)(uint32_t)r->scores_after[2] | ((uint64_t)(uint32_t)r->scores_after[3] << 32));
  }
  return d;
}

/* observe(current player) folded (device: rs_io.cuh digest_obs) */
static uint64_t o_digest_obs(uint64_t d, const orc_obs* o) {
  uint64_t lo = 0, hi = 0;
  for (int j = 0; j < 8; j++) lo |= (uint64_t)o->hand_tokens[j] << (8 * j);
  for (int j = 0; j < 6; j++) hi |= (uint64_t)o->hand_tokens[8 + j] << (8 * j);
  d = o_fold(d, lo);
  d = o_fold(d, hi);
  const uint8_t* ev = &o->event_tokens[0][0];
  for (int k = 0; k < 192; k += 8) {
    uint64_t w = 0;
    for (int j = 0; j < 8; j++) w |= (uint64_t)ev[k + j] << (8 * j);
    d = o_fold(d, w);
  }
  d = o_fold(d, o_pack4((uint16_t)(int16_t)o->scores[0], (uint16_t)(int16_t)o->scores[1],
                        (uint16_t)(int16_t)o->scores[2], (uint16_t)(int16_t)o->scores[3]));
  d = o_fold(d, (uint64_t)(uint8_t)(int8_t)o->shanten | ((uint64_t)(uint8_t)o->round_wind << 8) |
                    ((uint64_t)(uint8_t)o->seat_wind << 16) | ((uint64_t)(uint8_t)o->kyoku << 24) |
                    ((uint64_t)(uint16_t)(int16_t)o->honba << 32) | ((uint64_t)(uint16_t)(int16_t)o->deposits << 48));
  uint64_t w = 0;
  for (int j = 0; j < 5; j++) w |= (uint64_t)o->dora_tokens[j] << (8 * j);
  w |= (uint64_t)(uint8_t)o->live_wall << 40;
  for (int j = 0; j < 4; j++) w |= (uint64_t)(o->riichi_flags[j] & 1u) << (48 + j);
  return o_fold(d, w);
}

/* identical on the device (rs_io.cuh
 * digest_step + digest_state + digest_obs) */
uint64_t orc_digest_step(uint64_t d, int action, const orc_env* e) {
  d = o_digest_summary(d, action, e);
  d = o_digest_state(d, e);
  orc_obs o;
  orc_env_observe(e, e->current_player, &o);
  return o_digest_obs(d, &o);
}

/* the summary part: action, player, flags, round counters, legal mask,
 * scores, rewards, shanten, event count, wall counters */
static uint64_t o_digest_summary(uint64_t d, int action, const orc_env* e) {
  d = o_fold(d, (uint64_t)(uint32_t)action);
  d = o_fold(d, (uint64_t)(uint32_t)e->current_player | ((uint64_t)e->env_terminated << 8) |
                    ((uint64_t)e->env_truncated << 9) | ((uint64_t)e->phase << 12) |
                    ((uint64_t)(uint32_t)e->kyoku << 16) | ((uint64_t)(uint32_t)e->honba << 24) |
                    ((uint64_t)(uint32_t)e->deposits << 40));
  uint32_t m[4];
  for (int i = 0; i < 4; i++) m[i] = (e->env_terminated || e->env_truncated) ? 0u : e->mask[i];
  d = o_fold(d, (uint64_t)m[0] | ((uint64_t)m[1] << 32));
  d = o_fold(d, (uint64_t)m[2] | ((uint64_t)m[3] << 32));
  for (int s = 0; s < 4; s += 2)
    d = o_fold(d, (uint64_t)(uint32_t)e->scores[s] | ((uint64_t)(uint32_t)e->scores[s + 1] << 32));
  uint32_t rb[4];
  memcpy(rb, e->rewards, 16);
  d = o_fold(d, (uint64_t)rb[0] | ((uint64_t)rb[1] << 32));
  d = o_fold(d, (uint64_t)rb[2] | ((uint64_t)rb[3] << 32));
  uint64_t sh = 0;
  for (int s = 0; s < 4; s++) sh |= (uint64_t)(uint8_t)e->hands[s].shanten << (8 * s);
  sh |= (uint64_t)(uint32_t)(e->ev_base + e->nevents) << 32;
  d = o_fold(d, sh);
  d = o_fold(d, (uint64_t)(uint32_t)e->cursor | ((uint64_t)(uint32_t)e->kan_draws << 8) |
                    ((uint64_t)(uint32_t)e->dora_count << 16) | ((uint64_t)(uint32_t)e->step_count << 32));
  return d;
}

/* bench/runner.py:64-132 (run_shard one_pass) */
int64_t orc_run_shard(const rs_config* cfg, uint64_t seed, int64_t idx0, int64_t n, int32_t steps,
                      int32_t policy, uint64_t* digests) {
  orc_tables_build();
  orc_env* e = orc_env_new();
  int64_t games = 0;
  for (int64_t j = 0; j < n; j++) {
    uint64_t idx = (uint64_t)(idx0 + j);
    e->resets = 0;
    e->env_key = orc_derive_key(orc_seed_key(seed), idx);
    e->policy_key = orc_derive_key(e->env_key, 1);
    e->policy_counter = 0;
    orc_env_init(e, cfg, orc_derive_key(e->env_key, 2));
    uint64_t d = 0;
    for (int t = 0; t < steps; t++) {
      if (e->env_terminated || e->env_truncated) {
        e->resets++;
        orc_env_init(e, cfg, orc_derive_key(e->env_key, 2 + (uint64_t)e->resets));
      }
      int a;
      if (policy == 0) {
        uint64_t kc[2] = {e->policy_key, e->policy_counter};
        a = orc_random_policy(e, kc);
        e->policy_counter = kc[1];
      } else {
        a = orc_heuristic_policy(e);
      }
      orc_env_step(e, a);
      if (digests) d = orc_digest_step(d, a, e);
      if (e->env_terminated || e->env_truncated) games++;
    }
    if (digests) digests[j] = d;
  }
  orc_env_free(e);
  return games;
}

/* ------------------------------------------------- batched CPU baseline */

/* A persistent shard of envs stepped like bench/runner.py:97-121 one_pass
 * (auto-reset + random policy + step) plus observe(current player), the
 * same work per env step as the GPU bench step. */
struct orc_batch {
  rs_config cfg;
  int64_t n;
  orc_env** envs;
  orc_obs obs;
};

orc_batch* orc_batch_new(const rs_config* cfg, uint64_t seed, int64_t idx0, int64_t n) {
  orc_tables_build();
  orc_batch* b = (orc_batch*)calloc(1, sizeof(orc_batch));
  b->cfg = *cfg;
  b->n = n;
  b->envs = (orc_env**)calloc((size_t)n, sizeof(orc_env*));
  for (int64_t j = 0; j < n; j++) {
    orc_env* e = orc_env_new();
    e->env_key = orc_derive_key(orc_seed_key(seed), (uint64_t)(idx0 + j));
    e->policy_key = orc_derive_key(e->env_key, 1);
    e->policy_counter = 0;
    e->resets = 0;
    orc_env_init(e, cfg, orc_derive_key(e->env_key, 2));
    b->envs[j] = e;
  }
  return b;
}

void orc_batch_free(orc_batch* b) {
  if (!b) return;
  for (int64_t j = 0; j < b->n; j++) orc_env_free(b->envs[j]);
  free(b->envs);
  free(b);
}

int64_t orc_batch_step(orc_batch* b, int32_t steps, int32_t observe) {
  int64_t games = 0;
  for (int64_t j = 0; j < b->n; j++) {
    orc_env* e = b->envs[j];
    for (int t = 0; t < steps; t++) {
      if (e->env_terminated || e->env_truncated) {
        e->resets++;
        orc_env_init(e, &b->cfg, orc_derive_key(e->env_key, 2 + (uint64_t)e->resets));
      }
      uint64_t kc[2] = {e->policy_key, e->policy_counter};
      const int a = orc_random_policy(e, kc);
      e->policy_counter = kc[1];
      orc_env_step(e, a);
      if (observe) orc_env_observe(e, e->current_player, &b->obs);
      if (e->env_terminated || e->env_truncated) games++;
    }
  }
  return games;
}
