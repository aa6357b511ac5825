// rs_tables.cpp — host construction of the re-encoded shanten tables.
//
// Stage 1 reproduces the reference's per-suit statistics (hand/tables.py:
// _fill_stats :51-120 DP over ascending base-5 codes, _pack_words :123-147
// sub-entry selection, _values_from_words :169-178, illegal codes zeroed
// :191-209).  Stage 2 (new) deduplicates the 10-value rows into classes and
// precomputes the pairwise (max,+) merges so a device query needs no loop.
#include "rs_tables.h"

#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <map>
#include <mutex>

namespace rs {

namespace {

constexpr int NEGV = -99;

// DP state per code: best partial count for (head h, complete sets s),
// -1 when unreachable.  Codes are visited in ascending order so every
// removal of tiles refers to a solved code.
void suit_dp(int n_digits, bool runs, std::vector<int8_t>& dp) {
  const int ncodes = (int)dp.size() / 10;
  int p5[9];
  for (int i = n_digits - 1, p = 1; i >= 0; i--, p *= 5) p5[i] = p;
  std::fill(dp.begin(), dp.begin() + 10, (int8_t)-1);
  dp[0] = 0;
  int digit[9] = {0};
  for (int code = 1; code < ncodes; code++) {
    // increment the little-endian digit vector (digit n-1 least significant)
    for (int i = n_digits - 1; i >= 0; i--) {
      if (++digit[i] < 5) break;
      digit[i] = 0;
    }
    int lead = 0;
    while (digit[lead] == 0) lead++;
    int8_t* row = &dp[(size_t)code * 10];
    std::fill(row, row + 10, (int8_t)-1);
    auto relax_from = [&](int child_code, auto&& body) {
      const int8_t* ch = &dp[(size_t)child_code * 10];
      body(ch);
    };
    // one copy of the leading kind left unused
    relax_from(code - p5[lead], [&](const int8_t* ch) {
      for (int j = 0; j < 10; j++) row[j] = std::max(row[j], ch[j]);
    });
    auto pair_like = [&](const int8_t* ch, bool may_be_head) {
      for (int h = 0; h < 2; h++)
        for (int s = 0; s < 5; s++) {
          int q = ch[h * 5 + s];
          if (q < 0) continue;
          if (may_be_head && h == 0) row[5 + s] = (int8_t)std::max<int>(row[5 + s], q);
          row[h * 5 + s] = (int8_t)std::max<int>(row[h * 5 + s], std::min(q + 1, 4));
        }
    };
    auto set_like = [&](const int8_t* ch) {
      for (int h = 0; h < 2; h++)
        for (int s = 0; s < 4; s++) {
          int q = ch[h * 5 + s];
          if (q >= 0) row[h * 5 + s + 1] = (int8_t)std::max<int>(row[h * 5 + s + 1], q);
        }
    };
    const int d = digit[lead];
    if (d >= 2) relax_from(code - 2 * p5[lead], [&](const int8_t* ch) { pair_like(ch, true); });
    if (d >= 3) relax_from(code - 3 * p5[lead], set_like);
    if (runs) {
      const bool has1 = lead + 1 < n_digits && digit[lead + 1] > 0;
      const bool has2 = lead + 2 < n_digits && digit[lead + 2] > 0;
      if (has1 && has2) relax_from(code - p5[lead] - p5[lead + 1] - p5[lead + 2], set_like);
      if (has1) relax_from(code - p5[lead] - p5[lead + 1], [&](const int8_t* ch) { pair_like(ch, false); });
      if (has2) relax_from(code - p5[lead] - p5[lead + 2], [&](const int8_t* ch) { pair_like(ch, false); });
    }
  }
}

uint64_t pack_word(const int8_t* row) {
  uint64_t w = 0;
  for (int m = 0; m < 5; m++)
    for (int h = 0; h < 2; h++) {
      int bv = -1, bs = 0, bp = 0;
      for (int s = 0; s <= m; s++) {
        int q = row[h * 5 + s];
        if (q < 0) continue;
        int pe = std::min(q, m - s), v = 2 * s + pe;
        if (v > bv || (v == bv && s > bs)) { bv = v; bs = s; bp = pe; }
      }
      uint64_t sub = bv < 0 ? 0x3Fu : (uint64_t)(bs | (bp << 3));
      w |= sub << (6 * (m * 2 + h));
    }
  return w;
}

std::array<int8_t, 10> word_values(uint64_t w) {
  std::array<int8_t, 10> v;
  for (int i = 0; i < 10; i++) {
    uint64_t sub = (w >> (6 * i)) & 0x3F;
    v[i] = sub == 0x3F ? (int8_t)NEGV : (int8_t)(2 * (sub & 7) + (sub >> 3));
  }
  return v;
}

int digit_sum(int code) {
  int t = 0;
  while (code) { t += code % 5; code /= 5; }
  return t;
}

// dense words (zero for codes holding more than 14 tiles)
void dense_words(int n_digits, bool runs, std::vector<uint64_t>& dense, std::vector<uint64_t>& legal) {
  int ncodes = 1;
  for (int i = 0; i < n_digits; i++) ncodes *= 5;
  std::vector<int8_t> dp((size_t)ncodes * 10);
  suit_dp(n_digits, runs, dp);
  dense.assign(ncodes, 0);
  legal.clear();
  for (int c = 0; c < ncodes; c++)
    if (digit_sum(c) <= 14) {
      dense[c] = pack_word(&dp[(size_t)c * 10]);
      legal.push_back(dense[c]);
    }
}

// (max,+) merge of two 10-vectors [a0[b], a1[b]] interleaved (shanten.py:40-60)
std::array<int, 10> merge(const std::array<int, 10>& a, const std::array<int, 10>& r) {
  std::array<int, 10> n;
  n.fill(NEGV);
  for (int b = 0; b < 5; b++)
    for (int k = 0; k <= b; k++) {
      int v0 = r[2 * k], v1 = r[2 * k + 1], x0 = a[2 * (b - k)], x1 = a[2 * (b - k) + 1];
      if (v0 > NEGV) {
        if (x0 > NEGV) n[2 * b] = std::max(n[2 * b], x0 + v0);
        if (x1 > NEGV) n[2 * b + 1] = std::max(n[2 * b + 1], x1 + v0);
      }
      if (v1 > NEGV && x0 > NEGV) n[2 * b + 1] = std::max(n[2 * b + 1], x0 + v1);
    }
  return n;
}

void classify(const std::vector<uint64_t>& dense, std::vector<uint8_t>& cls, std::vector<int8_t>& vecs, int& ncls) {
  std::map<std::array<int8_t, 10>, int> ids;  // ordered -> deterministic numbering
  for (uint64_t w : dense) ids.emplace(word_values(w), 0);
  int next = 0;
  vecs.clear();
  for (auto& kv : ids) {
    kv.second = next++;
    vecs.insert(vecs.end(), kv.first.begin(), kv.first.end());
  }
  ncls = next;
  cls.resize(dense.size());
  for (size_t c = 0; c < dense.size(); c++) cls[c] = (uint8_t)ids[word_values(dense[c])];
}

std::array<int, 10> vec_of(const std::vector<int8_t>& v, int c) {
  std::array<int, 10> a;
  for (int i = 0; i < 10; i++) a[i] = v[(size_t)c * 10 + i];
  return a;
}

void finalize(HostTables& T, std::vector<uint64_t>& sd, std::vector<uint64_t>& hd) {
  classify(sd, T.suit_cls, T.suit_vec, T.ns);
  classify(hd, T.honor_cls, T.honor_vec, T.nh);
  std::map<std::array<int, 10>, int> amap, bmap;
  std::vector<std::array<int, 10>> avec, bvec;
  T.t1.assign((size_t)T.ns * T.ns, 0);
  T.t2.assign((size_t)T.ns * T.nh, 0);
  for (int i = 0; i < T.ns; i++)
    for (int j = 0; j < T.ns; j++) {
      auto m = merge(vec_of(T.suit_vec, i), vec_of(T.suit_vec, j));
      auto it = amap.find(m);
      if (it == amap.end()) { it = amap.emplace(m, (int)avec.size()).first; avec.push_back(m); }
      T.t1[(size_t)i * T.ns + j] = (uint8_t)it->second;
    }
  for (int i = 0; i < T.ns; i++)
    for (int j = 0; j < T.nh; j++) {
      auto m = merge(vec_of(T.suit_vec, i), vec_of(T.honor_vec, j));
      auto it = bmap.find(m);
      if (it == bmap.end()) { it = bmap.emplace(m, (int)bvec.size()).first; bvec.push_back(m); }
      T.t2[(size_t)i * T.nh + j] = (uint8_t)it->second;
    }
  T.na = (int)avec.size();
  T.nb = (int)bvec.size();
  T.t3.assign((size_t)T.na * T.nb, 0);
  for (int a = 0; a < T.na; a++)
    for (int b = 0; b < T.nb; b++) {
      auto m = merge(avec[a], bvec[b]);
      uint32_t packed = 0;
      for (int bud = 0; bud <= 4; bud++) {
        int best = m[2 * bud];
        if (m[2 * bud + 1] > NEGV && m[2 * bud + 1] + 1 > best) best = m[2 * bud + 1] + 1;
        // best >= 0 always: the empty reading (no sets, no head) exists
        packed |= (uint32_t)(best & 0xF) << (4 * bud);
      }
      T.t3[(size_t)a * T.nb + b] = packed;
    }
  uint8_t buf[8];
  uint32_t crc = 0;
  for (auto* words : {&T.suit_words, &T.honor_words})
    for (uint64_t w : *words) {
      for (int b = 0; b < 8; b++) buf[b] = (uint8_t)(w >> (8 * b));
      crc = crc32_bytes(buf, 8, crc);
    }
  T.crc = crc;
  T.ready = true;
}

HostTables g_tables;
std::mutex g_mu;

}  // namespace

uint32_t crc32_bytes(const uint8_t* data, int64_t n, uint32_t crc) {
  static uint32_t table[256];
  static std::once_flag once;
  std::call_once(once, [] {
    for (uint32_t i = 0; i < 256; i++) {
      uint32_t c = i;
      for (int k = 0; k < 8; k++) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[i] = c;
    }
  });
  crc = ~crc;
  for (int64_t i = 0; i < n; i++) crc = table[(crc ^ data[i]) & 0xFF] ^ (crc >> 8);
  return ~crc;
}

const HostTables& host_tables() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_tables.ready) {
    std::vector<uint64_t> sd, hd;
    dense_words(9, true, sd, g_tables.suit_words);
    dense_words(7, false, hd, g_tables.honor_words);
    finalize(g_tables, sd, hd);
    if (g_tables.ns != NS || g_tables.nh != NH || g_tables.na != NA || g_tables.nb != NB) abort();
  }
  return g_tables;
}

int host_tables_load(const uint8_t* blob, int64_t size) {
  if (size < 24 || memcmp(blob, "MJSUIT1\0", 8) != 0) return -4;
  uint32_t hdr[4];
  for (int i = 0; i < 4; i++) {
    hdr[i] = 0;
    for (int b = 0; b < 4; b++) hdr[i] |= (uint32_t)blob[8 + 4 * i + b] << (8 * b);
  }
  const int64_t ns = hdr[0], nh = hdr[1];
  if (ns != 405350 || nh != 43130 || size != 24 + 8 * (ns + nh)) return -4;
  if (crc32_bytes(blob + 24, size - 24, 0) != hdr[2]) return -4;
  HostTables T;
  auto rd = [&](int64_t i) {
    uint64_t w = 0;
    for (int b = 0; b < 8; b++) w |= (uint64_t)blob[24 + 8 * i + b] << (8 * b);
    return w;
  };
  std::vector<uint64_t> sd(SUIT_CODES, 0), hd(HONOR_CODES, 0);
  int64_t k = 0;
  for (int c = 0; c < SUIT_CODES; c++)
    if (digit_sum(c) <= 14) { sd[c] = rd(k); T.suit_words.push_back(sd[c]); k++; }
  for (int c = 0; c < HONOR_CODES; c++)
    if (digit_sum(c) <= 14) { hd[c] = rd(k); T.honor_words.push_back(hd[c]); k++; }
  finalize(T, sd, hd);
  if (T.ns != NS || T.nh != NH || T.na != NA || T.nb != NB) return -4;
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_tables.ready) {
    // tables already built / loaded: host_tables() hands out references and
    // device copies are made once per device, so the live tables are never
    // replaced; an identical blob is a no-op, a different one an error
    const bool same = T.suit_words == g_tables.suit_words && T.honor_words == g_tables.honor_words;
    return same ? 0 : -5;
  }
  g_tables = std::move(T);
  return 0;
}

int64_t host_tables_blob(uint8_t* out, int64_t cap) {
  const HostTables& T = host_tables();
  const int64_t size = 24 + 8 * (int64_t)(T.suit_words.size() + T.honor_words.size());
  if (!out || cap < size) return size;
  memcpy(out, "MJSUIT1\0", 8);
  const uint32_t hdr[4] = {(uint32_t)T.suit_words.size(), (uint32_t)T.honor_words.size(), T.crc, 0};
  for (int i = 0; i < 4; i++)
    for (int b = 0; b < 4; b++) out[8 + 4 * i + b] = (uint8_t)(hdr[i] >> (8 * b));
  uint8_t* p = out + 24;
  for (auto* words : {&T.suit_words, &T.honor_words})
    for (uint64_t w : *words)
      for (int b = 0; b < 8; b++) *p++ = (uint8_t)(w >> (8 * b));
  return size;
}

}  // namespace rs
