// rs_tables.h — shanten tables re-encoded for the B200 memory hierarchy.
//
// The reference evaluates the standard-form shanten with one dense int8
// row per suit code (hand/tables.py:181-188: 5^9 x 10 suit rows, 5^7 x 10
// honor rows, 19.5 MB) and a sequential budget-split merge per query
// (hand/shanten.py:30-63).  Here the same values are factored once on the
// host into:
//   suit_cls  u8[5^9]   code -> class of its 10-value row   (1.95 MB, L2)
//   honor_cls u8[5^7]   code -> class                        (78 KB,  L2)
//   t1        u8[NS*NS] (class_m, class_p) -> merged-pair id A (smem)
//   t2        u8[NS*NH] (class_s, class_z) -> merged-pair id B (smem)
//   t3        u32[NA*NB] (A, B) -> best value per block budget 0..4,
//             4 bits each (smem)
// The merge is a truncated (max,+) convolution, so merging (m,p) and (s,z)
// first and combining the two halves equals the reference's left fold at
// every budget <= 4; a query is 4 class loads + 3 smem loads.
#pragma once

#include <stdint.h>

#include <vector>

namespace rs {

constexpr int SUIT_CODES = 1953125;  // 5^9
constexpr int HONOR_CODES = 78125;   // 5^7
// Geometry of the factored tables.  These are facts of the reference's
// DP (checked at build time by host_tables()); fixing them makes every
// shared-memory offset a compile-time constant on the device.
constexpr int NS = 70;  // distinct suit rows (69 legal + the zeroed illegal row)
constexpr int NH = 25;  // distinct honor rows
constexpr int NA = 95;  // distinct (m, p) merges
constexpr int NB = 84;  // distinct (s, z) merges
constexpr int T3_BYTES = 4 * NA * NB;
constexpr int T1_OFF = T3_BYTES;
constexpr int T2_OFF = T1_OFF + NS * NS;
constexpr int POW_OFF = (T2_OFF + NS * NH + 3) & ~3;  // u32[34]: code delta per kind
constexpr int SMEM_TABLE_BYTES = POW_OFF + 4 * 34;
// The stepping kernels read the factored tables through L1 from global
// memory (the default; every CTA used to wait ~3 us for its 38.7 KB copy at
// the start of a K=1 launch) or, built with -DRS_TABLES_SMEM, from a copy
// staged into shared memory by one TMA bulk copy per CTA (optionally
// multicast over a thread-block cluster).  The deal's shuffle scratch
// starts the dynamic shared memory, after the staged tables if any.
#if defined(RS_TABLES_SMEM)
constexpr int WALL_SLOT_OFF = (SMEM_TABLE_BYTES + 15) & ~15;
#else
constexpr int WALL_SLOT_OFF = 0;
#endif

struct HostTables {
  bool ready = false;
  std::vector<uint8_t> suit_cls, honor_cls;
  int ns = 0, nh = 0, na = 0, nb = 0;
  std::vector<int8_t> suit_vec, honor_vec;  // [class][10]
  std::vector<uint8_t> t1, t2;
  std::vector<uint32_t> t3;
  std::vector<uint64_t> suit_words, honor_words;  // legal codes only (blob order)
  uint32_t crc = 0;
};

// device/host view used by the engine
struct Tabs {
  const uint8_t* suit_cls;
  const uint8_t* honor_cls;
  const uint8_t* t1;
  const uint8_t* t2;
  const uint32_t* t3;
};

// builds (once) from scratch; returns nullptr-free reference
const HostTables& host_tables();
// replaces the singleton from a reference blob (docs/formats.md:54-74);
// returns 0 or a negative error
int host_tables_load(const uint8_t* blob, int64_t size);
int64_t host_tables_blob(uint8_t* out, int64_t cap);
uint32_t crc32_bytes(const uint8_t* data, int64_t n, uint32_t crc);

}  // namespace rs
