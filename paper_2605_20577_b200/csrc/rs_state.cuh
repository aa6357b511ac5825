// rs_state.cuh — env state in HBM and its shared-memory stage.
//
// The state a step touches on every transition (packed game header, scores,
// the four hands' tile sets / suit codes / classes / flags / waits / river
// kinds / observation tokens, the legal mask and the wall) is one
// contiguous 544-byte block per env in HBM.  A stepping kernel moves an
// env's block into shared memory with one TMA bulk copy, runs the
// transition against shared memory (every access a ~30-cycle LDS/STS, and
// shared-memory traffic cannot alias the global stores of the step, so the
// dependent chain of a transition never waits on L2 / HBM), and moves the
// block back with one bulk copy.  Rarely touched or write-mostly fields
// (melds, river, event rings, kyoku result) stay field-major in HBM.
//
// Field inventory follows the reference GameState / HandState
// (engine/types.py:72-158); `canonical_state_bytes()` is the S of the roofline.
#pragma once

#include <stdint.h>
#include <string.h>

#include "../../include/rinshan.h"
#include "rs_common.cuh"

namespace rs {

constexpr int WALL_STRIDE = 144;  // 136 tiles padded to 9 x 16 B
// per-thread shuffle scratch in shared memory: 37 words, odd, so the 32 lanes
// of a warp touching the same byte offset of their own copies hit 32
// different banks (a 36-word stride put 4 lanes on every bank)
constexpr int SCRATCH_STRIDE = 148;
// with lane groups (G > 1) one shuffle scratch per env instead: the wall
// copy, then the 135 swap targets the group's lanes draw in parallel
constexpr int ENV_SCRATCH = 288;  // 148 + 136, 16-byte multiple
// shuffle scratch bytes of a CTA of `block` threads at 2^glog2 lanes per env
RS_HD constexpr int scratch_bytes(int block, int glog2) {
  return glog2 == 0 ? block * SCRATCH_STRIDE : (block >> glog2) * ENV_SCRATCH;
}

// ------------------------------------------------ the env block (HBM)
// 132 words then the 144-byte wall; in shared memory each env's slot adds
// its mbarrier (the bulk copy's completion) and pads to 16 bytes
constexpr uint32_t W_HDR = 0;      // 4 x uint4 packed game scalars (Game::pack)
constexpr uint32_t W_SCORES = 16;  // int4
constexpr uint32_t W_HTOK = 20;    // 4 seats x uint4 sorted hand tokens (observe.py:89-90), pad 37
constexpr uint32_t W_HWAITS = 36;  // 4 seats x u64 34-bit wait mask (13-form tenpai)
constexpr uint32_t W_HRKIND = 44;  // 4 seats x u64 kinds present in the river
constexpr uint32_t W_HMASK = 52;   // 4 seats x 5 words: 136-bit concealed tile-id set
constexpr uint32_t W_HCODE = 72;   // 4 seats x 4 base-5 codes m, p, s, z
constexpr uint32_t W_HCLS = 88;    // 4 seats: table class per suit (4 x u8)
constexpr uint32_t W_HINFO = 92;   // 4 seats: packed HandState flags
constexpr uint32_t W_LEGAL = 96;   // 4 words env-view legal mask
// melds: seat s, meld i at words W_MELD + 2 (4 s + i): tile ids (4 x u8),
// then type | n | from | called -- a seat's four melds are one 32-byte
// sector, prefetched with the rest of the block (they used to be
// field-major arrays: a DRAM round trip per meld read at large batches)
constexpr uint32_t W_MELD = 100;
constexpr uint32_t W_WORDS = 132;
constexpr uint32_t BLK_WALL = 4 * W_WORDS;               // 528: wall bytes
constexpr uint32_t BLK_BYTES = BLK_WALL + WALL_STRIDE;   // 672 per env in HBM (42 x 16 B)
constexpr uint32_t SLOT_BAR = BLK_BYTES;                 // mbarrier of the slot
constexpr uint32_t SLOT_BYTES = BLK_BYTES + 16;          // 688 per env in shared memory

struct Soa {
  int n;
  uint8_t* blk;      // [n][672] env blocks (layout above)
  uint16_t* river;   // [4 seat][40][n] tile | flags << 8
  // [n][64] ring (256 B per env) of event words (rs_engine.cuh event_word):
  // the event and its observer-independent tokens; observe() reads the
  // window slots (len + i) & 63 and synthesizes pads
  uint32_t* events;
  rs_result_rec* results;  // [n] last kyoku result (written at kyoku end)
};

// An engine addresses its env's block through one base pointer: the
// stage slot in shared memory (stepping kernels at small batches) or the
// block in HBM; every field is an immediate offset from it.
#if defined(__CUDACC__)
extern __shared__ __align__(16) uint8_t g_smem[];
#endif
RS_HD uint32_t& sword(const uint8_t* b, uint32_t i) { return const_cast<uint32_t*>(reinterpret_cast<const uint32_t*>(b))[i]; }
RS_HD uint64_t& sdword(const uint8_t* b, uint32_t i) {
  return *const_cast<uint64_t*>(reinterpret_cast<const uint64_t*>(b + 4 * i));
}
RS_HD uint4& squad(const uint8_t* b, uint32_t i) { return *const_cast<uint4*>(reinterpret_cast<const uint4*>(b + 4 * i)); }
RS_HD uint8_t* swall(const uint8_t* b) { return const_cast<uint8_t*>(b) + BLK_WALL; }

// S of the roofline: the fields that define one env's game (header, scores,
// wall, concealed sets, flags, waits, river kinds, melds, river, event ring,
// legal mask); excludes derived caches (suit codes / classes, per-observer
// event streams) and the kyoku-result output record
constexpr int64_t canonical_state_bytes() {
  return 4 * 16 + 16 + WALL_STRIDE + 4 * 5 * 4 + 4 * 4 + 4 * 8 + 4 * 8 + 4 * 4 * 4 + 4 * 4 * 4 +
         4 * RS_MAX_RIVER * 2 + RS_EVENT_WINDOW * 2 + 4 * 4;
}

inline int64_t bytes_per_env() {
  return BLK_BYTES + 4 * RS_MAX_RIVER * 2 + RS_EVENT_WINDOW * 4 + (int64_t)sizeof(rs_result_rec);
}

struct Cfg {
  int rule, mode, reward_scheme;
  float illegal_penalty;
  int max_steps, kazoe, double_yakuman, agari_yame, renchan_cap;
};

// --------------------------------------------------------- packed fields
// HandState flag word (hinfo)
namespace hi {
RS_HD int riichi(uint32_t x) { return x & 3; }
RS_HD int riichi_index(uint32_t x) { return (int)((x >> 2) & 63) - 1; }
RS_HD int ippatsu(uint32_t x) { return (x >> 8) & 1; }
RS_HD int temp(uint32_t x) { return (x >> 9) & 1; }
RS_HD int perm(uint32_t x) { return (x >> 10) & 1; }
RS_HD int shanten(uint32_t x) { return (int)((x >> 11) & 15) - 1; }
RS_HD int nmelds(uint32_t x) { return (x >> 15) & 7; }
RS_HD int nriver(uint32_t x) { return (x >> 18) & 63; }
RS_HD int nconc(uint32_t x) { return (x >> 24) & 15; }
RS_HD uint32_t set(uint32_t x, int shift, int width, int v) {
  uint32_t m = ((1u << width) - 1u) << shift;
  return (x & ~m) | (((uint32_t)v << shift) & m);
}
RS_HD uint32_t set_riichi(uint32_t x, int v) { return set(x, 0, 2, v); }
RS_HD uint32_t set_riichi_index(uint32_t x, int v) { return set(x, 2, 6, v + 1); }
RS_HD uint32_t set_ippatsu(uint32_t x, int v) { return set(x, 8, 1, v); }
RS_HD uint32_t set_temp(uint32_t x, int v) { return set(x, 9, 1, v); }
RS_HD uint32_t set_perm(uint32_t x, int v) { return set(x, 10, 1, v); }
RS_HD uint32_t set_shanten(uint32_t x, int v) { return set(x, 11, 4, v + 1); }
RS_HD uint32_t set_nmelds(uint32_t x, int v) { return set(x, 15, 3, v); }
RS_HD uint32_t set_nriver(uint32_t x, int v) { return set(x, 18, 6, v); }
RS_HD uint32_t set_nconc(uint32_t x, int v) { return set(x, 24, 4, v); }
}  // namespace hi

// meld info word
namespace mi {
RS_HD int type(uint32_t x) { return x & 7; }
RS_HD int ntiles(uint32_t x) { return (x >> 3) & 7; }
RS_HD int from(uint32_t x) { return (int)((x >> 6) & 7) - 1; }
RS_HD int called(uint32_t x) { return (int)((x >> 9) & 255) - 1; }
RS_HD uint32_t make(int type, int n, int from, int called) {
  return (uint32_t)type | ((uint32_t)n << 3) | ((uint32_t)(from + 1) << 6) | ((uint32_t)(called + 1) << 9);
}
}  // namespace mi

// ------------------------------------------------------- game scalars
// GameState scalars (engine/types.py:124-158) + env wrapper + rollout keys,
// held in registers for the duration of one step.
// The scalars are bit-fields laid out exactly as the block's four header
// words: load / store are word copies, and the live header is 16 words of
// registers instead of ~35 unpacked ones (accesses become bit-field
// extracts / inserts, cheap on an issue-idle SM).  Measured against
// unpacked fields at the same 128-register cap: 4,096 envs +4 %, fused
// 100-step +5 %, 1 M envs +7 %; k_rollout's stack frame 832 -> 720 B.
// Widths: every value the engine stores fits (kyoku <= 7, cursor <= 122,
// drawn / call_tile -1..135, honba / deposits / repeats / results <= 255).
struct Game {
  uint32_t phase : 2, actor : 2, kyoku : 3, riichi_pending : 1, rinshan_pending : 1, call_chankan : 1,
      four_kan_pending : 1, any_call_made : 1, terminated : 1, truncated : 1, env_terminated : 1, env_truncated : 1,
      pending_dora : 3, dora_count : 3, kan_draws : 3;
  int call_from : 3;
  uint32_t current_player : 2, status : 2;
  int drawn : 9, call_tile : 9, kakan_kind : 7;
  uint32_t cursor : 7;
  uint32_t queue : 23, rons : 9;
  uint32_t honba : 8, deposits : 8, repeats : 8, n_results : 8;
  uint32_t step_count, events_len, rng_counter, resets;
  uint64_t rng_key, policy_counter, policy_key, env_key;
  int scores[4];

  RS_HD void unpack(uint4 a, uint4 b, uint4 c, uint4 d, int4 sc) {
    uint4 w[4] = {a, b, c, d};
    memcpy(this, w, 64);
    scores[0] = sc.x; scores[1] = sc.y; scores[2] = sc.z; scores[3] = sc.w;
  }
  RS_HD void pack(uint4& a, uint4& b, uint4& c, uint4& d, int4& sc) const {
    uint4 w[4];
    memcpy(w, this, 64);
    a = w[0]; b = w[1]; c = w[2]; d = w[3];
    sc.x = scores[0]; sc.y = scores[1]; sc.z = scores[2]; sc.w = scores[3];
  }

  // call queue helpers (engine/types.py:143-144)
  RS_HD int qn() const { return queue & 7; }
  RS_HD int qseat(int i) const { return (queue >> (3 + 4 * i)) & 3; }
  RS_HD int qstage(int i) const { return (queue >> (5 + 4 * i)) & 3; }
  RS_HD void qset(int n, const int* seats, const int* stages) {
    RS_CHECK(n >= 0 && n <= 5);
    uint32_t q = (uint32_t)n;
    for (int i = 0; i < n; i++) q |= ((uint32_t)seats[i] | ((uint32_t)stages[i] << 2)) << (3 + 4 * i);
    queue = q;
  }
  RS_HD void qpop() {
    int n = qn();
    RS_CHECK(n > 0);
    uint32_t entries = (queue >> 7) & 0xFFFFu;
    queue = (uint32_t)(n - 1) | (entries << 3);
  }
  RS_HD int rn() const { return rons & 3; }
  RS_HD int rseat(int i) const { return (rons >> (2 + 2 * i)) & 3; }
  RS_HD void rpush(int s) {
    int n = rn();
    RS_CHECK(n < 3 && (unsigned)s < 4u);
    rons = (rons & ~3u) | (uint32_t)(n + 1) | ((uint32_t)s << (2 + 2 * n));
  }
  RS_HD int dealer() const { return kyoku % 4; }
  RS_HD int round_wind() const { return kyoku >= 4 ? 28 : 27; }
  RS_HD int seat_wind(int s) const { return 27 + ((s - dealer()) & 3); }
  RS_HD int live() const { return 122 - kan_draws - cursor; }
};
static_assert(sizeof(Game) == 80, "Game: the four header words + scores");

}  // namespace rs
