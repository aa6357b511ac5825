// rs_common.cuh — shared primitives of the B200 env-step engine.
//
// Everything here is __host__ __device__ so the identical engine source can
// also be compiled by g++ for the test-only host harness (tests/hostcheck),
// which exercises the transition logic without a GPU; the shipped library
// is the nvcc sm_100a build.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#include <cuda_runtime.h>
#define RS_HD __host__ __device__ inline
#define RS_HOT __host__ __device__ __forceinline__
#if defined(RS_ALL_INLINE)  // (measured alternative: -5 % at 4,096 envs, -18 % fused, -4 % at 1 M)
#define RS_COLD __host__ __device__ inline
#else
#define RS_COLD __host__ __device__ __noinline__
#endif
#define RS_DEV_ONLY __device__
#else
#define RS_HD inline
#define RS_HOT inline
#define RS_COLD
#define RS_DEV_ONLY
// host-only build (test harness): the CUDA vector types the state uses
struct alignas(16) uint4 { uint32_t x, y, z, w; };
struct alignas(16) int4 { int x, y, z, w; };
inline uint4 make_uint4(uint32_t x, uint32_t y, uint32_t z, uint32_t w) { return uint4{x, y, z, w}; }
#endif

// -DRS_BOUNDS: bounds checks on every state-array index, wall position,
// meld / river slot and shared-memory scratch / stage offset; a violation
// traps the kernel (abort() in the host build).  compute-sanitizer is not
// available on the measurement pool, so the parity suite runs against this
// build (tools/bounds_check.sh) and the host build runs under ASan / UBSan
// (tests/test_hostcheck_sanitized.py).  Off in the shipped library.
#if defined(RS_BOUNDS)
#if defined(__CUDA_ARCH__)
#define RS_CHECK(c) \
  do {              \
    if (!(c)) __trap(); \
  } while (0)
#else
#include <stdlib.h>
#define RS_CHECK(c) \
  do {              \
    if (!(c)) abort(); \
  } while (0)
#endif
#else
#define RS_CHECK(c) ((void)0)
#endif

// Measured alternatives kept buildable (tools/build_variant.sh -D...):
//   -DRS_AB_OFF_WIN16   observation window over 4 lanes instead of 8 / 16
//   -DRS_NO_CLAIM_LANES the opponents' claim checks on every lane of the
//                       env's group instead of one opponent per lane (lanes
//                       1-3, combined by one warp reduction: the default
//                       since the cold paths shrank, DESIGN §4 items 31, 56)
//   -DRS_SWAP5          the deal's swap chain five swaps per load round
//                       (neutral to -0.7 %: resets are not the launch tail)
#if defined(RS_AB_OFF_WIN16)
#define RS_WIN16 0
#else
#define RS_WIN16 1
#endif
#if defined(RS_NO_CLAIM_LANES)
#define RS_CLAIM_LANES_ON 0
#else
#define RS_CLAIM_LANES_ON 1
#endif
#if defined(RS_SWAP5)
#define RS_SWAP5_ON 1
#else
#define RS_SWAP5_ON 0
#endif

namespace rs {

#if defined(__CUDACC__)
// dynamic shared memory of the running CTA (RS_BOUNDS checks of scratch /
// stage offsets)
__device__ __forceinline__ uint32_t dyn_smem_bytes() {
#if defined(__CUDA_ARCH__)
  uint32_t v;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
#else
  return 0u;
#endif
}
#endif

// -DRS_PROFILE_MARKS=3: per-thread cycle accumulators of selected functions
// (profiling builds only; g_marks[thread][8])
#if defined(RS_PROFILE_MARKS) && defined(__CUDACC__)
__device__ unsigned long long* g_marks;
#endif
#if defined(RS_PROFILE_MARKS) && RS_PROFILE_MARKS == 3 && defined(__CUDA_ARCH__)
struct AccTimer {
  int slot;
  long long t0;
  __device__ explicit AccTimer(int i) : slot(i), t0(clock64()) {}
  __device__ ~AccTimer() {
    if (g_marks) g_marks[(size_t)(blockIdx.x * blockDim.x + threadIdx.x) * 8 + slot] += clock64() - t0;
  }
};
#define RS_ACC(i) ::rs::AccTimer _acc_timer_##i(i)
#else
#define RS_ACC(i) do {} while (0)
#endif

constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;

// ------------------------------------------------------- lane groups
// At small batches a warp holds fewer envs than lanes; the stepping kernels
// then give each env a group of G = 2^s_grp_log2 consecutive lanes that run
// the engine redundantly (identical data, identical control flow) and
// split the long loops of the rare paths (wait scans, riichi filters,
// the observation window) between them, combining with warp reductions.
// G = 1 everywhere else (and on the host).
#if defined(__CUDACC__)
__shared__ int s_grp_log2;
#endif
RS_HD int grp_size() {
#if defined(__CUDA_ARCH__)
  return 1 << s_grp_log2;
#else
  return 1;
#endif
}
RS_HD int grp_sub() {
#if defined(__CUDA_ARCH__)
  return (int)(threadIdx.x & 31) & (grp_size() - 1);
#else
  return 0;
#endif
}
RS_HD uint32_t grp_mask() {
#if defined(__CUDA_ARCH__)
  const int G = grp_size();
  return G == 32 ? 0xFFFFFFFFu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(uint32_t)(G - 1)));
#else
  return 1u;
#endif
}
// memory ordering between the lanes of the env's group (a lane reads what
// another lane of the group wrote: the observer streams, emit_event_impl)
RS_HD void grp_sync() {
#if defined(__CUDA_ARCH__)
  if (grp_size() > 1) __syncwarp(grp_mask());
#endif
}
RS_HD uint32_t grp_or32(uint32_t x) {
#if defined(__CUDA_ARCH__)
  if (grp_size() == 1) return x;
  return __reduce_or_sync(grp_mask(), x);
#else
  return x;
#endif
}
RS_HD uint64_t grp_or64(uint64_t x) {
#if defined(__CUDA_ARCH__)
  if (grp_size() == 1) return x;
  const uint32_t m = grp_mask();
  return (uint64_t)__reduce_or_sync(m, (uint32_t)x) | ((uint64_t)__reduce_or_sync(m, (uint32_t)(x >> 32)) << 32);
#else
  return x;
#endif
}

// ---------------------------------------------------------------- bit ops
RS_HD int popc32(uint32_t x) {
#if defined(__CUDA_ARCH__)
  return __popc(x);
#else
  return __builtin_popcount(x);
#endif
}
RS_HD int popc64(uint64_t x) {
#if defined(__CUDA_ARCH__)
  return __popcll(x);
#else
  return __builtin_popcountll(x);
#endif
}
RS_HD int ctz32(uint32_t x) {  // x != 0
#if defined(__CUDA_ARCH__)
  return __ffs((int)x) - 1;
#else
  return __builtin_ctz(x);
#endif
}
RS_HD int ctz64(uint64_t x) {  // x != 0
#if defined(__CUDA_ARCH__)
  return __ffsll((long long)x) - 1;
#else
  return __builtin_ctzll(x);
#endif
}
RS_HD int clz32(uint32_t x) {  // x != 0
#if defined(__CUDA_ARCH__)
  return __clz((int)x);
#else
  return __builtin_clz(x);
#endif
}
RS_HD uint64_t umulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// PRMT: byte i of the result is byte (s >> 4i) & 7 of {x (0-3), y (4-7)}
RS_HD uint32_t byte_perm(uint32_t x, uint32_t y, uint32_t s) {
#if defined(__CUDA_ARCH__)
  return __byte_perm(x, y, s);
#else
  const uint64_t v = (uint64_t)x | ((uint64_t)y << 32);
  uint32_t r = 0;
  for (int i = 0; i < 4; i++) r |= (uint32_t)((v >> (8 * ((s >> (4 * i)) & 7))) & 0xFF) << (8 * i);
  return r;
#endif
}

// ---------------------------------------------- counter RNG (rng.py:18-65)
// SplitMix64 finalizer; key/counter streams; randbelow = high word of x*n.
RS_HD uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
RS_HD uint64_t derive_key(uint64_t key, uint64_t stream) {
  return mix64((key ^ GOLDEN) + mix64(stream));
}
// value number `c` (1-based) of stream `key`
RS_HD uint64_t stream_value(uint64_t key, uint64_t c) { return mix64(key + c * GOLDEN); }
RS_HD uint32_t randbelow_from(uint64_t x, uint32_t n) { return (uint32_t)umulhi64(x, (uint64_t)n); }

// --------------------------------------- per-nibble tile-count arithmetic
// A hand is a 136-bit set of tile ids held in five 32-bit words; kind k owns
// the nibble (k & 7) of word k >> 3.  SWAR turns words into per-kind counts.
RS_HD uint32_t nib_counts(uint32_t x) {  // 8 nibbles of 4 bits -> 8 counts 0..4
  uint32_t v = x - ((x >> 1) & 0x55555555u);
  return (v & 0x33333333u) + ((v >> 2) & 0x33333333u);
}
// gather bit 0 of each nibble (positions 0,4,...,28) into bits 0..7
RS_HD uint32_t nib_gather(uint32_t x) {
  x &= 0x11111111u;
  x = (x | (x >> 3)) & 0x03030303u;
  x = (x | (x >> 6)) & 0x000F000Fu;
  x = (x | (x >> 12)) & 0xFFu;
  return x;
}
// bit i of the result set iff nibble count i >= t (t in 1..4)
RS_HD uint32_t nib_ge(uint32_t counts, int t) {
  uint32_t add = (uint32_t)(8 - t) * 0x11111111u;
  return nib_gather(((counts + add) & 0x88888888u) >> 3);
}
RS_HD uint32_t nib_eq(uint32_t counts, int t) {
  return t >= 4 ? nib_ge(counts, 4) : (nib_ge(counts, t) & ~nib_ge(counts, t + 1));
}

// ------------------------------------------------------------ tile facts
RS_HD bool is_orphan(int k) { return k >= 27 || k % 9 == 0 || k % 9 == 8; }
RS_HD bool is_terminal(int k) { return k < 27 && (k % 9 == 0 || k % 9 == 8); }
constexpr uint64_t ORPHAN_MASK = (1ull << 0) | (1ull << 8) | (1ull << 9) | (1ull << 17) | (1ull << 18) |
                                 (1ull << 26) | (0x7Full << 27);
constexpr uint64_t GREEN_MASK = (1ull << 19) | (1ull << 20) | (1ull << 21) | (1ull << 23) | (1ull << 25) |
                                (1ull << 32);
constexpr uint64_t HONOR_MASK = 0x7Full << 27;
constexpr uint64_t TERMINAL_MASK = ORPHAN_MASK & ~HONOR_MASK;
constexpr uint64_t KINDS_MASK = (1ull << 34) - 1;

RS_HD int dora_kind(int ind) {  // tiles.py:108-115
  if (ind < 27) return ind - ind % 9 + (ind % 9 + 1) % 9;
  if (ind < 31) return 27 + (ind - 27 + 1) % 4;
  return 31 + (ind - 31 + 1) % 3;
}
RS_HD bool is_red_tile(int t) { return t == 16 || t == 52 || t == 88; }
RS_HD int red_index_of_kind(int k) { return k == 4 ? 0 : (k == 13 ? 1 : (k == 22 ? 2 : -1)); }

RS_HD uint32_t pow5(int i) {  // 5^i, i in 0..8, without memory
  uint32_t p = 1;
  for (int j = 0; j < i; j++) p *= 5u;
  return p;
}
// code delta of one tile of kind k, and the suit slot (0 m, 1 p, 2 s, 3 z)
RS_HD uint32_t kind_pow_calc(int k) {
  return k < 27 ? pow5(8 - k % 9) : pow5(6 - (k - 27));
}
RS_HD int kind_suit(int k) { return k < 27 ? k / 9 : 3; }
// 5^d for d in 0..8 from the bits of d: selects and two multiplies, no
// memory (the per-kind table was a dependent load in every hand update)
RS_HD uint32_t pow5_bits(int d) {
  uint32_t p = (d & 1) ? 5u : 1u;
  p *= (d & 2) ? 25u : 1u;
  p *= (d & 4) ? 625u : 1u;
  return (d & 8) ? 390625u : p;  // d == 8
}

}  // namespace rs
