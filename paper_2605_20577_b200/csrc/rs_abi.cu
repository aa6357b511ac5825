// rs_abi.cu — sm_100a kernels and the extern "C" boundary (include/rinshan.h).
//
// Kernels (one thread per env, 128-thread CTAs; the pre-merged shanten
// tables are staged into shared memory at CTA start):
//   k_init      init(seed)                         env/core.py:81-82
//   k_step      step(state, action) + legal mask   env/core.py:85-94
//   k_observe   observe(state, seat)               env/observe.py:81-124
//   k_policy    random_policy(legal, rng)          env/policies.py:17-22
//   k_rollout   fused {auto-reset, random policy, step, observe} x K
//               (bench/runner.py:97-121 one_pass)
//   k_expand    packed legal bits -> bool[n][115] (coalesced)
//   k_export / k_import  projection records for the parity harness
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <new>
#include <string>

#include <cub/device/device_radix_sort.cuh>

#include "rs_check.cuh"
#include "rs_io.cuh"

using namespace rs;

namespace {

constexpr int BLOCK = 128;
// k_rollout CTA shape: one staged table copy is shared by ROLL_BLOCK
// threads; ROLL_MINB CTAs per SM caps the registers (occupancy)
#ifndef ROLL_BLOCK
#define ROLL_BLOCK 256  // large batches: 2 CTAs x 8 warps per SM
#endif
#ifndef ROLL_MINB
#define ROLL_MINB 2  // <= 128 registers, no spills
#endif
// dynamic shared memory of a CTA: staged tables + one 144-byte wall slot
// per thread for the deal (rs_engine.cuh start_kyoku)
// dynamic shared memory: the staged tables, then either one stage slot per
// env of the CTA (staged stepping kernels) or a 144-byte shuffle scratch
// per thread (kernels working on the blocks in HBM)
// -DRS_ENGINE_SMEM (measured alternative): the stepping kernels' Engine
// objects (the game header and the env context, addressed through `this`
// by the out-of-line members) live in a per-thread shared-memory slot
// instead of the thread's local memory, which misses L1 at large batches
// (ncu: ~100 local loads per warp-step at 262 K envs, 32 % L1 hits).
// 26 % slower at 4,096 envs, 4 % at 1 M: in local memory the compiler
// keeps most header fields in registers between the out-of-line calls.
#if defined(RS_ENGINE_SMEM)
constexpr int ENGINE_SLOT = (int)((sizeof(Engine) + 15) & ~(size_t)15);
#else
constexpr int ENGINE_SLOT = 0;
#endif
constexpr int smem_staged(int block, int slots, int glog2 = 0) {
  return WALL_SLOT_OFF + scratch_bytes(block, glog2) + block * ENGINE_SLOT + slots * (int)SLOT_BYTES;
}
constexpr int smem_for(int block, int glog2 = 0) {
  return WALL_SLOT_OFF + scratch_bytes(block, glog2) + block * ENGINE_SLOT;
}
// bytes of the staged t3 | t1 | t2 block (a TMA bulk copy is a multiple of 16 B)
constexpr uint32_t STAGE_BYTES = (SMEM_TABLE_BYTES + 15u) & ~15u;

thread_local std::string g_err;
int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess) return set_err((int)_e, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

struct DevTables {
  const uint8_t* suit_cls;
  const uint8_t* honor_cls;
  const uint8_t* t1;
  const uint8_t* t2;
  const uint32_t* t3;
  int ns, nh, na, nb;
  int smem;  // bytes of the staged copy
};

// one copy of the tables per device, shared by every handle on it (the
// class-map pointers live in __constant__ memory of the module)
struct DeviceTables {
  void* mem = nullptr;
  size_t bytes = 0;
  DevTables D{};
  // L2 residency of the whole table block (class maps + the staged image,
  // ~2.1 MB of the 126 MB L2): the stepping kernels launch with an access
  // policy window marking it persisting, so the class-map lookups and the
  // per-CTA staging copy stay L2 hits even when everything else (the env
  // state, a policy network between steps) streams through L2.
  // RINSHAN_L2_PERSIST=0 turns it off.
  cudaAccessPolicyWindow window{};
  bool persist = false;
};
std::mutex g_dev_mu;
DeviceTables g_dev_tables[64];

int device_tables(int device, DevTables* out) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (device < 0 || device >= 64) return set_err(RS_E_ARG, "device id out of range");
  DeviceTables& dt = g_dev_tables[device];
  if (!dt.mem) {
    const HostTables& H = host_tables();
    // block layout: t3 | t1 | t2 (exactly the shared-memory image) | suit | honor
    const size_t blk = ((size_t)SMEM_TABLE_BYTES + 255) & ~(size_t)255;
    const size_t sz = blk + H.suit_cls.size() + 256 + H.honor_cls.size();
    void* mem = nullptr;
    CUDA_TRY(cudaMalloc(&mem, sz));
    uint8_t* base = (uint8_t*)mem;
    uint8_t* suit = base + blk;
    uint8_t* honor = suit + ((H.suit_cls.size() + 255) & ~(size_t)255);
    CUDA_TRY(cudaMemset(base, 0, blk));
    CUDA_TRY(cudaMemcpy(base, H.t3.data(), H.t3.size() * 4, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(base + T1_OFF, H.t1.data(), H.t1.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(base + T2_OFF, H.t2.data(), H.t2.size(), cudaMemcpyHostToDevice));
    uint32_t pw[34];
    for (int k = 0; k < 34; k++) pw[k] = kind_pow_calc(k);
    CUDA_TRY(cudaMemcpy(base + POW_OFF, pw, sizeof(pw), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(suit, H.suit_cls.data(), H.suit_cls.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(honor, H.honor_cls.data(), H.honor_cls.size(), cudaMemcpyHostToDevice));
    const uint8_t* sp = suit;
    const uint8_t* hp = honor;
    CUDA_TRY(cudaMemcpyToSymbol(c_suit_cls, &sp, sizeof(sp)));
    CUDA_TRY(cudaMemcpyToSymbol(c_honor_cls, &hp, sizeof(hp)));
    const uint8_t* tb = base;
    CUDA_TRY(cudaMemcpyToSymbol(c_tblock, &tb, sizeof(tb)));
    dt.D.suit_cls = suit;
    dt.D.honor_cls = honor;
    dt.D.t3 = reinterpret_cast<const uint32_t*>(base);
    dt.D.t1 = base + T1_OFF;
    dt.D.t2 = base + T2_OFF;
    dt.D.ns = NS; dt.D.nh = NH; dt.D.na = NA; dt.D.nb = NB;
    dt.D.smem = (int)STAGE_BYTES;
    dt.mem = mem;
    dt.bytes = sz;
    const char* pe = getenv("RINSHAN_L2_PERSIST");
    int max_persist = 0, max_window = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, device);
    if (!(pe && pe[0] == '0') && max_persist > 0 && max_window > 0) {
      size_t cur = 0;
      cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
      const size_t want = std::min((size_t)max_persist, std::max(cur, sz));
      if (cur >= want || cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) {
        dt.window.base_ptr = mem;
        dt.window.num_bytes = std::min(sz, (size_t)max_window);
        dt.window.hitRatio = 1.0f;
        dt.window.hitProp = cudaAccessPropertyPersisting;
        dt.window.missProp = cudaAccessPropertyStreaming;
        dt.persist = true;
      }
      cudaGetLastError();  // a refused limit only disables the window
    }
  }
  *out = dt.D;
  return 0;
}

struct StepOut {
  uint32_t* legal_bits;
  int8_t* current_player;
  float* rewards;
  uint8_t* terminated;
  uint8_t* truncated;
  uint8_t* status;
};

// -DRS_TABLES_SMEM: stage the packed t3 | t1 | t2 block into shared memory;
// the engine reads it at compile-time offsets (rs_hand.cuh t1_at / t2_at /
// t3_at).  Default build: the tables stay in global memory (read through
// L1, kept in L2 by the persisting window) and these are no-ops.
// One elected thread issues a single TMA bulk copy (cp.async.bulk, no tensor
// map needed for a contiguous block) completing on an mbarrier; the other
// warps spend no instructions on the copy and wait on the barrier phase.
__shared__ __align__(8) uint64_t s_tables_bar;
__device__ __forceinline__ void tables_wait() {
#if !defined(RS_TABLES_SMEM)
  return;
#endif
  const uint32_t bar_addr = (uint32_t)__cvta_generic_to_shared(&s_tables_bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar_addr)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ncta() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// issue the copy; the caller waits (tables_wait) before the first table read.
// Launched as a thread-block cluster (RINSHAN_CLUSTER, stepping kernels), the
// CTAs of the cluster split the block: CTA r fetches slice r once from L2 and
// multicasts it into every CTA of the cluster, so the launch-start burst of
// table reads (every CTA at once) shrinks by the cluster size.  Each CTA's
// barrier expects the whole block; the cluster barrier orders the barrier
// initialisations before any peer's slice can complete on them.  A CTA must
// wait on its barrier before exiting (peers write into its shared memory).
__device__ __forceinline__ void tables_begin(const DevTables& D, int grp_log2) {
  const uint32_t bar_addr = (uint32_t)__cvta_generic_to_shared(&s_tables_bar);
#if !defined(RS_TABLES_SMEM)
  if (threadIdx.x == 0) s_grp_log2 = grp_log2;
  __syncthreads();
  return;
#endif
  const uint32_t nc = cluster_ncta();
  const uint32_t dst = (uint32_t)__cvta_generic_to_shared(g_smem);
  if (threadIdx.x == 0) {
    s_grp_log2 = grp_log2;  // lanes per env (rs_common.cuh), published by the barrier below
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_addr) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_addr), "r"(STAGE_BYTES)
                 : "memory");
    if (nc == 1)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
          "l"(D.t3), "r"(STAGE_BYTES), "r"(bar_addr)
          : "memory");
  }
  if (nc == 1) {
    __syncthreads();
    return;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t chunk = ((STAGE_BYTES + nc - 1) / nc + 15u) & ~15u;
    const uint32_t off = cluster_rank() * chunk;
    if (off < STAGE_BYTES) {
      const uint32_t bytes = min(chunk, STAGE_BYTES - off);
      const uint16_t mask = (uint16_t)((1u << nc) - 1u);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, "
          "[%3], %4;" ::"r"(dst + off),
          "l"(reinterpret_cast<const uint8_t*>(D.t3) + off), "r"(bytes), "r"(bar_addr), "h"(mask)
          : "memory");
    }
  }
}
__device__ __forceinline__ Tabs stage_tables(const DevTables& D, int grp_log2 = 0) {
  tables_begin(D, grp_log2);
  tables_wait();
  return Tabs{};
}

// ------------------------------------------------------------ prefetch
// RINSHAN_PREFETCH (default 2): before an env's first step, the lanes of
// its group issue L1 prefetches for the lines the step will touch first --
// the 672-byte block (6-7 lines) and, with mode 2, the env's 256-byte event
// ring that observe() reads -- one line per lane, so the dependent first
// touches of the step find them in L1 instead of waiting on HBM one after
// another
__device__ __forceinline__ void prefetch_env(const Soa& S, int e, int sub, int G, int mode) {
  const uintptr_t b0 = (uintptr_t)(S.blk + (size_t)e * BLK_BYTES) & ~(uintptr_t)127;
  const uintptr_t b1 = ((uintptr_t)(S.blk + (size_t)e * BLK_BYTES) + BLK_BYTES - 1) & ~(uintptr_t)127;
  const int nb = (int)((b1 - b0) >> 7) + 1;
  const int total = nb + (mode >= 2 ? RS_EVENT_WINDOW * 4 / 128 : 0);
  for (int k = sub; k < total; k += G) {
    const uintptr_t a = k < nb ? b0 + ((uintptr_t)k << 7)
                               : (uintptr_t)(S.events + (size_t)e * RS_EVENT_WINDOW) + ((uintptr_t)(k - nb) << 7);
    asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
  }
}

// --------------------------------------------------------------- stage
// Each env a CTA works on owns a SLOT_BYTES slot after the staged tables
// (rs_state.cuh): its 544-byte block moves HBM -> slot with one TMA bulk
// copy completing on the slot's mbarrier, the step runs on shared memory,
// and the block moves back with one bulk copy (bulk_group).
__device__ __forceinline__ uint32_t slot_off(int slot, int glog2) {  // after the shuffle scratch
  const uint32_t o = (uint32_t)WALL_SLOT_OFF + (uint32_t)scratch_bytes((int)blockDim.x, glog2) +
                     blockDim.x * (uint32_t)ENGINE_SLOT + (uint32_t)slot * SLOT_BYTES;
  return o;
}
// this thread's Engine slot (RS_ENGINE_SMEM), after the shuffle scratch
__device__ __forceinline__ uint8_t* engine_slot(int glog2) {
  return g_smem + WALL_SLOT_OFF + scratch_bytes((int)blockDim.x, glog2) + threadIdx.x * ENGINE_SLOT;
}
#if defined(RS_ENGINE_SMEM)
#define RS_ENGINE(name, glog2, ...) Engine& name = *new (engine_slot(glog2)) Engine(__VA_ARGS__)
#else
#define RS_ENGINE(name, glog2, ...) Engine name(__VA_ARGS__)
#endif
__device__ __forceinline__ uint32_t smem_addr(uint32_t off) {
  return (uint32_t)__cvta_generic_to_shared(g_smem) + off;
}
// once per kernel and slot; the caller tracks the phase parity
__device__ __forceinline__ void slot_bar_init(uint32_t sb) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(sb + SLOT_BAR)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one thread of the env's lane group issues the copy ...
__device__ __forceinline__ void stage_issue(const Soa& S, int e, uint32_t sb) {
  RS_CHECK((unsigned)e < (unsigned)S.n && sb % 16u == 0 && sb + SLOT_BYTES <= rs::dyn_smem_bytes());
  const uint32_t dst = smem_addr(sb), bar = smem_addr(sb + SLOT_BAR);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(BLK_BYTES) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(S.blk + (size_t)e * BLK_BYTES), "r"(BLK_BYTES), "r"(bar)
               : "memory");
}
// ... and every lane of the group waits for the phase
__device__ __forceinline__ void stage_wait(uint32_t sb, uint32_t phase) {
  const uint32_t bar = smem_addr(sb + SLOT_BAR);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void stage_out(const Soa& S, int e, uint32_t sb) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> bulk copy
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(S.blk + (size_t)e * BLK_BYTES),
               "r"(smem_addr(sb)), "r"(BLK_BYTES)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// the slot's previous stage_out has read shared memory (slot reusable)
__device__ __forceinline__ void stage_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// every stage_out of this thread has completed
__device__ __forceinline__ void stage_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ uint32_t globaltimer_lo() {
  uint32_t t;
  asm volatile("mov.u32 %0, %%globaltimer_lo;" : "=r"(t));
  return t;
}

__device__ __forceinline__ void write_step_out(const StepOut& o, int64_t e, const Engine& E, const Mask115& m,
                                               const float* r, int status) {
  if (o.legal_bits) {
    reinterpret_cast<uint4*>(o.legal_bits)[e] = make_uint4(m.m[0], m.m[1], m.m[2], m.m[3]);
  }
  if (o.current_player) o.current_player[e] = (int8_t)E.g.current_player;
  if (o.rewards) reinterpret_cast<float4*>(o.rewards)[e] = make_float4(r[0], r[1], r[2], r[3]);
  if (o.terminated) o.terminated[e] = (uint8_t)E.g.env_terminated;
  if (o.truncated) o.truncated[e] = (uint8_t)E.g.env_truncated;
  if (o.status) o.status[e] = (uint8_t)status;
}

// the kind of an env's next step, for grouping envs with the same branch
// structure into the same warps (large batches).  RS_KIND_BITS 2: 0
// auto-reset, 1 call phase, 2 turn with a drawn tile, 3 other turn (after
// a call).  RS_KIND_BITS 3 also splits the call phase by the head of the
// queue (ron: a win evaluation) and the drawn turns by the actor's hand --
// in riichi (tsumogiri or a kan only), tenpai or complete and closed (the
// riichi discard filter, the tsumo check), open, other.
#ifndef RS_KIND_BITS
#define RS_KIND_BITS 2
#endif
__device__ __forceinline__ uint8_t next_kind(const Engine& E) {
  if (E.g.env_terminated || E.g.env_truncated) return 0;
#if RS_KIND_BITS == 2
  if (E.g.phase == PH_CALL) return 1;
  return E.g.drawn >= 0 ? 2 : 3;
#else
  if (E.g.phase == PH_CALL) return E.g.qstage(0) == ST_RON ? 1 : 2;
  if (E.g.drawn < 0) return 7;
  const uint32_t inf = E.info(E.g.actor);
  if (hi::riichi(inf)) return 3;
  if (hi::nmelds(inf)) return 6;
  return hi::shanten(inf) <= 0 ? 4 : 5;
#endif
}

__global__ void k_iota(int32_t* a, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

__global__ void __launch_bounds__(BLOCK) k_init(const __grid_constant__ Soa S, const __grid_constant__ DevTables D,
    const __grid_constant__ Cfg C, const uint64_t* seeds, uint64_t seed,
                                                int64_t base, int indexed, StepOut out) {
  const Tabs T = stage_tables(D);
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= S.n) return;
  Engine E(S, T, C, e, S.blk + (size_t)e * BLK_BYTES);
  uint64_t game_seed;
  if (indexed) {
    // bench/runner.py:25-33
    E.g.env_key = derive_key(mix64(seed), (uint64_t)(base + e));
    E.g.policy_key = derive_key(E.g.env_key, 1);
    game_seed = derive_key(E.g.env_key, 2);
  } else {
    game_seed = seeds[e];
    E.g.env_key = game_seed;
    E.g.policy_key = derive_key(game_seed, 1);
  }
  E.g.policy_counter = 0;
  E.g.resets = 0;
  float r[4];
  E.init_game(game_seed, r);
  E.store();
  write_step_out(out, e, E, E.load_legal(), r, 0);
}

// step (+ optional auto-reset, observation and next random action) in one
// pass over the env's state.  With RS_STEP_AUTORESET the rewards / flags
// describe the transition while the legal mask, current player and
// observation already belong to the next game (Pgx auto_reset convention).
// Env <-> thread mapping: `epw` envs per warp, each env run by a group of
// 2^glog2 lanes (rs_common.cuh lane groups).  At small batches a few envs
// per warp spread the batch over many more warps (the step is a long
// dependent chain; the SMs' issue slots are idle), fewer envs per warp also
// means fewer divergent paths per warp, and the idle lanes join their env.

// Completion signal of a step launch in mapped host memory
// (rs_set_done_flag): a host thread waiting for the step's results polls
// one word instead of sleeping in a stream synchronize.  Every working
// warp publishes its stores system-wide and counts itself in; the last one
// bumps the sequence number the host watches and re-arms the counter for
// the next launch (launches on one stream are ordered).
struct Done {
  uint32_t* ctr;                 // device: [0] warps done this launch, [1] sequence
  volatile uint32_t* host_flag;  // mapped pinned host word: the last sequence completed
  uint32_t warps;                // working warps of the launch
};
__device__ __noinline__ void signal_done(const Done& d, uint32_t working, int lane) {
  __threadfence_system();  // this lane's record / observation stores, before the count
  __syncwarp(working);
  if (lane == (int)(__ffs(working) - 1)) {
    if (atomicAdd(d.ctr, 1u) == d.warps - 1) {
      __threadfence();  // every other warp's count (and so its fenced stores) happened before
      const uint32_t seq = d.ctr[1] + 1u;
      d.ctr[1] = seq;
      d.ctr[0] = 0u;
      __threadfence_system();
      *d.host_flag = seq;
    }
  }
}

// rs_signal_done: the completion word after the work queued before it on
// the stream (e.g. a copy of the observations to the host)
__global__ void k_signal(Done done) { signal_done(done, 0xFFFFFFFFu, (int)(threadIdx.x & 31)); }

// Instruction warm-up for the win path (DESIGN §4 item 55): at small
// batches a K=1 launch runs the scoring code (win input, the reading search,
// settlement, the result record) on at most a few envs, after the L2 flush
// that precedes every launch, so its instructions come from HBM one line at
// a time (~40 K cycles for a win).  One extra CTA runs the two largest
// single-copy (out-of-line) pieces at the start of the launch on a constant
// closed riichi tsumo, one piece per warp so they are fetched in parallel
// and ahead of any env (its scratch block in its own shared memory, nothing
// written outside the CTA); by the time an env reaches a win or a yaku
// check those lines are in L2.
__device__ __noinline__ void warm_win_path(int piece, const Soa& S, const Tabs& T, const Cfg& C, uint8_t* scratch,
                                           volatile int* sink) {
  // 234m 567m 345p 678s 55z (+ the drawn 3m)
  constexpr uint8_t tiles[14] = {4, 8, 12, 16, 20, 24, 48, 52, 56, 96, 100, 104, 128, 129};
  if (piece == 0) {  // the reading search (the largest piece)
    WinIn w;
    for (int j = 0; j < 5; j++) w.conc.c[j] = 0;
    for (int i = 0; i < 14; i++) w.conc.add(tiles[i] >> 2, 1);
    w.nmelds = 0;
    for (int m = 0; m < 4; m++) w.mtype[m] = w.mbase[m] = 0;
    w.win_kind = 3;
    w.tsumo = true;
    w.seat_wind = 27;
    w.round_wind = 27;
    w.riichi = 1;
    w.ippatsu = w.last_tile = w.rinshan = w.chankan = w.first_draw = false;
    w.closed = true;
    w.dora = w.ura = w.reds = 0;
    w.double_yakuman = w.kazoe = false;
    Reading rd;
    score_win(w, rd, false);
    *sink = rd.han + rd.fu;
  } else if (piece == 1) {  // the win input of an engine over a zeroed block
    for (int i = 0; i < (int)BLK_BYTES / 4; i++) reinterpret_cast<uint32_t*>(scratch)[i] = 0u;
    Engine E(S, T, C, 0, scratch);
    E.g = Game{};
    E.g.dora_count = 1;
    Hand h;
    h.w0 = h.w1 = h.w2 = h.w3 = h.w4 = 0;
    h.cm = h.cp = h.cs = h.cz = 0;
    for (int i = 0; i < 14; i++) deal_tile(h, tiles[i]);
    h.info = hi::set_riichi(hi::set_nconc(hi::set_riichi_index(0u, -1), 14), 1);
    WinIn w;
    E.win_input(0, h, 12, true, false, w);
    *sink = w.dora + w.win_kind;
  }
}

// the warm-up CTA's body: warp w runs piece w (piece 1's scratch block in
// the CTA's dynamic shared memory when it fits)
__device__ __forceinline__ void warm_cta(const Soa& S, const Tabs& T, const Cfg& C) {
  __shared__ int s_sink;
  const int wp = threadIdx.x >> 5;
#if defined(__CUDA_ARCH__)
  if (wp == 2 && grp_size() >= 4) {
    // the reset's deal (deal_group, the lane-group path): every lane of the
    // warp, one scratch block + identity wall per lane group, after the
    // tables; it runs ~7 us into a reset, so the warm copy gets ahead
    const int G = grp_size(), grp = (threadIdx.x & 31) / G, sub = grp_sub();
    const uint32_t base = (uint32_t)WALL_SLOT_OFF + (uint32_t)grp * 1024u;
    if (base + 1024u <= dyn_smem_bytes()) {
      uint8_t* bp = g_smem + base;
      uint8_t* w = bp + 768;
      for (int i = sub; i < (int)BLK_BYTES / 4; i += G) reinterpret_cast<uint32_t*>(bp)[i] = 0u;
      for (int i = sub; i < 36; i += G) reinterpret_cast<uint32_t*>(w)[i] = 0x03020100u + 0x04040404u * (uint32_t)i;
      __syncwarp(grp_mask());
      Engine E(S, T, C, 0, bp);
      E.g = Game{};
      E.deal_group(w, 0);
      if (sub == 0) s_sink = (int)reinterpret_cast<const uint32_t*>(bp)[W_HINFO];
    }
    return;
  }
#endif
  // piece 1's scratch block after the staged tables (-DRS_TABLES_SMEM: their
  // bulk copy lands first; WALL_SLOT_OFF is 0 otherwise)
  const uint32_t need = wp == 1 ? (uint32_t)WALL_SLOT_OFF + BLK_BYTES : 0u;
  if ((threadIdx.x & 31) == 0 && wp < 2 && need <= dyn_smem_bytes())
    warm_win_path(wp, S, T, C, g_smem + WALL_SLOT_OFF, &s_sink);
}

__global__ void __launch_bounds__(ROLL_BLOCK, ROLL_MINB) k_step(const __grid_constant__ Soa S, const __grid_constant__ DevTables D,
    const __grid_constant__ Cfg C, const int32_t* actions, int flags, rs_obs_out obs, int32_t* next_actions,
    StepOut out, int epw, int staged, int glog2, int check, rs_step_rec* recs, const int32_t* order,
    uint8_t* kind_out, int prefetch, Done done, int warm) {
  tables_begin(D, glog2);  // the action and header loads overlap the table copy
  const Tabs T{};
  if (warm && blockIdx.x == gridDim.x - 1) {  // the warm-up CTA (no envs)
    tables_wait();
    warm_cta(S, T, C);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int q = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * epw + (lane >> glog2);
  const bool idle = (lane >> glog2) >= epw || q >= S.n;
  const uint32_t working = done.host_flag ? __ballot_sync(0xFFFFFFFFu, !idle) : 0u;
  if (idle) {
    tables_wait();  // (cluster launches: peers may still be writing this CTA's tables)
    return;
  }
  const int e = order ? order[q] : q;  // envs grouped by the kind of their step (large batches)
  // one stage slot per env, shared by the env's lane group
  const uint32_t sb = slot_off((threadIdx.x >> 5) * epw + (lane >> glog2), glog2);
  const int sub = lane & ((1 << glog2) - 1);
  const uint32_t gm = glog2 >= 5 ? 0xFFFFFFFFu : (((1u << (1 << glog2)) - 1u) << (lane - sub));
  if (staged) {
    if (sub == 0) {
      slot_bar_init(sb);
      stage_issue(S, e, sb);
    }
    __syncwarp(gm);  // the slot's barrier is initialised for the whole group
    stage_wait(sb, 0);
  }
  if ((prefetch & 3) && !staged) prefetch_env(S, e, sub, 1 << glog2, prefetch & 3);
  const int action = actions[e];  // may live in mapped host memory (HostStepper)
  RS_ENGINE(E, glog2, S, T, C, e, staged ? g_smem + sb : S.blk + (size_t)e * BLK_BYTES);
  E.load();
  tables_wait();
  Mask115 m;
  float r[4];
  // RS_ACTION_SKIP: the env is not stepped (actors that have not decided
  // yet); its outputs describe its current state with zero rewards
  const bool skip = action == RS_ACTION_SKIP;
  int st = 0;
  int act = action;
  if (!skip && (flags & RS_STEP_RESET_FIRST) && (E.g.env_terminated || E.g.env_truncated)) {
    // runner.py:107-113: the finished env's next game, then its own policy
    // draw and the step (the host action is ignored)
    E.g.resets++;
    E.init_game(derive_key(E.g.env_key, 2 + (uint64_t)E.g.resets), r);
    const Mask115 lm = E.load_legal();
    act = (flags & RS_STEP_HEURISTIC) ? E.heuristic_action(lm) : E.random_action(lm);
  }
  if (skip) {
    if (E.g.env_terminated || E.g.env_truncated) m.clear();
    else m = E.load_legal();
    r[0] = r[1] = r[2] = r[3] = 0.f;
  } else {
    st = E.step(act, m, r);  // one inlined copy of the transition (cold code, §4 item 49)
  }
  const int term = E.g.env_terminated, trunc = E.g.env_truncated;
  bool dirty = !skip && st != RS_STATUS_CONTRACT;
  if (!skip && (flags & RS_STEP_AUTORESET) && (term || trunc)) {
    float r2[4];
    E.g.resets++;
    E.init_game(derive_key(E.g.env_key, 2 + (uint64_t)E.g.resets), r2);
    m = E.load_legal();
    dirty = true;
  }
  if (flags & RS_STEP_OBSERVE) write_obs(E, E.g.current_player, obs, e);
  int next = -1;
  if (next_actions || recs) {
    const bool done = E.g.env_terminated || E.g.env_truncated;
    next = skip ? RS_ACTION_SKIP
                : done ? -1 : (flags & RS_STEP_HEURISTIC) ? E.heuristic_action(m) : E.random_action(m);
    if (next_actions) next_actions[e] = next;
    dirty |= !done && !skip;
  }
  int st_out = st;
  if (check && check_invariants(E, true)) st_out |= (int)RS_STATUS_INVARIANT;  // debug: every step
  if (dirty) {
    E.store();
    if (staged) {
      __syncwarp(gm);  // every lane's writes to the slot precede the bulk store
      if (sub == 0) stage_out(S, e, sb);
    }
  }
  if (kind_out && (lane & ((1 << glog2) - 1)) == 0) kind_out[e] = next_kind(E);
  if (out.legal_bits) reinterpret_cast<uint4*>(out.legal_bits)[e] = make_uint4(m.m[0], m.m[1], m.m[2], m.m[3]);
  if (out.current_player) out.current_player[e] = (int8_t)E.g.current_player;
  if (out.rewards) reinterpret_cast<float4*>(out.rewards)[e] = make_float4(r[0], r[1], r[2], r[3]);
  if (out.terminated) out.terminated[e] = (uint8_t)term;
  if (out.truncated) out.truncated[e] = (uint8_t)trunc;
  if (out.status) out.status[e] = (uint8_t)st_out;
  if (recs) {
    // the record's 10 words from the lanes of the env's group (one store
    // instruction per 10 lanes: the env's 40 bytes leave as one burst)
    auto word = [&](int i) -> uint32_t {
      union { float f; uint32_t u; } cv;
      if (i < 4) { cv.f = r[i]; return cv.u; }
      if (i < 8) return m.m[i - 4];
      if (i == 8) return (uint32_t)next;
      return (uint32_t)(uint8_t)E.g.current_player | ((uint32_t)(uint8_t)term << 8) | ((uint32_t)(uint8_t)trunc << 16) |
             ((uint32_t)(uint8_t)st_out << 24);
    };
    uint32_t* dst = reinterpret_cast<uint32_t*>(recs + e);
    for (int i = lane & ((1 << glog2) - 1); i < 10; i += 1 << glog2) dst[i] = word(i);
  }
  if (staged && dirty && sub == 0) stage_wait_all();
  if (done.host_flag) signal_done(done, working, lane);
}

__global__ void __launch_bounds__(BLOCK) k_policy(const __grid_constant__ Soa S, const __grid_constant__ DevTables D,
    const __grid_constant__ Cfg C, int32_t* actions, int policy) {
  const Tabs T = stage_tables(D);
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= S.n) return;
  Engine E(S, T, C, e, S.blk + (size_t)e * BLK_BYTES);
  E.load();
  if (E.g.env_terminated || E.g.env_truncated) { actions[e] = -1; return; }
  if (policy == RS_POLICY_HEURISTIC) {
    actions[e] = E.heuristic_action(E.load_legal());
    return;
  }
  actions[e] = E.random_action(E.load_legal());
  E.store();
}

__global__ void __launch_bounds__(BLOCK) k_observe(const __grid_constant__ Soa S, const __grid_constant__ DevTables D,
    const __grid_constant__ Cfg C, const int8_t* seats, rs_obs_out obs) {
  const Tabs T = stage_tables(D);
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= S.n) return;
  Engine E(S, T, C, e, S.blk + (size_t)e * BLK_BYTES);
  E.load();
  write_obs(E, seats ? (int)seats[e] : E.g.current_player, obs, e);
}

// the wide trajectory digest of one step (tests, rs_rollout digests): the
// summary, every state field, then the current player's observation as
// write_obs encodes it into the env's scratch record (the lane group's
// lanes write quarters of the window, so the group syncs around it)
__device__ __noinline__ uint64_t digest_wide(uint64_t d, int a, const Engine& E, const Mask115& m, const float* r,
                                             const rs_obs_out& dobs, uint32_t gm) {
  __syncwarp(gm);  // the ring entries other lanes of the group wrote
  d = digest_state(digest_step(d, a, E, m, r), E);
  write_obs(E, E.g.current_player, dobs, E.e);
  __syncwarp(gm);
  d = digest_obs(d, dobs, E.e);
  __syncwarp(gm);
  return d;
}

// the fused rollout: the packed header stays in registers for all K steps.
// Persistent grid (at most the resident CTA count): each CTA stages the
// tables once and walks env tiles grid-stride.
// WIDE: the test / debug instantiation -- the wide digest (digest_wide)
// when `digests` is given, the invariant checker after every step with
// RINSHAN_CHECK; the production instantiation has none of that code
// (-2.5 % launch time at 4,096 envs when it shared the digest)
template <bool WIDE>
__global__ void __launch_bounds__(ROLL_BLOCK, ROLL_MINB) k_rollout(const __grid_constant__ Soa S, const __grid_constant__ DevTables D,
    const __grid_constant__ Cfg C, int steps, rs_obs_out obs,
                                                   int obs_slots, int16_t* actions_log, int8_t* actors_log,
                                                   StepOut traj, rs_rollout_stats* stats,
                                                   uint64_t* digests, rs_obs_out dobs, StepOut out, int epw,
                                                   uint32_t* prof, int staged, int policy, int glog2,
                                                   int check, const int32_t* order, uint8_t* kind_out,
                                                   int prefetch, int warm) {
  const uint32_t g_entry = prof ? globaltimer_lo() : 0u;
  tables_begin(D, glog2);  // the first env tile's header loads overlap the copy
  const Tabs T{};
  if (warm && blockIdx.x == gridDim.x - 1) {  // the warm-up CTA (no envs)
    tables_wait();
    warm_cta(S, T, C);
    return;
  }
  bool tables_ready = false;
  uint32_t g_staged = 0u;
  unsigned long long games = 0;
  const int lane = threadIdx.x & 31;
  const int warps = ((gridDim.x - (warm ? 1 : 0)) * blockDim.x) >> 5;
  const int sub = lane & ((1 << glog2) - 1);  // the lane's index in its env's group
  const uint32_t gm = glog2 >= 5 ? 0xFFFFFFFFu : (((1u << (1 << glog2)) - 1u) << (lane - sub));
  // one stage slot per env, shared by the env's lane group
  const uint32_t sb = slot_off((threadIdx.x >> 5) * epw + (lane >> glog2), glog2);
  if (staged && (lane >> glog2) < epw && sub == 0) slot_bar_init(sb);
  uint32_t phase = 0;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w * epw < S.n; w += warps) {
    const int q = w * epw + (lane >> glog2);
    if ((lane >> glog2) >= epw || q >= S.n) continue;
    const int e = order ? order[q] : q;  // envs grouped by the kind of their step (large batches)
    if (staged) {
      if (sub == 0) {
        stage_wait_read();  // the slot's previous block has left
        stage_issue(S, e, sb);
      }
      __syncwarp(gm);  // (first tile: the slot's barrier is initialised)
      stage_wait(sb, phase);
      phase ^= 1u;
    }
    if ((prefetch & 3) && !staged) prefetch_env(S, e, sub, 1 << glog2, prefetch & 3);
    RS_ENGINE(E, glog2, S, T, C, e, staged ? g_smem + sb : S.blk + (size_t)e * BLK_BYTES);
    E.load();
    uint64_t d = digests ? digests[e] : 0ull;
    if (!tables_ready) {
      tables_wait();
      tables_ready = true;
      if (prof) g_staged = globaltimer_lo();
    }
    float r[4] = {0.f, 0.f, 0.f, 0.f};
    Mask115 m;
    int st = 0;
    bool inv = false;
    const uint32_t g_first = prof ? globaltimer_lo() : 0u;
    for (int t = 0; t < steps; t++) {
      const long long t0 = prof ? clock64() : 0;
      const bool reset = E.g.env_terminated || E.g.env_truncated;
      if (reset) {  // runner.py:107-109
        E.g.resets++;
        E.init_game(derive_key(E.g.env_key, 2 + (uint64_t)E.g.resets), r);
      }
      const long long t1 = prof ? clock64() : 0;
      RS_SMARK(0);
      const int a = policy == RS_POLICY_HEURISTIC ? E.heuristic_action(E.load_legal()) : E.random_action(E.load_legal());
      const int actor = E.g.current_player;
      st = E.step(a, m, r);
      if (WIDE && check && check_invariants(E, true)) inv = true;  // debug: every step
      if (actions_log) actions_log[(size_t)t * S.n + e] = (int16_t)a;
      if (actors_log) actors_log[(size_t)t * S.n + e] = (int8_t)(actor | (reset ? 4 : 0));
      // per-step outputs into [steps][n] trajectory buffers (rs_rollout_policy traj)
      if (traj.legal_bits || traj.rewards || traj.current_player || traj.terminated || traj.status)
        write_step_out(traj, (int64_t)t * S.n + e, E, m, r, st);
      if ((E.g.env_terminated || E.g.env_truncated) && sub == 0) games++;
      if (WIDE && digests) d = digest_wide(d, a, E, m, r, dobs, gm);
      if (obs_slots > 0 && (obs_slots > 1 || t == steps - 1)) {
        const int slot = obs_slots > 1 ? t % obs_slots : 0;
        write_obs(E, E.g.current_player, obs, (int64_t)slot * S.n + e);
      }
      RS_SMARK(6);
      if (prof) {  // debug hook (rs_debug_rollout_cycles): reset / step+observe cycles, action
        const long long t2 = clock64();
        uint32_t* p = prof + ((size_t)t * S.n + e) * 4;
        p[0] = (uint32_t)(t1 - t0);
        p[1] = (uint32_t)(t2 - t1);
        p[2] = (uint32_t)a | ((uint32_t)reset << 8);
        p[3] = (uint32_t)E.g.phase | ((uint32_t)E.g.env_terminated << 4);
      }
    }
    E.store();
    if (staged) {
      __syncwarp(gm);  // every lane's writes to the slot precede the bulk store
      if (sub == 0) stage_out(S, e, sb);
    }
    if (kind_out && sub == 0) kind_out[e] = next_kind(E);
    if (digests) digests[e] = d;
    write_step_out(out, e, E, m, r, st | (inv ? (int)RS_STATUS_INVARIANT : 0));
    RS_SMARK(7);
    if (prof) {
      uint32_t* p = prof + ((size_t)steps * S.n + e) * 4;
      p[0] = g_entry; p[1] = g_staged; p[2] = g_first; p[3] = globaltimer_lo();
    }
  }
  if (staged && sub == 0) stage_wait_all();
  if (!tables_ready) tables_wait();  // a CTA without envs (cluster padding) still receives the tables
  if (stats) {
    unsigned long long g = games;
    for (int off = 16; off > 0; off >>= 1) g += __shfl_down_sync(0xffffffffu, g, off);
    if ((threadIdx.x & 31) == 0 && g) atomicAdd(reinterpret_cast<unsigned long long*>(&stats->games_completed), g);
    if (blockIdx.x == 0 && threadIdx.x == 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(&stats->steps), (unsigned long long)S.n * steps);
  }
}

// bench/runner.py:107-109: a finished env starts its next game from
// env_game_seed(seed, index, resets + 1); unfinished envs are untouched
__global__ void __launch_bounds__(BLOCK) k_autoreset(const __grid_constant__ Soa S,
    const __grid_constant__ DevTables D, const __grid_constant__ Cfg C, StepOut out) {
  stage_tables(D);
  const Tabs T{};
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= S.n) return;
  Engine E(S, T, C, e, S.blk + (size_t)e * BLK_BYTES);
  E.load();
  float r[4];
  int st = 0;
  if (E.g.env_terminated || E.g.env_truncated) {
    E.g.resets++;
    E.init_game(derive_key(E.g.env_key, 2 + (uint64_t)E.g.resets), r);
    E.store();
  } else {
    E.current_rewards(r);
  }
  write_step_out(out, e, E, E.load_legal(), r, st);
}

__global__ void __launch_bounds__(BLOCK) k_check(const __grid_constant__ Soa S, const __grid_constant__ DevTables D,
    const __grid_constant__ Cfg C, int fast, uint32_t* flags) {
  const Tabs T = stage_tables(D);
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= S.n) return;
  Engine E(S, T, C, e, S.blk + (size_t)e * BLK_BYTES);
  E.load();
#if defined(RS_BOUNDS)
  if (fast == 2) (void)E.wall(RS_NUM_TILES);  // bounds-build canary: must trap (tools/bounds_check.sh)
#endif
  const uint32_t bad = check_invariants(E, fast != 0);
  if (bad) flags[e] |= bad;
}

__global__ void k_expand(const uint32_t* bits, uint8_t* bools, int n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * RS_NUM_ACTIONS) return;
  const int64_t e = i / RS_NUM_ACTIONS;
  const int a = (int)(i - e * RS_NUM_ACTIONS);
  bools[i] = (uint8_t)((bits[e * 4 + (a >> 5)] >> (a & 31)) & 1u);
}

// the projection records of envs[0..count) (export_env reads no tables):
// one thread per listed env, so many envs cost one launch and one copy
__global__ void k_export_many(const __grid_constant__ Soa S, const __grid_constant__ Cfg C, const int64_t* envs,
                              int64_t count, rs_env_rec* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int e = (int)envs[i];
  Engine E(S, Tabs{}, C, e, S.blk + (size_t)e * BLK_BYTES);
  export_env(E, C, out[i]);
}

__global__ void k_import(const __grid_constant__ Soa S, const __grid_constant__ DevTables D,
    const __grid_constant__ Cfg C, int e, const rs_env_rec* in) {
  const Tabs T = stage_tables(D);
  if (threadIdx.x != 0) return;
  Engine E(S, T, C, e, S.blk + (size_t)e * BLK_BYTES);
  E.load();
  import_env(E, *in);
}

// score_win over WinContext records (rs_debug_score): the WinIn the
// engine's win_input builds from a state, built here from the context
// (scoring/context.py:19-57, dora parts as scoring/dora.py:9-22 counts them
// over all_tile_ids), then the engine's scorer and result-record writer
__global__ void k_debug_score(const rs_winctx* ctx, int64_t count, rs_win_rec* out, int32_t* ok) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const rs_winctx& c = ctx[i];
  WinIn w;
  for (int j = 0; j < 5; j++) w.conc.c[j] = 0;
  for (int k = 0; k < 34; k++) w.conc.add(k, c.concealed[k]);
  w.nmelds = c.n_melds;
  w.closed = true;
  for (int m = 0; m < 4; m++) {
    w.mtype[m] = m < c.n_melds ? c.melds[m].type : 0;
    w.mbase[m] = m < c.n_melds ? c.melds[m].tiles[0] >> 2 : 0;
    if (m < c.n_melds && c.melds[m].type != M_KAN_CLOSED) w.closed = false;
  }
  w.win_kind = c.win_tile >> 2;
  w.tsumo = c.tsumo != 0;
  w.seat_wind = c.seat_wind;
  w.round_wind = c.round_wind;
  w.riichi = c.riichi;
  w.ippatsu = c.ippatsu != 0;
  w.last_tile = c.last_tile != 0;
  w.rinshan = c.rinshan != 0;
  w.chankan = c.chankan != 0;
  w.first_draw = c.first_draw != 0;
  Counts all;
  for (int j = 0; j < 5; j++) all.c[j] = 0;
  int reds = 0;
  for (int j = 0; j < c.n_ids; j++) {
    all.add(c.ids[j] >> 2, 1);
    if (c.rule == RS_RULE_RED && is_red_tile(c.ids[j])) reds++;
  }
  int dora = 0, ura = 0;
  for (int j = 0; j < c.n_dora; j++) dora += all.get(dora_kind(c.dora[j] >> 2));
  if (c.riichi)
    for (int j = 0; j < c.n_ura; j++) ura += all.get(dora_kind(c.ura[j] >> 2));
  w.dora = dora;
  w.ura = ura;
  w.reds = reds;
  w.kazoe = c.kazoe != 0;
  w.double_yakuman = c.double_yakuman != 0;
  Reading r;
  rs_win_rec rec;
  memset(&rec, 0, sizeof(rec));
  const bool scored = score_win(w, r, false);
  if (scored) fill_win_rec(rec, r, w);
  out[i] = rec;
  ok[i] = scored ? 1 : 0;
}

}  // namespace

struct rs_handle {
  int device;
  int n;
  Cfg cfg;
  Soa S;
  DevTables D;
  void* mem;
  size_t mem_bytes;
  uint32_t* legal_bits_tmp;  // step output when the caller asks only for bools
  rs_env_rec* rec_dev;
  void* export_buf = nullptr;  // rs_export_envs: records + env list, grown on demand
  std::mutex export_mu;        // export_buf / rec_dev: export and import calls from several threads
  size_t export_cap = 0;
  int num_sms;
  int occ_key[16], occ_val[16];  // resident stepping-kernel CTAs per SM per (block, smem)
  // stepping kernels on a shared-memory stage (RINSHAN_STAGE): 0 = never
  // (default), 1 = below 32 envs per warp, 2 = always.  Measured on B200 the
  // stage cuts the mean per-env step latency by ~35% at 4096 envs but not
  // the launch time (set by the rare long transitions), and halves the
  // resident warps at large batches (4096 envs: 83 M steps/s unstaged vs
  // 78 M staged; 1M envs: 880 M vs 501 M)
  int stage_mode;
  int groups;  // idle lanes of small-batch warps join their env (RINSHAN_GROUPS=0: off)
  int check_steps;  // RINSHAN_CHECK=1: fast invariants after every step -> RS_STATUS_INVARIANT
  int block_override;  // RINSHAN_BLOCK (tuning experiments): stepping-kernel CTA size
  // env ordering (large batches): each stepping launch records the kind of
  // every env's next step; the next launch first sorts the envs by kind
  // (CUB radix sort, 2 key bits) so a warp's envs share a branch structure
  int ordering;            // RINSHAN_ORDER: 0 off, 1 at >= 131072 envs (default), 2 always
  uint8_t* kind;           // [n] next-step kind per env (k_rollout / k_step write it)
  uint8_t* kind_sorted;    // [n] sort scratch
  int32_t* iota;           // [n] 0..n-1
  int32_t* order;          // [n] env processed by slot q
  void* sort_tmp;
  size_t sort_tmp_bytes;
  int epw_override;         // RINSHAN_EPW (tuning experiments), 0 = heuristic
  bool persist;             // launch with the tables' L2 persisting window
  cudaAccessPolicyWindow window;
  // stepping kernels as thread-block clusters of this many CTAs, the table
  // block multicast over the cluster (tables_begin); RINSHAN_CLUSTER
  int cluster;
  int occ_cl_key[8], occ_cl_val[8];  // co-resident clusters per (block, smem)
  int prefetch;  // RINSHAN_PREFETCH: L1 prefetch of an env's lines before its step (prefetch_env)
  int warm;      // RINSHAN_WARM (default 1): the win-path warm-up CTA at small batches (warm_win_path)
  // rs_set_done_flag: the step launches' completion word in mapped host
  // memory and its device-side counter / sequence
  uint32_t* done_flag = nullptr;
  uint32_t* done_ctr = nullptr;
  // per-env observation scratch of the wide trajectory digest (digest_obs),
  // allocated by the first rollout that asks for digests
  void* dig_obs_mem = nullptr;
  rs_obs_out dig_obs{};
};

namespace {

Cfg to_cfg(const rs_config* c) {
  return Cfg{c->rule, c->mode, c->reward_scheme, c->illegal_penalty, c->max_steps,
             c->kazoe, c->double_yakuman, c->agari_yame, c->renchan_cap};
}
int grid_of(int n) { return (n + BLOCK - 1) / BLOCK; }

// grid of `block`-thread CTAs covering n envs at `epw` envs per warp, capped
// at `max_ctas` (the grid-stride kernels then loop)
int warp_grid(const rs_handle* h, int epw, int block, int max_ctas) {
  const int64_t warps = (h->n + epw - 1) / epw;
  const int64_t ctas = (warps * 32 + block - 1) / block;
  return (int)std::min<int64_t>(ctas, max_ctas > 0 ? max_ctas : ctas);
}

// Launch shape of the stepping kernels (k_step, k_rollout) at `epw` envs per
// warp: 128-thread CTAs while the batch fills under ROLL_BLOCK threads per SM
// (spread over every SM), else ROLL_BLOCK-thread CTAs; one stage slot per
// env of the CTA.  `ctas` = resident CTAs per SM (occupancy, cached).
struct Launch {
  int grid, block, smem, epw, ctas, staged, glog2, ordered, cluster;
};
int resident_ctas(rs_handle* h, int block, int smem) {
  const int key = block * 1048576 + smem;
  for (int i = 0; i < 16; i++)
    if (h->occ_key[i] == key) return h->occ_val[i];
  int ctas = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, k_rollout<false>, block, smem) != cudaSuccess) {
    cudaGetLastError();
    ctas = 1;
  }
  ctas = std::max(ctas, 1);
  for (int i = 0; i < 16; i++)
    if (h->occ_key[i] == 0) {
      h->occ_key[i] = key;
      h->occ_val[i] = ctas;
      break;
    }
  return ctas;
}
Launch launch_at(rs_handle* h, int epw) {
  Launch L;
  L.epw = epw;
  const int64_t warps = (h->n + epw - 1) / epw;
  L.block = warps * 32 >= (int64_t)h->num_sms * ROLL_BLOCK ? ROLL_BLOCK : BLOCK;
  // large batches (the batch-sized grid, item 57): 128-thread CTAs give the
  // block scheduler finer units (131 K +1.7 %, 262 K +4.2 %, 1 M +2.0 %)
  if (h->n >= (1 << 17)) L.block = BLOCK;
  if (h->block_override > 0) L.block = h->block_override;
  L.staged = h->stage_mode == 2 || (h->stage_mode == 1 && epw < 32);
  // idle lanes join their env as a lane group (not with the stage: one slot per lane)
  L.glog2 = 0;
  if (h->groups)
    while ((epw << (L.glog2 + 1)) <= 32) L.glog2++;
  // measured on B200, round-2 final build with the batch-sized grid, K=1
  // launches at the plateau (launches 800-1200 from fresh games,
  // tools/drift_probe.py; unsorted envs drift apart for ~800 steps, sorted
  // ones hold): 262 K envs sorted 355 vs 468 us, 131 K 205 vs 250 us, 64 K
  // 138 vs 141 us, 16 K 75 vs 66 us
  L.ordered = h->ordering == 2 || (h->ordering == 1 && h->n >= (1 << 17));
  L.smem = L.staged ? smem_staged(L.block, L.block / 32 * epw, L.glog2) : smem_for(L.block, L.glog2);
  L.ctas = resident_ctas(h, L.block, L.smem);
  L.grid = warp_grid(h, epw, L.block, 0);
  L.cluster = h->cluster;
  L.grid = (L.grid + L.cluster - 1) / L.cluster * L.cluster;
  return L;
}
// the win-path warm-up CTA (warm_win_path): lane-group launches (small
// batches, where a launch holds few wins) without clusters
int warm_of(const rs_handle* h, const Launch& L) { return h->warm && L.cluster <= 1 && L.glog2 > 0 ? 1 : 0; }
// CTAs of the persistent grid: every resident CTA, or with clusters every
// CTA of the clusters that fit at once (cudaOccupancyMaxActiveClusters)
int persistent_ctas(rs_handle* h, const Launch& L) {
  if (L.cluster <= 1) return h->num_sms * L.ctas;
  const int key = L.block * 1048576 + L.smem;
  for (int i = 0; i < 8; i++)
    if (h->occ_cl_key[i] == key) return h->occ_cl_val[i];
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)L.grid);
  cfg.blockDim = dim3((unsigned)L.block);
  cfg.dynamicSmemBytes = (size_t)L.smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)L.cluster;
  at[0].val.clusterDim.y = at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, k_rollout<false>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    clusters = h->num_sms * L.ctas / L.cluster;
  }
  const int ctas = std::max(clusters, 1) * L.cluster;
  for (int i = 0; i < 8; i++)
    if (h->occ_cl_key[i] == 0) {
      h->occ_cl_key[i] = key;
      h->occ_cl_val[i] = ctas;
      break;
    }
  return ctas;
}
// envs per warp: the fewest (power of two) whose warps all fit in one wave
// (7/8 of the resident warps).  A step is a long dependent chain per env and
// the envs of a warp run their divergent paths one after another, so fewer
// envs per warp is faster as long as no second wave is needed (measured on
// B200 before the shared-memory stage: 4096 envs 79 M steps/s at 2 envs per
// warp vs 70 M at 4 and 54 M at 32; 16384 envs 217 M at 8 vs 149 M at 4)
int envs_per_warp(rs_handle* h) {
  if (h->epw_override > 0) return h->epw_override;
  int epw = 1;
  while (epw < 32) {
    const Launch L = launch_at(h, epw);
    const int64_t capacity = (int64_t)h->num_sms * L.ctas * (L.block / 32) * 7 / 8;
    if ((h->n + epw - 1) / epw <= capacity) break;
    epw *= 2;
  }
  return epw;
}
// `persistent` caps the grid at the resident CTAs (k_rollout walks env tiles)
// `persistent`: the rollout's grid-stride loop over the resident CTAs only
// when every CTA stages the tables (-DRS_TABLES_SMEM: one copy per CTA);
// with the tables read through L1 one env group per warp and the hardware
// block scheduler balancing the uneven steps is faster (DESIGN §4 item 57:
// 1 M envs +7-8 %, 262 K +10 %)
Launch step_launch(rs_handle* h, bool persistent) {
  Launch L = launch_at(h, envs_per_warp(h));
#if defined(RS_TABLES_SMEM)
  if (persistent) L.grid = std::min(L.grid, persistent_ctas(h, L));
#else
  (void)persistent;
#endif
  return L;
}

// the envs of the coming launch, sorted by the kind of their next step
int order_envs(rs_handle* h, cudaStream_t st) {
  size_t bytes = h->sort_tmp_bytes;
  CUDA_TRY(cub::DeviceRadixSort::SortPairs(h->sort_tmp, bytes, h->kind, h->kind_sorted, h->iota, h->order, h->n, 0,
                                           RS_KIND_BITS, st));
  return 0;
}

// launch with the table block's L2 access policy window (DeviceTables)
template <typename... KArgs, typename... Args>
cudaError_t launch_tables(const rs_handle* h, void (*kernel)(KArgs...), int grid, int block, int smem,
                          cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (h->persist) {
    at[na].id = cudaLaunchAttributeAccessPolicyWindow;
    at[na++].val.accessPolicyWindow = h->window;
  }
  if (h->cluster > 1) {  // the grid is a multiple of the cluster size (launch_at)
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = (unsigned)h->cluster;
    at[na].val.clusterDim.y = at[na].val.clusterDim.z = 1;
    na++;
  }
  cfg.attrs = na ? at : nullptr;
  cfg.numAttrs = (unsigned)na;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// launches go to the handle's device whatever the caller's current device
// (restored afterwards: the entry points are stream-ordered calls the
// caller may make from a thread working with another device)
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int device) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != device) cudaSetDevice(device);
    else prev = -1;
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

Done done_of(const rs_handle* h, const Launch& L, int flags) {
  if (!h->done_flag || !(flags & RS_STEP_SIGNAL)) return Done{nullptr, nullptr, 0u};
  return Done{h->done_ctr, h->done_flag, (uint32_t)((h->n + L.epw - 1) / L.epw)};
}

// observation slot t of [slots][n] observation buffers (rs_obs_out fields)
rs_obs_out obs_slot(const rs_obs_out& o, size_t t, size_t n) {
  rs_obs_out r{};
  auto at = [&](auto* p, size_t per) { return p ? p + t * n * per : p; };
  r.hand_tokens = at(o.hand_tokens, 14);
  r.event_tokens = at(o.event_tokens, 192);
  r.shanten = at(o.shanten, 1);
  r.scores = at(o.scores, 4);
  r.round_wind = at(o.round_wind, 1);
  r.seat_wind = at(o.seat_wind, 1);
  r.kyoku = at(o.kyoku, 1);
  r.honba = at(o.honba, 1);
  r.deposits = at(o.deposits, 1);
  r.dora_tokens = at(o.dora_tokens, 5);
  r.live_wall = at(o.live_wall, 1);
  r.riichi_flags = at(o.riichi_flags, 4);
  return r;
}

StepOut step_out(rs_handle* h, const rs_step_out* o) {
  StepOut s{};
  if (!o) return s;
  s.legal_bits = o->legal_bits ? o->legal_bits : (o->legal_mask ? h->legal_bits_tmp : nullptr);
  s.current_player = o->current_player;
  s.rewards = o->rewards;
  s.terminated = o->terminated;
  s.truncated = o->truncated;
  s.status = o->status;
  return s;
}
int finish_step_out(rs_handle* h, const rs_step_out* o, cudaStream_t st) {
  if (o && o->legal_mask) {
    const uint32_t* bits = o->legal_bits ? o->legal_bits : h->legal_bits_tmp;
    const int64_t total = (int64_t)h->n * RS_NUM_ACTIONS;
    k_expand<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(bits, o->legal_mask, h->n);
  }
  CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace

// the fields of an imported record must fit the device layout (bit widths
// of the packed header, array slots): the name of the first that does not
namespace {
const char* record_out_of_range(const rs_env_rec& r) {
  auto tile_or_none = [](int t) { return t >= -1 && t < RS_NUM_TILES; };
  for (int i = 0; i < RS_NUM_TILES; i++)
    if (r.wall[i] >= RS_NUM_TILES) return "wall";
  if (r.kan_draws < 0 || r.kan_draws > 4) return "kan_draws";
  if (r.cursor < 0 || r.cursor > 122 - r.kan_draws) return "cursor";
  if (r.dora_count < 1 || r.dora_count > 5) return "dora_count";
  for (int s = 0; s < 4; s++) {
    const rs_hand_rec& hr = r.hands[s];
    if (hr.n_concealed > 14) return "hands.n_concealed";
    for (int i = 0; i < hr.n_concealed; i++)
      if (hr.concealed[i] >= RS_NUM_TILES) return "hands.concealed";
    if (hr.n_melds > 4) return "hands.n_melds";
    for (int i = 0; i < hr.n_melds; i++) {
      const rs_meld_rec& m = hr.melds[i];
      if (m.type < 0 || m.type > 4 || m.n_tiles < 3 || m.n_tiles > 4 || m.from_seat < -1 || m.from_seat > 3 ||
          !tile_or_none(m.called_tile))
        return "hands.melds";
      for (int j = 0; j < m.n_tiles; j++)
        if (m.tiles[j] >= RS_NUM_TILES) return "hands.melds.tiles";
    }
    // a discard appends one entry: keep a free slot
    if (hr.n_river < 0 || hr.n_river >= RS_MAX_RIVER) return "hands.n_river";
    for (int i = 0; i < hr.n_river; i++)
      if (hr.river_tile[i] >= RS_NUM_TILES || hr.river_flags[i] > 7) return "hands.river";
    if (hr.riichi < 0 || hr.riichi > 2 || hr.riichi_index < -1 || hr.riichi_index >= RS_MAX_RIVER) return "hands.riichi";
  }
  if (r.kyoku < 0 || r.kyoku > 7) return "kyoku";
  if (r.honba < 0 || r.honba > 255 || r.deposits < 0 || r.deposits > 255 || r.repeats < 0 || r.repeats > 255)
    return "honba / deposits / repeats";
  if (r.phase < 0 || r.phase > 2 || r.actor < 0 || r.actor > 3 || r.current_player < 0 || r.current_player > 3)
    return "phase / actor";
  if (!tile_or_none(r.drawn) || !tile_or_none(r.call_tile) || r.call_from < -1 || r.call_from > 3 ||
      r.kakan_kind < -1 || r.kakan_kind >= RS_NUM_KINDS)
    return "drawn / call state";
  if (r.n_queue < 0 || r.n_queue > 5) return "n_queue";
  for (int i = 0; i < r.n_queue; i++)
    if (r.queue_seat[i] < 0 || r.queue_seat[i] > 3 || r.queue_stage[i] < 0 || r.queue_stage[i] > 2) return "queue";
  if (r.n_rons < 0 || r.n_rons > 3) return "n_rons";
  for (int i = 0; i < r.n_rons; i++)
    if (r.rons[i] < 0 || r.rons[i] > 3) return "rons";
  if (r.pending_dora < 0 || r.pending_dora > 4) return "pending_dora";
  if (r.n_results < 0 || r.n_results > 255 || r.events_len < 0 || r.step_count < 0) return "counters";
  const int cnt = r.events_len < RS_EVENT_WINDOW ? r.events_len : RS_EVENT_WINDOW;
  for (int i = 0; i < cnt; i++)
    if (r.events[i][0] < 0 || r.events[i][0] > 11 || r.events[i][1] < -1 || r.events[i][1] > 3 ||
        !tile_or_none(r.events[i][2]))
      return "events";
  return nullptr;
}
}  // namespace

extern "C" {

const char* rs_last_error(void) { return g_err.c_str(); }
int rs_abi_version(void) { return RS_ABI_VERSION; }

int rs_tables_build(void) {
  host_tables();
  return 0;
}
int rs_tables_load(const uint8_t* blob, int64_t size) {
  const int rc = host_tables_load(blob, size);
  if (rc == -5) return set_err(RS_E_TABLES, "suit tables already in use (built or loaded); a different blob must be "
                                         "loaded before the first handle or table query");
  return rc ? set_err(rc, "suit-table blob rejected (magic, cardinality or crc)") : 0;
}
int rs_tables_blob(uint8_t* out, int64_t cap, int64_t* size) {
  const int64_t s = host_tables_blob(out, cap);
  if (size) *size = s;
  return 0;
}
int rs_tables_crc(uint32_t* crc) {
  *crc = host_tables().crc;
  return 0;
}
int rs_tables_info(int32_t* ns, int32_t* nh, int32_t* na, int32_t* nb) {
  const HostTables& T = host_tables();
  if (ns) *ns = T.ns;
  if (nh) *nh = T.nh;
  if (na) *na = T.na;
  if (nb) *nb = T.nb;
  return 0;
}
int rs_tables_shanten_std(uint32_t cm, uint32_t cp, uint32_t cs, uint32_t cz, int32_t melds, int32_t* out) {
  const HostTables& H = host_tables();
  if (cm >= (uint32_t)SUIT_CODES || cp >= (uint32_t)SUIT_CODES || cs >= (uint32_t)SUIT_CODES ||
      cz >= (uint32_t)HONOR_CODES || melds < 0 || melds > 4)
    return set_err(RS_E_ARG, "code or meld count out of range");
  Tabs T{H.suit_cls.data(), H.honor_cls.data(), H.t1.data(), H.t2.data(), H.t3.data()};
  const uint32_t cls = (uint32_t)H.suit_cls[cm] | ((uint32_t)H.suit_cls[cp] << 8) | ((uint32_t)H.suit_cls[cs] << 16) |
                       ((uint32_t)H.honor_cls[cz] << 24);
  *out = std_shanten_cls(T, cls, melds);
  return 0;
}

int64_t rs_state_bytes(const rs_handle* h) { return h ? (int64_t)h->mem_bytes : canonical_state_bytes(); }
int64_t rs_num_envs(const rs_handle* h) { return h ? h->n : 0; }

int rs_create(rs_handle** out, int64_t n_envs, const rs_config* cfg, int32_t device) {
  if (!out || !cfg || n_envs <= 0 || n_envs > (1 << 23)) return set_err(RS_E_ARG, "bad rs_create arguments (1 <= n <= 2^23)");
  if (cfg->rule != RS_RULE_RED && cfg->rule != RS_RULE_NO_RED) return set_err(RS_E_ARG, "bad rule");
  if (cfg->mode < 0 || cfg->mode > 2) return set_err(RS_E_ARG, "bad mode");
  if (cfg->illegal_penalty > 0.f) return set_err(RS_E_ARG, "illegal penalty must be <= 0");
  if (cfg->max_steps <= 0 || cfg->max_steps > 65535) return set_err(RS_E_ARG, "max_steps out of range");
  const HostTables& H = host_tables();
  const DeviceScope device_scope(device);
  rs_handle* h = new rs_handle();
  h->device = device;
  h->n = (int)n_envs;
  h->cfg = to_cfg(cfg);
  const size_t n = (size_t)n_envs;
  struct Part { void** p; size_t bytes; };
  Soa& S = h->S;
  S.n = (int)n;
  const int trc = device_tables(device, &h->D);
  if (trc == 0) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    h->persist = g_dev_tables[device].persist;
    h->window = g_dev_tables[device].window;
  }
  if (trc) {
    delete h;
    return trc;
  }
  Part parts[] = {
      {(void**)&S.blk, (size_t)BLK_BYTES * n},
      {(void**)&S.river, 4 * RS_MAX_RIVER * 2 * n},
      {(void**)&S.events, 64 * 4 * n},
      {(void**)&S.results, sizeof(rs_result_rec) * n},
      {(void**)&h->legal_bits_tmp, 16 * n},  {(void**)&h->rec_dev, sizeof(rs_env_rec)},
      {(void**)&h->kind, n},                 {(void**)&h->kind_sorted, n},
      {(void**)&h->iota, 4 * n},             {(void**)&h->order, 4 * n},
  };
  size_t total = 0;
  for (auto& p : parts) total += (p.bytes + 255) & ~(size_t)255;
  cudaError_t err = cudaMalloc(&h->mem, total);
  if (err != cudaSuccess) {
    delete h;
    return set_err((int)err, "cudaMalloc(%zu): %s", total, cudaGetErrorString(err));
  }
  h->mem_bytes = total;
  size_t off = 0;
  for (auto& p : parts) {
    *p.p = (char*)h->mem + off;
    off += (p.bytes + 255) & ~(size_t)255;
  }
  auto cleanup = [&](cudaError_t e2, const char* what) {
    cudaFree(h->mem);
    cudaFree(h->sort_tmp);  // (value-initialised: null until allocated)
    delete h;
    return set_err((int)e2, "%s: %s", what, cudaGetErrorString(e2));
  };
  if ((err = cudaMemset(h->mem, 0, total))) return cleanup(err, "state clear");
  if ((err = cudaMemset(h->kind, 2, n))) return cleanup(err, "kind init");
  k_iota<<<(unsigned)((n + 255) / 256), 256>>>(h->iota, (int)n);
  if ((err = cudaGetLastError())) return cleanup(err, "iota");
  h->sort_tmp = nullptr;
  h->sort_tmp_bytes = 0;
  if ((err = cub::DeviceRadixSort::SortPairs(nullptr, h->sort_tmp_bytes, h->kind, h->kind_sorted, h->iota, h->order,
                                             (int)n, 0, RS_KIND_BITS)))
    return cleanup(err, "sort size query");
  if ((err = cudaMalloc(&h->sort_tmp, std::max<size_t>(h->sort_tmp_bytes, 16)))) return cleanup(err, "sort scratch");
  const void* kernels[] = {(const void*)k_init, (const void*)k_step, (const void*)k_policy,
                           (const void*)k_observe, (const void*)k_rollout<false>, (const void*)k_rollout<true>,
                           (const void*)k_import, (const void*)k_autoreset, (const void*)k_check};
  // the largest launch (the stage mode's slots) may exceed the opt-in limit
  // in a -DRS_TABLES_SMEM build (tables + scratch + 256 slots): allow what
  // the device allows; a launch that needs more fails at launch
  int optin = 0;
  if ((err = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device)))
    return cleanup(err, "device query");
  for (const void* k : kernels) {
    cudaFuncAttributes fa{};
    if ((err = cudaFuncGetAttributes(&fa, k))) return cleanup(err, "cudaFuncGetAttributes");
    const int want = std::min(smem_staged(ROLL_BLOCK, ROLL_BLOCK), optin - (int)fa.sharedSizeBytes);
    if ((err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, want)))
      return cleanup(err, "cudaFuncSetAttribute");
  }
  if ((err = cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device)))
    return cleanup(err, "device query");
  for (int i = 0; i < 16; i++) h->occ_key[i] = h->occ_val[i] = 0;
  for (int i = 0; i < 8; i++) h->occ_cl_key[i] = h->occ_cl_val[i] = 0;
  const char* cluster_env = getenv("RINSHAN_CLUSTER");
  h->cluster = cluster_env ? std::max(1, std::min(8, atoi(cluster_env))) : 1;
  if (h->cluster & (h->cluster - 1)) h->cluster = 1;
  const char* prefetch_env_s = getenv("RINSHAN_PREFETCH");
  // measured on B200 (tools/prefetch_ab.sh): block lines +1-1.5 % at 4,096-16,384 envs, neutral at 1 M;
  // the observer streams too (2) cost HBM traffic at large batches (1 M envs -7 %)
  // the next observer's stream alone (after the header load, k_rollout): neutral at 4,096 envs, -1 % at 1 M
  // round 2: with the observer streams replaced by the 256-byte event ring, mode 2 (block + ring) is the
  // default: +1-1.7 % at 262 K-1 M envs, neutral at 4,096-64 K
  h->prefetch = prefetch_env_s ? std::max(0, std::min(2, atoi(prefetch_env_s))) : 2;
  const char* warm_env_s = getenv("RINSHAN_WARM");
  h->warm = warm_env_s ? (atoi(warm_env_s) != 0) : 1;
  const char* stage_env = getenv("RINSHAN_STAGE");
  h->stage_mode = stage_env ? std::max(0, std::min(2, atoi(stage_env))) : 0;
  const char* groups_env = getenv("RINSHAN_GROUPS");
  h->groups = groups_env ? (atoi(groups_env) != 0) : 1;
  const char* check_env = getenv("RINSHAN_CHECK");
  h->check_steps = check_env ? (atoi(check_env) != 0) : 0;
  const char* order_env = getenv("RINSHAN_ORDER");
  h->ordering = order_env ? std::max(0, std::min(2, atoi(order_env))) : 1;
  const char* block_env = getenv("RINSHAN_BLOCK");
  h->block_override = block_env ? std::max(0, std::min(ROLL_BLOCK, atoi(block_env) & ~31)) : 0;
  const char* epw_env = getenv("RINSHAN_EPW");
  h->epw_override = epw_env ? std::max(0, std::min(32, atoi(epw_env))) : 0;
  *out = h;
  return 0;
}

int rs_destroy(rs_handle* h) {
  if (!h) return 0;
  const DeviceScope device_scope(h->device);
  cudaFree(h->mem);
  cudaFree(h->sort_tmp);
  cudaFree(h->export_buf);
  cudaFree(h->dig_obs_mem);
  cudaFree(h->done_ctr);
  delete h;
  return 0;
}

int rs_init(rs_handle* h, const uint64_t* seeds_dev, const rs_step_out* out, void* stream) {
  if (!h || !seeds_dev) return set_err(RS_E_ARG, "rs_init: null argument");
  const DeviceScope device_scope(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  k_init<<<grid_of(h->n), BLOCK, smem_for(BLOCK), st>>>(h->S, h->D, h->cfg, seeds_dev, 0, 0, 0, step_out(h, out));
  return finish_step_out(h, out, st);
}

int rs_init_indexed(rs_handle* h, uint64_t seed, int64_t index_base, const rs_step_out* out, void* stream) {
  if (!h) return set_err(RS_E_ARG, "rs_init_indexed: null handle");
  const DeviceScope device_scope(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  k_init<<<grid_of(h->n), BLOCK, smem_for(BLOCK), st>>>(h->S, h->D, h->cfg, nullptr, seed, index_base, 1,
                                                  step_out(h, out));
  return finish_step_out(h, out, st);
}

int rs_step(rs_handle* h, const int32_t* actions_dev, const rs_step_out* out, void* stream) {
  return rs_step_ex(h, actions_dev, 0, out, nullptr, nullptr, stream);
}

int rs_step_ex(rs_handle* h, const int32_t* actions_dev, int32_t flags, const rs_step_out* out,
               const rs_obs_out* obs, int32_t* next_actions_dev, void* stream) {
  if (!h || !actions_dev) return set_err(RS_E_ARG, "rs_step: null argument");
  if ((flags & RS_STEP_OBSERVE) && !obs) return set_err(RS_E_ARG, "RS_STEP_OBSERVE needs obs buffers");
  if ((flags & RS_STEP_RESET_FIRST) && ((flags & RS_STEP_AUTORESET) || !next_actions_dev))
    return set_err(RS_E_ARG, "RS_STEP_RESET_FIRST needs next_actions and excludes RS_STEP_AUTORESET");
  const DeviceScope device_scope(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  rs_obs_out o{};
  if (obs) o = *obs;
  const Launch L = step_launch(h, false);
  if (L.ordered) {
    const int rc = order_envs(h, st);
    if (rc) return rc;
  }
  CUDA_TRY(launch_tables(h, k_step, L.grid + warm_of(h, L), L.block, L.smem, st, h->S, h->D, h->cfg, actions_dev,
                         flags, o, next_actions_dev, step_out(h, out), L.epw, L.staged, L.glog2, h->check_steps,
                         (rs_step_rec*)nullptr, L.ordered ? (const int32_t*)h->order : nullptr,
                         L.ordered ? h->kind : nullptr, h->prefetch, done_of(h, L, flags), warm_of(h, L)));
  return finish_step_out(h, out, st);
}

int rs_step_rec_out(rs_handle* h, const int32_t* actions, int32_t flags, rs_step_rec* recs,
                    const rs_obs_out* obs, int32_t* next_actions, void* stream) {
  if (!h || !actions || !recs) return set_err(RS_E_ARG, "rs_step_rec_out: null argument");
  if ((flags & RS_STEP_OBSERVE) && !obs) return set_err(RS_E_ARG, "RS_STEP_OBSERVE needs obs buffers");
  if ((flags & RS_STEP_RESET_FIRST) && (flags & RS_STEP_AUTORESET))
    return set_err(RS_E_ARG, "RS_STEP_RESET_FIRST excludes RS_STEP_AUTORESET");
  const DeviceScope device_scope(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  rs_obs_out o{};
  if (obs) o = *obs;
  const Launch L = step_launch(h, false);
  if (L.ordered) {
    const int rc = order_envs(h, st);
    if (rc) return rc;
  }
  CUDA_TRY(launch_tables(h, k_step, L.grid + warm_of(h, L), L.block, L.smem, st, h->S, h->D, h->cfg, actions,
                         flags, o, next_actions, StepOut{}, L.epw, L.staged, L.glog2, h->check_steps, recs,
                         L.ordered ? (const int32_t*)h->order : nullptr, L.ordered ? h->kind : nullptr,
                         h->prefetch, done_of(h, L, flags), warm_of(h, L)));
  return 0;
}

int rs_signal_done(rs_handle* h, void* stream) {
  if (!h || !h->done_flag) return set_err(RS_E_ARG, "rs_signal_done: no completion word (rs_set_done_flag)");
  const DeviceScope device_scope(h->device);
  k_signal<<<1, 32, 0, (cudaStream_t)stream>>>(Done{h->done_ctr, h->done_flag, 1u});
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int rs_set_done_flag(rs_handle* h, uint32_t* host_flag) {
  if (!h) return set_err(RS_E_ARG, "rs_set_done_flag: null handle");
  const DeviceScope device_scope(h->device);
  if (host_flag && !h->done_ctr) {
    CUDA_TRY(cudaMalloc(&h->done_ctr, 2 * sizeof(uint32_t)));
    CUDA_TRY(cudaMemset(h->done_ctr, 0, 2 * sizeof(uint32_t)));
  }
  if (host_flag) {
    // the sequence starts again from the host word's current value
    CUDA_TRY(cudaDeviceSynchronize());
    const uint32_t init[2] = {0u, *host_flag};
    CUDA_TRY(cudaMemcpy(h->done_ctr, init, sizeof(init), cudaMemcpyHostToDevice));
  }
  h->done_flag = host_flag;
  return 0;
}

int rs_observe(rs_handle* h, const int8_t* seats_dev, const rs_obs_out* obs, void* stream) {
  if (!h || !obs) return set_err(RS_E_ARG, "rs_observe: null argument");
  const DeviceScope device_scope(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  k_observe<<<grid_of(h->n), BLOCK, smem_for(BLOCK), st>>>(h->S, h->D, h->cfg, seats_dev, *obs);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int rs_policy_random(rs_handle* h, int32_t* actions_dev, void* stream) {
  if (!h || !actions_dev) return set_err(RS_E_ARG, "rs_policy_random: null argument");
  const DeviceScope device_scope(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  k_policy<<<grid_of(h->n), BLOCK, smem_for(BLOCK), st>>>(h->S, h->D, h->cfg, actions_dev, RS_POLICY_RANDOM);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int rs_policy_heuristic(rs_handle* h, int32_t* actions_dev, void* stream) {
  if (!h || !actions_dev) return set_err(RS_E_ARG, "rs_policy_heuristic: null argument");
  const DeviceScope device_scope(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  k_policy<<<grid_of(h->n), BLOCK, smem_for(BLOCK), st>>>(h->S, h->D, h->cfg, actions_dev, RS_POLICY_HEURISTIC);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int rs_rollout(rs_handle* h, int32_t steps, const rs_obs_out* obs, int32_t obs_slots, int16_t* actions_log,
               rs_rollout_stats* stats_dev, uint64_t* digests_dev, const rs_step_out* out, void* stream) {
  return rs_rollout_policy(h, steps, RS_POLICY_RANDOM, obs, obs_slots, actions_log, nullptr, nullptr, stats_dev,
                           digests_dev, out, stream);
}

int rs_rollout_policy(rs_handle* h, int32_t steps, int32_t policy, const rs_obs_out* obs, int32_t obs_slots,
                      int16_t* actions_log, int8_t* actors_log, const rs_step_out* traj,
                      rs_rollout_stats* stats_dev, uint64_t* digests_dev, const rs_step_out* out, void* stream) {
  if (traj && traj->legal_mask) return set_err(RS_E_ARG, "rs_rollout: traj takes packed legal_bits, not legal_mask");
  if (!h || steps < 0) return set_err(RS_E_ARG, "rs_rollout: bad arguments");
  if (policy != RS_POLICY_RANDOM && policy != RS_POLICY_HEURISTIC) return set_err(RS_E_ARG, "rs_rollout: unknown policy");
  if (obs_slots < 0 || (obs_slots > 1 && obs_slots != steps)) return set_err(RS_E_ARG, "obs_slots must be 0, 1 or steps");
  if (obs_slots > 0 && !obs) return set_err(RS_E_ARG, "obs_slots > 0 needs obs buffers");
  const DeviceScope device_scope(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  rs_obs_out o{};
  if (obs) o = *obs;
  // persistent grid of the resident CTA count (tables staged once per CTA,
  // envs walked grid-stride)
  if (digests_dev && !h->dig_obs_mem) {
    const size_t n = (size_t)h->n;
    uint8_t* p = nullptr;
    CUDA_TRY(cudaMalloc(&p, n * 256));
    h->dig_obs_mem = p;
    rs_obs_out& d = h->dig_obs;
    d.event_tokens = p; d.hand_tokens = p + 192 * n; d.shanten = (int8_t*)(p + 206 * n);  // window: uint4 stores
    d.scores = (int16_t*)(p + 208 * n); d.honba = (int16_t*)(p + 216 * n); d.deposits = (int16_t*)(p + 218 * n);
    d.round_wind = p + 220 * n; d.seat_wind = p + 221 * n; d.kyoku = p + 222 * n; d.live_wall = p + 223 * n;
    d.dora_tokens = p + 224 * n; d.riichi_flags = p + 229 * n;
  }
  const Launch L = step_launch(h, true);
  auto kern = (digests_dev || h->check_steps) ? k_rollout<true> : k_rollout<false>;
  if (L.ordered && steps > 1) {
    // large batches: one launch per step, the envs re-sorted by the kind
    // of their next step before each (within one fused launch the envs of
    // a warp drift apart: 1 M envs ran 603 M env steps/s fused 100 steps
    // per launch vs 946 M one sorted step per launch); outputs indexed by
    // step go to slot t of the caller's [steps][n] buffers
    const size_t n = (size_t)h->n;
    StepOut tr = step_out(h, traj);
    for (int t = 0; t < steps; t++) {
      if (const int rc = order_envs(h, st)) return rc;
      rs_obs_out ot{};
      int slots = 0;
      if (obs && obs_slots > 1) {
        ot = obs_slot(o, (size_t)t, n);
        slots = 1;
      } else if (obs && obs_slots == 1 && t == steps - 1) {
        ot = o;
        slots = 1;
      }
      StepOut trt{};
      if (tr.legal_bits) trt.legal_bits = tr.legal_bits + (size_t)t * n * 4;
      if (tr.current_player) trt.current_player = tr.current_player + (size_t)t * n;
      if (tr.rewards) trt.rewards = tr.rewards + (size_t)t * n * 4;
      if (tr.terminated) trt.terminated = tr.terminated + (size_t)t * n;
      if (tr.truncated) trt.truncated = tr.truncated + (size_t)t * n;
      if (tr.status) trt.status = tr.status + (size_t)t * n;
      CUDA_TRY(launch_tables(h, kern, L.grid + warm_of(h, L), L.block, L.smem, st, h->S, h->D, h->cfg, 1, ot, slots,
                             actions_log ? actions_log + (size_t)t * n : nullptr,
                             actors_log ? actors_log + (size_t)t * n : nullptr, trt, stats_dev, digests_dev,
                             h->dig_obs, step_out(h, out), L.epw, nullptr, L.staged, policy, L.glog2,
                             h->check_steps, (const int32_t*)h->order, h->kind, h->prefetch, warm_of(h, L)));
    }
    return finish_step_out(h, out, st);
  }
  if (L.ordered) {
    const int rc = order_envs(h, st);
    if (rc) return rc;
  }
  CUDA_TRY(launch_tables(h, kern, L.grid + warm_of(h, L), L.block, L.smem, st, h->S, h->D, h->cfg, steps, o,
                         obs ? obs_slots : 0, actions_log, actors_log, step_out(h, traj), stats_dev, digests_dev,
                         h->dig_obs, step_out(h, out), L.epw, nullptr, L.staged, policy, L.glog2, h->check_steps,
                         L.ordered ? (const int32_t*)h->order : nullptr, L.ordered ? h->kind : nullptr,
                         h->prefetch, warm_of(h, L)));
  return finish_step_out(h, out, st);
}

// debug / profiling hook: one rollout of `steps` with per-env per-step
// clock64 cycles of the auto-reset and of policy+step+observe, the action
// and flags, into prof_dev[steps][n][4] (u32)
int rs_debug_rollout_cycles(rs_handle* h, int32_t steps, const rs_obs_out* obs, uint32_t* prof_dev, void* stream) {
  if (!h || !prof_dev || steps < 1) return set_err(RS_E_ARG, "rs_debug_rollout_cycles: bad arguments");
  const DeviceScope device_scope(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  rs_obs_out o{};
  if (obs) o = *obs;
  const Launch L = step_launch(h, true);
  CUDA_TRY(launch_tables(h, k_rollout<false>, L.grid, L.block, L.smem, st, h->S, h->D, h->cfg, steps, o, obs ? 1 : 0,
                         nullptr, nullptr, StepOut{}, nullptr, nullptr, rs_obs_out{}, StepOut{}, L.epw, prof_dev, L.staged,
                         (int)RS_POLICY_RANDOM, L.glog2, 0, (const int32_t*)nullptr, (uint8_t*)nullptr,
                         h->prefetch, 0));
  CUDA_TRY(cudaGetLastError());
  return 0;
}

#if defined(RS_PROFILE_MARKS)
extern "C" int rs_debug_set_marks(void* marks) {
  return (int)cudaMemcpyToSymbol(g_marks, &marks, sizeof(marks));
}
#endif

int rs_check_invariants(rs_handle* h, int32_t fast, uint32_t* flags_dev, void* stream) {
  if (!h || !flags_dev) return set_err(RS_E_ARG, "rs_check_invariants: null argument");
  const DeviceScope device_scope(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  k_check<<<grid_of(h->n), BLOCK, smem_for(BLOCK), st>>>(h->S, h->D, h->cfg, fast, flags_dev);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int rs_autoreset(rs_handle* h, const rs_step_out* out, void* stream) {
  if (!h) return set_err(RS_E_ARG, "rs_autoreset: null handle");
  const DeviceScope device_scope(h->device);
  cudaStream_t st = (cudaStream_t)stream;
  k_autoreset<<<grid_of(h->n), BLOCK, smem_for(BLOCK), st>>>(h->S, h->D, h->cfg, step_out(h, out));
  return finish_step_out(h, out, st);
}

int rs_export_env(rs_handle* h, int64_t env, rs_env_rec* out) {
  if (!h || !out || env < 0 || env >= h->n) return set_err(RS_E_ARG, "rs_export_env: bad arguments");
  return rs_export_envs(h, &env, 1, out);
}

int rs_export_envs(rs_handle* h, const int64_t* envs, int64_t count, rs_env_rec* out) {
  if (!h || count < 0 || (count > 0 && (!envs || !out)) || count > INT32_MAX)
    return set_err(RS_E_ARG, "rs_export_envs: bad arguments");
  for (int64_t i = 0; i < count; i++)
    if (envs[i] < 0 || envs[i] >= h->n) return set_err(RS_E_ARG, "rs_export_envs: env %lld out of range", (long long)envs[i]);
  if (count == 0) return 0;
  const DeviceScope device_scope(h->device);
  std::lock_guard<std::mutex> lk(h->export_mu);  // the export buffer is shared by the handle's callers
  // steps may have been launched on any stream, blocking or not
  CUDA_TRY(cudaDeviceSynchronize());
  const size_t rec_bytes = (size_t)count * sizeof(rs_env_rec);
  const size_t need = rec_bytes + (size_t)count * sizeof(int64_t);
  if (need > h->export_cap) {
    CUDA_TRY(cudaFree(h->export_buf));
    h->export_buf = nullptr;
    h->export_cap = 0;
    CUDA_TRY(cudaMalloc(&h->export_buf, need));
    h->export_cap = need;
  }
  rs_env_rec* d_out = (rs_env_rec*)h->export_buf;
  int64_t* d_envs = (int64_t*)((char*)h->export_buf + rec_bytes);
  cudaError_t e = cudaMemcpy(d_envs, envs, (size_t)count * sizeof(int64_t), cudaMemcpyHostToDevice);
  // fields export_env leaves unwritten (padding, slots past the counts) read as zero
  if (e == cudaSuccess) e = cudaMemset(d_out, 0, rec_bytes);
  if (e == cudaSuccess) {
    k_export_many<<<(unsigned)((count + 127) / 128), 128>>>(h->S, h->cfg, d_envs, count, d_out);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, d_out, rec_bytes, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return set_err((int)e, "rs_export_envs: %s", cudaGetErrorString(e));
  return 0;
}

int rs_import_env(rs_handle* h, int64_t env, const rs_env_rec* in) {
  if (!h || !in || env < 0 || env >= h->n) return set_err(RS_E_ARG, "rs_import_env: bad arguments");
  if (in->abi_version != RS_ABI_VERSION) return set_err(RS_E_ARG, "record abi version mismatch");
  if (const char* bad = record_out_of_range(*in)) return set_err(RS_E_ARG, "rs_import_env: %s out of range", bad);
  const DeviceScope device_scope(h->device);
  std::lock_guard<std::mutex> lk(h->export_mu);  // rec_dev
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(h->rec_dev, in, sizeof(rs_env_rec), cudaMemcpyHostToDevice));
  k_import<<<1, 32, smem_for(32)>>>(h->S, h->D, h->cfg, (int)env, h->rec_dev);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaDeviceSynchronize());
  return 0;
}

int rs_debug_score(const rs_winctx* ctx, int64_t count, rs_win_rec* out, int32_t* ok, int32_t device) {
  if (count < 0 || (count && (!ctx || !out || !ok))) return set_err(RS_E_ARG, "bad rs_debug_score arguments");
  if (!count) return 0;
  for (int64_t i = 0; i < count; i++) {
    const rs_winctx& c = ctx[i];
    if (c.n_melds < 0 || c.n_melds > 4 || c.n_ids < 0 || c.n_ids > 18 || c.n_dora < 0 || c.n_dora > 5 ||
        c.n_ura < 0 || c.n_ura > 5 || c.win_tile < 0 || c.win_tile >= RS_NUM_TILES)
      return set_err(RS_E_ARG, "rs_winctx field out of range");
  }
  const DeviceScope device_scope(device);
  rs_winctx* dctx = nullptr;
  rs_win_rec* dout = nullptr;
  int32_t* dok = nullptr;
  int rc = 0;
  cudaError_t e = cudaMalloc(&dctx, sizeof(rs_winctx) * count);
  if (e == cudaSuccess) e = cudaMalloc(&dout, sizeof(rs_win_rec) * count);
  if (e == cudaSuccess) e = cudaMalloc(&dok, sizeof(int32_t) * count);
  if (e == cudaSuccess) e = cudaMemcpy(dctx, ctx, sizeof(rs_winctx) * count, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    k_debug_score<<<(unsigned)((count + 127) / 128), 128>>>(dctx, count, dout, dok);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, dout, sizeof(rs_win_rec) * count, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(ok, dok, sizeof(int32_t) * count, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) rc = set_err((int)e, cudaGetErrorString(e));
  cudaFree(dctx);
  cudaFree(dout);
  cudaFree(dok);
  return rc;
}

int rs_record_sizes(int32_t* out /*[7]*/) {
  out[0] = (int32_t)sizeof(rs_config);
  out[1] = (int32_t)sizeof(rs_meld_rec);
  out[2] = (int32_t)sizeof(rs_hand_rec);
  out[3] = (int32_t)sizeof(rs_win_rec);
  out[4] = (int32_t)sizeof(rs_result_rec);
  out[5] = (int32_t)sizeof(rs_env_rec);
  out[6] = (int32_t)sizeof(rs_step_rec);
  return 0;
}

}  // extern "C"
