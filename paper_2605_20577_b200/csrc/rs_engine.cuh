// rs_engine.cuh — the kyoku/game state machine, one thread per env.
//
// Mirrors the reference transition function (engine/engine.py:105-891) and
// env facade (env/core.py:65-94) over the SoA state of rs_state.cuh.  The
// game scalars live in registers (`Game`) for the whole step; per-seat
// hands are loaded into registers (`Hand`) where a transition reads or
// rewrites them and stored back once.
#pragma once

#include "rs_hand.cuh"
#include "rs_score.cuh"

namespace rs {

// phase timestamps for build-time profiling experiments (-DRS_PROFILE_MARKS)
// RS_PROFILE_MARKS=1: phases of init_game (RS_MARK); =2: phases of a step (RS_SMARK);
// =4: phases of a win (RS_WMARK)
#if defined(RS_PROFILE_MARKS) && defined(__CUDA_ARCH__)
#define RS_MARK_AT(i)                                                                        \
  do {                                                                                       \
    if (g_marks) g_marks[(size_t)(blockIdx.x * blockDim.x + threadIdx.x) * 8 + (i)] = clock64(); \
  } while (0)
#else
#define RS_MARK_AT(i) \
  do {                \
  } while (0)
#endif
#if defined(RS_PROFILE_MARKS) && RS_PROFILE_MARKS == 4
#define RS_WMARK(i) RS_MARK_AT(i)
#else
#define RS_WMARK(i) do {} while (0)
#endif
#if defined(RS_PROFILE_MARKS) && RS_PROFILE_MARKS == 2
#define RS_MARK(i) do {} while (0)
#define RS_SMARK(i) RS_MARK_AT(i)
#elif defined(RS_PROFILE_MARKS) && RS_PROFILE_MARKS == 1
#define RS_MARK(i) RS_MARK_AT(i)
#define RS_SMARK(i) do {} while (0)
#else
#define RS_MARK(i) do {} while (0)
#define RS_SMARK(i) do {} while (0)
#endif

enum : int { PH_ACT = 0, PH_CALL = 1, PH_GAME_END = 2 };
enum : int { ST_RON = 0, ST_PONKAN = 1, ST_CHI = 2 };
enum : int {
  EV_DRAW = 0, EV_DISCARD, EV_CHI, EV_PON, EV_KAN_OPEN, EV_KAN_CLOSED, EV_KAN_ADDED,
  EV_RIICHI, EV_RON, EV_TSUMO, EV_DRAW_END, EV_NEW_DORA
};
enum : int {
  A_RIICHI = 37, A_TSUMO = 38, A_RON = 39, A_PON = 40, A_CHI_LOW = 41, A_CHI_MID = 42,
  A_CHI_HIGH = 43, A_KAN_OPEN = 44, A_KAN_CLOSED = 45, A_KAN_ADDED = 79, A_PASS = 113, A_NINE = 114
};
enum : int { M_CHI = 0, M_PON = 1, M_KAN_OPEN = 2, M_KAN_CLOSED = 3, M_KAN_ADDED = 4 };

struct Mask115 {
  uint32_t m[4];
  RS_HD void clear() { m[0] = m[1] = m[2] = m[3] = 0; }
  // dynamic word index as selects (no branches)
  RS_HD void set(int a) {
    const uint32_t b = 1u << (a & 31);
    const int w = a >> 5;
    m[0] |= w == 0 ? b : 0u;
    m[1] |= w == 1 ? b : 0u;
    m[2] |= w == 2 ? b : 0u;
    m[3] |= w >= 3 ? b : 0u;
  }
  RS_HD bool test(int a) const {
    const int i = a >> 5;
    uint32_t w = m[3];
    w = i == 2 ? m[2] : w;
    w = i == 1 ? m[1] : w;
    w = i == 0 ? m[0] : w;
    return (w >> (a & 31)) & 1u;
  }
  RS_HD int count() const { return popc32(m[0]) + popc32(m[1]) + popc32(m[2]) + popc32(m[3]); }
  // the i-th set bit (ascending ids, engine.py:258); -1 when i >= count().
  // Branch-free (the 32 envs of a warp have different masks and ranks at
  // large batches): the word by prefix counts, then a binary search over
  // half / byte / nibble / pair popcounts (__fns is emulated in software on
  // sm_100)
  RS_HD int nth(int i) const {
    const int c0 = popc32(m[0]), c1 = popc32(m[1]), c2 = popc32(m[2]);
    int w = 0;
    uint32_t x = m[0];
    if (i >= c0) { i -= c0; w = 1; x = m[1]; }
    if (w == 1 && i >= c1) { i -= c1; w = 2; x = m[2]; }
    if (w == 2 && i >= c2) { i -= c2; w = 3; x = m[3]; }
    if (i >= popc32(x)) return -1;
    int pos = 0;
#pragma unroll
    for (int half = 16; half >= 1; half >>= 1) {
      const uint32_t lo = x & ((1u << half) - 1u);
      const int c = popc32(lo);
      const bool up = i >= c;
      i -= up ? c : 0;
      x = up ? x >> half : lo;
      pos += up ? half : 0;
    }
    return 32 * w + pos;
  }
};

// engine.py:100-102 event, written into the env's 64-slot ring as one word
// laid out for observe() (observe.py:92-106), which decodes four slots at a
// time with byte permutes (rs_io.cuh view4):
//   byte 0: observation type token (ron / tsumo share 8) | bit 4 + s: the
//           tile is hidden from observer s (an opponent's draw)
//   byte 1: bits 2s..2s+1: the actor relative to observer s (0 without one)
//   byte 2: visible tile token (red fives 34-36, none 37) | bit 6: has an actor
//   byte 3: tile copy (tile & 3) | bit 2: has a tile | bits 3-6: event type
// -- the event itself (type, actor, tile) stays recoverable (event_raw) for
// export, import and the digest.  One store per event (round 1 also kept
// the event pre-encoded for each of the four observers: four more
// scattered sector writes per event, 1 KB per env).
RS_HD uint32_t event_word(int rule, int type, int actor, int tile) {
  const uint32_t ty = (uint32_t)(type <= 8 ? type : type - 1);
  const uint32_t tok = tile < 0 ? 37u
                       : (rule == RS_RULE_RED && is_red_tile(tile)) ? (uint32_t)(34 + red_index_of_kind(tile >> 2))
                                                                    : (uint32_t)(tile >> 2);
  uint32_t hid = 0, rel = 0;
  if (actor >= 0) {
    if (type == EV_DRAW) hid = 0xFu & ~(1u << actor);
    for (int o = 0; o < 4; o++) rel |= (uint32_t)((actor - o) & 3) << (2 * o);
  }
  return ty | (hid << 4) | (rel << 8) | (tok << 16) | ((actor >= 0 ? 1u : 0u) << 22) |
         ((uint32_t)(tile >= 0 ? tile & 3 : 0) << 24) | ((tile >= 0 ? 1u : 0u) << 26) | ((uint32_t)type << 27);
}
// the canonical event (type | (actor + 1) << 4 | (tile + 1) << 7)
RS_HD uint32_t event_raw(uint32_t x) {
  const uint32_t type = (x >> 27) & 15u;
  const uint32_t a1 = ((x >> 22) & 1u) ? ((x >> 8) & 3u) + 1u : 0u;
  const uint32_t tok = (x >> 16) & 63u;
  const int tile = ((x >> 26) & 1u) ? (tok >= 34 ? 16 + 36 * (int)(tok - 34) : (int)(4 * tok + ((x >> 24) & 3u))) : -1;
  return type | (a1 << 4) | ((uint32_t)(tile + 1) << 7);
}
// a window pad slot: (0, 0, 37) for every observer
constexpr uint32_t EVENT_PAD = 37u << 16;
// out of line, called with scalars (19 emit sites; DESIGN §4 item 25)
RS_COLD void emit_event(uint32_t* ring, uint32_t p, int rule, int type, int actor, int tile) {
  ring[p] = event_word(rule, type, actor, tile);
}

// engine members that can go out of line for a smaller hot code footprint
// (DESIGN §4 items 23-26): draw() is (gains at every batch size); these
// switches keep the measured alternatives reproducible (mixed results, off)
#if defined(RS_OL_LEGAL)
#define RS_OL_LEGAL_Q RS_COLD
#else
#define RS_OL_LEGAL_Q RS_HD
#endif
#if defined(RS_OL_CALL)
#define RS_OL_CALL_Q RS_COLD
#else
#define RS_OL_CALL_Q RS_HD
#endif
#if defined(RS_OL_STANDS)
#define RS_OL_STANDS_Q RS_COLD
#else
#define RS_OL_STANDS_Q RS_HD
#endif

// Five consecutive Fisher-Yates swaps (rng.py:59-65) i, i-1, .., i-4 with
// targets j[0..4] on a byte array: the ten positions are loaded at once,
// the swaps are resolved in registers (a later swap reads what an earlier
// one of the batch wrote: a target j[v] can equal a later position i-u or a
// later target), and the ten stores issue in swap order, so the chain costs
// one load round trip per five swaps instead of one per swap.
RS_HD void swap5(uint8_t* w, int i, const int* j) {
  if (!RS_SWAP5_ON) {  // the plain chain (default; -DRS_SWAP5: batched)
    for (int u = 0; u < 5; u++) {
      const uint8_t t = w[i - u];
      w[i - u] = w[j[u]];
      w[j[u]] = t;
    }
    return;
  }
  int x[5], y[5];
#pragma unroll
  for (int u = 0; u < 5; u++) {
    x[u] = w[i - u];
    y[u] = w[j[u]];
  }
  int av[5], bv[5];
#pragma unroll
  for (int u = 0; u < 5; u++) {
    int ca = x[u], cb = y[u];
#pragma unroll
    for (int v = 0; v < u; v++) {
      if (j[v] == i - u) ca = bv[v];
      if (j[v] == j[u]) cb = bv[v];
    }
    if (j[u] == i - u) cb = ca;
    av[u] = cb;
    bv[u] = ca;
  }
#pragma unroll
  for (int u = 0; u < 5; u++) {
    w[i - u] = (uint8_t)av[u];
    w[j[u]] = (uint8_t)bv[u];
  }
}

struct Engine {
  const Soa& S;
  const Tabs& T;
  const Cfg& C;
  int e;
  uint8_t* bp;  // the env's block: its shared-memory stage slot or its HBM copy (rs_state.cuh)
  Game g;

  RS_HD Engine(const Soa& s, const Tabs& t, const Cfg& c, int env, uint8_t* block)
      : S(s), T(t), C(c), e(env), bp(block) {}

  // ------------------------------------------------------------- memory
  // 32-bit index math: rs_create bounds n so that 160 * n < 2^31
  RS_HD uint32_t at(int f) const {
    RS_CHECK((unsigned)f < 4u * RS_MAX_RIVER && (unsigned)e < (unsigned)S.n);
    return (uint32_t)f * (uint32_t)S.n + (uint32_t)e;
  }
  RS_HD void load() {
    const int4 sc = *reinterpret_cast<const int4*>(&squad(bp, W_SCORES));
    g.unpack(squad(bp, W_HDR), squad(bp, W_HDR + 4), squad(bp, W_HDR + 8), squad(bp, W_HDR + 12), sc);
  }
  RS_HD void store() const {
    uint4 a, b, c, d;
    int4 sc;
    g.pack(a, b, c, d, sc);
    squad(bp, W_HDR) = a; squad(bp, W_HDR + 4) = b; squad(bp, W_HDR + 8) = c; squad(bp, W_HDR + 12) = d;
    *reinterpret_cast<int4*>(&squad(bp, W_SCORES)) = sc;
  }
  RS_HD int wall(int pos) const {
    RS_CHECK((unsigned)pos < (unsigned)RS_NUM_TILES);
    return swall(bp)[pos];
  }
  RS_HD int tok() const { return C.rule == RS_RULE_RED ? 1 : 0; }  // hand_put / hand_take token mode
  RS_HD uint32_t info(int s) const { return sword(bp, W_HINFO + s); }
  RS_HD void set_info(int s, uint32_t v) const { sword(bp, W_HINFO + s) = v; }
  RS_HD uint64_t waits(int s) const { return sdword(bp, W_HWAITS + 2 * s); }
  RS_HD int count_of(int s, int k) const {
    return popc32((sword(bp, W_HMASK + 5 * s + (k >> 3)) >> ((k & 7) * 4)) & 0xFu);
  }
  RS_HD uint32_t meld_info(int s, int i) const {
    RS_CHECK((unsigned)s < 4u && (unsigned)i < 4u);
    return sword(bp, W_MELD + 2 * (4 * s + i) + 1);
  }
  RS_HD uint32_t meld_tiles(int s, int i) const {
    RS_CHECK((unsigned)s < 4u && (unsigned)i < 4u);
    return sword(bp, W_MELD + 2 * (4 * s + i));
  }

  // engine.py:100-102 (64-slot ring; the full history is reconstructed by
  // the host while stepping)
  RS_HD void emit(int type, int actor, int tile) {
    emit_event(S.events + (uint32_t)e * RS_EVENT_WINDOW, g.events_len & 63u, C.rule, type, actor, tile);
    g.events_len++;
  }

  // ------------------------------------------------------ rng / dealing
  // deal 4-4-4 then 1 from the dealer (engine.py:142-151): the seat at
  // offset i = (s - dealer) & 3 receives wall positions 16r + 4i .. +3 and
  // 48 + i (its 4-tile blocks are aligned words of the shuffled wall)
  RS_HD Hand dealt_hand(const uint8_t* w, int i) const {
    Hand h;
    h.w0 = h.w1 = h.w2 = h.w3 = h.w4 = 0;
    h.cm = h.cp = h.cs = h.cz = 0;
    const uint32_t* w32 = reinterpret_cast<const uint32_t*>(w);
#pragma unroll 1
    for (int r = 0; r < 3; r++) {
      const uint32_t q = w32[4 * r + i];
#pragma unroll 1
      for (int j = 0; j < 4; j++) deal_tile(h, (int)((q >> (8 * j)) & 255u));
    }
    deal_tile(h, w[48 + i]);
    h.cls = class_of(T, 0, h.cm) | (class_of(T, 1, h.cp) << 8) | (class_of(T, 2, h.cs) << 16) |
            (class_of(T, 3, h.cz) << 24);
    tokens_from_set(h, C.rule == RS_RULE_RED);
    h.info = hi::set_nconc(hi::set_riichi_index(0u, -1), 13);
    return h;
  }
#if defined(__CUDA_ARCH__)
  // lane group of 4+: lane sub builds seat sub & 3 (the four deals' table
  // lookups in parallel instead of one seat after the other); the waits of
  // a 13-tile tenpai deal (rare) are then scanned by the whole group
  RS_COLD void deal_group(const uint8_t* w, int dealer) {  // one copy (warm_cta warms it)
    const int sub = grp_sub();
    const uint32_t gm = grp_mask();
    const int s = sub & 3;
    Hand h = dealt_hand(w, (s - dealer) & 3);
    RS_MARK(6);
    const int sh = full_shanten(T, h, 0);
    h.info = hi::set_shanten(h.info, sh);
    h.waits = 0ull;
    if (sub < 4) {
      store_hand(bp, s, h);
      sdword(bp, W_HRKIND + 2 * s) = 0ull;
    }
    RS_MARK(7);
    uint32_t tenpai = __ballot_sync(gm, sub < 4 && sh == 0);
    tenpai = (tenpai >> ((threadIdx.x & 31) - sub)) & 15u;
    __syncwarp(gm);
    while (tenpai) {
      const int t = __ffs(tenpai) - 1;
      tenpai &= tenpai - 1;
      const uint64_t wv = compute_waits(T, load_hand(bp, t), 0);
      if (sub == 0) sdword(bp, W_HWAITS + 2 * t) = wv;
      __syncwarp(gm);
    }
  }
#endif

  // engine.py:139-164 (_start_kyoku) with tiles.py:142-144 / rng.py:59-65
  RS_COLD void start_kyoku() {
    // the swap chain is a dependent load / store sequence: it runs in shared
    // memory, in place when the block is staged, else in the thread's
    // 144-byte scratch after the tables (copied to the block afterwards)
    uint8_t* const wall_dst = swall(bp);
    // Fisher-Yates (rng.py:59-65) on a shared-memory scratch (pointers derived
    // from the shared array alone keep the swap chain on LDS / STS), copied
    // to the block afterwards; the draws are counter-based: draw u of the
    // deal (position 135 - u) uses counter rng_counter + 1 + u
    uint64_t c = g.rng_counter;
#if defined(__CUDA_ARCH__)
    const int G = grp_size();
    uint8_t* const w = G > 1 ? g_smem + WALL_SLOT_OFF + (threadIdx.x >> s_grp_log2) * ENV_SCRATCH
                             : g_smem + WALL_SLOT_OFF + threadIdx.x * SCRATCH_STRIDE;
    RS_CHECK((uint32_t)(w - g_smem) + (uint32_t)(G > 1 ? ENV_SCRATCH : SCRATCH_STRIDE) <= dyn_smem_bytes());
    if (G > 1) {
      // lane group: one wall copy per env; the lanes draw the 135 targets in
      // parallel, then lane 0 runs the swap chain alone (no redundant copies,
      // a tenth of the shared memory per env)
      const int sub = grp_sub();
      const uint32_t gm = grp_mask();
      uint32_t* w32 = reinterpret_cast<uint32_t*>(w);
      for (int k = sub; k < 36; k += G) w32[k] = k < 34 ? 0x03020100u + 0x04040404u * (uint32_t)k : 0u;
      uint8_t* const J = w + SCRATCH_STRIDE;
      for (int i = 135 - sub; i > 0; i -= G)
        J[i] = (uint8_t)randbelow_from(stream_value(g.rng_key, c + 1 + (uint64_t)(135 - i)), (uint32_t)(i + 1));
      __syncwarp(gm);
      RS_MARK(0);
      if (sub == 0) {
        for (int i = 135; i > 0; i -= 5) {  // 135 = 27 x 5
          int j[5];
#pragma unroll
          for (int u = 0; u < 5; u++) j[u] = J[i - u];
          swap5(w, i, j);
        }
      }
      __syncwarp(gm);
      c += 135;
      for (int k = sub; k < WALL_STRIDE / 16; k += G)
        reinterpret_cast<uint4*>(wall_dst)[k] = make_uint4(w32[4 * k], w32[4 * k + 1], w32[4 * k + 2], w32[4 * k + 3]);
    } else
#else
    uint8_t* const w = wall_dst;
#endif
    {
      uint32_t* w32 = reinterpret_cast<uint32_t*>(w);
#pragma unroll
      for (int i = 0; i < 34; i++) w32[i] = 0x03020100u + 0x04040404u * (uint32_t)i;
      w32[34] = w32[35] = 0;
      for (int i = 135; i > 0; i -= 5) {
        int j[5];
#pragma unroll
        for (int u = 0; u < 5; u++)
          j[u] = (int)randbelow_from(stream_value(g.rng_key, c + 1 + u), (uint32_t)(i - u + 1));
        c += 5;
        swap5(w, i, j);
      }
#if defined(__CUDA_ARCH__)
      for (int k = 0; k < WALL_STRIDE / 16; k++)  // (scratch: 4-byte aligned)
        reinterpret_cast<uint4*>(wall_dst)[k] = make_uint4(w32[4 * k], w32[4 * k + 1], w32[4 * k + 2], w32[4 * k + 3]);
#endif
    }
    g.rng_counter = (uint32_t)c;
    RS_MARK(2);
    const int dealer = g.dealer();
#if defined(__CUDA_ARCH__)
    if (G >= 4) {
      deal_group(w, dealer);
    } else
#endif
    {
      for (int s = 0; s < 4; s++) {
        Hand h = dealt_hand(w, (s - dealer) & 3);
        finish_hand(T, h);
        store_hand(bp, s, h);
        sdword(bp, W_HRKIND + 2 * s) = 0ull;
      }
    }
    g.cursor = 52;
    g.kan_draws = 0;
    g.dora_count = 1;
    g.riichi_pending = 0;
    g.rinshan_pending = 0;
    g.call_tile = -1;
    g.call_from = -1;
    g.queue = 0;
    g.rons = 0;
    g.call_chankan = 0;
    g.kakan_kind = -1;
    g.pending_dora = 0;
    g.four_kan_pending = 0;
    g.any_call_made = 0;
    RS_MARK(3);
    draw(dealer);
    RS_MARK(4);
  }

  // engine.py:167-178
  RS_COLD void draw(int seat) {  // out of line: DESIGN §4 item 26
    Hand h = load_hand(bp, seat);
    h.info = hi::set_temp(h.info, 0);
    const int tile = wall(g.cursor);
    g.cursor++;
    hand_put(T, h, tile, tok());
    finish_hand(T, h);
    store_hand(bp, seat, h);
    g.drawn = tile;
    g.rinshan_pending = 0;
    g.phase = PH_ACT;
    g.actor = seat;
    emit(EV_DRAW, seat, tile);
  }
  // engine.py:181-189 (temp furiten is NOT cleared here)
  RS_HD void rinshan_draw(int seat, Hand& h) {
    const int tile = wall(135 - g.kan_draws);
    g.kan_draws++;
    hand_put(T, h, tile, tok());
    finish_hand(T, h);
    store_hand(bp, seat, h);
    g.drawn = tile;
    g.rinshan_pending = 1;
    g.phase = PH_ACT;
    g.actor = seat;
    emit(EV_DRAW, seat, tile);
  }

  // ------------------------------------------------------ win evaluation
  // engine.py:345-375 (_win_context)
  // one out-of-line copy for its four callers (cold: win checks and settlements)
  // `value`: also the dora / ura / red counts (the settlement); the legality
  // checks only ask whether a reading carries a yaku, which they never change
  RS_COLD void win_input(int seat, const Hand& h, int win_tile, bool tsumo, bool chankan, WinIn& w,
                         bool value = true) const {
    const uint32_t inf = h.info;
    w.conc.c[0] = nib_counts(h.w0);
    w.conc.c[1] = nib_counts(h.w1);
    w.conc.c[2] = nib_counts(h.w2);
    w.conc.c[3] = nib_counts(h.w3);
    w.conc.c[4] = nib_counts(h.w4);
    if (!tsumo) w.conc.add(win_tile >> 2, 1);
    w.nmelds = hi::nmelds(inf);
    w.closed = true;
    Counts all = w.conc;
    int reds = 0;
    if (value && C.rule == RS_RULE_RED) {
      reds = (int)h.has(16) + (int)h.has(52) + (int)h.has(88);
      if (!tsumo && is_red_tile(win_tile)) reds++;
    }
    // cold code: loops kept rolled (an instruction of a path run once per
    // launch costs its fetch, DESIGN §4 item 49)
    #pragma unroll 1
    for (int i = 0; i < 4; i++) {
      if (i < w.nmelds) {
        const uint32_t mf = meld_info(seat, i), mt = meld_tiles(seat, i);
        w.mtype[i] = mi::type(mf);
        w.mbase[i] = (mt & 255) >> 2;
        if (w.mtype[i] != M_KAN_CLOSED) w.closed = false;
        const int nt = value ? mi::ntiles(mf) : 0;
        #pragma unroll 1
        for (int j = 0; j < 4; j++)
          if (j < nt) {
            const int t = (mt >> (8 * j)) & 255;
            all.add(t >> 2, 1);
            if (C.rule == RS_RULE_RED && is_red_tile(t)) reds++;
          }
      }
    }
    w.win_kind = win_tile >> 2;
    w.tsumo = tsumo;
    w.seat_wind = g.seat_wind(seat);
    w.round_wind = g.round_wind();
    w.riichi = hi::riichi(inf);
    w.ippatsu = hi::ippatsu(inf);
    if (tsumo) {
      w.last_tile = g.live() == 0 && !g.rinshan_pending;
      w.rinshan = g.rinshan_pending;
      w.first_draw = hi::nriver(inf) == 0 && !g.any_call_made && w.nmelds == 0 && !w.rinshan;
      w.chankan = false;
    } else {
      w.last_tile = g.live() == 0 && !chankan;
      w.rinshan = false;
      w.first_draw = false;
      w.chankan = chankan;
    }
    // dora.py:9-26
    int dora = 0, ura = 0;
    const int nd = value ? (int)g.dora_count : 0;
#pragma unroll 1
    for (int i = 0; i < nd; i++) {
      dora += all.get(dora_kind(wall(122 + 2 * i) >> 2));
      if (w.riichi) ura += all.get(dora_kind(wall(123 + 2 * i) >> 2));
    }
    w.dora = dora;
    w.ura = ura;
    w.reds = reds;
    w.double_yakuman = C.double_yakuman != 0;
    w.kazoe = C.kazoe != 0;
  }

  // engine.py:386-390: the cheap shanten test inline, the yaku search cold
  RS_HOT bool can_tsumo(int seat, const Hand& h) const {
    if (hi::shanten(h.info) != -1) return false;
    // a complete hand always has a reading (shanten -1 is exactly "some
    // standard / seven-pairs / orphans form"), and every reading carries a
    // yaku when the hand is in riichi, closed (menzen tsumo), drawn from the
    // dead wall (rinshan) or the last live tile (haitei): yaku.py:239-310,
    // :353-369 add those before any other; the search runs otherwise
    if (hi::riichi(h.info) || hi::nmelds(h.info) == 0 || g.rinshan_pending || g.live() == 0) return true;
    return tsumo_has_yaku(seat, h);
  }
  RS_COLD bool tsumo_has_yaku(int seat, const Hand& h) const {
    WinIn w;
    win_input(seat, h, g.drawn, true, false, w, false);
    Reading r;
    return score_win(w, r, true);
  }
  // engine.py:393-399 + types.py:93-100 (furiten): the wait / furiten
  // rejections inline (they decide almost every call), the yaku search cold
  RS_HOT bool can_ron(int seat, int tile, bool chankan) const {
    const uint32_t inf = info(seat);
    if (hi::shanten(inf) != 0) return false;
    const uint64_t wt = waits(seat);
    if (!((wt >> (tile >> 2)) & 1)) return false;
    if (hi::temp(inf) || hi::perm(inf)) return false;
    if (wt & sdword(bp, W_HRKIND + 2 * seat)) return false;
    // the tile completes the hand (it is a wait), so a reading exists; riichi,
    // chankan and houtei (last live tile) make every reading valid
    if (hi::riichi(inf) || chankan || g.live() == 0) return true;
    return ron_has_yaku(seat, tile, chankan);
  }
  RS_COLD bool ron_has_yaku(int seat, int tile, bool chankan) const {
    const Hand h = load_hand(bp, seat);
    WinIn w;
    win_input(seat, h, tile, false, chankan, w, false);
    Reading r;
    return score_win(w, r, true);
  }

  // --------------------------------------------------------- legality
  RS_HD bool kan_draw_ok() const { return g.live() >= 1 && g.kan_draws < 4; }

  // engine.py:230-246
  RS_HD void discard_bits(const Hand& h, bool only_tenpai, Mask115& m) const {
    uint64_t present = h.kinds_ge(1);
    if (only_tenpai) {
      // lane `sub` of the group takes held kinds sub, sub + G, ... (one
      // evaluation per lane and round: the same instructions, different kinds)
      const int G = grp_size(), sub = grp_sub();
      uint64_t keep = 0, p = present;
      for (int j = 0; j < sub && p; j++) p &= p - 1;  // drop the kinds of the lanes before
      while (p) {
        const int k = ctz64(p);
        if (shanten_minus_kind(T, h, k) == 0) keep |= 1ull << k;
        for (int j = 0; j < G && p; j++) p &= p - 1;  // this lane's next kind
      }
      present = grp_or64(keep);
    }
    uint64_t kinds = present;
    if (C.rule == RS_RULE_RED) {
      const int reds[3] = {16, 52, 88};
      for (int i = 0; i < 3; i++) {
        const int k = reds[i] >> 2;
        if (((present >> k) & 1) && h.has(reds[i])) {
          m.set(34 + i);
          if (h.count(k) <= 1) kinds &= ~(1ull << k);
        }
      }
    }
    m.m[0] |= (uint32_t)kinds;
    m.m[1] |= (uint32_t)(kinds >> 32) & 3u;
  }

  // engine.py:331-339
  RS_COLD bool kan_keeps_waits(const Hand& h, int kind) const {
    const int melds = hi::nmelds(h.info);
    Hand before = h;
    hand_take(T, before, before.lowest_of_kind(kind), -1);
    const uint64_t old = compute_waits(T, before, melds);
    Hand after = h;
    for (int j = 0; j < 4; j++) hand_take(T, after, after.lowest_of_kind(kind), -1);
    const uint64_t nw = compute_waits(T, after, melds + 1);
    return old == nw && !((old >> kind) & 1);
  }

  // engine.py:265-306
  RS_HD void legal_act(Mask115& m) const {
    const int seat = g.actor;
    const Hand h = load_hand(bp, seat);
    if (g.riichi_pending) { discard_bits(h, true, m); return; }
    if (hi::riichi(h.info)) {
      if (can_tsumo(seat, h)) m.set(A_TSUMO);
      const int kind = g.drawn >> 2;
      if (C.rule == RS_RULE_RED && is_red_tile(g.drawn)) m.set(34 + red_index_of_kind(kind));
      else m.set(kind);
      if (h.count(kind) == 4 && kan_draw_ok() && kan_keeps_waits(h, kind)) m.set(A_KAN_CLOSED + kind);
      return;
    }
    discard_bits(h, false, m);
    if (g.drawn < 0) return;
    const int nm = hi::nmelds(h.info);
    bool closed = true;
    uint64_t pon_kinds = 0;
    for (int i = 0; i < 4; i++)
      if (i < nm) {
        const uint32_t mf = meld_info(seat, i);
        if (mi::type(mf) != M_KAN_CLOSED) closed = false;
        if (mi::type(mf) == M_PON) pon_kinds |= 1ull << ((meld_tiles(seat, i) & 255) >> 2);
      }
    if (closed && g.scores[seat] >= 1000 && g.live() >= 4 && hi::shanten(h.info) <= 0) m.set(A_RIICHI);
    if (can_tsumo(seat, h)) m.set(A_TSUMO);
    if (kan_draw_ok()) {
      uint64_t quads = h.kinds_ge(4);
      while (quads) { const int k = ctz64(quads); quads &= quads - 1; m.set(A_KAN_CLOSED + k); }
      uint64_t adds = pon_kinds & h.kinds_ge(1);
      while (adds) { const int k = ctz64(adds); adds &= adds - 1; m.set(A_KAN_ADDED + k); }
    }
    if (C.rule == RS_RULE_RED && !g.any_call_made && hi::nriver(h.info) == 0 && nm == 0 &&
        popc64(h.kinds_ge(1) & ORPHAN_MASK) >= 9)
      m.set(A_NINE);
  }

  // engine.py:309-328
  RS_HD void legal_call(Mask115& m) const {
    const int seat = g.qseat(0), stage = g.qstage(0);
    const int kind = g.call_tile >> 2;
    m.set(A_PASS);
    if (stage == ST_RON) {
      m.set(A_RON);
    } else if (stage == ST_PONKAN) {
      m.set(A_PON);
      if (count_of(seat, kind) >= 3 && kan_draw_ok()) m.set(A_KAN_OPEN);
    } else {
      const uint32_t c = chi_bits(seat, kind);
      if (c & 1u) m.set(A_CHI_LOW);
      if (c & 2u) m.set(A_CHI_MID);
      if (c & 4u) m.set(A_CHI_HIGH);
    }
  }

  // engine.py:105-122 + 253-262
  RS_OL_LEGAL_Q void compute_legal(Mask115& m) const {
    m.clear();
    if (g.terminated || g.truncated) return;
    if (g.phase == PH_CALL) legal_call(m);
    else legal_act(m);
  }

  // ------------------------------------------------------ kyoku endings
  RS_HD rs_result_rec& result() const { return S.results[e]; }
  RS_COLD void begin_result(int kind) const {
    rs_result_rec& r = result();
    r.kyoku = g.kyoku;
    r.honba = g.honba;
    r.kind = kind;
    r.n_winners = 0;
    r.loser = -1;
    r.n_settlements = 0;
    r.tenpai_mask = 0;
  }
  RS_COLD void end_result() const {
    rs_result_rec& r = result();
    for (int s = 0; s < 4; s++) r.scores_after[s] = g.scores[s];
  }
  RS_COLD void write_win(int i, const Reading& rd, const WinIn& w) const { fill_win_rec(result().wins[i], rd, w); }


  RS_HD int final_kyoku() const { return C.mode == RS_MODE_SINGLE ? 0 : (C.mode == RS_MODE_EAST ? 3 : 7); }
  RS_HD void end_game() {
    g.phase = PH_GAME_END;
    g.terminated = 1;
    g.queue = 0;
  }
  // engine.py:842-872
  RS_COLD void advance_round(bool dealer_repeat, bool reset_honba) {
    g.n_results++;
    g.drawn = -1;
    if (dealer_repeat && g.repeats >= C.renchan_cap) dealer_repeat = false;
    if (dealer_repeat) g.repeats++;
    const bool bankrupt = g.scores[0] < 0 || g.scores[1] < 0 || g.scores[2] < 0 || g.scores[3] < 0;
    const int next_honba = reset_honba ? 0 : g.honba + 1;
    if (C.mode == RS_MODE_SINGLE || bankrupt) { end_game(); return; }
    if (dealer_repeat) {
      int leader = 0;
      for (int s = 1; s < 4; s++) if (g.scores[s] > g.scores[leader]) leader = s;
      if (g.kyoku == final_kyoku() && C.agari_yame && leader == g.dealer()) { end_game(); return; }
      g.honba = next_honba;
      start_kyoku();
      return;
    }
    if (g.kyoku + 1 > final_kyoku()) { end_game(); return; }
    g.kyoku++;
    g.honba = next_honba;
    start_kyoku();
  }
  RS_HD void clear_call() {
    g.call_tile = -1;
    g.call_from = -1;
    g.queue = 0;
    g.rons = 0;
    g.call_chankan = 0;
    g.kakan_kind = -1;
  }
  // engine.py:829-839
  RS_COLD void abort_kyoku(int kind) {
    #pragma unroll 1
    for (int s = 0; s < 4; s++)
      if (hi::riichi(info(s))) { g.scores[s] += 1000; g.deposits -= 1; }
    begin_result(kind);
    end_result();
    clear_call();
    advance_round(true, false);
  }
  // engine.py:810-826
  RS_COLD void exhaustive() {
    emit(EV_DRAW_END, -1, -1);
    int tmask = 0, n = 0;
    #pragma unroll 1
    for (int s = 0; s < 4; s++)
      if (hi::shanten(info(s)) == 0) { tmask |= 1 << s; n++; }
    int d[4] = {0, 0, 0, 0};
    if (n > 0 && n < 4) {
      const int gain = 3000 / n, loss = 3000 / (4 - n);
      #pragma unroll 1
      for (int s = 0; s < 4; s++) d[s] = ((tmask >> s) & 1) ? gain : -loss;
    }
    #pragma unroll 1
    for (int s = 0; s < 4; s++) g.scores[s] += d[s];
    begin_result(RS_RES_EXHAUSTIVE);
    rs_result_rec& r = result();
    r.tenpai_mask = tmask;
    r.n_settlements = 1;
    #pragma unroll 1
    for (int s = 0; s < 4; s++) r.deltas[0][s] = d[s];
    r.honba_component[0] = 0;
    r.deposits_claimed[0] = 0;
    end_result();
    advance_round((tmask >> g.dealer()) & 1, false);
  }
  // engine.py:764-779
  RS_COLD void apply_tsumo(int seat) {
    RS_WMARK(0);
    const Hand h = load_hand(bp, seat);
    WinIn w;
    win_input(seat, h, g.drawn, true, false, w);
    RS_WMARK(1);
    Reading rd;
    score_win(w, rd, false);
    RS_WMARK(2);
    begin_result(RS_RES_TSUMO);
    rs_result_rec& r = result();
    int deltas[4], hc;
    settle(true, rd.base, g.dealer(), seat, -1, g.honba, g.deposits, deltas, &hc);
    for (int s = 0; s < 4; s++) { r.deltas[0][s] = deltas[s]; g.scores[s] += deltas[s]; }
    r.honba_component[0] = hc;
    r.deposits_claimed[0] = g.deposits;
    r.n_winners = 1;
    r.winners[0] = (int8_t)seat;
    r.n_settlements = 1;
    write_win(0, rd, w);
    g.deposits = 0;
    emit(EV_TSUMO, seat, g.drawn);
    end_result();
    const int dealer = g.dealer();
    RS_WMARK(3);
    advance_round(seat == dealer, seat != dealer);
    RS_WMARK(4);
  }
  // engine.py:782-807
  RS_COLD void apply_ron_wins() {
    RS_WMARK(0);
    const int loser = g.call_from;
    const int nw = g.rn();
    int w4[3];
    #pragma unroll 1
    for (int i = 0; i < nw; i++) w4[i] = g.rseat(i);
    #pragma unroll 1
    for (int i = 1; i < nw; i++)
      #pragma unroll 1
      for (int j = i; j > 0 && ((w4[j - 1] - loser) & 3) > ((w4[j] - loser) & 3); j--) {
        const int t = w4[j]; w4[j] = w4[j - 1]; w4[j - 1] = t;
      }
    begin_result(RS_RES_RON);
    rs_result_rec& r = result();
    r.loser = loser;
    r.n_winners = nw;
    r.n_settlements = nw;
    const int dealer = g.dealer();
    bool dealer_won = false;
    #pragma unroll 1
    for (int i = 0; i < nw; i++) {
      const int seat = w4[i];
      r.winners[i] = (int8_t)seat;
      const Hand h = load_hand(bp, seat);
      WinIn w;
      win_input(seat, h, g.call_tile, false, g.call_chankan, w);
      RS_WMARK(1);
      Reading rd;
      score_win(w, rd, false);
      RS_WMARK(2);
      const int honba = i == 0 ? g.honba : 0, dep = i == 0 ? g.deposits : 0;
      int deltas[4], hc;
      settle(false, rd.base, dealer, seat, loser, honba, dep, deltas, &hc);
      #pragma unroll 1
      for (int s = 0; s < 4; s++) { r.deltas[i][s] = deltas[s]; g.scores[s] += deltas[s]; }
      r.honba_component[i] = hc;
      r.deposits_claimed[i] = dep;
      write_win(i, rd, w);
      emit(EV_RON, seat, g.call_tile);
      if (seat == dealer) dealer_won = true;
    }
    g.deposits = 0;
    end_result();
    clear_call();
    RS_WMARK(3);
    advance_round(dealer_won, !dealer_won);
    RS_WMARK(4);
  }

  // ------------------------------------------------------ call handling
  // engine.py:580-591
  RS_HD void mark_passed_furiten(int kind, int discarder) {
#pragma unroll
    for (int s = 0; s < 4; s++) {
      const uint32_t inf = info(s);
      // (the waits load for every seat: no branch on the shanten)
      const bool hit = s != discarder && hi::shanten(inf) == 0 && ((waits(s) >> kind) & 1);
      if (hit) set_info(s, hi::riichi(inf) ? hi::set_perm(inf, 1) : hi::set_temp(inf, 1));
    }
  }
  // engine.py:594-615
  RS_OL_STANDS_Q void discard_stands() {
    const int discarder = g.phase == PH_CALL ? g.call_from : g.actor;
    g.phase = PH_ACT;
    const uint32_t inf = info(discarder);
    if (hi::riichi(inf) && hi::riichi_index(inf) == hi::nriver(inf) - 1 && !hi::ippatsu(inf)) {
      set_info(discarder, hi::set_ippatsu(inf, 1));
      if (C.rule == RS_RULE_RED && hi::riichi(info(0)) && hi::riichi(info(1)) && hi::riichi(info(2)) &&
          hi::riichi(info(3))) {
        emit(EV_DRAW_END, discarder, -1);
        abort_kyoku(RS_RES_ABORT_FOUR_RIICHI);
        return;
      }
    }
    if (g.four_kan_pending && C.rule == RS_RULE_RED) {
      emit(EV_DRAW_END, discarder, -1);
      abort_kyoku(RS_RES_ABORT_FOUR_KAN);
      return;
    }
    g.call_tile = -1;
    g.call_from = -1;
    g.queue = 0;
    g.rons = 0;
    if (g.live() == 0) { exhaustive(); return; }
    draw((discarder + 1) & 3);
  }
  // engine.py:489-495
  RS_HD void reveal_pending_dora() {
    while (g.pending_dora > 0 && g.dora_count < 5) {
      g.dora_count++;
      g.pending_dora--;
      emit(EV_NEW_DORA, -1, wall(122 + 2 * (g.dora_count - 1)));
    }
    g.pending_dora = 0;
  }
  // the chi variants seat s could make with a discarded suit tile of
  // `kind` (bit 0 low, 1 mid, 2 high; engine.py:320-327): presence of kinds
  // kind-2 .. kind+2 from at most two words of the seat's tile set
  RS_HD uint32_t chi_bits(int s, int kind) const {
    const int n = kind % 9;
    const int base = kind >= 2 ? kind - 2 : 0, j = base >> 3;  // j <= 3 for a suit kind
    const uint64_t v = (uint64_t)sword(bp, W_HMASK + 5 * s + j) | ((uint64_t)sword(bp, W_HMASK + 5 * s + j + 1) << 32);
    const uint64_t x = v >> (4 * (base - 8 * j));
    const uint32_t pm = (uint32_t)((x | (x >> 1) | (x >> 2) | (x >> 3)) & 0x11111ull);  // a bit per nibble
    const int off = kind - base;  // kind's nibble in x
    // (branch-free: a shift below the window reads bit 0 and is masked off)
    auto has = [&](int d) -> uint32_t { return (pm >> (4 * (off + d > 0 ? off + d : 0))) & 1u; };
    const uint32_t lo = (uint32_t)(n <= 6) & has(1) & has(2);
    const uint32_t mid = (uint32_t)(n >= 1 && n <= 7) & has(-1) & has(1);
    const uint32_t hi = (uint32_t)(n >= 2) & has(-2) & has(-1);
    return lo | (mid << 1) | (hi << 2);
  }
  RS_HD bool can_chi(int s, int kind) const { return chi_bits(s, kind) != 0; }
  // engine.py:498-531
  RS_OL_CALL_Q bool begin_call_phase(int tile, int discarder, bool chankan) {
    const int kind = tile >> 2;
    // the queue is packed as it is built (Game::queue layout): no arrays,
    // so nothing goes through local memory
    uint32_t q = 0;
    int n = 0;
    auto push = [&](int s, int stage) {
      q |= ((uint32_t)s | ((uint32_t)stage << 2)) << (3 + 4 * n);
      n++;
    };
    // claims of the three opponents: bit 3 (off - 1) ron, + 1 pon / kan,
    // + 2 chi (the left seat only)
    const bool open_ok = !chankan && g.live() >= 1;
    auto claims_of = [&](int off) -> uint32_t {
      const int s = (discarder + off) & 3;
      uint32_t b = can_ron(s, tile, chankan) ? 1u : 0u;
      if (open_ok && !hi::riichi(info(s))) {
        if (count_of(s, kind) >= 2) b |= 2u;
        if (off == 1 && kind < 27 && can_chi(s, kind)) b |= 4u;
      }
      return b << (3 * (off - 1));
    };
    uint32_t claims = 0;
    if (RS_CLAIM_LANES_ON && grp_size() >= 4) {
      // lane group: lanes 1-3 of the env's group check one opponent each
      // and the group combines the claim bits with one warp reduction
      const int sub = grp_sub();
      claims = grp_or32(sub >= 1 && sub <= 3 ? claims_of(sub) : 0u);
    } else {
      claims = claims_of(1) | claims_of(2) | claims_of(3);
    }
    // queue order (engine.py:498-531): rons from the discarder's right,
    // then pon / kan in seat order, then chi
    for (int off = 1; off <= 3; off++)
      if ((claims >> (3 * (off - 1))) & 1u) push((discarder + off) & 3, ST_RON);
    for (int off = 1; off <= 3; off++)
      if ((claims >> (3 * (off - 1) + 1)) & 1u) push((discarder + off) & 3, ST_PONKAN);
    if (claims & 4u) push((discarder + 1) & 3, ST_CHI);
    if (!n) return false;
    g.phase = PH_CALL;
    g.call_tile = tile;
    g.call_from = discarder;
    g.queue = q | (uint32_t)n;
    g.rons = 0;
    g.call_chankan = chankan;
    g.actor = (int)((q >> 3) & 3);
    return true;
  }

  // engine.py:447-455
  RS_HD int pick_discard(const Hand& h, int action) const {
    const int kind = action < 34 ? action : (action == 34 ? 4 : action == 35 ? 13 : 22);
    const bool want_red = action >= 34;
    const bool red_rule = C.rule == RS_RULE_RED;
    // both candidates computed and selected (no branch)
    const bool drawn_ok = g.drawn >= 0 && (g.drawn >> 2) == kind && (red_rule && is_red_tile(g.drawn)) == want_red;
    uint32_t nib = h.nibble(kind);
    const uint32_t keep = want_red ? 1u : ~1u;
    nib = (red_rule && red_index_of_kind(kind) >= 0) ? (nib & keep) : nib;
    return drawn_ok ? g.drawn : 4 * kind + ctz32(nib);
  }
  // engine.py:458-486
  RS_HD void apply_discard(int seat, int action) {
    Hand h = load_hand(bp, seat);
    const int tile = pick_discard(h, action);
    const bool tsumogiri = tile == g.drawn;
    const bool declaring = g.riichi_pending;
    int riichi_val = hi::riichi(h.info), riichi_index = hi::riichi_index(h.info);
    const int nriver = hi::nriver(h.info);
    if (declaring) {
      riichi_val = (nriver == 0 && !g.any_call_made) ? 2 : 1;
      riichi_index = nriver;
      g.riichi_pending = 0;
    }
    int ipp = hi::ippatsu(h.info);
    if (hi::riichi(h.info) && !declaring && ipp) ipp = 0;
    RS_CHECK((unsigned)seat < 4u && (unsigned)nriver < (unsigned)RS_MAX_RIVER);
    S.river[at(seat * RS_MAX_RIVER + nriver)] =
        (uint16_t)(tile | ((tsumogiri ? RS_RIVER_TSUMOGIRI : 0) | (declaring ? RS_RIVER_RIICHI : 0)) << 8);
    sdword(bp, W_HRKIND + 2 * seat) |= 1ull << (tile >> 2);
    hand_take(T, h, tile, tok());
    h.info = hi::set_nriver(h.info, nriver + 1);
    h.info = hi::set_riichi(h.info, riichi_val);
    h.info = hi::set_riichi_index(h.info, riichi_index);
    h.info = hi::set_ippatsu(h.info, ipp);
    finish_hand(T, h);
    RS_SMARK(1);
    store_hand(bp, seat, h);
    g.drawn = -1;
    g.rinshan_pending = 0;
    emit(EV_DISCARD, seat, tile);
    reveal_pending_dora();
    if (!begin_call_phase(tile, seat, false)) {
      mark_passed_furiten(tile >> 2, seat);
      RS_SMARK(2);
      discard_stands();
      RS_SMARK(3);
    }
  }

  RS_HD void clear_all_ippatsu() {
    for (int s = 0; s < 4; s++) {
      const uint32_t inf = info(s);
      if (hi::ippatsu(inf)) set_info(s, hi::set_ippatsu(inf, 0));
    }
  }
  // engine.py:631-636
  RS_HD void mark_called_tile() {
    const int d = g.call_from;
    const int idx = hi::nriver(info(d)) - 1;
    RS_CHECK((unsigned)d < 4u && (unsigned)idx < (unsigned)RS_MAX_RIVER);
    uint16_t& rt = S.river[at(d * RS_MAX_RIVER + idx)];
    rt = (uint16_t)(rt | (RS_RIVER_CALLED << 8));
  }
  // engine.py:639-644
  RS_COLD void check_four_kans() {
    if (C.rule != RS_RULE_RED) return;
    int total = 0, seats = 0;
    #pragma unroll 1
    for (int s = 0; s < 4; s++) {
      const int nm = hi::nmelds(info(s));
      int c = 0;
      #pragma unroll 1
      for (int i = 0; i < 4; i++)
        if (i < nm && mi::type(meld_info(s, i)) >= M_KAN_OPEN) c++;
      total += c;
      if (c) seats++;
    }
    if (total == 4 && seats >= 2) g.four_kan_pending = 1;
  }
  // append a meld of sorted ids (melds.py:17-34)
  RS_HD void add_meld(int seat, Hand& h, int type, const int* ids, int nids, int called, int from) {
    int t[4];
    #pragma unroll 1
    for (int i = 0; i < nids; i++) t[i] = ids[i];
    #pragma unroll 1
    for (int i = 1; i < nids; i++)
      #pragma unroll 1
      for (int j = i; j > 0 && t[j - 1] > t[j]; j--) { const int x = t[j]; t[j] = t[j - 1]; t[j - 1] = x; }
    uint32_t packed = 0;
    #pragma unroll 1
    for (int i = 0; i < nids; i++) packed |= (uint32_t)t[i] << (8 * i);
    const int nm = hi::nmelds(h.info);
    RS_CHECK((unsigned)seat < 4u && (unsigned)nm < 4u && nids >= 3 && nids <= 4);
    sword(bp, W_MELD + 2 * (4 * seat + nm)) = packed;
    sword(bp, W_MELD + 2 * (4 * seat + nm) + 1) = mi::make(type, nids, from, called);
    h.info = hi::set_nmelds(h.info, nm + 1);
  }
  // engine.py:696-702
  RS_HD void finish_meld_call(int seat) {
    g.any_call_made = 1;
    clear_all_ippatsu();
    g.phase = PH_ACT;
    g.actor = seat;
    g.drawn = -1;
    g.rinshan_pending = 0;
  }
  // engine.py:647-693 (pon / chi / open kan share the claim prologue)
  RS_COLD void apply_claim(int seat, int action) {
    const int kind = g.call_tile >> 2;
    mark_passed_furiten(kind, g.call_from);
    mark_called_tile();
    Hand h = load_hand(bp, seat);
    int ids[4], n = 0;
    if (action == A_PON || action == A_KAN_OPEN) {
      const int need = action == A_PON ? 2 : 3;
      uint32_t nib = h.nibble(kind);
      #pragma unroll 1
      for (int j = 0; j < need; j++) { const int b = ctz32(nib); nib &= nib - 1; ids[n++] = 4 * kind + b; }
    } else {
      int k0, k1;
      if (action == A_CHI_LOW) { k0 = kind + 1; k1 = kind + 2; }
      else if (action == A_CHI_MID) { k0 = kind - 1; k1 = kind + 1; }
      else { k0 = kind - 2; k1 = kind - 1; }
      ids[n++] = h.lowest_of_kind(k0);
      ids[n++] = h.lowest_of_kind(k1);
    }
    #pragma unroll 1
    for (int j = 0; j < n; j++) hand_take(T, h, ids[j], tok());
    ids[n] = g.call_tile;
    const int type = action == A_PON ? M_PON : (action == A_KAN_OPEN ? M_KAN_OPEN : M_CHI);
    add_meld(seat, h, type, ids, n + 1, g.call_tile, g.call_from);
    finish_hand(T, h);
    const int called = g.call_tile;
    if (action == A_KAN_OPEN) {
      store_hand(bp, seat, h);
      g.any_call_made = 1;
      clear_all_ippatsu();
      g.pending_dora++;
      emit(EV_KAN_OPEN, seat, called);
      clear_call();
      check_four_kans();
      h.info = info(seat);  // ippatsu may have been cleared above
      rinshan_draw(seat, h);
      return;
    }
    store_hand(bp, seat, h);
    finish_meld_call(seat);
    emit(action == A_PON ? EV_PON : EV_CHI, seat, called);
    clear_call();
  }
  // engine.py:714-727
  RS_COLD void apply_closed_kan(int seat, int kind) {
    Hand h = load_hand(bp, seat);
    int ids[4];
    uint32_t nib = h.nibble(kind);
    #pragma unroll 1
    for (int j = 0; j < 4; j++) { ids[j] = 4 * kind + ctz32(nib); nib &= nib - 1; }
    #pragma unroll 1
    for (int j = 0; j < 4; j++) hand_take(T, h, ids[j], tok());
    add_meld(seat, h, M_KAN_CLOSED, ids, 4, -1, -1);
    finish_hand(T, h);
    store_hand(bp, seat, h);
    g.any_call_made = 1;
    clear_all_ippatsu();
    g.dora_count = g.dora_count + 1 < 5 ? g.dora_count + 1 : 5;
    emit(EV_KAN_CLOSED, seat, ids[0]);
    emit(EV_NEW_DORA, -1, wall(122 + 2 * (g.dora_count - 1)));
    check_four_kans();
    h.info = info(seat);
    rinshan_draw(seat, h);
  }
  // engine.py:742-758
  RS_COLD void complete_added_kan(int seat, int kind) {
    Hand h = load_hand(bp, seat);
    const int tile = h.lowest_of_kind(kind);
    const int nm = hi::nmelds(h.info);
    #pragma unroll 1
    for (int i = 0; i < 4; i++)
      if (i < nm) {
        const uint32_t mf = meld_info(seat, i), mt = meld_tiles(seat, i);
        if (mi::type(mf) == M_PON && ((mt & 255) >> 2) == kind) {
          int t[4] = {(int)(mt & 255), (int)((mt >> 8) & 255), (int)((mt >> 16) & 255), tile};
          #pragma unroll 1
          for (int a = 1; a < 4; a++)
            #pragma unroll 1
            for (int b = a; b > 0 && t[b - 1] > t[b]; b--) { const int x = t[b]; t[b] = t[b - 1]; t[b - 1] = x; }
          sword(bp, W_MELD + 2 * (4 * seat + i)) = (uint32_t)t[0] | ((uint32_t)t[1] << 8) | ((uint32_t)t[2] << 16) |
                                       ((uint32_t)t[3] << 24);
          sword(bp, W_MELD + 2 * (4 * seat + i) + 1) = mi::make(M_KAN_ADDED, 4, mi::from(mf), mi::called(mf));
        }
      }
    hand_take(T, h, tile, tok());
    finish_hand(T, h);
    store_hand(bp, seat, h);
    g.any_call_made = 1;
    clear_all_ippatsu();
    g.pending_dora++;
    clear_call();
    check_four_kans();
    h.info = info(seat);
    rinshan_draw(seat, h);
  }
  // engine.py:730-739
  RS_COLD void apply_added_kan(int seat, int kind) {
    const int tile = 4 * kind + ctz32((sword(bp, W_HMASK + 5 * seat + (kind >> 3)) >> ((kind & 7) * 4)) & 0xFu);
    emit(EV_KAN_ADDED, seat, tile);
    if (begin_call_phase(tile, seat, true)) { g.kakan_kind = kind; return; }
    mark_passed_furiten(kind, seat);
    complete_added_kan(seat, kind);
  }
  // engine.py:561-577
  RS_COLD void resolve_call_end() {
    if (g.rn()) {
      if (g.rn() >= 3 && C.rule == RS_RULE_RED) {
        emit(EV_DRAW_END, g.call_from, -1);
        abort_kyoku(RS_RES_ABORT_TRIPLE_RON);
        return;
      }
      apply_ron_wins();
      return;
    }
    mark_passed_furiten(g.call_tile >> 2, g.call_from);
    if (g.call_chankan) {
      const int seat = g.call_from;
      g.call_chankan = 0;
      g.phase = PH_ACT;
      g.actor = seat;
      complete_added_kan(seat, g.kakan_kind);
      return;
    }
    discard_stands();
  }
  // engine.py:552-558
  RS_HD void advance_call_queue() {
    if (g.rn()) {
      uint32_t q = 0;
      int n = 0;
      for (int i = 0; i < g.qn(); i++)
        if (g.qstage(i) == ST_RON) {
          q |= ((uint32_t)g.qseat(i) | ((uint32_t)ST_RON << 2)) << (3 + 4 * n);
          n++;
        }
      g.queue = q | (uint32_t)n;
    }
    if (g.qn()) { g.actor = g.qseat(0); return; }
    resolve_call_end();
  }
  // engine.py:534-549
  RS_HD void apply_call_action(int action) {
    const int seat = g.qseat(0);
    g.qpop();
    if (action == A_RON) { g.rpush(seat); advance_call_queue(); }
    else if (action == A_PASS) advance_call_queue();
    else apply_claim(seat, action);
  }
  // engine.py:425-444
  RS_HD void apply_turn_action(int action) {
    const int seat = g.actor;
    if (action <= 36) apply_discard(seat, action);
    else if (action == A_RIICHI) {
      g.scores[seat] -= 1000;
      g.deposits += 1;
      g.riichi_pending = 1;
      emit(EV_RIICHI, seat, -1);
    } else if (action == A_TSUMO) apply_tsumo(seat);
    else if (action < A_KAN_ADDED) apply_closed_kan(seat, action - A_KAN_CLOSED);
    else if (action < A_PASS) apply_added_kan(seat, action - A_KAN_ADDED);
    else {
      emit(EV_DRAW_END, seat, -1);
      abort_kyoku(RS_RES_ABORT_NINE);
    }
  }

  // ------------------------------------------------------------ env API
  RS_HD void store_legal(const Mask115& m) const {
    for (int i = 0; i < 4; i++) sword(bp, W_LEGAL + i) = m.m[i];
  }
  RS_HD Mask115 load_legal() const {
    Mask115 m;
    for (int i = 0; i < 4; i++) m.m[i] = sword(bp, W_LEGAL + i);
    return m;
  }
  // env/core.py:81-94 (_wrap, _terminal_rewards) -> rewards into r[4]
  RS_HD void wrap(float* r) {
    g.current_player = g.actor;
    g.env_terminated = g.terminated;
    g.env_truncated = g.truncated;
    if (g.terminated || g.truncated) terminal_rewards(r);
    else r[0] = r[1] = r[2] = r[3] = 0.0f;
  }
  RS_COLD void terminal_rewards(float* r) const {  // game end only
    if (C.reward_scheme == RS_REWARD_RANK) {
      const double RR[4] = {1.0, 0.333, -0.333, -1.0};
      #pragma unroll 1
      for (int s = 0; s < 4; s++) {
        int rank = 0;
        #pragma unroll 1
        for (int t = 0; t < 4; t++)
          if (g.scores[t] > g.scores[s] || (g.scores[t] == g.scores[s] && t < s)) rank++;
        r[s] = (float)RR[rank];
      }
    } else {
      #pragma unroll 1
      for (int s = 0; s < 4; s++) r[s] = (float)((double)(g.scores[s] - 25000) / 25000.0);
    }
  }
  // current rewards of a stored env (illegal penalty or terminal rewards)
  RS_HD void current_rewards(float* r) const {
    if (g.status & RS_STATUS_ILLEGAL) {
      r[0] = r[1] = r[2] = r[3] = 0.0f;
      r[g.current_player] = C.illegal_penalty;
    } else if (g.env_terminated || g.env_truncated) {
      terminal_rewards(r);
    } else {
      r[0] = r[1] = r[2] = r[3] = 0.0f;
    }
  }

  // engine.py:128-136 + core.py:81-82: fresh game from `seed`; rollout
  // keys (env_key, policy stream, resets) are preserved
  RS_HD void init_game(uint64_t seed, float* r) {
    RS_ACC(5);
    {
      const uint64_t ek = g.env_key, pk = g.policy_key, pc = g.policy_counter;
      const uint32_t rs = g.resets;
      g = Game{};
      g.env_key = ek; g.policy_key = pk; g.policy_counter = pc; g.resets = rs;
    }
    g.phase = PH_ACT; g.actor = 0; g.kyoku = 0;
    g.terminated = g.truncated = 0;
    g.env_terminated = g.env_truncated = 0;
    g.status = 0;
    g.honba = g.deposits = g.repeats = g.n_results = 0;
    g.step_count = 0;
    g.events_len = 0;
    g.drawn = -1;
    for (int s = 0; s < 4; s++) g.scores[s] = 25000;
    g.rng_key = mix64(seed);
    g.rng_counter = 0;
    RS_MARK(1);
    start_kyoku();
    Mask115 m;
    compute_legal(m);
    RS_MARK(5);
    store_legal(m);
    wrap(r);
  }

  // env/core.py:85-94 + engine.py:405-422.  Returns status bits.
  RS_HD int step(int action, Mask115& legal, float* r) {
    RS_ACC(0);
    if (g.env_terminated || g.env_truncated) {
      // contract violation: nothing changes (core.py:87-88 raises)
      legal.clear();
      current_rewards(r);
      return RS_STATUS_CONTRACT;
    }
    legal = load_legal();
    if (action < 0 || action >= RS_NUM_ACTIONS || !legal.test(action)) {
      r[0] = r[1] = r[2] = r[3] = 0.0f;
      r[g.current_player] = C.illegal_penalty;
      g.env_terminated = 1;
      g.env_truncated = 0;
      g.status = RS_STATUS_ILLEGAL;
      legal.clear();
      // the stored mask is the game's cached list; the env view is empty
      return RS_STATUS_ILLEGAL;
    }
    g.status = 0;
    g.step_count++;
    if (g.phase == PH_CALL) apply_call_action(action);
    else apply_turn_action(action);
    if (!g.terminated && g.step_count >= (uint32_t)C.max_steps) g.truncated = 1;
    RS_SMARK(4);
    compute_legal(legal);
    RS_SMARK(5);
    store_legal(legal);
    wrap(r);
    return 0;
  }

  // env/policies.py:51-109 (heuristic_policy).  The reference rebuilds the
  // current player's counts from its observation tokens and finds the
  // called tile as the last discard / added-kan event of the window; here
  // both come from the state: the concealed set of the actor and call_tile.
  RS_HD int heuristic_action(const Mask115& legal) const {
    if (legal.test(A_TSUMO)) return A_TSUMO;
    if (legal.test(A_RON)) return A_RON;
    if (legal.test(A_RIICHI)) return A_RIICHI;
    const Hand h = load_hand(bp, g.current_player);
    const int n = h.ntiles();
    const int melds = n % 3 == 2 ? (14 - n) / 3 : (13 - n) / 3;  // policies.py:34-35
    // discards (policies.py:67-78): minimise (shanten, honor/terminal/other,
    // kind, red) over the legal discard ids
    const uint64_t disc = (uint64_t)legal.m[0] | ((uint64_t)(legal.m[1] & 0x1Fu) << 32);
    if (disc) {
      int best_a = -1;
      uint32_t best_key = 0xFFFFFFFFu;
      uint64_t d = disc;
      while (d) {
        const int a = ctz64(d);
        d &= d - 1;
        const int kind = a < 34 ? a : (a == 34 ? 4 : a == 35 ? 13 : 22);
        Hand x = h;
        hand_take(T, x, x.lowest_of_kind(kind), -1);
        const int sh = full_shanten(T, x, melds);
        const uint32_t cls = kind >= 27 ? 0u : (is_terminal(kind) ? 1u : 2u);
        const uint32_t key = ((uint32_t)(sh + 1) << 9) | (cls << 7) | ((uint32_t)kind << 1) | (a >= 34 ? 1u : 0u);
        if (key < best_key) { best_key = key; best_a = a; }
      }
      return best_a;
    }
    // calls (policies.py:80-107): the first call (ascending ids) reaching
    // the lowest shanten, only when strictly below the current one
    if (legal.test(A_PASS)) {
      const int current = full_shanten(T, h, melds);
      const int ck = g.call_tile >> 2;
      int best_call = -1, best_sh = 0;
      for (int a = A_PON; a <= A_KAN_OPEN; a++) {
        if (!legal.test(a)) continue;
        Hand x = h;
        const int take = a == A_PON ? 2 : (a == A_KAN_OPEN ? 3 : 0);
        for (int j = 0; j < take; j++) hand_take(T, x, x.lowest_of_kind(ck), -1);
        if (a == A_CHI_LOW) { hand_take(T, x, x.lowest_of_kind(ck + 1), -1); hand_take(T, x, x.lowest_of_kind(ck + 2), -1); }
        if (a == A_CHI_MID) { hand_take(T, x, x.lowest_of_kind(ck - 1), -1); hand_take(T, x, x.lowest_of_kind(ck + 1), -1); }
        if (a == A_CHI_HIGH) { hand_take(T, x, x.lowest_of_kind(ck - 2), -1); hand_take(T, x, x.lowest_of_kind(ck - 1), -1); }
        const int sh = full_shanten(T, x, melds + 1);
        if (sh < current && (best_call < 0 || sh < best_sh)) { best_sh = sh; best_call = a; }
      }
      return best_call >= 0 ? best_call : A_PASS;
    }
    return legal.nth(0);
  }

  // env/policies.py:17-22 over the env-view mask
  RS_HD int random_action(const Mask115& legal) {
    RS_ACC(6);
    const int n = legal.count();
    g.policy_counter++;
    const int i = (int)randbelow_from(stream_value(g.policy_key, g.policy_counter), (uint32_t)n);
    return legal.nth(i);
  }
};

}  // namespace rs
