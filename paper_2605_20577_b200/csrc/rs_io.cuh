// rs_io.cuh — observation encoding, trajectory digest and record import /
// export for one env (device code, also usable on host memory).
#pragma once

#include "rs_engine.cuh"

namespace rs {

// tile token (observe.py:43-46)
RS_HD int tile_token(int t, int rule) {
  if (rule == RS_RULE_RED && is_red_tile(t)) return 34 + red_index_of_kind(t >> 2);
  return t >> 2;
}
RS_HD int ev_token(int type) { return type <= 8 ? type : type - 1; }  // win events merge (observe.py:26-39)

// four window slots (event words, rs_engine.cuh event_word) as observer
// `seat` sees them, packed as write_obs emits them: 4 x (type token,
// relative actor, visible tile token) in 3 words.  Byte-parallel: the
// slots' bytes are gathered into one word per field and decoded four at a
// time (~5.5 instructions per slot instead of ~12).
RS_HD void view4(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3, int seat, uint32_t& w0, uint32_t& w1,
                 uint32_t& w2) {
  const uint32_t p = byte_perm(x0, x1, 0x5140), q = byte_perm(x2, x3, 0x5140);
  const uint32_t b0 = byte_perm(p, q, 0x5410), b1 = byte_perm(p, q, 0x7632);
  const uint32_t b2 = byte_perm(byte_perm(x0, x1, 0x7362), byte_perm(x2, x3, 0x7362), 0x5410);
  const uint32_t ty = b0 & 0x0F0F0F0Fu;
  const uint32_t hid = (b0 >> (4 + seat)) & 0x01010101u;
  const uint32_t rel = (b1 >> (2 * seat)) & 0x03030303u;
  const uint32_t m = hid * 0xFFu;  // 0x00 / 0xFF per byte
  const uint32_t tok = ((b2 & 0x3F3F3F3Fu) & ~m) | (0x25252525u & m);  // hidden: 37
  const uint32_t yr = byte_perm(ty, rel, 0x5140), yr2 = byte_perm(ty, rel, 0x7362);
  w0 = byte_perm(yr, tok, 0x2410);                          // y0 r0 t0 y1
  w1 = byte_perm(byte_perm(yr, tok, 0x0053), yr2, 0x5410);  // r1 t1 y2 r2
  w2 = byte_perm(tok, yr2, 0x3762);                         // t2 y3 r3 t3
}

// observe(state, seat) (observe.py:81-124), written into slot `o` of `obs`
RS_HD void write_obs(const Engine& E, int seat, const rs_obs_out& obs, int64_t o) {
  RS_ACC(4);
  const Soa& S = E.S;
  const Game& g = E.g;
  const int rule = E.C.rule;
  const Hand h = load_hand(E.bp, seat);
  // every block read of the observation before its first store (the output
  // stores could alias the block as far as the compiler knows)
  const uint32_t inf0 = E.info(seat), inf1 = E.info((seat + 1) & 3), inf2 = E.info((seat + 2) & 3),
                 inf3 = E.info((seat + 3) & 3);
  const uint32_t* wall_w = reinterpret_cast<const uint32_t*>(swall(E.bp));
  const uint32_t dw0 = wall_w[30], dw1 = wall_w[31], dw2 = wall_w[32];  // wall bytes 120..131
  if (obs.hand_tokens) {
    // sorted tokens (kinds ascending, then the held red fives 34..36), padded
    // with 37: the hand keeps them sorted incrementally (rs_hand.cuh
    // tok_insert / tok_remove); written as 7 u16 stores
    const uint64_t lo = h.tlo, hi8 = h.thi;
    uint16_t* ht = reinterpret_cast<uint16_t*>(obs.hand_tokens + o * 14);
    ht[0] = (uint16_t)lo; ht[1] = (uint16_t)(lo >> 16); ht[2] = (uint16_t)(lo >> 32); ht[3] = (uint16_t)(lo >> 48);
    ht[4] = (uint16_t)hi8; ht[5] = (uint16_t)(hi8 >> 16); ht[6] = (uint16_t)(hi8 >> 32);
  }
  if (obs.event_tokens) {
    // 64 x (type, rel actor, token), oldest first, padded (0,0,37): slot i
    // of the window is ring entry (len + i) & 63 seen by this observer,
    // pads while i < 64 - len; 4 slots decode and pack into 3 words at a
    // time (view4)
    const uint32_t* ring = S.events + (uint32_t)E.e * RS_EVENT_WINDOW;
    const uint32_t len = g.events_len;
    const int pad = len >= 64u ? 0 : 64 - (int)len;
    uint4* dst = reinterpret_cast<uint4*>(obs.event_tokens + o * 192);
    // four quarters of 16 slots, each loaded completely before its stores
    // (stores to the output could alias the ring as far as the compiler
    // knows); with a lane group, lanes 0-3 of the group take one quarter
    // each -- the same instructions on different data, so the warp runs
    // the quarter body once
    const int G = grp_size(), sub = grp_sub();
    // slot i: ring entry (len + i) & 63, or a pad while i < pad (also right
    // when len < 64: (len + i) & 63 = i - pad)
    auto ev = [&](int i) -> uint32_t { return i < pad ? EVENT_PAD : ring[(len + (uint32_t)i) & 63u]; };
    if (G >= 8 && RS_WIN16) {
      // 8+ lanes per env: lane `sub` encodes slots [per * sub, per * (sub + 1))
      // (per = 4 at 16+ lanes, 8 at 8), stored as u32 -- the group's stores
      // form one 192-byte burst
      const int L = G >= 16 ? 16 : 8, per = 64 / L;
      if (sub < L) {
        uint32_t* d32 = reinterpret_cast<uint32_t*>(obs.event_tokens + o * 192) + sub * (3 * per / 4);
        for (int c = 0; c < per; c += 4) {
          const int i0 = per * sub + c;
          uint32_t w0, w1, w2;
          view4(ev(i0), ev(i0 + 1), ev(i0 + 2), ev(i0 + 3), seat, w0, w1, w2);
          d32[3 * c / 4] = w0;
          d32[3 * c / 4 + 1] = w1;
          d32[3 * c / 4 + 2] = w2;
        }
      }
    } else {
      // four quarters of 16 slots, each loaded completely before its stores
      // (stores to the output could alias the ring as far as the compiler
      // knows); with 2 or 4 lanes, lane `sub` takes quarters sub, sub + G
      for (int q = sub; q < 4; q += G) {
        uint32_t v[16];
#pragma unroll
        for (int j = 0; j < 16; j++) v[j] = ev(16 * q + j);
        uint32_t w[12];
#pragma unroll
        for (int r = 0; r < 4; r++) view4(v[4 * r], v[4 * r + 1], v[4 * r + 2], v[4 * r + 3], seat, w[3 * r], w[3 * r + 1], w[3 * r + 2]);
        uint4* d = dst + 3 * q;
        d[0] = make_uint4(w[0], w[1], w[2], w[3]);
        d[1] = make_uint4(w[4], w[5], w[6], w[7]);
        d[2] = make_uint4(w[8], w[9], w[10], w[11]);
      }
    }
  }
  if (obs.shanten) obs.shanten[o] = (int8_t)hi::shanten(h.info);
  if (obs.scores)
    for (int i = 0; i < 4; i++) {
      const int s = g.scores[(seat + i) & 3];
      obs.scores[o * 4 + i] = (int16_t)(s >= 0 ? s / 100 : -((-s + 99) / 100));  // floor division
    }
  if (obs.round_wind) obs.round_wind[o] = (uint8_t)g.round_wind();
  if (obs.seat_wind) obs.seat_wind[o] = (uint8_t)g.seat_wind(seat);
  if (obs.kyoku) obs.kyoku[o] = (uint8_t)g.kyoku;
  if (obs.honba) obs.honba[o] = (int16_t)g.honba;
  if (obs.deposits) obs.deposits[o] = (int16_t)g.deposits;
  if (obs.dora_tokens) {
    // indicators at wall positions 122, 124, ..., 130 (tiles.py:118-144)
    const int ind[5] = {(int)(dw0 >> 16) & 255, (int)dw1 & 255, (int)(dw1 >> 16) & 255, (int)dw2 & 255,
                        (int)(dw2 >> 16) & 255};
#pragma unroll
    for (int i = 0; i < 5; i++) obs.dora_tokens[o * 5 + i] = (uint8_t)(i < g.dora_count ? tile_token(ind[i], rule) : 37);
  }
  if (obs.live_wall) obs.live_wall[o] = (uint8_t)g.live();
  if (obs.riichi_flags) {
    obs.riichi_flags[o * 4 + 0] = (uint8_t)(hi::riichi(inf0) ? 1 : 0);
    obs.riichi_flags[o * 4 + 1] = (uint8_t)(hi::riichi(inf1) ? 1 : 0);
    obs.riichi_flags[o * 4 + 2] = (uint8_t)(hi::riichi(inf2) ? 1 : 0);
    obs.riichi_flags[o * 4 + 3] = (uint8_t)(hi::riichi(inf3) ? 1 : 0);
  }
}

// trajectory digest (identical to oracle/mjoracle.c orc_digest_step)
RS_HD uint64_t dfold(uint64_t d, uint64_t w) { return mix64((d ^ w) + GOLDEN); }
RS_HD uint64_t digest_step(uint64_t d, int action, const Engine& E, const Mask115& view, const float* r) {
  const Game& g = E.g;
  d = dfold(d, (uint64_t)(uint32_t)action);
  d = dfold(d, (uint64_t)(uint32_t)g.current_player | ((uint64_t)g.env_terminated << 8) |
                   ((uint64_t)g.env_truncated << 9) | ((uint64_t)g.phase << 12) |
                   ((uint64_t)(uint32_t)g.kyoku << 16) | ((uint64_t)(uint32_t)g.honba << 24) |
                   ((uint64_t)(uint32_t)g.deposits << 40));
  d = dfold(d, (uint64_t)view.m[0] | ((uint64_t)view.m[1] << 32));
  d = dfold(d, (uint64_t)view.m[2] | ((uint64_t)view.m[3] << 32));
  for (int s = 0; s < 4; s += 2)
    d = dfold(d, (uint64_t)(uint32_t)g.scores[s] | ((uint64_t)(uint32_t)g.scores[s + 1] << 32));
  uint32_t rb[4];
  for (int i = 0; i < 4; i++) {
    union { float f; uint32_t u; } cv;
    cv.f = r[i];
    rb[i] = cv.u;
  }
  d = dfold(d, (uint64_t)rb[0] | ((uint64_t)rb[1] << 32));
  d = dfold(d, (uint64_t)rb[2] | ((uint64_t)rb[3] << 32));
  uint64_t sh = 0;
  for (int s = 0; s < 4; s++) sh |= (uint64_t)(uint8_t)(int8_t)hi::shanten(E.info(s)) << (8 * s);
  sh |= (uint64_t)g.events_len << 32;
  d = dfold(d, sh);
  d = dfold(d, (uint64_t)(uint32_t)g.cursor | ((uint64_t)(uint32_t)g.kan_draws << 8) |
                   ((uint64_t)(uint32_t)g.dora_count << 16) | ((uint64_t)g.step_count << 32));
  return d;
}

// The wide part of the trajectory digest (identical to oracle/mjoracle.c
// o_digest_state / o_digest_obs): every state field of the env, folded in
// a canonical form after every step -- the four hands (136-bit concealed
// sets, HandState flags and waits, melds, river entries with their flags),
// the call state, the game and policy RNGs, the whole wall, the newest
// events and the last kyoku result with its win details
// (engine/types.py:72-179, engine/state.py:191-242) -- and the observation
// of the current player exactly as write_obs encodes it (observe.py:81-124).
RS_HD uint64_t dpack4(uint32_t a, uint32_t b, uint32_t c, uint32_t e) {
  return (uint64_t)(a & 0xFFFFu) | ((uint64_t)(b & 0xFFFFu) << 16) | ((uint64_t)(c & 0xFFFFu) << 32) |
         ((uint64_t)(e & 0xFFFFu) << 48);
}
RS_COLD uint64_t digest_state(uint64_t d, const Engine& E) {
  const Soa& S = E.S;
  const Game& g = E.g;
  for (int s = 0; s < 4; s++) {
    const Hand h = load_hand(E.bp, s);
    d = dfold(d, (uint64_t)h.w0 | ((uint64_t)h.w1 << 32));
    d = dfold(d, (uint64_t)h.w2 | ((uint64_t)h.w3 << 32));
    d = dfold(d, (uint64_t)(h.w4 & 0xFFu));
    const uint32_t inf = h.info;
    const int nm = hi::nmelds(inf), nr = hi::nriver(inf);
    d = dfold(d, (uint64_t)hi::riichi(inf) | ((uint64_t)(hi::riichi_index(inf) + 1) << 2) |
                     ((uint64_t)hi::ippatsu(inf) << 8) | ((uint64_t)hi::temp(inf) << 9) |
                     ((uint64_t)hi::perm(inf) << 10) | ((uint64_t)nm << 12) | ((uint64_t)nr << 16) |
                     ((uint64_t)hi::nconc(inf) << 24) | (E.waits(s) << 30));
    for (int i = 0; i < nm; i++) {
      const uint32_t mf = E.meld_info(s, i), mt = E.meld_tiles(s, i);
      const int nt = mi::ntiles(mf);
      const uint32_t tiles = nt >= 4 ? mt : (mt & ((1u << (8 * nt)) - 1u));
      d = dfold(d, (uint64_t)tiles | ((uint64_t)mi::type(mf) << 32) | ((uint64_t)nt << 36) |
                       ((uint64_t)(mi::from(mf) + 1) << 40) | ((uint64_t)(mi::called(mf) + 1) << 48));
    }
    for (int i = 0; i < nr; i += 4) {
      uint32_t v[4];
      for (int j = 0; j < 4; j++) v[j] = i + j < nr ? S.river[E.at(s * RS_MAX_RIVER + i + j)] : 0u;
      d = dfold(d, dpack4(v[0], v[1], v[2], v[3]));
    }
  }
  d = dfold(d, (uint64_t)(uint32_t)(g.drawn + 1) | ((uint64_t)(uint32_t)(g.call_tile + 1) << 8) |
                   ((uint64_t)(uint32_t)(g.kakan_kind + 1) << 16) | ((uint64_t)(uint32_t)(g.call_from + 1) << 24) |
                   ((uint64_t)g.actor << 28) | ((uint64_t)g.riichi_pending << 32) |
                   ((uint64_t)g.rinshan_pending << 33) | ((uint64_t)g.call_chankan << 34) |
                   ((uint64_t)g.four_kan_pending << 35) | ((uint64_t)g.any_call_made << 36) |
                   ((uint64_t)g.terminated << 37) | ((uint64_t)g.truncated << 38) |
                   ((uint64_t)g.pending_dora << 40) | ((uint64_t)g.repeats << 48) | ((uint64_t)g.n_results << 56));
  uint64_t q = (uint64_t)g.qn();
  for (int i = 0; i < g.qn(); i++) q |= (uint64_t)(g.qseat(i) | (g.qstage(i) << 2)) << (4 + 4 * i);
  q |= (uint64_t)g.rn() << 40;
  for (int i = 0; i < g.rn(); i++) q |= (uint64_t)g.rseat(i) << (44 + 2 * i);
  d = dfold(d, q);
  d = dfold(d, g.rng_key);
  d = dfold(d, (uint64_t)g.rng_counter);
  d = dfold(d, g.policy_key);
  d = dfold(d, g.policy_counter);
  const uint8_t* wl = swall(E.bp);
  for (int i = 0; i < 136; i += 8) {
    uint64_t w = 0;
    for (int j = 0; j < 8; j++) w |= (uint64_t)wl[i + j] << (8 * j);
    d = dfold(d, w);
  }
  // the newest 8 events (type | (actor + 1) << 4 | (tile + 1) << 7)
  for (int j = 0; j < 8; j += 4) {
    uint32_t v[4];
    for (int k = 0; k < 4; k++) {
      const int idx = (int)g.events_len - 1 - (j + k);
      v[k] = idx >= 0 ? event_raw(S.events[(size_t)E.e * RS_EVENT_WINDOW + (idx & 63)]) : 0u;
    }
    d = dfold(d, dpack4(v[0], v[1], v[2], v[3]));
  }
  if (g.n_results > 0) {
    const rs_result_rec& r = S.results[E.e];
    uint64_t wn = 0;
    for (int i = 0; i < r.n_winners; i++) wn |= (uint64_t)(uint8_t)r.winners[i] << (2 * i);
    d = dfold(d, (uint64_t)(uint32_t)r.kyoku | ((uint64_t)(uint32_t)r.honba << 8) | ((uint64_t)(uint32_t)r.kind << 16) |
                     ((uint64_t)(uint32_t)r.n_winners << 24) | ((uint64_t)(uint32_t)r.n_settlements << 28) |
                     ((uint64_t)(uint32_t)(r.loser + 1) << 32) | ((uint64_t)(uint32_t)r.tenpai_mask << 40) |
                     (wn << 48));
    for (int i = 0; i < r.n_settlements; i++) {
      d = dfold(d, (uint64_t)(uint32_t)r.deltas[i][0] | ((uint64_t)(uint32_t)r.deltas[i][1] << 32));
      d = dfold(d, (uint64_t)(uint32_t)r.deltas[i][2] | ((uint64_t)(uint32_t)r.deltas[i][3] << 32));
      d = dfold(d, (uint64_t)(uint32_t)r.honba_component[i] | ((uint64_t)(uint32_t)r.deposits_claimed[i] << 32));
    }
    for (int i = 0; i < r.n_winners; i++) {
      const rs_win_rec& w = r.wins[i];
      for (int k = 0; k < 40; k += 8) {
        uint64_t y = 0;
        for (int j = 0; j < 8; j++) y |= (uint64_t)(uint8_t)w.yaku_han[k + j] << (8 * j);
        d = dfold(d, y);
      }
      d = dfold(d, (uint64_t)(uint32_t)w.yakuman | ((uint64_t)(uint32_t)w.han << 8) | ((uint64_t)(uint32_t)w.fu << 16) |
                       ((uint64_t)(uint32_t)w.base << 32));
      d = dfold(d, (uint64_t)(uint32_t)w.dora | ((uint64_t)(uint32_t)w.ura << 8) | ((uint64_t)(uint32_t)w.reds << 16) |
                       ((uint64_t)(uint32_t)w.form << 24));
    }
    d = dfold(d, (uint64_t)(uint32_t)r.scores_after[0] | ((uint64_t)(uint32_t)r.scores_after[1] << 32));
    d = dfold(d, (uint64_t)(uint32_t)r.scores_after[2] | ((uint64_t)(uint32_t)r.scores_after[3] << 32));
  }
  return d;
}
// the observation record i of `o` (as write_obs wrote it)
RS_COLD uint64_t digest_obs(uint64_t d, const rs_obs_out& o, int64_t i) {
  const uint8_t* ht = o.hand_tokens + i * 14;
  uint64_t lo = 0, hi8 = 0;
  for (int j = 0; j < 8; j++) lo |= (uint64_t)ht[j] << (8 * j);
  for (int j = 0; j < 6; j++) hi8 |= (uint64_t)ht[8 + j] << (8 * j);
  d = dfold(d, lo);
  d = dfold(d, hi8);
  const uint8_t* ev = o.event_tokens + i * 192;
  for (int k = 0; k < 192; k += 8) {
    uint64_t w = 0;
    for (int j = 0; j < 8; j++) w |= (uint64_t)ev[k + j] << (8 * j);
    d = dfold(d, w);
  }
  const int16_t* sc = o.scores + i * 4;
  d = dfold(d, dpack4((uint16_t)sc[0], (uint16_t)sc[1], (uint16_t)sc[2], (uint16_t)sc[3]));
  d = dfold(d, (uint64_t)(uint8_t)o.shanten[i] | ((uint64_t)o.round_wind[i] << 8) | ((uint64_t)o.seat_wind[i] << 16) |
                   ((uint64_t)o.kyoku[i] << 24) | ((uint64_t)(uint16_t)o.honba[i] << 32) |
                   ((uint64_t)(uint16_t)o.deposits[i] << 48));
  uint64_t w = 0;
  for (int j = 0; j < 5; j++) w |= (uint64_t)o.dora_tokens[i * 5 + j] << (8 * j);
  w |= (uint64_t)o.live_wall[i] << 40;
  for (int j = 0; j < 4; j++) w |= (uint64_t)(o.riichi_flags[i * 4 + j] & 1u) << (48 + j);
  return dfold(d, w);
}

// projection record (include/rinshan.h rs_env_rec) of env e
RS_COLD void export_env(Engine& E, const Cfg& C, rs_env_rec& r) {
  const Soa& S = E.S;
  E.load();
  const Game& g = E.g;
  r.abi_version = RS_ABI_VERSION;
  r.cfg.rule = C.rule; r.cfg.mode = C.mode; r.cfg.reward_scheme = C.reward_scheme;
  r.cfg.illegal_penalty = C.illegal_penalty; r.cfg.max_steps = C.max_steps; r.cfg.kazoe = C.kazoe;
  r.cfg.double_yakuman = C.double_yakuman; r.cfg.agari_yame = C.agari_yame; r.cfg.renchan_cap = C.renchan_cap;
  for (int i = 0; i < 136; i++) r.wall[i] = (uint8_t)E.wall(i);
  r.cursor = g.cursor; r.kan_draws = g.kan_draws; r.dora_count = g.dora_count;
  for (int s = 0; s < 4; s++) {
    const Hand h = load_hand(E.bp, s);
    rs_hand_rec& hr = r.hands[s];
    int n = 0;
    for (int t = 0; t < 136; t++)
      if (h.has(t)) hr.concealed[n++] = (uint8_t)t;
    for (int i = n; i < 14; i++) hr.concealed[i] = 0;
    hr.n_concealed = (uint8_t)n;
    const int nm = hi::nmelds(h.info);
    hr.n_melds = (uint8_t)nm;
    for (int i = 0; i < 4; i++) {
      rs_meld_rec& m = hr.melds[i];
      const uint32_t mf = i < nm ? E.meld_info(s, i) : 0u, mt = i < nm ? E.meld_tiles(s, i) : 0u;
      m.type = (int8_t)(i < nm ? mi::type(mf) : 0);
      m.n_tiles = (int8_t)(i < nm ? mi::ntiles(mf) : 0);
      m.from_seat = (int8_t)(i < nm ? mi::from(mf) : 0);
      m.pad0 = 0;
      for (int j = 0; j < 4; j++) m.tiles[j] = (uint8_t)(j < m.n_tiles ? (mt >> (8 * j)) & 255 : 0);
      m.called_tile = (int16_t)(i < nm ? mi::called(mf) : 0);
      m.pad1 = 0;
    }
    const int nr = hi::nriver(h.info);
    for (int i = 0; i < RS_MAX_RIVER; i++) {
      const uint16_t v = i < nr ? S.river[(size_t)(s * RS_MAX_RIVER + i) * S.n + E.e] : (uint16_t)0;
      hr.river_tile[i] = (uint8_t)(v & 255);
      hr.river_flags[i] = (uint8_t)(v >> 8);
    }
    hr.n_river = nr;
    hr.riichi = (int8_t)hi::riichi(h.info);
    hr.riichi_index = (int8_t)hi::riichi_index(h.info);
    hr.ippatsu = (int8_t)hi::ippatsu(h.info);
    hr.temp_furiten = (int8_t)hi::temp(h.info);
    hr.perm_furiten = (int8_t)hi::perm(h.info);
    hr.shanten = (int8_t)hi::shanten(h.info);
    hr.pad = 0;
    hr.waits = h.waits;
  }
  for (int s = 0; s < 4; s++) r.scores[s] = g.scores[s];
  r.kyoku = g.kyoku; r.honba = g.honba; r.deposits = g.deposits; r.repeats = g.repeats;
  r.phase = g.phase; r.actor = g.actor; r.drawn = g.drawn;
  r.riichi_pending = g.riichi_pending; r.rinshan_pending = g.rinshan_pending;
  r.call_tile = g.call_tile; r.call_from = g.call_from;
  r.n_queue = g.qn();
  for (int i = 0; i < RS_MAX_QUEUE; i++) {
    r.queue_seat[i] = (int8_t)(i < r.n_queue ? g.qseat(i) : 0);
    r.queue_stage[i] = (int8_t)(i < r.n_queue ? g.qstage(i) : 0);
  }
  r.n_rons = g.rn();
  for (int i = 0; i < 4; i++) r.rons[i] = (int8_t)(i < r.n_rons ? g.rseat(i) : 0);
  r.call_chankan = g.call_chankan; r.kakan_kind = g.kakan_kind; r.pending_dora = g.pending_dora;
  r.four_kan_pending = g.four_kan_pending; r.any_call_made = g.any_call_made;
  r.rng_key = g.rng_key; r.rng_counter = g.rng_counter;
  r.step_count = (int32_t)g.step_count; r.terminated = g.terminated; r.truncated = g.truncated;
  r.events_len = (int32_t)g.events_len;
  const int cnt = g.events_len < 64 ? (int)g.events_len : 64;
  for (int i = 0; i < 64; i++) {
    if (i < cnt) {
      const uint32_t idx = (g.events_len - (uint32_t)cnt + (uint32_t)i) & 63u;
      const uint32_t ev = event_raw(S.events[(uint32_t)E.e * RS_EVENT_WINDOW + idx]);
      r.events[i][0] = (int16_t)(ev & 15);
      r.events[i][1] = (int16_t)((int)((ev >> 4) & 7) - 1);
      r.events[i][2] = (int16_t)((int)((ev >> 7) & 255) - 1);
    } else {
      r.events[i][0] = r.events[i][1] = r.events[i][2] = 0;
    }
  }
  r.n_results = g.n_results;
  r.last_result = S.results[E.e];
  const bool done = g.env_terminated || g.env_truncated;
  for (int i = 0; i < 4; i++) r.legal_mask[i] = done ? 0u : sword(E.bp, W_LEGAL + i);
  r.current_player = g.current_player;
  r.env_terminated = g.env_terminated;
  r.env_truncated = g.env_truncated;
  r.status = g.status;
  float rw[4];
  E.current_rewards(rw);
  for (int i = 0; i < 4; i++) r.rewards[i] = rw[i];
  r.env_key = g.env_key; r.policy_key = g.policy_key; r.policy_counter = g.policy_counter;
  r.resets = (int32_t)g.resets;
  r.pad = 0;
}

// crafted states (tests/engine_helpers.py:58-105 craft()); shanten / waits /
// codes / classes are derived, the legal mask is recomputed
RS_COLD void import_env(Engine& E, const rs_env_rec& r) {
  const Soa& S = E.S;
  const Tabs& T = E.T;
  Game& g = E.g;
  uint8_t* w = swall(E.bp);
  for (int i = 0; i < 136; i++) w[i] = r.wall[i];
  for (int i = 136; i < WALL_STRIDE; i++) w[i] = 0;
  g.cursor = r.cursor; g.kan_draws = r.kan_draws; g.dora_count = r.dora_count;
  for (int s = 0; s < 4; s++) {
    const rs_hand_rec& hr = r.hands[s];
    Hand h;
    h.w0 = h.w1 = h.w2 = h.w3 = h.w4 = 0;
    h.cm = h.cp = h.cs = h.cz = 0;
    for (int i = 0; i < hr.n_concealed; i++) {
      const int t = hr.concealed[i], k = t >> 2;
      h.set_word(t >> 5, h.word(t >> 5) | (1u << (t & 31)));
      h.set_code(kind_suit(k), h.code(kind_suit(k)) + kind_pow(k));
    }
    h.cls = class_of(T, 0, h.cm) | (class_of(T, 1, h.cp) << 8) | (class_of(T, 2, h.cs) << 16) |
            (class_of(T, 3, h.cz) << 24);
    uint32_t inf = 0;
    inf = hi::set_riichi(inf, hr.riichi);
    inf = hi::set_riichi_index(inf, hr.riichi_index);
    inf = hi::set_ippatsu(inf, hr.ippatsu);
    inf = hi::set_temp(inf, hr.temp_furiten);
    inf = hi::set_perm(inf, hr.perm_furiten);
    inf = hi::set_nmelds(inf, hr.n_melds);
    inf = hi::set_nriver(inf, hr.n_river);
    inf = hi::set_nconc(inf, hr.n_concealed);
    h.info = inf;
    tokens_from_set(h, E.C.rule == RS_RULE_RED);
    for (int i = 0; i < hr.n_melds; i++) {
      const rs_meld_rec& m = hr.melds[i];
      uint32_t packed = 0;
      for (int j = 0; j < m.n_tiles; j++) packed |= (uint32_t)m.tiles[j] << (8 * j);
      sword(E.bp, W_MELD + 2 * (4 * s + i)) = packed;
      sword(E.bp, W_MELD + 2 * (4 * s + i) + 1) = mi::make(m.type, m.n_tiles, m.from_seat, m.called_tile);
    }
    uint64_t rk = 0;
    for (int i = 0; i < hr.n_river; i++) {
      S.river[(size_t)(s * RS_MAX_RIVER + i) * S.n + E.e] =
          (uint16_t)(hr.river_tile[i] | ((uint16_t)hr.river_flags[i] << 8));
      rk |= 1ull << (hr.river_tile[i] >> 2);
    }
    sdword(E.bp, W_HRKIND + 2 * s) = rk;
    finish_hand(T, h);
    store_hand(E.bp, s, h);
  }
  for (int s = 0; s < 4; s++) g.scores[s] = r.scores[s];
  g.kyoku = r.kyoku; g.honba = r.honba; g.deposits = r.deposits; g.repeats = r.repeats;
  g.phase = r.phase; g.actor = r.actor; g.drawn = r.drawn;
  g.riichi_pending = r.riichi_pending; g.rinshan_pending = r.rinshan_pending;
  g.call_tile = r.call_tile; g.call_from = r.call_from;
  int qs[5], qt[5];
  const int nq = r.n_queue < 5 ? r.n_queue : 5;
  for (int i = 0; i < nq; i++) { qs[i] = r.queue_seat[i]; qt[i] = r.queue_stage[i]; }
  g.qset(nq, qs, qt);
  g.rons = 0;
  for (int i = 0; i < r.n_rons && i < 3; i++) g.rpush(r.rons[i]);
  g.call_chankan = r.call_chankan; g.kakan_kind = r.kakan_kind; g.pending_dora = r.pending_dora;
  g.four_kan_pending = r.four_kan_pending; g.any_call_made = r.any_call_made;
  g.rng_key = r.rng_key; g.rng_counter = (uint32_t)r.rng_counter;
  g.step_count = (uint32_t)r.step_count; g.terminated = r.terminated; g.truncated = r.truncated;
  const int cnt = r.events_len < 64 ? r.events_len : 64;
  g.events_len = (uint32_t)(r.events_len - cnt);
  for (int i = 0; i < cnt; i++) E.emit(r.events[i][0], r.events[i][1], r.events[i][2]);
  g.n_results = r.n_results;
  S.results[E.e] = r.last_result;
  g.env_key = r.env_key; g.policy_key = r.policy_key; g.policy_counter = r.policy_counter;
  g.resets = (uint32_t)r.resets;
  g.status = 0;
  Mask115 m;
  E.compute_legal(m);
  E.store_legal(m);
  float rw[4];
  E.wrap(rw);
  E.store();
}

}  // namespace rs
