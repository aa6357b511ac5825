// hostcheck.cpp — TEST-ONLY host build of the device engine source.
//
// Compiles paper_2605_20577_b200/csrc/rs_*.cuh with g++ over host-memory
// SoA buffers so the transition logic can be diffed against the CPU oracle
// without a GPU (tests/test_hostcheck.py).  It is never loaded by the
// product package, smoke() or bench.py; the shipped path is the nvcc
// sm_100a library (_rinshan.so).
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "../../paper_2605_20577_b200/csrc/rs_check.cuh"
#include "../../paper_2605_20577_b200/csrc/rs_io.cuh"

using namespace rs;

struct HC {
  Soa S;
  Tabs T;
  Cfg C;
  // one allocation per array, so the sanitized build
  // (tests/test_hostcheck_sanitized.py) sees an overrun of any of them
  std::vector<void*> parts;
  ~HC() {
    for (void* p : parts) free(p);
  }
};

extern "C" {

void* hc_create(int n, const rs_config* cfg) {
  const HostTables& ht = host_tables();
  HC* h = new HC();
  h->C = Cfg{cfg->rule, cfg->mode, cfg->reward_scheme, cfg->illegal_penalty, cfg->max_steps,
             cfg->kazoe, cfg->double_yakuman, cfg->agari_yame, cfg->renchan_cap};
  h->T = Tabs{ht.suit_cls.data(), ht.honor_cls.data(), ht.t1.data(), ht.t2.data(), ht.t3.data()};
  std::vector<std::pair<void**, size_t>> plan;
  Soa& S = h->S;
  S.n = n;
  plan.push_back({(void**)&S.blk, (size_t)BLK_BYTES * n});
  plan.push_back({(void**)&S.river, 4 * RS_MAX_RIVER * 2 * (size_t)n});
  plan.push_back({(void**)&S.events, 64 * 4 * (size_t)n});
  plan.push_back({(void**)&S.results, sizeof(rs_result_rec) * (size_t)n});
  for (auto& p : plan) {
    void* m = nullptr;
    if (posix_memalign(&m, 256, p.second)) abort();  // exact size: no slack past the array
    memset(m, 0, p.second);
    *p.first = m;
    h->parts.push_back(m);
  }
  return h;
}

void hc_free(void* p) { delete (HC*)p; }


// bench seeding (bench/runner.py:25-33)
void hc_init_indexed(void* p, uint64_t seed, int64_t base, float* rewards) {
  HC* h = (HC*)p;
  for (int e = 0; e < h->S.n; e++) {
    Engine E(h->S, h->T, h->C, e, h->S.blk + (size_t)e * BLK_BYTES);
    E.g.env_key = derive_key(mix64(seed), (uint64_t)(base + e));
    E.g.policy_key = derive_key(E.g.env_key, 1);
    E.g.policy_counter = 0;
    E.g.resets = 0;
    E.init_game(derive_key(E.g.env_key, 2), rewards + 4 * e);
    E.store();
  }
}

void hc_init_seeds(void* p, const uint64_t* seeds, float* rewards) {
  HC* h = (HC*)p;
  for (int e = 0; e < h->S.n; e++) {
    Engine E(h->S, h->T, h->C, e, h->S.blk + (size_t)e * BLK_BYTES);
    E.g.env_key = seeds[e];
    E.g.policy_key = derive_key(seeds[e], 1);
    E.g.policy_counter = 0;
    E.g.resets = 0;
    E.init_game(seeds[e], rewards + 4 * e);
    E.store();
  }
}

void hc_step(void* p, const int32_t* actions, uint8_t* status, float* rewards) {
  HC* h = (HC*)p;
  for (int e = 0; e < h->S.n; e++) {
    Engine E(h->S, h->T, h->C, e, h->S.blk + (size_t)e * BLK_BYTES);
    E.load();
    Mask115 m;
    status[e] = (uint8_t)E.step(actions[e], m, rewards + 4 * e);
    E.store();
  }
}

void hc_random_actions(void* p, int32_t* actions) {
  HC* h = (HC*)p;
  for (int e = 0; e < h->S.n; e++) {
    Engine E(h->S, h->T, h->C, e, h->S.blk + (size_t)e * BLK_BYTES);
    E.load();
    actions[e] = E.random_action(E.load_legal());
    E.store();
  }
}

void hc_export(void* p, int e, rs_env_rec* out) {
  HC* h = (HC*)p;
  Engine E(h->S, h->T, h->C, e, h->S.blk + (size_t)e * BLK_BYTES);
  export_env(E, h->C, *out);
}

void hc_import(void* p, int e, const rs_env_rec* in) {
  HC* h = (HC*)p;
  Engine E(h->S, h->T, h->C, e, h->S.blk + (size_t)e * BLK_BYTES);
  E.load();
  import_env(E, *in);
}

void hc_observe(void* p, int e, int seat, uint8_t* hand, uint8_t* events, int8_t* sh, int16_t* scores,
                uint8_t* misc /*round, seat, kyoku, live*/, int16_t* hd /*honba, deposits*/, uint8_t* dora,
                uint8_t* riichi) {
  HC* h = (HC*)p;
  Engine E(h->S, h->T, h->C, e, h->S.blk + (size_t)e * BLK_BYTES);
  E.load();
  rs_obs_out o;
  o.hand_tokens = hand; o.event_tokens = events; o.shanten = sh; o.scores = scores;
  o.round_wind = misc; o.seat_wind = misc + 1; o.kyoku = misc + 2; o.live_wall = misc + 3;
  o.honba = hd; o.deposits = hd + 1; o.dora_tokens = dora; o.riichi_flags = riichi;
  write_obs(E, seat, o, 0);
}

// fused rollout restated on the host: auto-reset + random policy + step
int64_t hc_rollout(void* p, int steps, uint64_t* digests, int16_t* actions_log, int policy) {
  HC* h = (HC*)p;
  int64_t games = 0;
  for (int e = 0; e < h->S.n; e++) {
    Engine E(h->S, h->T, h->C, e, h->S.blk + (size_t)e * BLK_BYTES);
    E.load();
    uint64_t d = digests ? digests[e] : 0;
    float r[4];
    for (int t = 0; t < steps; t++) {
      if (E.g.env_terminated || E.g.env_truncated) {
        E.g.resets++;
        E.init_game(derive_key(E.g.env_key, 2 + (uint64_t)E.g.resets), r);
      }
      const int a = policy ? E.heuristic_action(E.load_legal()) : E.random_action(E.load_legal());
      Mask115 m;
      E.step(a, m, r);
      if (actions_log) actions_log[(size_t)t * h->S.n + e] = (int16_t)a;
      if (E.g.env_terminated || E.g.env_truncated) games++;
      if (digests) {  // the wide digest, as k_rollout folds it
        uint8_t ht[14], ev[192], misc[4], dora[5], riichi[4];
        int8_t sh;
        int16_t sc[4], hd[2];
        rs_obs_out o;
        o.hand_tokens = ht; o.event_tokens = ev; o.shanten = &sh; o.scores = sc;
        o.round_wind = misc; o.seat_wind = misc + 1; o.kyoku = misc + 2; o.live_wall = misc + 3;
        o.honba = hd; o.deposits = hd + 1; o.dora_tokens = dora; o.riichi_flags = riichi;
        d = digest_state(digest_step(d, a, E, m, r), E);
        write_obs(E, E.g.current_player, o, 0);
        d = digest_obs(d, o, 0);
      }
    }
    if (digests) digests[e] = d;
    E.store();
  }
  return games;
}

uint32_t hc_check(void* p, int e, int fast) {
  HC* h = (HC*)p;
  Engine E(h->S, h->T, h->C, e, h->S.blk + (size_t)e * BLK_BYTES);
  E.load();
  return check_invariants(E, fast != 0);
}

}  // extern "C"
