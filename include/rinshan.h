/*
 * rinshan.h — C ABI of the B200-native batched Riichi-Mahjong environment step.
 *
 * This is the drop-in boundary for the reference's Pgx-style env path
 * (mjsim.init / mjsim.step / mjsim.observe + the random-policy rollout
 * harness).  Every entry point takes plain pointers and sizes; device
 * pointers are CUDA global-memory addresses (e.g. torch tensor data_ptr()),
 * `stream` is a cudaStream_t passed as void*.  No torch types cross this ABI.
 *
 * Reference interfaces each entry point replaces (paths under the
 * reference's pkg/src/mjsim/):
 *   rs_tables_build   hand/tables.py:212-224   build_tables()   (+ get_tables :278-291)
 *   rs_tables_load    hand/tables.py:243-265   load_tables(path) blob format
 *   rs_create         env/core.py:26-46        EnvConfig -> GameConfig (batched)
 *   rs_init           env/core.py:81-82        init(seed, config) for n envs
 *   rs_init_indexed   bench/runner.py:25-33,76-84  env_game_seed/env_policy_state + init
 *   rs_step           env/core.py:85-94      step(state, action) for n envs
 *                     (engine/engine.py:405-422 apply_action, :105-122 _finish)
 *   rs_observe        env/observe.py:81-124   observe(state, seat)
 *   rs_policy_random  env/policies.py:17-22    random_policy(legal, rng)
 *   rs_policy_heuristic env/policies.py:51-109 heuristic_policy(obs, legal)
 *   rs_rollout_policy bench/runner.py:97-121   one_pass, random or heuristic policy
 *   rs_rollout        bench/runner.py:97-121   run_shard.one_pass (auto-reset +
 *                                              random_policy + step), fused
 *   rs_autoreset      bench/runner.py:107-109  auto-reset of finished envs
 *   rs_check_invariants engine/state.py:105-180 check_invariants (+ runner.py soak gates)
 *   rs_export_env     engine/state.py:191-242  serialize_state (projection record)
 *   rs_export_envs    engine/state.py:191-242  serialize_state of many envs (one
 *                                              launch + one copy; service/sessions.py
 *                                              state reads, batched sessions)
 *   rs_import_env     tests/engine_helpers.py:58-105 craft() (crafted states)
 *   rs_set_done_flag, rs_signal_done (no counterpart: the reference steps
 *                                              in-process) completion word of host-driven
 *                                              steps (HostStepper)
 *   rs_debug_score    scoring/score.py:45-82   score_win(ctx, kazoe, double_yakuman)
 *                                              over WinContext (scoring/context.py:19-57),
 *                                              the device scorer alone (parity harness)
 *
 * Error convention: every function returns 0 on success, a negative RS_E*
 * code on contract violations and a positive cudaError_t value when a CUDA
 * call fails; rs_last_error() gives a message.  Per-env contract outcomes
 * (illegal action, stepping a finished env) are reported in the per-env
 * status byte, never as a global error (reference env/core.py:85-94).
 */
#ifndef RINSHAN_H
#define RINSHAN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 1

#define RS_NUM_TILES 136
#define RS_NUM_KINDS 34
#define RS_NUM_ACTIONS 115
#define RS_EVENT_WINDOW 64
#define RS_MAX_RIVER 40
#define RS_MAX_QUEUE 8
#define RS_MASK_WORDS 4

/* rules / modes / schemes (reference tiles.py:18-19, engine/types.py:12-14) */
#define RS_RULE_RED 0
#define RS_RULE_NO_RED 1
#define RS_MODE_SINGLE 0
#define RS_MODE_EAST 1
#define RS_MODE_HALF 2
#define RS_REWARD_SCORE_DELTA 0
#define RS_REWARD_RANK 1

/* per-env status bits written by rs_step (reference env/core.py:85-94) */
#define RS_STATUS_ILLEGAL 1u  /* masked-off action: penalty, episode ends   */
#define RS_STATUS_CONTRACT 2u /* stepped a finished env: state unchanged   */
#define RS_STATUS_INVARIANT 4u /* check_invariants failed after the step
                                  (only when the handle checks every step:
                                  RINSHAN_CHECK=1 at rs_create)            */

/* rs_check_invariants violation bits (engine/state.py:105-180,
 * bench/runner.py:226-284) */
#define RS_INV_SCORE_SUM 1u         /* scores + 1000 x deposits != 100000        */
#define RS_INV_TILES 2u             /* the 136 tiles are not each held once      */
#define RS_INV_EMPTY_LEGAL 4u       /* live game with no legal action            */
#define RS_INV_TERMINAL_LEGAL 8u    /* finished game with legal actions          */
#define RS_INV_FURITEN_RON 16u      /* ron offered to a furiten seat             */
#define RS_INV_HAND_SYNC 32u        /* codes / classes / tokens / shanten /
                                       waits / river kinds out of sync (full)   */
#define RS_INV_HAND_SIZE 64u        /* tile-equivalents held != 13 / 14 (full)  */
#define RS_INV_RIICHI_NOT_TENPAI 128u /* riichi with shanten > 0 (full)         */

/* error codes */
#define RS_OK 0
#define RS_E_ARG (-1)
#define RS_E_TABLES (-2)
#define RS_E_STATE (-3)
#define RS_E_CORRUPT (-4)

typedef struct rs_config {
  int32_t rule;           /* RS_RULE_*                                       */
  int32_t mode;           /* RS_MODE_*                                       */
  int32_t reward_scheme;  /* RS_REWARD_*                                     */
  float illegal_penalty;  /* <= 0                                            */
  int32_t max_steps;      /* truncation (engine/types.py:56)                 */
  int32_t kazoe;          /* engine/types.py:53                              */
  int32_t double_yakuman; /* engine/types.py:54                              */
  int32_t agari_yame;     /* engine/types.py:55                              */
  int32_t renchan_cap;    /* engine/types.py:57                              */
} rs_config;

/* ---- projection records (host side, import/export, parity harness) ---- */

typedef struct rs_meld_rec {
  int8_t type;        /* 0 chi 1 pon 2 kan_open 3 kan_closed 4 kan_added   */
  int8_t n_tiles;
  int8_t from_seat;   /* -1 for closed kan                                 */
  int8_t pad0;
  uint8_t tiles[4];   /* sorted tile ids                                   */
  int16_t called_tile;
  int16_t pad1;
} rs_meld_rec;

#define RS_RIVER_TSUMOGIRI 1u
#define RS_RIVER_RIICHI 2u
#define RS_RIVER_CALLED 4u

typedef struct rs_hand_rec {
  uint8_t concealed[14]; /* sorted tile ids                                */
  uint8_t n_concealed;
  uint8_t n_melds;
  rs_meld_rec melds[4];
  uint8_t river_tile[RS_MAX_RIVER];
  uint8_t river_flags[RS_MAX_RIVER];
  int32_t n_river;
  int8_t riichi;       /* 0 / 1 / 2 (double)                               */
  int8_t riichi_index;
  int8_t ippatsu;
  int8_t temp_furiten;
  int8_t perm_furiten;
  int8_t shanten;
  int16_t pad;
  uint64_t waits;      /* bit k: kind k completes the hand                 */
} rs_hand_rec;

/* kyoku result kinds (engine/engine.py: "tsumo", "ron", "exhaustive",
 * "abort_nine_terminals", "abort_triple_ron", "abort_four_riichi",
 * "abort_four_kan") */
#define RS_RES_TSUMO 0
#define RS_RES_RON 1
#define RS_RES_EXHAUSTIVE 2
#define RS_RES_ABORT_NINE 3
#define RS_RES_ABORT_TRIPLE_RON 4
#define RS_RES_ABORT_FOUR_RIICHI 5
#define RS_RES_ABORT_FOUR_KAN 6

#define RS_FORM_STANDARD 0
#define RS_FORM_SEVEN_PAIRS 1
#define RS_FORM_KOKUSHI 2

typedef struct rs_win_rec {
  int8_t yaku_han[40]; /* han (or yakuman multiplicity) per yaku id, 0 = absent */
  int32_t yakuman;     /* yakuman count                                     */
  int32_t han, fu, base, dora, ura, reds, form;
} rs_win_rec;

typedef struct rs_result_rec {
  int32_t kyoku, honba, kind;
  int32_t n_winners;
  int8_t winners[4];
  int32_t loser;
  int32_t n_settlements;
  int32_t deltas[3][4];
  int32_t honba_component[3];
  int32_t deposits_claimed[3];
  rs_win_rec wins[3];
  int32_t tenpai_mask; /* exhaustive draw: bit s = seat s tenpai            */
  int32_t scores_after[4];
} rs_result_rec;

typedef struct rs_env_rec {
  int32_t abi_version;
  rs_config cfg;
  uint8_t wall[RS_NUM_TILES];
  int32_t cursor, kan_draws, dora_count;
  rs_hand_rec hands[4];
  int32_t scores[4];
  int32_t kyoku, honba, deposits, repeats, phase, actor, drawn;
  int32_t riichi_pending, rinshan_pending, call_tile, call_from;
  int32_t n_queue;
  int8_t queue_seat[RS_MAX_QUEUE];
  int8_t queue_stage[RS_MAX_QUEUE];
  int32_t n_rons;
  int8_t rons[4];
  int32_t call_chankan, kakan_kind, pending_dora, four_kan_pending, any_call_made;
  uint64_t rng_key, rng_counter;
  int32_t step_count, terminated, truncated;
  int32_t events_len;          /* total events emitted so far            */
  int16_t events[RS_EVENT_WINDOW][3]; /* last min(64, len), oldest first  */
  int32_t n_results;
  rs_result_rec last_result;
  uint32_t legal_mask[RS_MASK_WORDS];
  /* env wrapper (env/core.py:49-62) */
  int32_t current_player;
  int32_t env_terminated, env_truncated;
  int32_t status;
  float rewards[4];
  /* rollout bookkeeping (bench/runner.py:25-33, 80-82) */
  uint64_t env_key, policy_key, policy_counter;
  int32_t resets;
  int32_t pad;
} rs_env_rec;

/* ---- device buffers supplied by the caller ---- */

typedef struct rs_step_out {
  uint8_t* legal_mask;   /* [n][115] bool, may be NULL                      */
  uint32_t* legal_bits;  /* [n][4] packed mask, may be NULL                 */
  int8_t* current_player;/* [n]                                             */
  float* rewards;        /* [n][4]                                          */
  uint8_t* terminated;   /* [n]                                             */
  uint8_t* truncated;    /* [n]                                             */
  uint8_t* status;       /* [n] RS_STATUS_* bits, may be NULL               */
} rs_step_out;

/* one env's step result as one 40-byte record (rs_step_rec_out): what a
 * host-driven actor reads back per step, packed so the writes of an env
 * are contiguous (e.g. into mapped pinned host memory) */
typedef struct rs_step_rec {
  float rewards[4];
  uint32_t legal_bits[4];
  int32_t next_action;   /* the policy's next action, -1 for finished envs  */
  int8_t current_player;
  uint8_t terminated;
  uint8_t truncated;
  uint8_t status;
} rs_step_rec;

/* observation tensors (reference docs/formats.md:32-52, env/observe.py:50-62) */
typedef struct rs_obs_out {
  uint8_t* hand_tokens;  /* [n][14]                                         */
  uint8_t* event_tokens; /* [n][64][3]                                      */
  int8_t* shanten;       /* [n]                                             */
  int16_t* scores;       /* [n][4] points // 100, observer first            */
  uint8_t* round_wind;   /* [n]                                             */
  uint8_t* seat_wind;    /* [n]                                             */
  uint8_t* kyoku;        /* [n]                                             */
  int16_t* honba;        /* [n]                                             */
  int16_t* deposits;     /* [n]                                             */
  uint8_t* dora_tokens;  /* [n][5]                                          */
  uint8_t* live_wall;    /* [n]                                             */
  uint8_t* riichi_flags; /* [n][4]                                          */
} rs_obs_out;

typedef struct rs_rollout_stats {
  /* accumulated on device over a rollout (reduced over envs by the host)  */
  uint64_t steps;
  uint64_t games_completed;
  uint64_t illegal;
} rs_rollout_stats;

typedef struct rs_handle rs_handle;

const char* rs_last_error(void);
int rs_abi_version(void);

/* tables (host-built once per process, uploaded per handle).  A blob is
 * loaded before the tables are first used (built, queried or uploaded by
 * rs_create); afterwards an identical blob is a no-op and a different one
 * is rejected with RS_E_TABLES (live tables are never replaced). */
int rs_tables_build(void);
int rs_tables_load(const uint8_t* blob, int64_t size);
int rs_tables_blob(uint8_t* out, int64_t cap, int64_t* size);
int rs_tables_crc(uint32_t* crc);
int rs_tables_info(int32_t* n_suit_classes, int32_t* n_honor_classes,
                   int32_t* n_pair_mp, int32_t* n_pair_sz);
/* host-side query of the re-encoded tables (unit tests of the encoding) */
int rs_tables_shanten_std(uint32_t cm, uint32_t cp, uint32_t cs, uint32_t cz,
                          int32_t melds, int32_t* out);

int rs_create(rs_handle** out, int64_t n_envs, const rs_config* cfg, int32_t device);
int rs_destroy(rs_handle* h);
int64_t rs_num_envs(const rs_handle* h);
/* h != NULL: bytes of the handle's device allocation; h == NULL: canonical
 * bytes of one env's game state (the S of the roofline B_step = 2S+O+M+R+A) */
int64_t rs_state_bytes(const rs_handle* h);

/* seeds_dev: device u64[n] game seeds; policy streams are derived from them */
int rs_init(rs_handle* h, const uint64_t* seeds_dev, const rs_step_out* out, void* stream);
/* bench seeding: env i uses env_game_seed(seed, index_base + i, 0) and
 * env_policy_state(seed, index_base + i) */
int rs_init_indexed(rs_handle* h, uint64_t seed, int64_t index_base,
                    const rs_step_out* out, void* stream);
int rs_step(rs_handle* h, const int32_t* actions_dev, const rs_step_out* out, void* stream);
/* an action id for rs_step / rs_step_ex / rs_step_rec_out: the env is not
 * stepped (state untouched: no transition, no auto-reset, no policy draw);
 * its outputs describe its current state with zero rewards and status 0,
 * and its next action is RS_ACTION_SKIP.  For actors that decide at
 * different times (game sessions, asynchronous agents); the reference steps
 * one env at a time and has no counterpart. */
#define RS_ACTION_SKIP (-2147483647 - 1)

/* rs_step fused with what an actor loop does next, in the same kernel:
 *   RS_STEP_AUTORESET  finished envs start their next game (auto-reset,
 *                      bench/runner.py:107-109); rewards / terminated /
 *                      truncated / status describe the transition while the
 *                      legal mask, current player and observation belong to
 *                      the new game (Pgx auto_reset convention)
 *   RS_STEP_OBSERVE    observe(current player) into `obs` (observe.py:81)
 * next_actions_dev (may be NULL) receives random_policy's next action from
 * each env's policy stream (policies.py:17-22), -1 for finished envs. */
#define RS_STEP_AUTORESET 1
#define RS_STEP_OBSERVE 2
/* next_actions_dev from heuristic_policy instead of random_policy */
#define RS_STEP_HEURISTIC 4
/* bump the completion word (rs_set_done_flag) once every output of the
 * step is visible to the host */
#define RS_STEP_SIGNAL 8
/* instead of RS_STEP_AUTORESET, the reference runner's order
 * (bench/runner.py:107-113, Gymnasium's next-step autoreset): a finished
 * env starts its next game at the beginning of the following step, acts
 * with its own policy stream there (random, or heuristic with
 * RS_STEP_HEURISTIC; its host action is ignored) and steps.  The step that
 * finishes an env leaves it finished (its outputs describe the final
 * state, next action -1).  Per-env trajectories equal rs_rollout's.  Needs
 * a policy output (next_actions or recs); exclusive with
 * RS_STEP_AUTORESET.  An env whose action is RS_ACTION_SKIP is left
 * untouched (not reset). */
#define RS_STEP_RESET_FIRST 16
int rs_step_ex(rs_handle* h, const int32_t* actions_dev, int32_t flags, const rs_step_out* out,
               const rs_obs_out* obs, int32_t* next_actions_dev, void* stream);
/* rs_step_ex with the per-env outputs and the next action (random, or
 * heuristic with RS_STEP_HEURISTIC) written as one rs_step_rec per env into
 * recs[n] (device or mapped pinned host memory); next_actions (may be
 * NULL): the next actions also as one contiguous int32[n] (what a host
 * loop feeding them back reads: 4 bytes per env instead of a strided
 * gather over the records) */
int rs_step_rec_out(rs_handle* h, const int32_t* actions, int32_t flags, rs_step_rec* recs,
                    const rs_obs_out* obs, int32_t* next_actions, void* stream);
/* Completion word for host-driven stepping: after an rs_step_ex /
 * rs_step_rec_out launch with RS_STEP_SIGNAL, once all of its per-env
 * outputs are visible to the host, the kernel writes an incremented
 * sequence number into *host_flag (mapped pinned host memory), so a host
 * thread can poll one word instead of sleeping in a stream synchronize;
 * rs_signal_done bumps it after whatever precedes it on `stream` (a copy of
 * device outputs to the host).  The sequence continues from the word's
 * value at this call; NULL turns it off. */
int rs_set_done_flag(rs_handle* h, uint32_t* host_flag);
int rs_signal_done(rs_handle* h, void* stream);
/* seats_dev: device int8[n] or NULL for each env's current player */
int rs_observe(rs_handle* h, const int8_t* seats_dev, const rs_obs_out* obs, void* stream);
/* random policy over each env's legal list using its policy stream */
int rs_policy_random(rs_handle* h, int32_t* actions_dev, void* stream);
/* heuristic_policy (policies.py:51-109): win, riichi, else the discard
 * minimising shanten (honors, terminals, then kind; plain before red), else
 * the call that strictly lowers shanten, else pass; -1 for finished envs.
 * Uses no randomness (the policy stream is untouched). */
int rs_policy_heuristic(rs_handle* h, int32_t* actions_dev, void* stream);
/* fused rollout: `steps` iterations of {auto-reset, random policy, step,
 * observe} per env (bench/runner.py:97-121).  obs (may be NULL) receives
 * the current player's observation: obs_slots = 1 keeps only the final
 * one, obs_slots = steps writes slot t of [steps][n] every step (a
 * trajectory buffer).  actions_log (may be NULL) is [steps][n] int16;
 * stats_dev (may be NULL) is a device rs_rollout_stats accumulated
 * atomically; digests_dev (may be NULL) is u64[n] per-env trajectory
 * digests chained across calls; out (may be NULL) gets the final step's
 * outputs. */
int rs_rollout(rs_handle* h, int32_t steps, const rs_obs_out* obs, int32_t obs_slots,
               int16_t* actions_log, rs_rollout_stats* stats_dev, uint64_t* digests_dev,
               const rs_step_out* out, void* stream);
/* rs_rollout with the acting policy chosen: RS_POLICY_RANDOM (= rs_rollout)
 * or RS_POLICY_HEURISTIC (the one_pass loop with heuristic_policy acting:
 * tenpai / riichi / win branches at scale) */
#define RS_POLICY_RANDOM 0
#define RS_POLICY_HEURISTIC 1
/* actors_log (may be NULL): [steps][n] int8, the seat that acted at each
 * step (engine state.actor, the mjlog-lite [seat, action] pair) | 4 when
 * the env was auto-reset just before that step (a new game starts there).
 * traj (may be NULL): the per-step outputs of every step (packed
 * legal_bits [steps][n][4], current_player [steps][n], rewards
 * [steps][n][4], terminated / truncated / status [steps][n]; any field may
 * be NULL, legal_mask must be), i.e. with obs_slots = steps a complete
 * trajectory buffer of the rollout. */
int rs_rollout_policy(rs_handle* h, int32_t steps, int32_t policy, const rs_obs_out* obs, int32_t obs_slots,
                      int16_t* actions_log, int8_t* actors_log, const rs_step_out* traj,
                      rs_rollout_stats* stats_dev, uint64_t* digests_dev, const rs_step_out* out, void* stream);

/* auto-reset (bench/runner.py:107-109): every finished env starts its next
 * game from env_game_seed(seed, index, resets + 1); outputs for all envs */
int rs_autoreset(rs_handle* h, const rs_step_out* out, void* stream);

/* check_invariants (engine/state.py:105-180) of every env; fast != 0 runs
 * only conservation, the score identity, mask sanity and the furiten-ron
 * gate (the soak suite's per-step check).  The RS_INV_* bits found are
 * OR-ed into flags_dev[n] (u32, device), so calls accumulate. */
int rs_check_invariants(rs_handle* h, int32_t fast, uint32_t* flags_dev, void* stream);

/* Synchronous projection-record I/O (parity harness, sessions, crafted
 * states).  Each call first waits for all work on the handle's device
 * (cudaDeviceSynchronize, so steps launched on any stream, blocking or
 * not, are complete), then copies; the caller's current device is kept.
 * rs_export_envs: records of envs[0..count) (host indices) into
 * out[count] (host).  rs_import_env rejects a record whose fields do not
 * fit the device layout (counts, tile ids, packed-header widths) with
 * RS_E_ARG. */
int rs_export_env(rs_handle* h, int64_t env, rs_env_rec* out);
int rs_export_envs(rs_handle* h, const int64_t* envs, int64_t count, rs_env_rec* out);
int rs_import_env(rs_handle* h, int64_t env, const rs_env_rec* in);
/* WinContext (scoring/context.py:19-57) as plain data: the parity
 * harness's input to the device scorer.  `concealed` counts include the
 * winning tile; `ids` lists concealed plus meld tile ids (red fives and
 * dora are counted over them, scoring/dora.py:9-22). */
typedef struct rs_winctx {
  uint8_t concealed[34];
  int32_t n_melds;
  rs_meld_rec melds[4];
  int32_t win_tile;
  int32_t tsumo; /* 1 tsumo, 0 ron */
  int32_t seat_wind, round_wind; /* 27..30 */
  int32_t n_ids;
  uint8_t ids[18];
  int32_t riichi, ippatsu, last_tile, rinshan, chankan, first_draw;
  int32_t n_dora;
  uint8_t dora[5];
  int32_t n_ura;
  uint8_t ura[5];
  int32_t rule;
  int32_t kazoe, double_yakuman;
} rs_winctx;

/* score_win (scoring/score.py:45-82) of count contexts (host arrays) on
 * the device: the engine's own scorer (rs_score.cuh score_win, the result
 * record's win entry as settlements write it) in one kernel, one thread
 * per context.  ok[i] = 1 when scored, 0 on NoYakuError (out[i] zeroed).
 * Test and parity entry point; synchronous. */
int rs_debug_score(const rs_winctx* ctx, int64_t count, rs_win_rec* out, int32_t* ok, int32_t device);

/* sizeof of the records above, for binding checks: config, meld, hand,
 * win, result, env, step */
int rs_record_sizes(int32_t* out /*[7]*/);

/* profiling hook: a fused rollout recording, per env and step, the clock64
 * cycles of the auto-reset and of policy + step + observe, the action and
 * flags into prof_dev[steps][n][4] (u32), followed by [n][4] u32 per env:
 * %globaltimer (ns, low 32 bits) at kernel entry, after the table staging,
 * at the env's first step and after its last step */
int rs_debug_rollout_cycles(rs_handle* h, int32_t steps, const rs_obs_out* obs, uint32_t* prof_dev,
                            void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RINSHAN_H */
