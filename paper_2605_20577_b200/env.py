"""Batched Pgx-style env on B200: `BatchEnv`.

The batched counterpart of the reference env facade (env/core.py:26-94,
env/observe.py:50-124, env/policies.py:17-22, bench/runner.py:25-33,97-121).
State lives on the GPU in the library's structure-of-arrays; the tensors
exposed here (legal mask, current player, rewards, terminated, truncated,
observations) are torch CUDA tensors written in place by the kernels.
Every method is stream-ordered on the current torch stream; nothing is
copied to the host on the step path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import abi
from ._lib import check, lib

_RULES = {"red": abi.RULE_RED, "no-red": abi.RULE_NO_RED}
_MODES = {"single": abi.MODE_SINGLE, "east": abi.MODE_EAST, "half": abi.MODE_HALF}
_SCHEMES = {"score_delta": abi.REWARD_SCORE_DELTA, "rank": abi.REWARD_RANK}


@dataclass(frozen=True)
class EnvConfig:
    """reference env/core.py:26-46 (plus GameConfig flags, engine/types.py:49-57)"""

    rule: str = "red"
    mode: str = "single"
    illegal_penalty: float = -1.0
    reward_scheme: str = "score_delta"
    max_steps: int = 10_000
    kazoe: bool = False
    double_yakuman: bool = False
    agari_yame: bool = True
    renchan_cap: int = 32

    def __post_init__(self):
        if self.rule not in _RULES:
            raise ValueError(f"bad rule {self.rule!r}")
        if self.mode not in _MODES:
            raise ValueError(f"bad mode {self.mode!r}")
        if self.reward_scheme not in _SCHEMES:
            raise ValueError(f"bad reward scheme {self.reward_scheme!r}")
        if self.illegal_penalty > 0:
            raise ValueError("illegal penalty must be <= 0")

    def to_abi(self) -> abi.rs_config:
        return abi.rs_config(
            rule=_RULES[self.rule], mode=_MODES[self.mode], reward_scheme=_SCHEMES[self.reward_scheme],
            illegal_penalty=self.illegal_penalty, max_steps=self.max_steps, kazoe=int(self.kazoe),
            double_yakuman=int(self.double_yakuman), agari_yame=int(self.agari_yame),
            renchan_cap=self.renchan_cap)


def _policy_id(policy: str) -> int:
    ids = {"random": 0, "heuristic": 1}
    if policy not in ids:
        raise ValueError(f"unknown policy {policy!r} (random | heuristic)")
    return ids[policy]


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


OBS_BYTES = 232  # one observation record (rs_obs_out fields) per env


class Observations(dict):
    """Observation tensors keyed like Observation.to_dict() (docs/formats.md:32-52)."""


def alloc_observations(n: int, device, slots: int | None = None) -> Observations:
    lead = (n,) if slots is None else (slots, n)
    kw = dict(device=device)
    return Observations(
        hand_tokens=torch.empty(*lead, 14, dtype=torch.uint8, **kw),
        event_tokens=torch.empty(*lead, 64, 3, dtype=torch.uint8, **kw),
        shanten=torch.empty(*lead, dtype=torch.int8, **kw),
        scores=torch.empty(*lead, 4, dtype=torch.int16, **kw),
        round_wind=torch.empty(*lead, dtype=torch.uint8, **kw),
        seat_wind=torch.empty(*lead, dtype=torch.uint8, **kw),
        kyoku=torch.empty(*lead, dtype=torch.uint8, **kw),
        honba=torch.empty(*lead, dtype=torch.int16, **kw),
        deposits=torch.empty(*lead, dtype=torch.int16, **kw),
        dora_indicator_tokens=torch.empty(*lead, 5, dtype=torch.uint8, **kw),
        live_wall=torch.empty(*lead, dtype=torch.uint8, **kw),
        riichi_flags=torch.empty(*lead, 4, dtype=torch.uint8, **kw),
    )


def alloc_observations_block(n: int, pinned: bool = True, device=None) -> tuple[torch.Tensor, Observations]:
    """one contiguous 232-byte-per-env block (field-major) and the
    observation views into it: pinned host memory by default (the kernels
    write it directly over the host link), else device memory.  The event
    window comes first: write_obs stores it as 16-byte vectors."""
    kw = dict(pin_memory=True) if pinned else dict(device=device)
    buf = torch.zeros(OBS_BYTES * n, dtype=torch.uint8, **kw)
    o, off = {}, 0
    for name, shape, dt in (("event_tokens", (64, 3), torch.uint8), ("hand_tokens", (14,), torch.uint8),
                            ("scores", (4,), torch.int16), ("honba", (), torch.int16),
                            ("deposits", (), torch.int16), ("shanten", (), torch.int8),
                            ("round_wind", (), torch.uint8), ("seat_wind", (), torch.uint8),
                            ("kyoku", (), torch.uint8), ("dora_indicator_tokens", (5,), torch.uint8),
                            ("live_wall", (), torch.uint8), ("riichi_flags", (4,), torch.uint8)):
        size = torch.tensor([], dtype=dt).element_size()
        for d in shape:
            size *= d
        o[name] = buf[off:off + size * n].view(dt).view(n, *shape)
        off += size * n
    assert off == OBS_BYTES * n
    return buf, Observations(o)


def alloc_trajectory(steps: int, n: int, device) -> dict:
    """per-step output buffers of a fused rollout (BatchEnv.rollout traj=)"""
    kw = dict(device=device)
    return {
        "legal_bits": torch.empty(steps, n, 4, dtype=torch.int32, **kw),
        "current_player": torch.empty(steps, n, dtype=torch.int8, **kw),
        "rewards": torch.empty(steps, n, 4, dtype=torch.float32, **kw),
        "terminated": torch.empty(steps, n, dtype=torch.uint8, **kw),
        "truncated": torch.empty(steps, n, dtype=torch.uint8, **kw),
        "status": torch.empty(steps, n, dtype=torch.uint8, **kw),
    }


def obs_struct(o: Observations) -> abi.rs_obs_out:
    return abi.rs_obs_out(
        hand_tokens=_ptr(o["hand_tokens"]), event_tokens=_ptr(o["event_tokens"]),
        shanten=_ptr(o["shanten"]), scores=_ptr(o["scores"]), round_wind=_ptr(o["round_wind"]),
        seat_wind=_ptr(o["seat_wind"]), kyoku=_ptr(o["kyoku"]), honba=_ptr(o["honba"]),
        deposits=_ptr(o["deposits"]), dora_tokens=_ptr(o["dora_indicator_tokens"]),
        live_wall=_ptr(o["live_wall"]), riichi_flags=_ptr(o["riichi_flags"]))


class BatchEnv:
    """`n` independent envs on one GPU (the batched drop-in of mjsim.init/step/observe)."""

    def __init__(self, n: int, config: EnvConfig | None = None, device: str | torch.device = "cuda",
                 **kw):
        if config is None:
            config = EnvConfig(**kw)
        elif kw:
            raise TypeError("pass either config or keyword fields")
        self.config = config
        self.n = int(n)
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise ValueError("BatchEnv runs on a CUDA device (there is no CPU fallback)")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self._L = lib()
        self._cfg = config.to_abi()
        h = C.c_void_p()
        check(self._L.rs_create(C.byref(h), self.n, C.byref(self._cfg), self.device.index), "rs_create")
        self._h = h
        dev = self.device
        self.legal_action_mask = torch.zeros(self.n, abi.NUM_ACTIONS, dtype=torch.bool, device=dev)
        self.legal_bits = torch.zeros(self.n, 4, dtype=torch.int32, device=dev)
        self.current_player = torch.zeros(self.n, dtype=torch.int8, device=dev)
        self.rewards = torch.zeros(self.n, 4, dtype=torch.float32, device=dev)
        self.terminated = torch.zeros(self.n, dtype=torch.bool, device=dev)
        self.truncated = torch.zeros(self.n, dtype=torch.bool, device=dev)
        self.status = torch.zeros(self.n, dtype=torch.uint8, device=dev)
        self._out = abi.rs_step_out(
            legal_mask=_ptr(self.legal_action_mask), legal_bits=_ptr(self.legal_bits),
            current_player=_ptr(self.current_player), rewards=_ptr(self.rewards),
            terminated=_ptr(self.terminated), truncated=_ptr(self.truncated), status=_ptr(self.status))
        self._obs = None

    # -- lifecycle ---------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._L.rs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    @property
    def state_bytes(self) -> int:
        return int(self._L.rs_state_bytes(self._h))

    # -- env API -----------------------------------------------------------
    def init(self, seeds: torch.Tensor | None = None, *, seed: int | None = None,
             index_base: int = 0) -> "BatchEnv":
        """init(seed) for every env.  Either explicit u64 game seeds (a CUDA
        int64 tensor holding the bit patterns), or bench seeding: env i uses
        env_game_seed(seed, index_base + i) and env_policy_state(seed,
        index_base + i) (reference bench/runner.py:25-33)."""
        if seeds is not None:
            seeds = seeds.to(device=self.device, dtype=torch.int64).contiguous()
            if seeds.numel() != self.n:
                raise ValueError("need one seed per env")
            check(self._L.rs_init(self._h, seeds.data_ptr(), C.byref(self._out), self._stream()), "rs_init")
        else:
            s = 0 if seed is None else int(seed) & ((1 << 64) - 1)
            check(self._L.rs_init_indexed(self._h, s, int(index_base), C.byref(self._out), self._stream()),
                  "rs_init_indexed")
        return self

    def step(self, actions: torch.Tensor, *, autoreset: bool | str = False, observe: bool = False,
             next_actions: torch.Tensor | None = None, out: abi.rs_step_out | None = None,
             next_policy: str = "random") -> "BatchEnv":
        """step(state, action) for every env (env/core.py:85-94): illegal ids
        end the episode with the penalty at the offender; stepping a finished
        env sets RS_STATUS_CONTRACT in `status` and changes nothing.

        In the same kernel: `autoreset` restarts finished envs (rewards and
        flags still describe the transition, the mask / player / observation
        belong to the new game); `observe` fills `self.observe()`'s tensors
        for the current players; `next_actions` (int32[n]) receives the
        next action of `next_policy` ("random" or "heuristic"; -1 for
        finished envs).  `autoreset="next"` (needs `next_actions`) instead
        restarts an env finished by an earlier step at the start of this
        one, where it acts with `next_policy` (its action is ignored): the
        reference runner's order (bench/runner.py:107-113)."""
        actions = actions.to(device=self.device, dtype=torch.int32).contiguous()
        if actions.numel() != self.n:
            raise ValueError("need one action per env")
        if autoreset == "next":
            if next_actions is None:
                raise ValueError('autoreset="next" needs next_actions')
            flags = abi.STEP_RESET_FIRST
        else:
            flags = abi.STEP_AUTORESET if autoreset else 0
        flags |= (abi.STEP_OBSERVE if observe else 0) | (abi.STEP_HEURISTIC if _policy_id(next_policy) else 0)
        ost = None
        if observe:
            if self._obs is None:
                self._obs = alloc_observations(self.n, self.device)
            ost = obs_struct(self._obs)
        check(self._L.rs_step_ex(self._h, actions.data_ptr(), flags, C.byref(out if out is not None else self._out),
                                 C.byref(ost) if ost is not None else None, _ptr(next_actions), self._stream()),
              "rs_step_ex")
        return self

    @property
    def observations(self) -> Observations:
        """the tensors `observe()` / `step(observe=True)` write into"""
        if self._obs is None:
            self._obs = alloc_observations(self.n, self.device)
        return self._obs

    def observe(self, seats: torch.Tensor | None = None, out: Observations | None = None) -> Observations:
        """observe(state, seat) for every env; `seats` defaults to each env's
        current player (env/observe.py:81-124)."""
        if out is None:
            if self._obs is None:
                self._obs = alloc_observations(self.n, self.device)
            out = self._obs
        st = obs_struct(out)
        sp = None
        if seats is not None:
            seats = seats.to(device=self.device, dtype=torch.int8).contiguous()
            sp = seats.data_ptr()
        check(self._L.rs_observe(self._h, sp, C.byref(st), self._stream()), "rs_observe")
        return out

    def random_actions(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """random_policy over each env's legal list from its policy stream
        (env/policies.py:17-22); -1 for finished envs."""
        if out is None:
            out = torch.empty(self.n, dtype=torch.int32, device=self.device)
        check(self._L.rs_policy_random(self._h, out.data_ptr(), self._stream()), "rs_policy_random")
        return out

    def heuristic_actions(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """heuristic_policy for every env (env/policies.py:51-109): win,
        riichi, shanten-minimising discard, improving call, else pass; -1
        for finished envs.  Deterministic (no policy stream)."""
        if out is None:
            out = torch.empty(self.n, dtype=torch.int32, device=self.device)
        check(self._L.rs_policy_heuristic(self._h, out.data_ptr(), self._stream()), "rs_policy_heuristic")
        return out

    def check_invariants(self, fast: bool = False, flags: torch.Tensor | None = None) -> torch.Tensor:
        """check_invariants (engine/state.py:105-180) of every env on the
        device: RS_INV_* bits per env (abi.INV_*), OR-ed into `flags` (int32[n])
        when given.  `fast` = the soak suite's per-step subset."""
        if flags is None:
            flags = torch.zeros(self.n, dtype=torch.int32, device=self.device)
        check(self._L.rs_check_invariants(self._h, 1 if fast else 0, flags.data_ptr(), self._stream()),
              "rs_check_invariants")
        return flags

    def soak(self, steps: int, policy: str = "random", fast: bool = False) -> torch.Tensor:
        """bench/runner.py:226-284 play_games on the device: `steps` fused
        steps (auto-reset + policy + step), the invariants checked after
        every one; returns the OR of the RS_INV_* bits per env."""
        flags = self.check_invariants(fast)
        for _ in range(steps):
            self.rollout(1, policy=policy)
            self.check_invariants(fast, flags)
        return flags

    def autoreset(self) -> "BatchEnv":
        """Restart every finished env with its next bench seed
        (bench/runner.py:107-109); the output tensors are refreshed."""
        check(self._L.rs_autoreset(self._h, C.byref(self._out), self._stream()), "rs_autoreset")
        return self

    def rollout(self, steps: int, obs: Observations | None = None, obs_slots: int = 0,
                actions_log: torch.Tensor | None = None, stats: torch.Tensor | None = None,
                digests: torch.Tensor | None = None, policy: str = "random",
                actors_log: torch.Tensor | None = None, traj: dict | None = None) -> "BatchEnv":
        """Fused `steps` x {auto-reset, policy, step, observe} per env in one
        kernel (bench/runner.py:97-121); `policy` is "random" (the bench
        loop) or "heuristic".  stats: int64[3] CUDA tensor (steps,
        games_completed, illegal) accumulated; digests: int64[n];
        actions_log int16[steps, n] / actors_log int8[steps, n]: the action and
        the acting seat of every step (| 4 where an auto-reset preceded it);
        traj: per-step outputs, a dict of [steps, n, ...] CUDA tensors with any
        of legal_bits (int32 [.., 4]), current_player (int8), rewards
        (float32 [.., 4]), terminated / truncated / status (uint8) --
        `alloc_trajectory(steps, n)` makes one."""
        st = obs_struct(obs) if obs is not None else None
        tr = None
        if traj is not None:
            tr = abi.rs_step_out(legal_mask=None, legal_bits=_ptr(traj.get("legal_bits")),
                                 current_player=_ptr(traj.get("current_player")), rewards=_ptr(traj.get("rewards")),
                                 terminated=_ptr(traj.get("terminated")), truncated=_ptr(traj.get("truncated")),
                                 status=_ptr(traj.get("status")))
        check(self._L.rs_rollout_policy(
            self._h, int(steps), _policy_id(policy), C.byref(st) if st is not None else None,
            int(obs_slots if obs is not None else 0), _ptr(actions_log), _ptr(actors_log),
            C.byref(tr) if tr is not None else None, _ptr(stats), _ptr(digests),
            C.byref(self._out), self._stream()), "rs_rollout")
        return self

    # -- projection records (parity harness) ----------------------------------
    def export(self, i: int) -> abi.rs_env_rec:
        torch.cuda.current_stream(self.device).synchronize()
        r = abi.rs_env_rec()
        check(self._L.rs_export_env(self._h, int(i), C.byref(r)), "rs_export_env")
        return r

    def export_many(self, envs) -> list:
        """export() of every env in `envs` (host indices), one launch and one copy"""
        envs = [int(i) for i in envs]
        torch.cuda.current_stream(self.device).synchronize()
        recs = (abi.rs_env_rec * len(envs))()
        idx = (C.c_int64 * len(envs))(*envs)
        check(self._L.rs_export_envs(self._h, idx, len(envs), recs), "rs_export_envs")
        return list(recs)

    def load(self, i: int, rec: abi.rs_env_rec) -> None:
        torch.cuda.current_stream(self.device).synchronize()
        check(self._L.rs_import_env(self._h, int(i), C.byref(rec)), "rs_import_env")


class HostStepper:
    """Host-driven stepping through pinned memory, one CUDA graph per step.

    Per `step()`: the actions in `actions` (pinned int32[n], written by the
    caller) reach the device, one fused kernel steps every env (optionally
    auto-resetting, observing and sampling the random policy's next action),
    and the step result lands in pinned host buffers.  With `zero_copy`
    (default) the kernel reads the actions and writes the result block
    directly in the pinned host buffers (mapped host memory: the bytes cross
    the host link inside the kernel, no copy engines, a one-node graph);
    otherwise an H2D copy, the kernel and a D2H copy are captured into the
    graph.  Either way a step costs one graph launch.

    Host result views (valid after `step()` returns): rewards f32[n,4],
    legal_bits i32[n,4], next_actions i32[n] (contiguous), current_player i8[n],
    terminated / truncated / status u8[n]; with `obs_to_host` (and
    `observe`) also `observations`, the current player's observation of
    every env (observe.py:81-124) in pinned host memory: the kernel writes
    it to a device block and one copy moves the block (232 bytes per env)
    to the host inside the same graph (the kernel writing it over the host
    link directly was ~2x slower: small scattered stores).

    `autoreset`: True resets a finished env in the step that finishes it
    (its result shows the transition, its legal mask / observation / next
    action the new game); "next" (with `policy`) keeps it finished until the
    following step, which starts its next game, draws its action from its
    policy stream (the host action is ignored) and steps it -- the
    reference runner's order (bench/runner.py:107-113) and the same
    trajectories as `BatchEnv.rollout`; False never resets.
    """

    BYTES_PER_ENV = 40

    def __init__(self, env: BatchEnv, *, autoreset: bool = True, observe: bool = True, policy: bool = True,
                 graph: bool = True, zero_copy: bool | str = True, obs_to_host: bool = False):
        n, dev = env.n, env.device
        self.observations = None
        self._obs_host = None
        if obs_to_host:
            if not observe:
                raise ValueError("obs_to_host needs observe=True")
            self._obs_host, self.observations = alloc_observations_block(n, pinned=True)
            self._obs_dev_buf, self._obs_dev = alloc_observations_block(n, pinned=False, device=dev)
        if autoreset not in (True, False, "next"):
            raise ValueError(f"bad autoreset {autoreset!r}")
        if autoreset == "next" and not policy:
            raise ValueError('autoreset="next" needs policy=True (a reset env acts with its own policy)')
        self.env = env
        self.n = n
        self.autoreset, self.observe, self.policy = autoreset, observe, policy
        # "both" (True): actions and results through mapped pinned memory;
        # "actions": actions mapped, results copied D2H; "none" (False): copies
        mode = {True: "both", False: "none"}.get(zero_copy, zero_copy)
        if mode not in ("both", "actions", "none"):
            raise ValueError(f"bad zero_copy mode {zero_copy!r}")
        self.zero_copy = mode
        self.actions = torch.zeros(n, dtype=torch.int32, pin_memory=True)
        self._res_host = torch.zeros(n * self.BYTES_PER_ENV, dtype=torch.uint8, pin_memory=True)
        # the kernel addresses mapped pinned buffers directly (unified addressing)
        self._act_dev = self.actions if mode != "none" else torch.zeros(n, dtype=torch.int32, device=dev)
        self._res_dev = self._res_host if mode == "both" else torch.zeros(n * self.BYTES_PER_ENV, dtype=torch.uint8,
                                                                          device=dev)
        # "both": one rs_step_rec (40 B) per env, written as a burst per env;
        # otherwise field-major arrays (rs_step_out)
        self._packed = mode == "both" and policy  # (the record always carries the next action)
        views = self._rec_views if self._packed else self._views
        d, h = views(self._res_dev), views(self._res_host)
        self.rewards, self.legal_bits, self.next_actions = h["rewards"], h["legal_bits"], h["next_actions"]
        if self._packed:
            # the next actions also as one contiguous pinned int32[n] (what a
            # host loop feeding them back reads; the records hold them too)
            self._next_host = torch.zeros(n, dtype=torch.int32, pin_memory=True)
            self.next_actions = self._next_host
        self.current_player, self.terminated = h["current_player"], h["terminated"]
        self.truncated, self.status = h["truncated"], h["status"]
        self._dev_views = d
        self._out = abi.rs_step_out(
            legal_mask=None, legal_bits=d["legal_bits"].data_ptr(), current_player=d["current_player"].data_ptr(),
            rewards=d["rewards"].data_ptr(), terminated=d["terminated"].data_ptr(),
            truncated=d["truncated"].data_ptr(), status=d["status"].data_ptr())
        self.bytes_h2d = 4 * n
        self.bytes_d2h = self.BYTES_PER_ENV * n + (OBS_BYTES * n if obs_to_host else 0) + (4 * n if self._packed else 0)
        # completion word (rs_set_done_flag): when the kernel itself writes
        # every result into pinned memory, the host polls one word bumped
        # after the step's last store (rs_signal_done, a one-thread kernel in
        # the same graph) instead of sleeping in a stream synchronize (~15 us
        # less per step)
        self._flag = None
        if self._packed:
            self._flag = torch.zeros(1, dtype=torch.int32, pin_memory=True)
            self._flag_np = self._flag.numpy().view(np.uint32)
            check(env._L.rs_set_done_flag(env._h, self._flag.data_ptr()), "rs_set_done_flag")
            self._seq = 0
        self._graph = None
        if graph:
            # no eager warm-up: a step mutates the envs, and nothing in the
            # body needs lazy initialisation (capture does not execute)
            s = torch.cuda.Stream(device=dev)
            s.wait_stream(torch.cuda.current_stream(dev))
            torch.cuda.synchronize(dev)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                self._body()
            self._graph = g
            self._stream = s

    def _flags(self) -> int:
        f = abi.STEP_OBSERVE if self.observe else 0
        if self.autoreset == "next":
            return f | abi.STEP_RESET_FIRST
        return f | (abi.STEP_AUTORESET if self.autoreset else 0)

    def _rec_views(self, buf: torch.Tensor) -> dict:
        """views of an rs_step_rec[n] buffer (include/rinshan.h)"""
        n = self.n
        w = buf.view(torch.int32).view(n, 10)
        b = buf.view(n, 40)
        return {
            "rewards": buf.view(torch.float32).view(n, 10)[:, 0:4],
            "legal_bits": w[:, 4:8],
            "next_actions": w[:, 8],
            "current_player": b[:, 36].view(torch.int8),
            "terminated": b[:, 37],
            "truncated": b[:, 38],
            "status": b[:, 39],
        }

    def _views(self, buf: torch.Tensor) -> dict:
        n = self.n
        return {
            "rewards": buf[0:16 * n].view(torch.float32).view(n, 4),
            "legal_bits": buf[16 * n:32 * n].view(torch.int32).view(n, 4),
            "next_actions": buf[32 * n:36 * n].view(torch.int32),
            "current_player": buf[36 * n:37 * n].view(torch.int8),
            "terminated": buf[37 * n:38 * n],
            "truncated": buf[38 * n:39 * n],
            "status": buf[39 * n:40 * n],
        }

    def _obs_target(self) -> Observations:
        if self.observations is not None:
            return self._obs_dev
        env = self.env
        if env._obs is None:
            env._obs = alloc_observations(env.n, env.device)
        return env._obs

    def _body(self):
        if self._packed:
            env = self.env
            ost = obs_struct(self._obs_target()) if self.observe else None
            flags = self._flags()
            check(env._L.rs_step_rec_out(env._h, self.actions.data_ptr(), flags, self._res_host.data_ptr(),
                                         C.byref(ost) if ost is not None else None, self._next_host.data_ptr(),
                                         env._stream()),
                  "rs_step_rec_out")
            if self.observations is not None:
                self._obs_host.copy_(self._obs_dev_buf, non_blocking=True)
            # the completion word from a one-thread kernel after the step (and
            # the observation copy): the kernel boundary orders every record
            # store before it, cheaper than a system-scope fence in each of
            # the step's warps (RS_STEP_SIGNAL: e2e 86.3 -> 89.3 M, DESIGN §4
            # item 60)
            check(env._L.rs_signal_done(env._h, env._stream()), "rs_signal_done")
            return
        if self.zero_copy != "none":
            env = self.env
            ost = obs_struct(self._obs_target()) if self.observe else None
            flags = self._flags()
            check(env._L.rs_step_ex(env._h, self.actions.data_ptr(), flags, C.byref(self._out),
                                    C.byref(ost) if ost is not None else None,
                                    self._dev_views["next_actions"].data_ptr() if self.policy else None,
                                    env._stream()), "rs_step_ex")
            if self.zero_copy == "actions":
                self._res_host.copy_(self._res_dev, non_blocking=True)
            if self.observations is not None:
                self._obs_host.copy_(self._obs_dev_buf, non_blocking=True)
            return
        self._act_dev.copy_(self.actions, non_blocking=True)
        if self.observations is not None:
            self.env._obs = self._obs_dev
        self.env.step(self._act_dev, autoreset=self.autoreset, observe=self.observe,
                      next_actions=self._dev_views["next_actions"] if self.policy else None, out=self._out)
        self._res_host.copy_(self._res_dev, non_blocking=True)
        if self.observations is not None:
            self._obs_host.copy_(self._obs_dev_buf, non_blocking=True)

    def launch(self):
        """enqueue one step (graph replay) without waiting"""
        if self._graph is not None:
            self._graph.replay()
        else:
            self._body()

    def step(self):
        """one step; returns when the host result views are valid (graph
        replays run on the current stream)"""
        self.launch()
        self.wait()
        return self

    def wait(self):
        """until the launched step's results are in the host views"""
        stream = torch.cuda.current_stream(self.env.device)
        if self._flag is None:
            stream.synchronize()
            return
        target = (self._seq + 1) & 0xFFFFFFFF
        f = self._flag_np
        spins = 0
        while f[0] != target:
            spins += 1
            if spins & 0xFFFFF == 0 and stream.query():  # the stream is idle: surface any fault
                stream.synchronize()
                if f[0] != target:
                    raise RuntimeError("HostStepper: the step finished without signalling completion")
        self._seq = target

    def close(self):
        """drop the captured graph and the completion word (the pinned
        buffers go with the object)"""
        self._graph = None
        if self._flag is not None and getattr(self.env, "_h", None):
            torch.cuda.current_stream(self.env.device).synchronize()
            self.env._L.rs_set_done_flag(self.env._h, None)
            self._flag = None
