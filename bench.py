#!/usr/bin/env python
"""Throughput benchmark of the batched Riichi-Mahjong env step on B200.

Metric (BASELINE.json): env steps/sec, random-policy rollout, no-red rule
(`--rule red` for the red-dora rule).  N=1 workload = BASELINE configs[1]:
4096 envs, fused step + observe(current player) + legal mask.  One bench
"step" = one env step of every env in the batch (one launch of the fused
kernel `k_rollout` with K=1: auto-reset, on-device random policy, step,
legal mask, observation).  Multi-GPU: one process per GPU (torchrun),
envs sharded by global index (rank r owns [r*B, (r+1)*B)), no collective
on the step path, one NCCL all_reduce of episode statistics at the end.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "env steps/sec at 1/2/4/8 B200 (no-red & red rules), vs CPU oracle"
UNIT = "env steps/s"
PUBLISHED_8GPU = {"no-red": 2_000_000.0, "red": 1_000_000.0}  # PAPER.md:40,207 (8x A100)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--rule", choices=("no-red", "red"), default="no-red")
    p.add_argument("--mode", choices=("single", "east", "half"), default="single")
    p.add_argument("--batch", type=int, default=4096, help="envs per GPU")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-fused", action="store_true", help="skip the fused 100-step rollout timing")
    p.add_argument("--sweep", type=str, default="",
                   help="comma list of envs/GPU: one extra JSON line each (BASELINE configs[2])")
    p.add_argument("--fuse", type=int, default=1, help="env steps per k_rollout launch in --sweep")
    p.add_argument("--sweep-warm", type=int, default=0,
                   help="untimed env steps before a --sweep timing (0: fresh games, the reference's protocol)")
    return p.parse_args()


def sweep(args):
    """Batch sweep (BASELINE configs[2]): device-timed k_rollout launches of
    `--fuse` env steps each, L2 flushed between launches."""
    import ctypes as C

    import torch

    from paper_2605_20577_b200 import abi
    from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations, obs_struct

    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for n in [int(x) for x in args.sweep.split(",") if x]:
        env = BatchEnv(n, EnvConfig(rule=args.rule, mode=args.mode), device=dev).init(seed=args.seed)
        obs = alloc_observations(n, dev)
        ost = obs_struct(obs)
        out = abi.rs_step_out(legal_mask=None, legal_bits=env.legal_bits.data_ptr(),
                              current_player=env.current_player.data_ptr(), rewards=env.rewards.data_ptr(),
                              terminated=env.terminated.data_ptr(), truncated=env.truncated.data_ptr(),
                              status=env.status.data_ptr())
        stream = torch.cuda.current_stream(dev)
        k = args.fuse

        def launch():
            rc = env._L.rs_rollout(env._h, k, C.byref(ost), 1, None, None, None, C.byref(out), stream.cuda_stream)
            if rc:
                raise RuntimeError(env._L.rs_last_error().decode())

        if args.sweep_warm:
            env.rollout(args.sweep_warm, obs=obs, obs_slots=1)
        for _ in range(3):
            flush.fill_(1)
            launch()
        reps = max(3, min(args.steps, int(2e7 // (n * k)) + 1))
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        torch.cuda.synchronize()
        for i in range(reps):
            flush.fill_(i & 255)
            ev[i][0].record(stream)
            launch()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ev)
        sps = n * k * reps / (ms / 1000)
        S = state_bytes_per_env(env)
        gbs = (2 * S + 272) * n * k / (ms / reps / 1000) / 1e9
        print(json.dumps({"sweep": True, "rule": args.rule, "envs": n, "fuse": k, "warm_steps": args.sweep_warm,
                          "launches": reps,
                          "ms_per_launch": ms / reps, "env_steps_per_s": sps, "hbm_gbs_algorithmic": gbs}),
              flush=True)
        env.close()
        del env
    return 0


def workload(args, n_gpus):
    return {
        "workload": f"{args.rule} {args.mode}, {args.batch} envs/GPU random-policy rollout, fused "
                    f"step+observe+legal mask per env step (BASELINE configs[1])",
        "rule": args.rule,
        "mode": args.mode,
        "envs_per_gpu": args.batch,
        "global_batch": args.batch * n_gpus,
        "env_steps_per_bench_step": args.batch * n_gpus,
        "seed": args.seed,
        "l2": "flushed between timed steps (256 MiB write, untimed)",
        "parallelism": f"env-sharded x{n_gpus} (no step-path collective)",
    }


# ----------------------------------------------------------------- CPU side

def cpu_rollout(args, n_envs, seconds=None, steps=None, warmup=0):
    """The oracle port (oracle/, C) on all host cores: persistent shards of
    bench-seeded envs, each bench step = one env step + observe per env.
    Returns (steps/s, threads, steps done, wall)."""
    from oracle import mjoracle as O

    cfg = O.make_config(rule=args.rule, mode=args.mode)
    threads = max(1, min(os.cpu_count() or 1, n_envs))
    base, extra = divmod(n_envs, threads)
    shards, start = [], 0
    for w in range(threads):
        n = base + (1 if w < extra else 0)
        shards.append(O.OracleBatch(cfg, args.seed, start, n))
        start += n

    def run_all(k):
        ts = [threading.Thread(target=s.step, args=(k, True)) for s in shards]
        for t in ts:
            t.start()
        for t in ts:
            t.join()

    if warmup:
        run_all(warmup)
    done, wall = 0, 0.0
    per_step = []
    while True:
        t0 = time.perf_counter()
        run_all(1)
        dt = time.perf_counter() - t0
        per_step.append(dt)
        wall += dt
        done += 1
        if steps is not None and done >= steps:
            break
        if seconds is not None and wall >= seconds:
            break
    return n_envs * done / wall, threads, done, wall, per_step


def reference_arm(args, rank, world):
    """The reference's CPU path (the oracle port, all host threads) on this
    arm's whole-job workload: world x batch envs per bench step.  Under
    torchrun rank 0 alone runs it; the other ranks exit without work."""
    if rank != 0:
        return 0
    n = args.batch * world
    sps, threads, done, wall, per_step = cpu_rollout(args, n, steps=args.steps, warmup=args.warmup)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": sps,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 * wall / done,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic",
        "config": workload(args, world),
        "cpu_baseline": {
            "value": sps, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{n} envs x {done} bench steps (+{args.warmup} warm-up) of the C oracle "
                      f"port (oracle/mjoracle.c: auto-reset, random policy, step, observe), {threads} threads",
        },
        "e2e": {"value": sps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- GPU side

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def state_bytes_per_env(env):
    """canonical per-env game state S (rs_state_bytes(NULL)): header, scores,
    wall, hands, melds, river, event ring, legal mask"""
    return int(env._L.rs_state_bytes(None))


def ours_arm(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2605_20577_b200 import abi
    from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations, obs_struct

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n = args.batch
    env = BatchEnv(n, EnvConfig(rule=args.rule, mode=args.mode), device=dev)
    env.init(seed=args.seed, index_base=rank * n)
    obs = alloc_observations(n, dev)
    stats = torch.zeros(3, dtype=torch.int64, device=dev)
    # outputs of a bench step: packed legal mask, player, rewards, flags
    out = abi.rs_step_out(legal_mask=None, legal_bits=env.legal_bits.data_ptr(),
                          current_player=env.current_player.data_ptr(), rewards=env.rewards.data_ptr(),
                          terminated=env.terminated.data_ptr(), truncated=env.truncated.data_ptr(),
                          status=env.status.data_ptr())
    ost = obs_struct(obs)
    import ctypes as C
    L, h = env._L, env._h
    stream = torch.cuda.current_stream(dev)

    def launch():
        rc = L.rs_rollout(h, 1, C.byref(ost), 1, None, stats.data_ptr(), None, C.byref(out), stream.cuda_stream)
        if rc:
            raise RuntimeError(L.rs_last_error().decode())

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        flush.fill_(1)
        launch()
    torch.cuda.synchronize()
    stats.zero_()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            flush.fill_(i & 255)
            starts[i].record(stream)
            launch()
            ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    per_launch_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t_ms = sum(per_launch_ms)
    st = stats.clone()
    t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(st, op=dist.ReduceOp.SUM)  # the one NCCL collective: episode stats
    t_max_ms = float(t.item())
    total_steps = int(st[0].item())
    games = int(st[1].item())
    value = total_steps / (t_max_ms / 1000.0)

    # ---- e2e: public API, host-driven actions through pinned memory ----
    e2e = None
    if not args.no_e2e:
        e2e = e2e_run(args, env, dev, world)

    # ---- the same env steps fused 100 per launch ----
    fused = None if args.no_fused else fused_run(args, dev, rank, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sps, threads, done, wall, _ = cpu_rollout(args, n, seconds=args.cpu_seconds, warmup=2)
        cpu = {"value": sps, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{n} envs x {done} bench steps ({wall:.1f} s) of the C oracle port "
                         f"(oracle/mjoracle.c: auto-reset, random policy, step, observe) on {threads} host threads"}

    # ---- roofline of the dominant kernel (k_rollout, K=1) ----
    S = state_bytes_per_env(env)
    O_b, M_b, R_b, A_b = 232, 16, 22, 2  # obs, packed mask, rewards+flags+player+status, action
    b_step = 2 * S + O_b + M_b + R_b + A_b  # B_step = 2S + O + M + R + A
    avg_launch_s = (t_ms / args.steps) / 1000.0
    achieved = b_step * n / avg_launch_s / 1e9
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    traffic = ncu_extra = None
    prof = ROOT / "profiles" / "ncu_rollout_summary.json"
    if prof.exists():
        try:
            pj = json.loads(prof.read_text())
            if pj.get("rule") == args.rule and pj.get("batch") == n:
                traffic = pj.get("dram_bytes_per_launch")
                ls = pj.get("launches") or []
                if ls:  # instructions per step and warp execution efficiency beside the HBM fraction
                    inst = sum(float(x["metrics"]["Executed Instructions"][0]) for x in ls) / len(ls)
                    thr = sum(float(x["metrics"]["Avg. Active Threads Per Warp"][0]) for x in ls) / len(ls)
                    ncu_extra = {"warp_inst_per_env_step": inst / n, "warp_exec_efficiency": thr / 32.0,
                                 "source": "profiles/ncu_rollout_summary.json (" + str(pj.get("report")) + ")"}
        except Exception:
            traffic = ncu_extra = None

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": t_max_ms / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": (value / PUBLISHED_8GPU[args.rule]) if world == 8 else None,
            "dtype": "int32",
            "data": "synthetic",
            "config": workload(args, world),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k_rollout (K=1)", "bytes_per_env_step": b_step,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if peaks else "fallback 6650",
                         "ncu": ncu_extra},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "fused_rollout": fused,
            "clocks": clk.summary(),
            "gpu_launches": args.steps,
            "games_completed": games,
            "launch_ms": {"min": min(per_launch_ms), "median": statistics.median(per_launch_ms),
                          "max": max(per_launch_ms)},
        }
        print(json.dumps(line), flush=True)
    env.close()
    return 0


def fused_run(args, dev, rank, world, k=100):
    """The bench workload as the reference's bench runs it (100 batch steps,
    bench/runner.py:97-121) in one k_rollout launch of k env
    steps per env: auto-reset, random policy, step, legal mask and the
    current player's observation written EVERY step into a [k][n]
    trajectory buffer; fresh envs, a 10-step warm-up launch, then 2 timed
    launches (the same step range as the K=1 timing), L2 flushed between."""
    import torch
    import torch.distributed as dist

    from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations, alloc_trajectory

    n = args.batch
    env = BatchEnv(n, EnvConfig(rule=args.rule, mode=args.mode), device=dev).init(seed=args.seed,
                                                                                   index_base=rank * n)
    obs = alloc_observations(n, dev, slots=k)
    traj = alloc_trajectory(k, n, dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    env.rollout(10, obs=obs, obs_slots=1)
    reps = 2
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda.synchronize()
    for i in range(reps):
        flush.fill_(i & 255)
        ev[i][0].record(stream)
        env.rollout(k, obs=obs, obs_slots=k, traj=traj)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([sum(a.elapsed_time(b) for a, b in ev)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    env.close()
    return {"value": n * world * k * reps / (float(t.item()) / 1000.0), "unit": UNIT, "steps_per_launch": k,
            "launches": reps, "gpu_launches": reps,
            "work": "auto-reset + random policy + step, and every step's outputs (packed legal mask, "
                    "current player, rewards, flags, observation of the current player) written into "
                    "[k][n] trajectory buffers"}


def e2e_run(args, env, dev, world):
    """Same metric through the public API with host buffers
    (paper_2605_20577_b200.HostStepper): per step the host writes the
    actions into pinned memory, one fused kernel reads them across the host
    link, steps every env (auto-reset, observation of the current player,
    the random policy's next action) and writes the result (rewards, flags,
    player, packed legal mask, next action) into pinned host memory; one
    CUDA-graph replay and a stream sync per step.  The host feeds the next
    actions back."""
    import torch
    import torch.distributed as dist

    from paper_2605_20577_b200.env import HostStepper

    n = env.n
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    hs = HostStepper(env, autoreset=True, observe=True, policy=True)
    env.random_actions(out=hs._act_dev)
    hs.actions.copy_(hs._act_dev.cpu())

    def one():
        hs.step()
        hs.actions.copy_(hs.next_actions)  # host-side: the next step's inputs

    for _ in range(max(3, args.warmup)):
        one()
    steps = max(10, args.steps // 2)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(steps):
        flush.fill_(i & 255)
        starts[i].record(stream)
        one()
        ends[i].record(stream)
    torch.cuda.synchronize()
    t_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    value = n * world * steps / (float(t.item()) / 1000.0)
    return {"value": value, "unit": UNIT, "h2d_bytes_per_step": hs.bytes_h2d, "d2h_bytes_per_step": hs.bytes_d2h,
            "api": "HostStepper.step (one-node CUDA graph: the fused step+autoreset+observe+policy kernel "
                   "reads the actions from and writes the result block to mapped pinned host memory)",
            "steps": steps}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "gloo" if args.impl == "reference" else "nccl"
        if args.impl != "reference":
            import torch
            torch.cuda.set_device(local_rank)
        dist.init_process_group(backend=backend)
    try:
        if args.sweep:
            return sweep(args)
        if args.impl == "reference":
            return reference_arm(args, rank, world)
        return ours_arm(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
