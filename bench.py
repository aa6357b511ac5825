#!/usr/bin/env python
"""Throughput benchmark of the batched Riichi-Mahjong env step on B200.

Metric (BASELINE.json): env steps/sec, random-policy rollout, no-red rule
(`--rule red` for the red-dora rule).  N=1 workload = BASELINE configs[1]:
4096 envs, fused step + observe(current player) + legal mask.  One bench
"step" = one env step of every env in the batch (one launch of the fused
kernel `k_rollout` with K=1: auto-reset, on-device random policy, step,
legal mask, observation).  Before timing, every env is played
`--steady-warm` (default 300) untimed env steps, so the timed steps carry
the steady-state mix of auto-resets, calls and wins (fresh games are all
opening discards); the CPU arm warms the same way.

Multi-GPU: one process per GPU (torchrun; `--gpus N` without torchrun
launches it), envs sharded by global index (rank r owns [r*B, (r+1)*B),
paper_2605_20577_b200.dist), no collective on the step path, one
all_reduce of episode statistics and the max-over-ranks time at the end.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
OBS_BYTES = 232  # observation record (rs_obs_out) per env
# extra configurations measured beside the headline (BASELINE configs[2] /
# configs[3]: the red rule, and the saturating per-GPU batch)
ROWS = (("red", 4096), ("no-red", 1 << 20), ("red", 1 << 20))


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--rule", choices=("no-red", "red"), default="no-red")
    p.add_argument("--mode", choices=("single", "east", "half"), default="single")
    p.add_argument("--batch", type=int, default=4096, help="envs per GPU")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--steady-warm", type=int, default=300,
                   help="untimed env steps per env before timing (steady-state game mix), both arms")
    p.add_argument("--dist-backend", choices=("nccl", "gloo"), default=None,
                   help="torch.distributed backend at N>1 (default: nccl; the reference arm always uses gloo)")
    p.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU baseline sample budget (wall seconds)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-python-ref", action="store_true",
                   help="reference arm: skip timing the Python reference itself (baseline/_ref)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-autoreset", choices=("same", "next"), default="next",
                   help="HostStepper auto-reset in the e2e leg: in the finishing step, or at the start of the next "
                        "(the reference runner's order)")
    p.add_argument("--no-fused", action="store_true", help="skip the fused 100-step rollout timing")
    p.add_argument("--no-rows", action="store_true", help="skip the red / 1M-env extra rows")
    p.add_argument("--row-steps", type=int, default=20, help="timed K=1 launches per extra row")
    p.add_argument("--digests-out", type=str, default="",
                   help="after the bench, roll every env of every rank --digest-steps fused steps from fresh "
                        "games with the wide trajectory digest and write {global index: digest} here (rank 0)")
    p.add_argument("--digest-steps", type=int, default=120)
    p.add_argument("--sweep", type=str, default="",
                   help="comma list of envs/GPU: one extra JSON line each (BASELINE configs[2])")
    p.add_argument("--fuse", type=int, default=1, help="env steps per k_rollout launch in --sweep")
    p.add_argument("--sweep-warm", type=int, default=0,
                   help="untimed env steps before a --sweep timing (0: fresh games, the reference's protocol)")
    return p.parse_args(argv)


# ------------------------------------------------------------ K=1 timing

L2_BYTES = 126 << 20  # B200 L2


def state_exceeds_l2(env) -> bool:
    """the envs' device state alone is larger than L2 (the timing rules'
    alternative to flushing L2 between timed launches)"""
    return env.n * int(env._L.rs_state_bytes(None)) > 4 * L2_BYTES


def timed_launches(env, stats, steps: int, warmup: int, steady_warm: int, dev, barrier=None, flush_l2=True):
    """The bench step: one k_rollout launch of one env step per env (auto-
    reset, random policy, step, legal mask, observation of the current
    player into a device buffer), CUDA events on the launching stream around
    each launch, a 256 MiB write between launches flushing L2 (untimed;
    `flush_l2` False when the state itself is several times the L2).
    Returns the per-launch device times (ms)."""
    import ctypes as C

    import torch

    from paper_2605_20577_b200 import abi
    from paper_2605_20577_b200.env import alloc_observations, obs_struct

    n = env.n
    obs = alloc_observations(n, dev)
    ost = obs_struct(obs)
    out = abi.rs_step_out(legal_mask=None, legal_bits=env.legal_bits.data_ptr(),
                          current_player=env.current_player.data_ptr(), rewards=env.rewards.data_ptr(),
                          terminated=env.terminated.data_ptr(), truncated=env.truncated.data_ptr(),
                          status=env.status.data_ptr())
    L, h = env._L, env._h
    stream = torch.cuda.current_stream(dev)
    sp = stats.data_ptr() if stats is not None else None

    def launch():
        rc = L.rs_rollout(h, 1, C.byref(ost), 1, None, sp, None, C.byref(out), stream.cuda_stream)
        if rc:
            raise RuntimeError(L.rs_last_error().decode())

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    if steady_warm:
        env.rollout(steady_warm, obs=obs, obs_slots=1)  # one fused launch, untimed
    for _ in range(warmup):
        flush.fill_(1)
        launch()
    torch.cuda.synchronize()
    if stats is not None:
        stats.zero_()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    if barrier:
        barrier()
    torch.cuda.synchronize()
    for i in range(steps):
        if flush_l2:
            flush.fill_(i & 255)
        starts[i].record(stream)
        launch()
        ends[i].record(stream)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    del flush
    return [s.elapsed_time(e) for s, e in zip(starts, ends)]


def roofline(S: int, n: int, avg_launch_s: float, peak: float, peak_source: str, traffic=None, extra=None):
    O_b, M_b, R_b, A_b = OBS_BYTES, 16, 22, 2  # obs, packed mask, rewards+flags+player+status, action
    b_step = 2 * S + O_b + M_b + R_b + A_b  # B_step = 2S + O + M + R + A
    achieved = b_step * n / avg_launch_s / 1e9
    r = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
         "traffic": traffic, "kernel": "k_rollout (K=1)", "bytes_per_env_step": b_step, "envs_per_launch": n,
         "peak_source": peak_source}
    if extra:
        r.update(extra)
    return r


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (burst copy)"
    return 6650.0, "fallback 6650 GB/s (B200_PROFILING.md)"


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
        big = state_exceeds_l2(env)
        torch.cuda.synchronize()
        for i in range(reps):
            if not big:
                flush.fill_(i & 255)
            ev[i][0].record(stream)
            launch()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ev)
        sps = n * k * reps / (ms / 1000)
        S = int(env._L.rs_state_bytes(None))
        gbs = (2 * S + 272) * n * k / (ms / reps / 1000) / 1e9
        print(json.dumps({"sweep": True, "rule": args.rule, "envs": n, "fuse": k, "warm_steps": args.sweep_warm,
                          "launches": reps, "l2_flush": not big,
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
        "steady_warm_steps": args.steady_warm,
        "l2": "flushed between timed steps (256 MiB write, untimed)",
        "parallelism": f"env-sharded x{n_gpus} (no step-path collective)",
    }


# ----------------------------------------------------------------- CPU side

def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_rollout(args, n_envs, steps, warm):
    """The reference runner's protocol (bench/runner.py:64-121, 179-182) on
    the C oracle port: the batch split into one shard per host thread
    (runner.py:135-143 `_shards`), each worker steps its envs `warm`
    untimed steps, then runs its whole step budget in ONE call (env-major,
    like one_pass: auto-reset, random policy, step, observe(current
    player)); wall = the slowest worker's stepping section.
    Returns (steps/s, threads, wall, games)."""
    from oracle import mjoracle as O

    cfg = O.make_config(rule=args.rule, mode=args.mode)
    threads = max(1, min(host_threads(), n_envs))
    base, extra = divmod(n_envs, threads)
    shards, start = [], 0
    for w in range(threads):
        n = base + (1 if w < extra else 0)
        shards.append(O.OracleBatch(cfg, args.seed, start, n))
        start += n
    go = threading.Barrier(threads)
    times = [0.0] * threads
    games = [0] * threads

    def worker(i):
        if warm:
            shards[i].step(warm, True)
        go.wait()
        t0 = time.perf_counter()
        games[i] = shards[i].step(steps, True)  # ctypes releases the GIL
        times[i] = time.perf_counter() - t0

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    wall = max(times)
    return n_envs * steps / wall, threads, wall, sum(games)


def cpu_rollout_per_step(args, n_envs, steps, warm):
    """The same work with a barrier after every batch step (step-major: all
    workers finish env step t of every env before step t+1), the shape of
    the GPU's K=1 bench step.  Returns steps/s."""
    from oracle import mjoracle as O

    cfg = O.make_config(rule=args.rule, mode=args.mode)
    threads = max(1, min(host_threads(), n_envs))
    base, extra = divmod(n_envs, threads)
    shards, start = [], 0
    for w in range(threads):
        n = base + (1 if w < extra else 0)
        shards.append(O.OracleBatch(cfg, args.seed, start, n))
        start += n
    bar = threading.Barrier(threads)
    t_start = [0.0]

    def worker(i):
        if warm:
            shards[i].step(warm, True)
        bar.wait()
        if i == 0:
            t_start[0] = time.perf_counter()
        for _ in range(steps):
            shards[i].step(1, True)
            bar.wait()

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return n_envs * steps / (time.perf_counter() - t_start[0])


def cpu_sample_steps(args, n_envs, seconds):
    """steps per env of a CPU sample lasting about `seconds` (a short
    calibration pass first)"""
    sps, _, _, _ = cpu_rollout(args, n_envs, 4, 0)
    return max(5, int(sps * seconds / n_envs))


def reference_arm(args, rank, world):
    """The reference's CPU path (the oracle port, all host threads, the
    reference runner's protocol) on this arm's whole-job workload: world x
    batch envs, `--steady-warm` untimed steps, then --steps timed env steps
    per env.  Under torchrun rank 0 alone runs it; the other ranks exit
    without work."""
    if rank != 0:
        return 0
    n = args.batch * world
    warm = args.steady_warm + args.warmup
    sps, threads, wall, games = cpu_rollout(args, n, args.steps, warm)
    per_step = cpu_rollout_per_step(args, n, min(args.steps, 50), warm)
    pyref = None if args.no_python_ref else python_reference(args, n)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": sps,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 * wall / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic",
        "config": workload(args, world),
        "cpu_baseline": {
            "value": sps, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{n} envs x {args.steps} env steps each after {warm} untimed steps, the C oracle port "
                      f"(oracle/mjoracle.c: auto-reset, random policy, step, observe) in the reference "
                      f"runner's protocol (one shard per thread, env-major, one call per worker; wall = "
                      f"slowest worker), {threads} threads",
        },
        "per_step_barrier": {"value": per_step, "unit": UNIT,
                             "protocol": "the same shards step-major with a barrier after every batch step"},
        "games_completed": games,
        "python_reference": pyref,
        "e2e": {"value": sps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def python_reference(args, n):
    """The Python reference itself (mjsim, installed into baseline/_ref from
    /root/reference with pip --no-index), its own bench CLI on this box's
    cores: `python -m mjsim.cli bench --batch n --steps 100` (the paper's
    100 batch steps, fresh games, the runner's 0.25 s warm-up).  For
    context beside the oracle port, which is the arm's value."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "mjsim" / "__init__.py").exists():
        return {"unavailable": "baseline/_ref not installed (pip install --no-index --target baseline/_ref <reference>)"}
    threads = host_threads()
    env = dict(os.environ, PYTHONPATH=str(ref), MJSIM_TABLE_PATH="/tmp/mjsim_ref_tables/suit_tables.bin",
               NUMBA_CACHE_DIR="/tmp/mjsim_ref_numba")
    cmd = [sys.executable, "-m", "mjsim.cli", "bench", "--rule", args.rule, "--mode", args.mode, "--batch", str(n),
           "--steps", "100", "--seed", str(args.seed), "--threads", str(threads)]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=240, env=env).stdout
        row = [ln for ln in out.splitlines() if ln and not ln.startswith("#") and not ln.startswith("batch")][-1]
        batch, wall, sps, games = row.split(",")
        return {"value": float(sps), "unit": UNIT, "cores": threads, "wall_seconds": float(wall),
                "games_completed": int(games), "sample": f"{n} envs x 100 env steps, fresh games",
                "cmd": "python -m mjsim.cli bench --rule %s --mode %s --batch %d --steps 100 --threads %d"
                       % (args.rule, args.mode, n, threads)}
    except (subprocess.TimeoutExpired, IndexError, ValueError) as e:
        return {"unavailable": f"mjsim bench failed: {type(e).__name__}"}


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


def ncu_summary(rule: str, n: int):
    """DRAM traffic per launch and the divergence figures of the committed
    ncu capture of this configuration (profiles/ncu_rollout_summary.json)"""
    prof = ROOT / "profiles" / "ncu_rollout_summary.json"
    if not prof.exists():
        return None, None
    try:
        pj = json.loads(prof.read_text())
    except ValueError:
        return None, None
    if pj.get("rule") != rule or pj.get("batch") != n:
        return None, None
    extra = {k: pj[k] for k in ("warp_inst_per_env_step", "branch_efficiency", "divergence") if k in pj}
    extra["source"] = "profiles/ncu_rollout_summary.json (" + str(pj.get("report")) + ")"
    return pj.get("dram_bytes_per_launch"), {"ncu": extra}


def ours_arm(args, rank, world, local_rank):
    import torch

    from paper_2605_20577_b200 import dist as D
    from paper_2605_20577_b200.env import BatchEnv, EnvConfig

    dev = D.device(local_rank)
    torch.cuda.set_device(dev)
    base, n = D.shard(rank, world, args.batch)
    env = BatchEnv(n, EnvConfig(rule=args.rule, mode=args.mode), device=dev).init(seed=args.seed, index_base=base)
    stats = torch.zeros(3, dtype=torch.int64, device=dev)
    barrier = D.barrier if world > 1 else None
    with ClockSampler(dev.index) as clk:
        per_launch_ms = timed_launches(env, stats, args.steps, args.warmup, args.steady_warm, dev, barrier)
    t_ms = sum(per_launch_ms)
    t_max_ms = D.max_time(t_ms, dev)
    D.reduce_stats(stats)  # the one collective: episode statistics
    total_steps, games = int(stats[0].item()), int(stats[1].item())
    value = total_steps / (t_max_ms / 1000.0)
    S = int(env._L.rs_state_bytes(None))
    peak, peak_source = peaks()
    traffic, extra = ncu_summary(args.rule, n)
    line_roof = roofline(S, n, (t_ms / args.steps) / 1000.0, peak, peak_source, traffic, extra)

    # ---- e2e: public API, host buffers, copies inside the timed region ----
    e2e = None
    if not args.no_e2e:
        e2e = e2e_run(args, env, dev, world, obs_to_host=False)
        e2e["with_observation"] = e2e_run(args, env, dev, world, obs_to_host=True)
    env.close()

    # ---- the same env steps fused 100 per launch ----
    fused = None if args.no_fused else fused_run(args, dev, rank, world, base)

    # ---- red rule and the saturating batch (BASELINE configs[2], [3]) ----
    rows = None if args.no_rows else rows_run(args, dev, rank, world, peak, peak_source, barrier)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        k = cpu_sample_steps(args, n, args.cpu_seconds)
        sps, threads, wall, _ = cpu_rollout(args, n, k, args.steady_warm)
        cpu = {"value": sps, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{n} envs x {k} env steps each ({wall:.1f} s, after {args.steady_warm} untimed steps) "
                         f"of the C oracle port (oracle/mjoracle.c: auto-reset, random policy, step, observe) in "
                         f"the reference runner's protocol on {threads} host threads"}

    digests = None
    if args.digests_out:
        digests = digests_run(args, dev, rank, world, base, n)

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
            "roofline": line_roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "fused_rollout": fused,
            "rows": rows,
            "clocks": clk.summary(),
            "gpu_launches": args.steps,
            "games_completed": games,
            "env_steps": total_steps,
            "launch_ms": {"min": min(per_launch_ms), "median": statistics.median(per_launch_ms),
                          "max": max(per_launch_ms)},
            "dist": {"world": world, "backend": D.backend(), "index_base_rank0": 0},
        }
        if digests is not None:
            Path(args.digests_out).write_text(json.dumps(digests))
            line["digests_out"] = {"path": args.digests_out, "envs": len(digests), "steps": args.digest_steps}
    # the other ranks wait while rank 0 prints its line (no log lines of
    # theirs -- NCCL INFO goes to stdout -- can land inside it)
    if world > 1:
        D.barrier()
    if rank == 0:
        sys.stdout.flush()
        os.write(1, (json.dumps(line, separators=(",", ":")) + "\n").encode())
    if world > 1:
        D.barrier()
    return 0


def rows_run(args, dev, rank, world, peak, peak_source, barrier):
    """Extra K=1 rows beside the headline, each with its own roofline: the
    red rule at the bench batch and both rules at 2^20 envs/GPU (the
    saturating batch), same protocol (steady warm, L2 flushed, max over
    ranks)."""
    import torch

    from paper_2605_20577_b200 import dist as D
    from paper_2605_20577_b200.env import BatchEnv, EnvConfig

    out = []
    for rule, n in ROWS:
        if rule == args.rule and n == args.batch:
            continue
        env = BatchEnv(n, EnvConfig(rule=rule, mode=args.mode), device=dev).init(seed=args.seed,
                                                                                  index_base=rank * n)
        stats = torch.zeros(3, dtype=torch.int64, device=dev)
        big = state_exceeds_l2(env)
        ms = timed_launches(env, stats, args.row_steps, 3, args.steady_warm, dev, barrier, flush_l2=not big)
        t = D.max_time(sum(ms), dev)
        D.reduce_stats(stats)
        S = int(env._L.rs_state_bytes(None))
        traffic, _ = ncu_summary(rule, n)
        out.append({"rule": rule, "envs_per_gpu": n, "global_batch": n * world,
                    "l2": "state larger than L2 (%.1f GB), no flush" % (n * S / 1e9) if big
                          else "flushed between timed steps",
                    "value": int(stats[0].item()) / (t / 1000.0), "unit": UNIT,
                    "ms_per_step": t / args.row_steps, "steps": args.row_steps,
                    "games_completed": int(stats[1].item()),
                    "roofline": {k: v for k, v in roofline(S, n, (sum(ms) / args.row_steps) / 1000.0, peak, peak_source,
                                                           traffic).items()
                                 if k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "bytes_per_env_step")}})
        env.close()
        del env
        torch.cuda.empty_cache()
    return out


def fused_run(args, dev, rank, world, base, k=100):
    """The bench workload as the reference's bench runs it (100 batch steps,
    bench/runner.py:97-121) in one k_rollout launch of k env
    steps per env: auto-reset, random policy, step, legal mask and the
    current player's observation written EVERY step into a [k][n]
    trajectory buffer; steady-state envs, then 2 timed launches, L2
    flushed between."""
    import torch

    from paper_2605_20577_b200 import dist as D
    from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations, alloc_trajectory

    n = args.batch
    env = BatchEnv(n, EnvConfig(rule=args.rule, mode=args.mode), device=dev).init(seed=args.seed, index_base=base)
    obs = alloc_observations(n, dev, slots=k)
    traj = alloc_trajectory(k, n, dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    env.rollout(max(10, args.steady_warm), obs=obs, obs_slots=1)
    reps = 2
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda.synchronize()
    for i in range(reps):
        flush.fill_(i & 255)
        ev[i][0].record(stream)
        env.rollout(k, obs=obs, obs_slots=k, traj=traj)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    t = D.max_time(sum(a.elapsed_time(b) for a, b in ev), dev)
    env.close()
    return {"value": n * world * k * reps / (t / 1000.0), "unit": UNIT, "steps_per_launch": k,
            "launches": reps, "gpu_launches": reps,
            "work": "auto-reset + random policy + step, and every step's outputs (packed legal mask, "
                    "current player, rewards, flags, observation of the current player) written into "
                    "[k][n] trajectory buffers"}


def e2e_run(args, env, dev, world, obs_to_host: bool):
    """Same metric through the public API with host buffers
    (paper_2605_20577_b200.HostStepper): per step the host writes the
    actions into pinned memory, one fused kernel reads them across the host
    link, steps every env (auto-reset, observation of the current player,
    the random policy's next action) and writes the result (rewards, flags,
    player, packed legal mask, next action) -- and with `obs_to_host` the
    232-byte observation of every env -- into pinned host memory; one
    CUDA-graph replay per step, the host waiting on the completion word the
    kernel writes after its last result store.  The host feeds the next
    actions back.  >= 100 timed steps."""
    import torch

    from paper_2605_20577_b200 import dist as D
    from paper_2605_20577_b200.env import HostStepper

    n = env.n
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    autoreset = {"same": True, "next": "next"}[args.e2e_autoreset]
    hs = HostStepper(env, autoreset=autoreset, observe=True, policy=True, obs_to_host=obs_to_host)
    env.random_actions(out=hs._act_dev)
    hs.actions.copy_(hs._act_dev.cpu())
    acts, nxt = hs.actions.numpy(), hs.next_actions.numpy()  # views of the pinned buffers

    def one():
        hs.step()
        acts[:] = nxt  # host-side: the next step's inputs

    for _ in range(max(3, args.warmup)):
        one()
    steps = max(100, args.steps)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    if world > 1:
        D.barrier()
    torch.cuda.synchronize()
    for i in range(steps):
        flush.fill_(i & 255)
        starts[i].record(stream)
        one()
        ends[i].record(stream)
    torch.cuda.synchronize()
    t = D.max_time(sum(s.elapsed_time(e) for s, e in zip(starts, ends)), dev)
    value = n * world * steps / (t / 1000.0)
    res = {"value": value, "unit": UNIT, "h2d_bytes_per_step": hs.bytes_h2d, "d2h_bytes_per_step": hs.bytes_d2h,
           "steps": steps}
    if not obs_to_host:
        res["api"] = ("HostStepper.step: one CUDA-graph replay per step; the fused step+autoreset+observe+policy "
                      "kernel reads the actions from and writes its results to pinned host memory")
        res["autoreset"] = ("next step: a finished env starts its next game at the start of the following step, "
                            "the reference runner's order (bench/runner.py:107-113)" if autoreset == "next" else
                            "same step: a finished env starts its next game in the step that finishes it")
    hs.close()
    return res


def digests_run(args, dev, rank, world, base, n):
    """every env of this rank rolled --digest-steps fused steps from fresh
    games with the wide trajectory digest; gathered on rank 0 as {global
    index: digest} (the sharded run must equal one process over the whole
    index range)"""
    import torch

    from paper_2605_20577_b200 import dist as D
    from paper_2605_20577_b200.env import BatchEnv, EnvConfig

    env = BatchEnv(n, EnvConfig(rule=args.rule, mode=args.mode), device=dev).init(seed=args.seed, index_base=base)
    d = torch.zeros(n, dtype=torch.int64, device=dev)
    env.rollout(args.digest_steps, digests=d)
    torch.cuda.synchronize()
    mine = {base + i: int(x) & ((1 << 64) - 1) for i, x in enumerate(d.cpu().tolist())}
    env.close()
    parts = D.gather_objects(mine)
    if rank != 0:
        return None
    merged = {}
    for p in parts:
        merged.update(p)
    return {str(k): merged[k] for k in sorted(merged)}


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args) -> int:
    """`--gpus N` (N > 1) outside torchrun: run this script under
    torch.distributed.run with N local ranks (the driver's launch)"""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(Path(__file__).resolve())]
    cmd += sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    from paper_2605_20577_b200 import dist as D

    rank, world, local_rank = D.world()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    if args.gpus != world:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU "
              f"(torchrun --nproc-per-node {args.gpus}) or drop --gpus", file=sys.stderr)
        return 2
    if world > 1:
        backend = "gloo" if args.impl == "reference" else (args.dist_backend or "nccl")
        D.init(backend, local_rank)
    try:
        if args.sweep:
            return sweep(args)
        if args.impl == "reference":
            return reference_arm(args, rank, world)
        return ours_arm(args, rank, world, local_rank)
    finally:
        D.finish()


if __name__ == "__main__":
    sys.exit(main())
