"""Command line over the device engine, a drop-in for the reference's
`python -m mjsim.cli` (cli.py:1-140): `bench` (the throughput sweep with
the reference's CSV, bench/runner.py:161-226), `selfplay` (one game, its
mjlog-lite log) and `render` (a log position as SVG).  `serve` (the
FastAPI game service) is not provided: the HTTP layer is out of scope
(DESIGN.md §8); `sessions.py` holds the session layer it would serve.

    python -m paper_2605_20577_b200.cli bench --rule no-red --batch 4096 --steps 100
    python -m paper_2605_20577_b200.cli bench --rule red --sweep 1024..1048576
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
from dataclasses import dataclass, field


def parse_sweep(text: str) -> list[int]:
    """cli.py:11-21: 'lo..hi' doubles from lo to hi; 'a,b,c' lists sizes"""
    if ".." in text:
        lo, hi = (int(x) for x in text.split("..", 1))
        sizes = []
        b = lo
        while b <= hi:
            sizes.append(b)
            b *= 2
        return sizes
    return [int(x) for x in text.split(",")]


@dataclass(frozen=True)
class BenchRow:
    """bench/runner.py:48-53"""

    batch: int
    wall_seconds: float
    steps_per_second: float
    games_completed: int


@dataclass(frozen=True)
class BenchReport:
    rows: tuple
    metadata: dict = field(default_factory=dict)


def rollout(rule: str, mode: str, batch: int, steps: int, seed: int, min_duration: float = 0.8,
            device=None) -> BenchRow:
    """bench/runner.py:161-187 on the device: envs 0..batch-1 from their
    first game (env_game_seed / env_policy_state, runner.py:25-33), `steps`
    fused auto-reset + random policy + step per env in one launch.  The
    first pass counts the completed games; passes continue (same envs) until
    `min_duration` of device time accumulated, and the row reports the mean
    pass time, as the reference does with its worker wall time."""
    import torch

    from .env import BatchEnv, EnvConfig

    dev = torch.device(device if device is not None else "cuda")
    cfg = EnvConfig(rule=rule, mode=mode)
    # runner.py:83-94 warms up on a scratch env (index 2^32) outside the
    # measurement; here: module load and first launch
    BatchEnv(1, cfg, device=dev).init(seed=seed, index_base=1 << 32).rollout(2).close()
    env = BatchEnv(batch, cfg, device=dev).init(seed=seed, index_base=0)
    stats = torch.zeros(3, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def one_pass(count: bool) -> float:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        env.rollout(steps, stats=stats if count else None)
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b) / 1000.0

    elapsed = one_pass(True)
    games = int(stats[1].item())
    passes = 1
    while elapsed < min_duration:
        elapsed += one_pass(False)
        passes += 1
    env.close()
    wall = elapsed / passes
    return BenchRow(batch, wall, batch * steps / wall, games)


def sweep(sizes, rule: str = "red", mode: str = "single", steps: int = 100, seed: int = 0,
          min_duration: float = 0.8, device=None) -> BenchReport:
    """bench/runner.py:190-215 (one rollout per batch size), metadata keys
    of the reference plus the device"""
    import torch

    rows = tuple(rollout(rule, mode, b, steps, seed, min_duration, device) for b in sizes)
    dev = torch.device(device if device is not None else "cuda")
    meta = {
        "rule": rule,
        "mode": mode,
        "steps": steps,
        "seed": seed,
        "threads": 1,  # one host thread drives the GPU
        "cpu_count": os.cpu_count(),
        "platform": platform.platform(),
        "python": platform.python_version(),
        "device": torch.cuda.get_device_name(dev),
    }
    return BenchReport(rows, meta)


def report_to_csv(report: BenchReport) -> str:
    """bench/runner.py:218-223"""
    lines = [f"# {k}={v}" for k, v in sorted(report.metadata.items())]
    lines.append("batch,wall_seconds,steps_per_second,games_completed")
    for r in report.rows:
        lines.append(f"{r.batch},{r.wall_seconds:.6f},{r.steps_per_second:.2f},{r.games_completed}")
    return "\n".join(lines) + "\n"


def selfplay_log(rule: str, mode: str, seed: int, policy: str = "random") -> tuple[str, list]:
    """cli.py:38-60: one game from init(seed) with the env-0 policy stream,
    recorded -> (canonical log JSON, final scores)"""
    from . import mjlog, pgx
    from .env import EnvConfig

    config = EnvConfig(rule=rule, mode=mode)
    state = pgx.init(seed, config)
    recorder = mjlog.GameRecorder(config, seed)
    rng = pgx.env_policy_state(seed, 0)
    while not (state.terminated or state.truncated):
        if policy == "heuristic":
            action = pgx.heuristic_policy(state)
        else:
            action, rng = pgx.random_policy(state.legal, rng)
        recorder.record(state, action)
        state = pgx.step(state, action)
    return mjlog.log_to_json(recorder.to_log(state)), [int(x) for x in state.record.scores]


def render_log(log: dict, step: int | None = None, viewer: int | None = None, locale: str = "en") -> str:
    """cli.py:63-77: replay a log (up to `step` actions) and render it"""
    from . import mjlog, render

    state = mjlog.replay_log(log, upto=step)
    return render.to_svg(state, viewer=None if viewer is None or viewer < 0 else viewer, locale=locale)


def _cmd_bench(args) -> int:
    sizes = parse_sweep(args.sweep) if args.sweep else [args.batch]
    csv = report_to_csv(sweep(sizes, args.rule, args.mode, args.steps, args.seed))
    if args.out:
        with open(args.out, "w") as f:
            f.write(csv)
    sys.stdout.write(csv)
    return 0


def _cmd_selfplay(args) -> int:
    text, scores = selfplay_log(args.rule, args.mode, args.seed, args.policy)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text + "\n")
    print(f"scores: {scores}", file=sys.stderr)
    return 0


def _cmd_render(args) -> int:
    with open(args.log) as f:
        log = json.load(f)
    svg = render_log(log, args.step, args.viewer, args.locale)
    if args.out:
        with open(args.out, "w") as f:
            f.write(svg)
    else:
        sys.stdout.write(svg + "\n")
    return 0


def main(argv=None) -> int:
    """cli.py:80-136 (bench / selfplay / render)"""
    parser = argparse.ArgumentParser(prog="paper_2605_20577_b200.cli")
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("bench", help="throughput benchmark (device rollouts)")
    p.add_argument("--rule", choices=["red", "no-red"], default="red")
    p.add_argument("--mode", choices=["single", "east", "half"], default="single")
    p.add_argument("--batch", type=int, default=1024)
    p.add_argument("--sweep", help="e.g. 1024..1048576 (doubling) or 1024,4096")
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--threads", type=int, default=None, help="accepted for compatibility; unused")
    p.add_argument("--out", help="CSV output path")
    p.set_defaults(func=_cmd_bench)

    p = sub.add_parser("selfplay", help="play one game, write its log")
    p.add_argument("--rule", choices=["red", "no-red"], default="red")
    p.add_argument("--mode", choices=["single", "east", "half"], default="single")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--policy", choices=["random", "heuristic"], default="random")
    p.add_argument("--out", help="log JSON path")
    p.set_defaults(func=_cmd_selfplay)

    p = sub.add_parser("render", help="render a log position to SVG")
    p.add_argument("--log", required=True)
    p.add_argument("--step", type=int, default=None, help="actions to replay")
    p.add_argument("--viewer", type=int, default=None, help="seat, omit for omniscient")
    p.add_argument("--locale", choices=["en", "ja"], default="en")
    p.add_argument("--out", help="SVG output path")
    p.set_defaults(func=_cmd_render)

    args = parser.parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())
