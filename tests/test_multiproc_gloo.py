"""World-size-2 runs on CPU (gloo): the env sharding of the multi-GPU path
(paper_2605_20577_b200.dist) yields the same per-env trajectories as one
process, and the statistics reduction adds up.  The per-rank compute here
is the CPU oracle standing in for the GPU (there is none on this box)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, str(ROOT))
    from oracle import mjoracle as O
    from paper_2605_20577_b200 import dist as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    base, n = D.shard(rank, world, 64)
    cfg = O.make_config(rule="red")
    games, digests = O.run_shard(cfg, 13, base, n, 200, digests=True)
    stats = torch.tensor([n * 200, games, 0], dtype=torch.int64)
    D.reduce_stats(stats)
    gathered = [None] * world
    dist.all_gather_object(gathered, (base, digests))
    t = D.max_time(float(rank + 1), "cpu")
    if rank == 0:
        Path(out_path).write_text(json.dumps({"stats": stats.tolist(), "parts": gathered, "tmax": t}))
    dist.destroy_process_group()


def test_two_rank_sharding_matches_single_process(tmp_path):
    from oracle import mjoracle as O

    out = tmp_path / "r.json"
    port = 29500 + os.getpid() % 1000
    mp.spawn(_worker, args=(2, port, str(out)), nprocs=2, join=True)
    res = json.loads(out.read_text())
    games, ref = O.run_shard(O.make_config(rule="red"), 13, 0, 128, 200, digests=True)
    merged = {}
    for base, digests in res["parts"]:
        for j, d in enumerate(digests):
            merged[base + j] = d
    assert [merged[i] for i in range(128)] == ref
    assert res["stats"] == [128 * 200, games, 0]
    assert res["tmax"] == 2.0


def test_split_matches_runner_shards():
    from paper_2605_20577_b200.dist import split
    # runner.py:135-143: base, extra = divmod(batch, workers)
    for total in (1, 7, 64, 1000):
        for w in (1, 2, 3, 8):
            parts = [split(total, w, r) for r in range(w)]
            assert sum(n for _, n in parts) == total
            starts = [s for s, _ in parts]
            assert starts == sorted(starts) and starts[0] == 0
            for (s, n), (s2, _) in zip(parts, parts[1:]):
                assert s + n == s2


@pytest.mark.timeout(300)
def test_bench_reference_arm_under_torchrun():
    """`--impl reference` launched like the driver does for N>1: rank 0
    prints the JSON line, the other rank exits 0."""
    port = 30500 + os.getpid() % 1000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "3", "--warmup", "1", "--batch", "256"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=280, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "env steps/s"
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0
