"""bench.py's multi-rank harness (the N>1 path of BASELINE configs[3]):
rank discovery, the --gpus / WORLD_SIZE check, self-launch under
torch.distributed.run, the env shards (rank r owns global indices
[r*B, (r+1)*B), reference bench/runner.py:135-143), the stats reduction
and max-over-ranks timing, and per-env trajectories equal to one process
over the whole index range (reference tests/test_bench.py:26-42,51-57).
The CPU tests run the reference arm with world size 2 on gloo; the GPU
tests run the GPU arm with two ranks on one B200 over gloo (the ranks'
kernels never wait on each other: no collective on the step path)."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _lines(out: str) -> list[dict]:
    res = []
    for ln in out.splitlines():
        ln = ln.strip()
        if ln.startswith("{"):
            res.append(json.loads(ln))
    return res


def _torchrun(nproc: int, args: list[str], timeout=900) -> subprocess.CompletedProcess:
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py")] + args
    env = dict(os.environ, OMP_NUM_THREADS="1")
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)


def test_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2"], capture_output=True, text=True,
                       env=env, cwd=ROOT, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr


def test_reference_arm_two_ranks_on_gloo():
    """the driver launches --impl reference like our arm: rank 0 alone
    times the whole-job workload (world x batch envs), one JSON line"""
    r = _torchrun(2, ["--impl", "reference", "--gpus", "2", "--steps", "4", "--warmup", "1", "--steady-warm", "20",
                      "--batch", "96", "--no-python-ref"])
    assert r.returncode == 0, r.stderr[-2000:]
    ls = _lines(r.stdout)
    assert len(ls) == 1
    line = ls[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["global_batch"] == 192 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0
    # the same envs stepped by one process: identical games (trajectories
    # depend on the global index only)
    r1 = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "4", "--warmup",
                         "1", "--steady-warm", "20", "--batch", "192", "--no-python-ref"], capture_output=True, text=True,
                        cwd=ROOT, timeout=300)
    assert r1.returncode == 0
    assert _lines(r1.stdout)[0]["games_completed"] == line["games_completed"]


def test_dist_helpers_without_a_group():
    import torch

    from paper_2605_20577_b200 import dist as D

    assert D.shard(1, 4, 4096) == (4096, 4096)
    assert D.gather_objects({"a": 1}) == [{"a": 1}]
    assert D.max_time(3.5, "cpu") == 3.5
    t = torch.tensor([1, 2, 3])
    assert D.reduce_stats(t).tolist() == [1, 2, 3]
    assert D.backend() is None


_SMALL = ["--steps", "6", "--warmup", "2", "--steady-warm", "40", "--no-rows", "--no-cpu-baseline", "--no-fused",
          "--no-e2e", "--digest-steps", "90"]


@pytest.mark.gpu
def test_two_ranks_on_one_gpu_match_one_process(tmp_path):
    """torchrun --nproc-per-node 2 bench.py --gpus 2 --dist-backend gloo on
    one B200: n_gpus 2, global batch 2 x 4096, summed env steps and games,
    and every env's wide trajectory digest equal to a single process over
    the same 8192 global indices"""
    d2, d1 = tmp_path / "d2.json", tmp_path / "d1.json"
    r = _torchrun(2, ["--gpus", "2", "--dist-backend", "gloo", "--batch", "4096", "--digests-out", str(d2)] + _SMALL)
    assert r.returncode == 0, r.stderr[-3000:]
    ls = _lines(r.stdout)
    assert len(ls) == 1, r.stdout[-2000:]
    two = ls[0]
    assert two["n_gpus"] == 2 and two["config"]["global_batch"] == 8192
    assert two["env_steps"] == 8192 * 6 and two["dist"]["backend"] == "gloo"
    r1 = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--batch", "8192", "--digests-out", str(d1)] + _SMALL,
                        capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert r1.returncode == 0, r1.stderr[-3000:]
    one = _lines(r1.stdout)[0]
    assert one["n_gpus"] == 1 and one["env_steps"] == 8192 * 6
    assert one["games_completed"] == two["games_completed"]
    a, b = json.loads(d2.read_text()), json.loads(d1.read_text())
    assert len(a) == 8192 and a == b


@pytest.mark.gpu
def test_gpus_flag_self_launches_torchrun(tmp_path):
    """`python bench.py --gpus 2` outside torchrun launches the ranks itself"""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dist-backend", "gloo",
                        "--batch", "1024"] + _SMALL, capture_output=True, text=True, cwd=ROOT, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    ls = _lines(r.stdout)
    assert len(ls) == 1 and ls[0]["n_gpus"] == 2 and ls[0]["config"]["global_batch"] == 2048
