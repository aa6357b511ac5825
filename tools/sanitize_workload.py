#!/usr/bin/env python
"""Small workload for compute-sanitizer (tools/sanitize.sh): every kernel
family of the library on a few envs -- init, fused rollouts (random and
heuristic, digests, observation and trajectory outputs), k_step with
auto-reset + observe + next action, policy / observe / autoreset alone,
the invariant checker, the bool-mask expansion, export / import, the
device scorer -- under whatever RINSHAN_* knobs the environment sets.
Exits 0 when the oracle agrees (the sanitizer's own exit code carries its
verdict)."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from oracle import mjoracle as O  # noqa: E402
from paper_2605_20577_b200 import _lib  # noqa: E402
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations, alloc_trajectory  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96
steps = 40
for rule in ("no-red", "red"):
    env = BatchEnv(n, EnvConfig(rule=rule)).init(seed=5)
    d = torch.zeros(n, dtype=torch.int64, device="cuda")
    env.rollout(steps, digests=d)
    torch.cuda.synchronize()
    _, ref = O.run_shard(O.make_config(rule=rule), 5, 0, n, steps, digests=True)
    assert [int(x) & ((1 << 64) - 1) for x in d.cpu().tolist()] == ref, rule
    obs = alloc_observations(n, "cuda", slots=8)
    traj = alloc_trajectory(8, n, "cuda")
    env.rollout(8, obs=obs, obs_slots=8, traj=traj, policy="heuristic")
    for _ in range(4):
        env.step(env.random_actions(), autoreset=True, observe=True)
        env.step(env.heuristic_actions(), autoreset=True)
    env.observe()
    env.autoreset()
    flags = env.check_invariants(fast=False)
    mask = env.legal_action_mask
    torch.cuda.synchronize()
    assert int(flags.count_nonzero().item()) == 0
    assert int(mask.sum().item()) > 0
    rec = env.export(0)
    env.load(1, rec)
    recs = env.export_many([0, 1, n - 1])
    assert list(recs[0].scores) == list(recs[1].scores) and recs[0].cursor == recs[1].cursor
    env.close()
# the device scorer on a few fixture contexts
import gzip, json  # noqa: E401,E402
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from paritylib import ctx_from_json  # noqa: E402

cases = json.loads(gzip.open(Path(__file__).resolve().parent.parent / "tests/golden/scoring_rare.json.gz").read())
got = _lib.debug_score([ctx_from_json(c["ctx"], c["kazoe"], c["dy"]) for c in cases[:64]], 0)
assert [w is None for w in got] == [c["want"] is None for c in cases[:64]]
print("sanitize workload ok", n)
