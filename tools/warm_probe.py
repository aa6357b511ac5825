"""Profiling tool: what the L2 flush costs the K=1 rollout launch at the
bench config, split into code and data.  Median device time of one
k_rollout step (4,096 envs, steady state) after:
  flush        : the bench protocol (256 MiB write between launches)
  flush+data   : flush, then rs_check_invariants over the same envs
                 (their state and the tables back in L2, the rollout code cold)
  flush+code   : flush, then one rollout step of a second batch
                 (rollout code and tables in L2, the envs' state cold)
  no flush     : back-to-back launches
(not part of the product)"""
import statistics as st
import sys

import torch

sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
env = BatchEnv(n, EnvConfig(rule="no-red"), device=dev).init(seed=0)
env2 = BatchEnv(n, EnvConfig(rule="no-red"), device=dev).init(seed=1)
obs, obs2 = alloc_observations(n, dev), alloc_observations(n, dev)
env.rollout(300, obs=obs, obs_slots=1)
env2.rollout(300, obs=obs2, obs_slots=1)
flags = torch.zeros(n, dtype=torch.int32, device=dev)
s = torch.cuda.current_stream()


def run(pre):
    t = []
    for i in range(reps + 10):
        pre(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        env.rollout(1, obs=obs, obs_slots=1)
        b.record(s)
        b.synchronize()
        if i >= 10:
            t.append(a.elapsed_time(b) * 1000)
    return st.median(t), min(t)


modes = {
    "flush": lambda i: flush.fill_(i & 255),
    "flush+data": lambda i: (flush.fill_(i & 255), env.check_invariants(flags=flags)),
    "flush+code": lambda i: (flush.fill_(i & 255), env2.rollout(1, obs=obs2, obs_slots=1)),
    "no flush": lambda i: None,
}
for k, f in modes.items():
    med, mn = run(f)
    print("%-11s median %6.1f us  min %6.1f us" % (k, med, mn))
