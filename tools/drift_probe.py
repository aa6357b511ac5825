"""Profiling tool: K=1 launch time over a long run from fresh games (mean per
window of 100 launches, L2 not flushed), sorted (RINSHAN_ORDER=2) or not."""
import statistics as st
import sys

import torch

sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
total = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
env = BatchEnv(n, EnvConfig(rule="no-red")).init(seed=0)
obs = alloc_observations(n, env.device)
s = torch.cuda.current_stream()
times = []
for i in range(total):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    env.rollout(1, obs=obs, obs_slots=1)
    b.record(s)
    b.synchronize()
    times.append(a.elapsed_time(b) * 1000)
print(" ".join("%d:%.0f" % (w, st.mean(times[w:w + 100])) for w in range(0, total, 100)))
