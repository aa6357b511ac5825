"""Profiling tool: the host side of one e2e (HostStepper) step at the bench
config, steady state, L2 flushed before each step: host timestamps around
the graph replay, the completion-word wait, the actions copy and the end
event record, next to the device-timed step (not part of the product)."""
import statistics as st
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, HostStepper  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
env = BatchEnv(n, EnvConfig(rule="no-red"), device=dev).init(seed=0)
env.rollout(300)
hs = HostStepper(env, autoreset="next", observe=True, policy=True)
env.random_actions(out=hs._act_dev)
hs.actions.copy_(hs._act_dev.cpu())
acts, nxt = hs.actions.numpy(), hs.next_actions.numpy()
s = torch.cuda.current_stream()
rows = []
for i in range(120):
    flush.fill_(i & 255)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter_ns()
    hs.launch()
    t1 = time.perf_counter_ns()
    hs.wait()
    t2 = time.perf_counter_ns()
    acts[:] = nxt
    t3 = time.perf_counter_ns()
    e1.record(s)
    t4 = time.perf_counter_ns()
    e1.synchronize()
    rows.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3, e0.elapsed_time(e1) * 1e6))
rows = rows[20:]
for k, name in enumerate(("replay enqueue", "wait (flag)", "actions copy", "end record call", "device e2e")):
    print("%-16s median %7.1f us" % (name, st.median(r[k] for r in rows) / 1e3))
