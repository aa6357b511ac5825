"""Profiling tool: where a zero-copy HostStepper step's time goes (wall clock, 4096 envs)."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, HostStepper
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
hs = HostStepper(env)
hs.actions.copy_(env.random_actions().cpu())
s = torch.cuda.current_stream()
def timeit(f, k=300):
    for _ in range(20): f()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / k * 1e6
def full():
    hs.step(); hs.actions.copy_(hs.next_actions)
print('step + host copy      %.1f us' % timeit(full))
print('replay only (no sync) %.1f us' % timeit(lambda: hs._graph.replay()))
def rs():
    hs._graph.replay(); s.synchronize()
print('replay + sync         %.1f us' % timeit(rs))
print('empty sync            %.1f us' % timeit(lambda: s.synchronize()))
print('host actions copy     %.1f us' % timeit(lambda: hs.actions.copy_(hs.next_actions)))
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(100):
    ev0.record(); hs._graph.replay(); ev1.record(); ev1.synchronize(); ts.append(ev0.elapsed_time(ev1) * 1000)
ts.sort(); print('graph device time     %.1f us (median)' % ts[50])
