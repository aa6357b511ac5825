"""Profiling tool: where does the e2e step time go? (not part of the product)"""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, HostStepper
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
hs = HostStepper(env)
env.random_actions(out=hs._act_dev); hs.actions.copy_(hs._act_dev.cpu())
def timeit(f, k=200):
    for _ in range(20): f()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / k * 1e6
def full():
    hs.step(); hs.actions.copy_(hs.next_actions)
print('full step+host copy  %.1f us' % timeit(full))
print('graph replay + sync  %.1f us' % timeit(lambda: hs.step()))
s = torch.cuda.current_stream()
def kernel_only():
    env.step(hs._act_dev, autoreset=True, observe=True, next_actions=hs._dev_views['next_actions'], out=hs._out)
    s.synchronize()
print('kernel + sync        %.1f us' % timeit(kernel_only))
def copies():
    hs._act_dev.copy_(hs.actions, non_blocking=True); hs._res_host.copy_(hs._res_dev, non_blocking=True); s.synchronize()
print('H2D + D2H + sync     %.1f us' % timeit(copies))
print('empty sync           %.1f us' % timeit(lambda: s.synchronize()))
print('host actions copy    %.1f us' % timeit(lambda: hs.actions.copy_(hs.next_actions)))
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def kdev():
    ev0.record(); env.step(hs._act_dev, autoreset=True, observe=True, next_actions=hs._dev_views['next_actions'], out=hs._out); ev1.record(); ev1.synchronize(); return ev0.elapsed_time(ev1)
ts = [kdev() for _ in range(100)]
print('kernel device time   %.1f us (median)' % (sorted(ts)[50] * 1000))
from paper_2605_20577_b200.env import alloc_observations
obs = alloc_observations(n, env.device)
def rdev():
    ev0.record(); env.rollout(1, obs=obs, obs_slots=1); ev1.record(); ev1.synchronize(); return ev0.elapsed_time(ev1)
ts = [rdev() for _ in range(100)]
print('rollout K=1 device   %.1f us (median)' % (sorted(ts)[50] * 1000))
def sdev():
    ev0.record(); env.step(hs._act_dev, out=hs._out); ev1.record(); ev1.synchronize(); return ev0.elapsed_time(ev1)
ts = [sdev() for _ in range(100)]
print('plain step device    %.1f us (median)' % (sorted(ts)[50] * 1000))
