"""Profiling tool: steady-state device time of k_step (HostStepper kernel) and k_rollout K=1, L2 flushed."""
import sys, torch
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, HostStepper, alloc_observations
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
hs = HostStepper(env)
obs = alloc_observations(n, env.device)
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
env.rollout(300)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
env.random_actions(out=hs._act_dev)
def kstep():
    ev0.record(); env.step(hs._act_dev, autoreset=True, observe=True, next_actions=hs._act_dev, out=hs._out); ev1.record(); ev1.synchronize(); return ev0.elapsed_time(ev1)
def roll():
    ev0.record(); env.rollout(1, obs=obs, obs_slots=1); ev1.record(); ev1.synchronize(); return ev0.elapsed_time(ev1)
for name, f in (('k_step', kstep), ('rollout', roll), ('k_step', kstep), ('rollout', roll)):
    ts = []
    for i in range(150):
        flush.fill_(i & 255); torch.cuda.synchronize()
        ts.append(f())
    ts.sort()
    print('%-8s n=%d median %.1f us  p10 %.1f  p90 %.1f' % (name, n, ts[75] * 1000, ts[15] * 1000, ts[135] * 1000))
