"""Profiling tool: steady-state K=1 rollout launch time at large batches (after 150 warm steps), L2 flushed."""
import sys, torch
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
for n in [int(x) for x in (sys.argv[1].split(',') if len(sys.argv) > 1 else ['262144', '1048576'])]:
    env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
    obs = alloc_observations(n, env.device)
    for _ in range(150):
        env.rollout(1, obs=obs, obs_slots=1)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(30):
        flush.fill_(i & 255)
        ev0.record(); env.rollout(1, obs=obs, obs_slots=1); ev1.record(); ev1.synchronize()
        ts.append(ev0.elapsed_time(ev1))
    ts.sort()
    print('steady n=%d median %.0f us -> %.0f M env steps/s' % (n, ts[15] * 1000, n / ts[15] / 1000))
    env.close()
