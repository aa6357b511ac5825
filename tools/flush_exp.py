"""Profiling tool: K=1 k_rollout launch time after an L2 flush by writing 256 MB (dirty L2)
vs writing then reading another 256 MB (clean, still cold for the env state)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
obs = alloc_observations(n, env.device)
wbuf = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
rbuf = torch.ones(256 << 20 // 4, dtype=torch.int32, device='cuda')
sink = torch.zeros(1, dtype=torch.int64, device='cuda')
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
env.rollout(20, obs=obs, obs_slots=1)
for mode in ('write', 'write+read', 'none', 'write', 'write+read'):
    ts = []
    for i in range(60):
        if mode != 'none':
            wbuf.fill_(i & 255)
        if mode == 'write+read':
            sink += rbuf.sum()
        ev0.record(); env.rollout(1, obs=obs, obs_slots=1); ev1.record(); ev1.synchronize()
        ts.append(ev0.elapsed_time(ev1) * 1000)
    ts.sort()
    print('%-11s median %.1f us  p10 %.1f  p90 %.1f' % (mode, ts[30], ts[6], ts[54]))
