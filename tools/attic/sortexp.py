"""Profiling tool (needs the rs_debug_set_order hook, removed after the experiment): does processing envs grouped by their next step's kind
(reset / call phase / turn) cut warp divergence?  Host-side argsort between
launches (untimed) via the rs_debug_set_order hook."""
import sys, ctypes as C, torch
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations
n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
env.rollout(100)
obs = alloc_observations(n, env.device)
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
cls = torch.full((n,), 2, dtype=torch.uint8, device='cuda')
order = torch.arange(n, dtype=torch.int32, device='cuda')
L = env._L
L.rs_debug_set_order.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode in ('identity', 'sorted', 'identity', 'sorted'):
    ts = []
    for i in range(40):
        if mode == 'sorted':
            order.copy_(torch.argsort(cls, stable=True).int())
            L.rs_debug_set_order(env._h, order.data_ptr(), cls.data_ptr())
        else:
            L.rs_debug_set_order(env._h, None, cls.data_ptr())
        flush.fill_(i & 255)
        torch.cuda.synchronize()
        ev0.record(); env.rollout(1, obs=obs, obs_slots=1); ev1.record(); ev1.synchronize()
        ts.append(ev0.elapsed_time(ev1))
    ts.sort()
    c = torch.bincount(cls.long(), minlength=3).tolist()
    print('%-9s n=%d median %.1f us  classes %s' % (mode, n, ts[len(ts)//2] * 1000, c))
