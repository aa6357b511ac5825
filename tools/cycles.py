"""Profiling tool: per-env per-step cycle profile of the fused rollout (rs_debug_rollout_cycles)."""
import sys, ctypes as C, torch, collections
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations, obs_struct
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps = 40
env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
env.rollout(50)
obs = alloc_observations(n, env.device); ost = obs_struct(obs)
prof = torch.zeros((steps + 1) * n * 4, dtype=torch.int32, device='cuda')
rc = env._L.rs_debug_rollout_cycles(env._h, steps, C.byref(ost), prof.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
p = prof.view(steps + 1, n, 4)[:steps].cpu().long()
reset_c, step_c, act, flags = p[..., 0], p[..., 1], p[..., 2] & 255, (p[..., 2] >> 8) & 1
print('per env-step cycles: reset (when resetting) median %d max %d; step+obs median %d p99 %d max %d' % (
    reset_c[flags == 1].median(), reset_c[flags == 1].max(), step_c.median(), step_c.float().quantile(0.99), step_c.max()))
tot = reset_c + step_c
print('per-step max over envs (median over steps): %d cycles' % tot.max(dim=1).values.median())
# by action class
cls = collections.defaultdict(list)
for a_, c_ in zip(act.flatten().tolist(), step_c.flatten().tolist()):
    k = 'discard' if a_ <= 36 else ('pass' if a_ == 113 else ('ron/tsumo' if a_ in (38, 39) else ('call' if 40 <= a_ <= 44 else ('riichi' if a_ == 37 else 'kan/other'))))
    cls[k].append(c_)
for k, v in cls.items():
    v.sort(); print('  %-10s n=%6d median %6d p90 %6d max %6d' % (k, len(v), v[len(v)//2], v[int(len(v)*.9)], v[-1]))
