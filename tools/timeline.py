"""Profiling tool: per-env globaltimer timeline of one k_rollout K=1 launch (L2 flushed before)."""
import sys, ctypes as C, torch
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations, obs_struct
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
env.rollout(int(sys.argv[2]) if len(sys.argv) > 2 else 50)
obs = alloc_observations(n, env.device); ost = obs_struct(obs)
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
prof = torch.zeros(2 * n * 4, dtype=torch.int32, device='cuda')
rows = []
for it in range(20):
    flush.fill_(it & 255)
    torch.cuda.synchronize()
    env._L.rs_debug_rollout_cycles(env._h, 1, C.byref(ost), prof.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    p = prof.view(2, n, 4).cpu().long()
    cyc = p[0]
    tl = p[1] & 0xFFFFFFFF
    t0 = tl[:, 0].min()
    tl = (tl - t0) % (1 << 32)
    rows.append((tl, cyc))
import statistics as st
def q(x, f): x = sorted(x); return x[int(f * (len(x) - 1))]
for name, idx in (('entry', 0), ('staged', 1), ('first step', 2), ('end', 3)):
    med = [float(tl[:, idx].float().median()) for tl, _ in rows]
    mx = [float(tl[:, idx].max()) for tl, _ in rows]
    print('%-11s median-over-envs %7.0f ns   max-over-envs %7.0f ns' % (name, st.median(med), st.median(mx)))
stage = [float((tl[:, 1] - tl[:, 0]).float().median()) for tl, _ in rows]
print('staging (per CTA) median %.0f ns' % st.median(stage))
# the slowest envs: were they resetting?
for tl, cyc in rows[:6]:
    end = tl[:, 3]
    top = end.argsort(descending=True)[:5]
    print('slowest envs:', [(int(e), int(end[e]), int(cyc[e, 0]), int(cyc[e, 1]), int(cyc[e, 2]) & 255, (int(cyc[e, 2]) >> 8) & 1) for e in top])
