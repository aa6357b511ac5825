"""Profiling tool: what sets the K=1 launch time (the slowest warp) at steady state.
For each launch: the end time of the slowest env, the classes of the envs in its warp,
and the launch end if every warp holding an env of class X were as fast as the median."""
import sys, ctypes as C, torch, collections, statistics as st
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations, obs_struct
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
launches = int(sys.argv[2]) if len(sys.argv) > 2 else 200
env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
env.rollout(300)
obs = alloc_observations(n, env.device); ost = obs_struct(obs)
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
prof = torch.zeros(2 * n * 4, dtype=torch.int32, device='cuda')
def cls_of(a, reset, phase):
    c = 'reset+' if reset else ''
    if a <= 36: k = 'discard'
    elif a == 37: k = 'riichi'
    elif a in (38, 39): k = 'win'
    elif 40 <= a <= 44: k = 'call'
    elif 45 <= a <= 112: k = 'kan'
    elif a == 113: k = 'pass'
    else: k = 'nine'
    return c + k
top = collections.Counter(); ends = []; without = collections.defaultdict(list)
for it in range(launches):
    flush.fill_(it & 255)
    torch.cuda.synchronize()
    env._L.rs_debug_rollout_cycles(env._h, 1, C.byref(ost), prof.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    p = prof.view(2, n, 4).cpu().long()
    cyc, tl = p[0], p[1] & 0xFFFFFFFF
    t0 = tl[:, 0].min(); end = ((tl[:, 3] - t0) % (1 << 32)).tolist()
    a = (cyc[:, 2] & 255).tolist(); rs = ((cyc[:, 2] >> 8) & 1).tolist(); ph = (cyc[:, 3] & 15).tolist()
    cl = [cls_of(a[e], rs[e], ph[e]) for e in range(n)]
    emax = max(range(n), key=lambda e: end[e])
    ends.append(end[emax])
    # classes present in the slowest env's warp (2 envs per warp at 4096: neighbours share a warp)
    mate = emax ^ 1  # 2 envs per warp at 4096 envs: e and e^1 share a warp
    top[' & '.join(sorted((cl[emax], cl[mate])))] += 1
    for k in ('reset', 'win', 'kan', 'call'):
        without[k + ' (warps)'].append(max(end[e] for e in range(n) if k not in cl[e] and k not in cl[e ^ 1]))
    med = st.median(end)
    for k in set(cl):
        without[k].append(max(end[e] for e in range(n) if cl[e] != k))
print('n=%d launches=%d: slowest-env end median %.1f us (mean %.1f)' % (n, launches, st.median(ends) / 1e3, st.mean(ends) / 1e3))
print('classes of the slowest warp:', dict(top.most_common()))
print('mean launch end with that class removed (all its envs), us:')
for k, v in sorted(without.items(), key=lambda kv: st.mean(kv[1])):
    if len(v) == launches:
        print('  %-16s %.1f' % (k, st.mean(v) / 1e3))
