"""Profiling tool: per-env timing inside K=1 launches at steady state (the
bench protocol, L2 flushed before each launch), from rs_debug_rollout_cycles:
the distribution of env end times relative to the first warp's entry
(p50 / p90 / p99 / max per launch, averaged), when the warps start, and the
step+observe cycles per class (p50 / p99 / max).  (not part of the product)"""
import collections
import ctypes as C
import statistics as st
import sys

import torch

sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations, obs_struct  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
launches = int(sys.argv[2]) if len(sys.argv) > 2 else 100
no_flush = len(sys.argv) > 3 and sys.argv[3] == 'noflush'
env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
env.rollout(300)
obs = alloc_observations(n, env.device)
ost = obs_struct(obs)
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
prof = torch.zeros(2 * n * 4, dtype=torch.int32, device='cuda')


def cls_of(a, reset):
    k = ('discard' if a <= 36 else 'riichi' if a == 37 else 'win' if a in (38, 39) else 'call' if a <= 44
         else 'kan' if a <= 112 else 'pass' if a == 113 else 'nine')
    return ('reset+' if reset else '') + k


def q(xs, f):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(f * len(xs)))]


qs = collections.defaultdict(list)
cyc_by = collections.defaultdict(list)
for it in range(launches):
    if not no_flush:
        flush.fill_(it & 255)
    torch.cuda.synchronize()
    env._L.rs_debug_rollout_cycles(env._h, 1, C.byref(ost), prof.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    p = prof.view(2, n, 4).cpu().long()
    cyc, tl = p[0], p[1] & 0xFFFFFFFF
    t0 = int(tl[:, 0].min())
    rel = lambda col: [((int(x) - t0) % (1 << 32)) / 1000 for x in tl[:, col]]  # noqa: E731
    entry, first, end = rel(0), rel(2), rel(3)
    for name, xs in (("entry", entry), ("first step", first), ("end", end)):
        for f in (0.5, 0.9, 0.99, 1.0):
            qs[(name, f)].append(q(xs, f))
    a = (cyc[:, 2] & 255).tolist()
    rs = ((cyc[:, 2] >> 8) & 1).tolist()
    sc = cyc[:, 1].tolist()
    rc = cyc[:, 0].tolist()
    for e in range(n):
        cyc_by[cls_of(a[e], rs[e])].append(sc[e] + rc[e])
print("L2 %s; " % ("warm (no flush)" if no_flush else "flushed") + "n=%d, %d launches; times in us from the first warp's entry (mean over launches)" % (n, launches))
for name in ("entry", "first step", "end"):
    print("  %-10s " % name + "  ".join("p%s %6.2f" % (int(f * 100), st.mean(qs[(name, f)]))
                                        for f in (0.5, 0.9, 0.99, 1.0)))
print("reset+step+observe cycles by class (count/launch, p50, p99, max):")
for k, v in sorted(cyc_by.items(), key=lambda kv: -len(kv[1])):
    print("  %-16s %7.1f  %7d %7d %7d" % (k, len(v) / launches, q(v, 0.5), q(v, 0.99), max(v)))
