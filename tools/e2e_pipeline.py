"""Profiling tool: host-driven stepping of 4096 envs as one HostStepper vs two
pipelined half-batches (2 x 2048 envs on two streams: the host feeds one
half while the GPU steps the other)."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, HostStepper
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps = 200
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')

def single():
    env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
    hs = HostStepper(env)
    hs.actions.copy_(env.random_actions().cpu())
    for _ in range(10):
        hs.step(); hs.actions.copy_(hs.next_actions)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(steps):
        hs.step(); hs.actions.copy_(hs.next_actions)
    torch.cuda.synchronize()
    return n * steps / (time.perf_counter() - t)

def pipelined(parts=2):
    m = n // parts
    envs = [BatchEnv(m, EnvConfig(rule='no-red')).init(seed=0, index_base=i * m) for i in range(parts)]
    streams = [torch.cuda.Stream() for _ in range(parts)]
    hss = []
    for env, s in zip(envs, streams):
        with torch.cuda.stream(s):
            hs = HostStepper(env)
            hs.actions.copy_(env.random_actions().cpu())
        hss.append(hs)
    evs = [torch.cuda.Event() for _ in range(parts)]
    def launch(i):
        with torch.cuda.stream(streams[i]):
            hss[i].launch(); evs[i].record(streams[i])
    for i in range(parts): launch(i)
    def run(k):
        for _ in range(k):
            for i in range(parts):
                evs[i].synchronize()
                hss[i].actions.copy_(hss[i].next_actions)
                launch(i)
    run(10)
    torch.cuda.synchronize(); t = time.perf_counter()
    run(steps)
    torch.cuda.synchronize()
    return n * steps / (time.perf_counter() - t)

for rep in range(2):
    print('single     %.1f M env steps/s' % (single() / 1e6))
    print('pipelined2 %.1f M env steps/s' % (pipelined(2) / 1e6))
    print('pipelined4 %.1f M env steps/s' % (pipelined(4) / 1e6))
