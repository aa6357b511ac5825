"""Profiling tool: HostStepper step time per zero-copy mode (both / actions / none), L2 flushed."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, HostStepper
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
for rep in range(2):
    for mode in ("both", "actions", "none"):
        env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
        hs = HostStepper(env, zero_copy=mode)
        a = env.random_actions()
        hs.actions.copy_(a.cpu())
        for _ in range(10):
            hs.step(); hs.actions.copy_(hs.next_actions)
        s = torch.cuda.current_stream()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(100)]
        for i in range(100):
            flush.fill_(i & 255)
            ev[i][0].record(s); hs.step(); hs.actions.copy_(hs.next_actions); ev[i][1].record(s)
        torch.cuda.synchronize()
        ts = sorted(a.elapsed_time(b) for a, b in ev)
        print('%-8s median %.1f us  mean %.1f us  -> %.1f M env steps/s' % (mode, ts[50] * 1000, sum(ts) / len(ts) * 1000, n / (sum(ts) / len(ts) / 1000) / 1e6))
        env.close()
