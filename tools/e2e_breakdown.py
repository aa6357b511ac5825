"""Profiling tool: where the e2e (HostStepper) step's time goes at the bench
config, steady state, L2 flushed before every step (the bench protocol).
Device-timed with CUDA events on the current stream:
  rollout  : k_rollout K=1 (the bench `value` launch), device buffers
  step_dev : rs_step_rec_out (the HostStepper kernel) into device buffers
  step_map : the same kernel reading actions / writing results in mapped pinned memory (graph replay)
  e2e      : the bench's e2e step (replay + sync + host copy of the next actions)
  e2e_obs  : e2e with the observations also written to pinned host memory
(not part of the product)"""
import ctypes as C
import statistics as st
import sys

import torch

sys.path.insert(0, '.')
from paper_2605_20577_b200 import abi  # noqa: E402
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, HostStepper, alloc_observations, obs_struct  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream()


def timed(body, k=reps, pre=None):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    for _ in range(5):
        flush.fill_(1)
        body()
    torch.cuda.synchronize()
    for i in range(k):
        flush.fill_(i & 255)
        ev[i][0].record(s)
        body()
        ev[i][1].record(s)
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) * 1000 for a, b in ev]
    return st.mean(t), st.median(t)


env = BatchEnv(n, EnvConfig(rule="no-red"), device=dev).init(seed=0)
obs = alloc_observations(n, dev)
ost = obs_struct(obs)
env.rollout(300, obs=obs, obs_slots=1)
out = abi.rs_step_out(legal_mask=None, legal_bits=env.legal_bits.data_ptr(),
                      current_player=env.current_player.data_ptr(), rewards=env.rewards.data_ptr(),
                      terminated=env.terminated.data_ptr(), truncated=env.truncated.data_ptr(),
                      status=env.status.data_ptr())
res = {}
res["rollout"] = timed(lambda: env._L.rs_rollout(env._h, 1, C.byref(ost), 1, None, None, None, C.byref(out),
                                                 s.cuda_stream))
acts = env.random_actions()
recs = torch.empty(n * 40, dtype=torch.uint8, device=dev)


def step_dev():
    env._L.rs_step_rec_out(env._h, acts.data_ptr(), 18, recs.data_ptr(), C.byref(ost), None, s.cuda_stream)
    acts.copy_(recs.view(torch.int32).view(n, 10)[:, 8])


res["step_dev"] = timed(step_dev)
hs = HostStepper(env, autoreset="next", observe=True, policy=True)
env.random_actions(out=hs._act_dev)
hs.actions.copy_(hs._act_dev.cpu())
def step_map():
    hs.launch()
    s.synchronize()
    hs._seq = int(hs._flag_np[0])


res["step_map"] = timed(step_map)


acts_np, next_np = hs.actions.numpy(), hs.next_actions.numpy()


def e2e():
    hs.step()
    acts_np[:] = next_np


res["e2e"] = timed(e2e)
hs.close()
hs2 = HostStepper(env, autoreset="next", observe=True, policy=True, obs_to_host=True)
hs2.actions.copy_(hs.actions)
a2, n2 = hs2.actions.numpy(), hs2.next_actions.numpy()


def e2e_obs():
    hs2.step()
    a2[:] = n2


res["e2e_obs"] = timed(e2e_obs)
for k, (mean, med) in res.items():
    print("%-9s mean %6.1f us  median %6.1f us  -> %.1f M env steps/s" % (k, mean, med, n / mean))
