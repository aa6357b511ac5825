"""Profiling tool: one fused 100-step rollout launch at N envs with every per-step output (for ncu)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations, alloc_trajectory
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
k = 100
env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
obs = alloc_observations(n, env.device, slots=k)
traj = alloc_trajectory(k, n, env.device)
env.rollout(10, obs=obs, obs_slots=1)
for _ in range(3):
    env.rollout(k, obs=obs, obs_slots=k, traj=traj)
torch.cuda.synchronize()
print('ok')
