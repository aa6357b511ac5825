"""Profiling tool: phase timing of one step (variant build with -DRS_PROFILE_MARKS=2)."""
import os, sys, ctypes as C, torch
os.environ.setdefault('RINSHAN_LIB', 'build_variants/_rinshan_smarks.so')
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
env.rollout(300)
marks = torch.zeros(64 * n * 8 + 8 * 200000, dtype=torch.int64, device='cuda')
env._L.rs_debug_set_marks.argtypes = [C.c_void_p]
env._L.rs_debug_set_marks(marks.data_ptr())
obs = alloc_observations(n, env.device)
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
rows = []
for k in range(30):
    marks.zero_(); flush.fill_(k & 255)
    env.rollout(1, obs=obs, obs_slots=1)
    torch.cuda.synchronize()
    m = marks.view(-1, 8).cpu()
    rows.append(m[(m[:, 0] != 0) & (m[:, 7] != 0)])
mm = torch.cat(rows)
disc = mm[(mm[:, 1] != 0) & (mm[:, 3] != 0)]
def show(nm, a, b, x):
    d = (x[:, b] - x[:, a]).float()
    print('%-28s median %7.0f  p90 %7.0f  max %7.0f (n=%d)' % (nm, d.median(), d.quantile(0.9), d.max(), len(d)))
print('all steps:')
for nm, a, b in (('policy+apply (0-4)', 0, 4), ('legal (4-5)', 4, 5), ('obs+digest (5-6)', 5, 6), ('store+out (6-7)', 6, 7), ('total (0-7)', 0, 7)):
    show(nm, a, b, mm[mm[:, 4] != 0])
print('plain discards (no call phase):')
for nm, a, b in (('policy..finish_hand (0-1)', 0, 1), ('emit+calls+furiten (1-2)', 1, 2), ('discard_stands/draw (2-3)', 2, 3), ('3-4', 3, 4), ('legal (4-5)', 4, 5), ('obs (5-6)', 5, 6), ('store (6-7)', 6, 7), ('total', 0, 7)):
    show(nm, a, b, disc)
