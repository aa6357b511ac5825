"""Profiling tool: phase timing of win steps (variant build with -DRS_PROFILE_MARKS=4):
win_input, score_win, settlement + records, advance_round (clock64 cycles), L2 flushed
before each K=1 launch.  python tools/marks3.py [n] [launches]"""
import ctypes as C
import os
import sys

import torch

os.environ.setdefault('RINSHAN_LIB', 'build_variants/_rinshan_wmarks.so')
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
launches = int(sys.argv[2]) if len(sys.argv) > 2 else 400
env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
env.rollout(300)
marks = torch.zeros(64 * n * 8 + 8 * 200000, dtype=torch.int64, device='cuda')
env._L.rs_debug_set_marks.argtypes = [C.c_void_p]
env._L.rs_debug_set_marks(marks.data_ptr())
obs = alloc_observations(n, env.device)
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
rows = []
for k in range(launches):
    marks.zero_()
    flush.fill_(k & 255)
    env.rollout(1, obs=obs, obs_slots=1)
    torch.cuda.synchronize()
    m = marks.view(-1, 8).cpu()
    rows.append(m[(m[:, 0] != 0) & (m[:, 4] != 0)])
mm = torch.cat(rows)
print('win steps (lanes): %d' % len(mm))
for nm, a, b in (('win_input', 0, 1), ('score_win', 1, 2), ('settle+records', 2, 3), ('advance_round', 3, 4),
                 ('total', 0, 4)):
    d = (mm[:, b] - mm[:, a]).float()
    print('%-16s median %7.0f  p90 %7.0f  max %7.0f' % (nm, d.median(), d.quantile(0.9), d.max()))
