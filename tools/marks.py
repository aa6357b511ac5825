"""Profiling tool: phase timing inside init_game (variant build with -DRS_PROFILE_MARKS)."""
import os, sys, ctypes as C, torch
os.environ.setdefault('RINSHAN_LIB', 'build_variants/_rinshan_marks.so')
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations, obs_struct
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
env.rollout(300)
marks = torch.zeros(200000 * 8, dtype=torch.int64, device='cuda')
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
    sel = m[:, 1] != 0
    mm = m[sel]
    rows.append(mm)
mm = torch.cat(rows)
def show(nm, a, b):
    d = (mm[:, b] - mm[:, a]).float()
    print('%-22s median %8.0f  p90 %8.0f  (n=%d)' % (nm, d.median(), d.quantile(0.9), len(d)))
for nm, a, b in (('shuffle: draws', 1, 0), ('shuffle: swaps+copy', 0, 2), ('deal: hands', 2, 6),
                 ('deal: shanten+store', 6, 7), ('deal: tenpai waits', 7, 3), ('draw', 3, 4), ('legal', 4, 5)):
    show(nm, a, b)
