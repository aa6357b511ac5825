"""Profiling tool: per-function cycle accumulators (variant build -DRS_PROFILE_MARKS=3), steady state."""
import os, sys, ctypes as C, torch
os.environ.setdefault('RINSHAN_LIB', 'build_variants/_rinshan_acc.so')
sys.path.insert(0, '.')
from paper_2605_20577_b200.env import BatchEnv, EnvConfig, alloc_observations
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 300
env = BatchEnv(n, EnvConfig(rule='no-red')).init(seed=0)
env.rollout(warm)
marks = torch.zeros(8 * 400000, dtype=torch.int64, device='cuda')
env._L.rs_debug_set_marks.argtypes = [C.c_void_p]
env._L.rs_debug_set_marks(marks.data_ptr())
obs = alloc_observations(n, env.device)
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
rows = []
for k in range(40):
    marks.zero_(); flush.fill_(k & 255)
    env.rollout(1, obs=obs, obs_slots=1)
    torch.cuda.synchronize()
    m = marks.view(-1, 8).cpu()
    rows.append(m[m[:, 0] != 0])
mm = torch.cat(rows).double()
names = ['step()', 'score_win', 'compute_waits', 'shanten_minus_kind', 'write_obs', 'init_game', 'random_action', 'finish_hand']
print('n=%d warm=%d, %d env-steps; mean cycles per env-step (share of step()+obs+reset+policy):' % (n, warm, len(mm)))
tot = mm[:, 0] + mm[:, 4] + mm[:, 5] + mm[:, 6]
for i, nm in enumerate(names):
    print('  %-20s mean %8.0f  p99 %8.0f  max %8.0f  frac-nonzero %.3f  share %.3f' % (nm, mm[:, i].mean(), mm[:, i].quantile(0.99), mm[:, i].max(), (mm[:, i] > 0).double().mean(), mm[:, i].sum() / tot.sum()))
# per-warp critical path: max over envs of (step+obs+reset+policy)
print('  total per env-step   mean %8.0f  p99 %8.0f  max %8.0f' % (tot.mean(), tot.quantile(0.99), tot.max()))
# the slow warps: rows are per thread (g_marks[thread][8]); at 4,096 envs a
# warp holds envs 2w (lanes 0-15) and 2w+1 (lanes 16-31); a divergent warp
# runs both envs' paths, and each timer also sees the other env's cycles
if n == 4096:
    per = [m.double().view(-1, 32, 8)[:, [0, 16], :] for m in rows if len(m) == n * 16]
    W = torch.cat(per)                               # [warps][2 envs][8]
    tot_env = W[:, :, 0] + W[:, :, 4] + W[:, :, 5] + W[:, :, 6]
    wt = tot_env.max(1).values
    cut = wt.quantile(0.98)
    sel = W[wt >= cut]
    print('slowest 2%% of warps (%d): max-env total mean %.0f cycles vs all warps %.0f' % (len(sel), wt[wt >= cut].mean(), wt.mean()))
    for i, nm in enumerate(names):
        print('  %-20s slow warps: env-sum mean %8.0f  frac-nonzero %.2f   (all warps %8.0f)' % (
            nm, sel[:, :, i].sum(1).mean(), (sel[:, :, i].sum(1) > 0).double().mean(), W[:, :, i].sum(1).mean()))
