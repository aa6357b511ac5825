#!/bin/bash
# compute-sanitizer is closed on the measurement pool, so memory safety of
# the device paths is checked with a bounds-checked build instead: every
# state-array index, wall position, meld / river slot, hand insert /
# remove, call-queue push / pop and shared-memory scratch / stage offset
# traps on violation (-DRS_BOUNDS, rs_common.cuh RS_CHECK).  The GPU parity
# suite runs against that build under each optional launch path.
#   bash tools/bounds_check.sh  -> gpurun_out/bounds/{summary.txt,*.log}
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/bounds
mkdir -p $out
[ -f build_variants/bounds.so ] || bash tools/build_variant.sh bounds -DRS_BOUNDS
: > $out/summary.txt
T="tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_golden.py tests/test_gpu_scoring.py tests/test_scenarios.py tests/test_gpu_soak.py::test_lane_group_sizes_match_oracle tests/test_gpu_soak.py::test_env_ordering_matches_oracle"
for cfg in "default RINSHAN_X=0" "stage1 RINSHAN_STAGE=1" "stage2 RINSHAN_STAGE=2" "cluster2 RINSHAN_CLUSTER=2" \
           "cluster4 RINSHAN_CLUSTER=4" "order2 RINSHAN_ORDER=2" "nogroups RINSHAN_GROUPS=0" "check RINSHAN_CHECK=1" \
           "prefetch2 RINSHAN_PREFETCH=2"; do
  set -- $cfg
  env RINSHAN_LIB=build_variants/bounds.so RINSHAN_NO_BUILD=1 $2 timeout 900 python -m pytest $T -m gpu -q -x \
      -p no:cacheprovider > $out/$1.log 2>&1
  echo "$1 ($2) rc=$? $(tail -1 $out/$1.log)" | tee -a $out/summary.txt
done
# canary: the bounds build must trap on a deliberate out-of-range wall read
# (k_check with fast == 2 exists only under RS_BOUNDS)
env RINSHAN_LIB=build_variants/bounds.so RINSHAN_NO_BUILD=1 timeout 300 python - > $out/canary.log 2>&1 <<'PY'
import torch
from paper_2605_20577_b200.env import BatchEnv, EnvConfig
env = BatchEnv(64, EnvConfig()).init(seed=1)
flags = torch.zeros(64, dtype=torch.int32, device="cuda")
env._L.rs_check_invariants(env._h, 2, flags.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("canary NOT caught")
PY
rc=$?
if [ $rc -ne 0 ] && ! grep -q "NOT caught" $out/canary.log; then echo "canary trapped (rc=$rc): ok" | tee -a $out/summary.txt
else echo "canary NOT caught" | tee -a $out/summary.txt; fi
