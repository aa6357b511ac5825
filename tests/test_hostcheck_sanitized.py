"""The engine source under AddressSanitizer + UndefinedBehaviorSanitizer.

compute-sanitizer is closed on the GPU pool this repo is measured on ("runs
under it have left GPUs needing a reset"), so the memory and UB safety of
the transition code is checked on its host build instead: the same
rs_*.cuh source (tests/hostcheck, test only) compiled with
-fsanitize=address,undefined runs the whole hostcheck suite -- random and
heuristic rollouts over every rule and mode against the oracle's digests,
lockstep projections, crafted rare actions and illegal probes, the
invariant checker after every step -- and any heap / stack / global
overflow, use after free, misaligned access, signed overflow, invalid
shift or out-of-bounds index aborts the run.  A canary proves the
instrumentation is live.  (The GPU-only paths -- TMA bulk copies,
mbarriers, cluster multicast, lane-group shuffles -- are covered by the
parity suite under every RINSHAN_* option and the device invariant
checker.)"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HC = ROOT / "tests" / "hostcheck"
SANCXX = "/usr/bin/g++"


def _runtime():
    if not os.path.exists(SANCXX):
        pytest.skip("no system g++ with sanitizer runtimes")
    libs = []
    for name in ("libasan.so", "libubsan.so"):
        p = subprocess.run([SANCXX, f"-print-file-name={name}"], capture_output=True, text=True).stdout.strip()
        if not os.path.isabs(p) or not os.path.exists(p):
            pytest.skip(f"{name} not installed")
        libs.append(p)
    subprocess.check_call(["make", "-s", "-C", str(HC), "libhostcheck_asan.so"])
    return dict(os.environ, LD_PRELOAD=":".join(libs), ASAN_OPTIONS="detect_leaks=0:abort_on_error=1",
                UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1", HOSTCHECK_LIB="libhostcheck_asan.so")


def test_hostcheck_suite_clean_under_asan_ubsan():
    env = _runtime()
    r = subprocess.run([sys.executable, "-m", "pytest", str(ROOT / "tests" / "test_hostcheck.py"), "-x", "-q",
                        "-p", "no:cacheprovider"], capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "Sanitizer" not in r.stderr and "runtime error" not in r.stderr


def test_canary_out_of_bounds_is_caught():
    """exporting env n of an n-env host batch reads past the state
    allocation: the sanitized build must abort with an ASan report"""
    env = _runtime()
    code = (
        "import sys, ctypes as C; sys.path[:0] = [%r, %r]\n"
        "import hc\n"
        "from oracle import mjoracle as O\n"
        "from paper_2605_20577_b200 import abi\n"
        "hb = hc.HostBatch(4, O.make_config())\n"
        "hb.init_indexed(1, 0)\n"
        "rec = abi.rs_env_rec()\n"
        "hb.L.hc_export(hb.p, 4, C.byref(rec))\n"
        "print('not caught')\n" % (str(HC), str(ROOT)))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT, timeout=300)
    assert r.returncode != 0 and "AddressSanitizer" in r.stderr, (r.stdout[-500:], r.stderr[-2000:])
