#!/usr/bin/env python
"""Summarise ncu reports into the tracked evidence files of profiles/.

  python profiles/summarize.py gpurun_out/<report>.ncu-rep <tag> [--batch N --rule R]
      -> profiles/<tag>.json (key metrics, per launch)
  python profiles/summarize.py --launches gpurun_out/<launches>.csv <tag>
      -> profiles/<tag>.json (per-kernel launch counts / device-time shares)
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent

DETAILS = ("Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate",
           "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy",
           "Achieved Active Warps Per SM", "Theoretical Occupancy", "Registers Per Thread", "Grid Size",
           "Block Size", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
           "Executed Instructions", "Branch Efficiency", "Dynamic Shared Memory Per Block", "Stack Size")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "smsp__inst_executed.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
       "sm__warps_active.avg.pct_of_peak_sustained_active")


def ncu_csv(args):
    out = subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def report(rep: str, tag: str, batch: int | None, rule: str | None):
    rows = ncu_csv([rep, "--page", "details"])
    hdr = {h: i for i, h in enumerate(rows[0])}
    launches = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        lid = r[hdr["ID"]]
        names[lid] = r[hdr["Kernel Name"]]
        m = r[hdr["Metric Name"]]
        if m in DETAILS and m not in launches[lid]:
            launches[lid][m] = [r[hdr["Metric Value"]], r[hdr["Metric Unit"]]]
    raw = ncu_csv([rep, "--page", "raw"])
    rh = {h: i for i, h in enumerate(raw[0])}
    units = raw[1]
    for r in raw[2:]:
        lid = r[rh["ID"]]
        for k in RAW:
            if k in rh:
                launches[lid][k] = [r[rh[k]], units[rh[k]]]
    per = []
    for lid in sorted(launches, key=int):
        d = launches[lid]

        def num(k, scale=1.0):
            try:
                v = float(str(d[k][0]).replace(",", ""))
            except (KeyError, ValueError):
                return None
            unit = d[k][1]
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            return v * mult * scale
        per.append({"id": int(lid), "kernel": names[lid].split("(")[0], "metrics": d,
                    "dram_bytes": (num("dram__bytes_read.sum") or 0) + (num("dram__bytes_write.sum") or 0)})
    out = {"report": Path(rep).name, "batch": batch, "rule": rule, "launches": per,
           "dram_bytes_per_launch": sum(p["dram_bytes"] for p in per) / max(len(per), 1)}
    (HERE / f"{tag}.json").write_text(json.dumps(out, indent=1))
    print(json.dumps({k: v for k, v in out.items() if k != "launches"}))


def launch_list(path: str, tag: str):
    text = Path(path).read_text()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = {h: i for i, h in enumerate(rows[0])}
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        if len(r) < len(hdr) or r[hdr["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = r[hdr["Kernel Name"]].split("(")[0]
        v = float(r[hdr["Metric Value"]].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                 "ms": 1e3}.get(r[hdr["Metric Unit"]], 1.0)
        tot[k] += v * scale
        cnt[k] += 1
    total = sum(tot.values())
    out = {"source": Path(path).name, "kernels": [
        {"kernel": k, "launches": cnt[k], "total_us": tot[k], "share": tot[k] / total} for k, _ in tot.most_common()]}
    (HERE / f"{tag}.json").write_text(json.dumps(out, indent=1))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("tag")
    ap.add_argument("--launches", action="store_true")
    ap.add_argument("--batch", type=int)
    ap.add_argument("--rule")
    a = ap.parse_args()
    if a.launches:
        launch_list(a.path, a.tag)
    else:
        report(a.path, a.tag, a.batch, a.rule)
