#!/usr/bin/env python
"""Per-function divergence of a kernel from an ncu capture (--set full,
--import-source on, -lineinfo build): the source page's per-line warp
instructions executed and thread instructions executed, attributed to the
enclosing function of the engine source, averaged over the captured
launches.

  python tools/ncu_regions.py gpurun_out/<rep>.ncu-rep --lanes 16 --epw 2 \
      [--out profiles/<tag>.json] [--summary profiles/ncu_rollout_summary.json --batch N --rule R]

For a function, `threads_per_inst` = thread instructions / warp
instructions.  With lane groups (`--lanes` G lanes per env, `--epw` envs
per warp) the G lanes of an env execute together (the same instructions,
redundantly or on split data), so `envs_per_inst` = threads_per_inst / G
is the number of the warp's envs active per warp instruction and
`env_efficiency` = envs_per_inst / epw the fraction of the warp's envs
doing useful work: 1.0 means no divergence between the envs of a warp.
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
FUNC = re.compile(r"^\s{0,2}(?:template\s*<[^>]*>\s*)?(?:RS_HD|RS_HOT|RS_COLD|__device__|__global__|static|inline)"
                  r"[\w\s:<>,\*&()]*?\b(\w+)\s*\(")
REGIONS = {
    # call (claim) resolution: engine.py:498-615
    "claims": ("begin_call_phase", "can_ron", "ron_has_yaku", "apply_call_action", "advance_call_queue",
               "resolve_call_end", "mark_passed_furiten", "discard_stands", "legal_call", "can_chi"),
    # win evaluation and settlement: scoring/*.py, engine.py:764-809
    "scoring": ("score_win", "standard_reading", "seven_pairs_reading", "kokushi_reading", "finalize_reading",
                "make_blocks", "chuuren", "mask_han", "yaku_han_of", "base_points", "situational", "settle",
                "fill_win_rec", "write_win", "win_input", "tsumo_has_yaku", "apply_tsumo", "apply_ron_wins"),
}


def functions_of(path: Path) -> list[tuple[int, str]]:
    out = []
    for i, line in enumerate(path.read_text().splitlines(), 1):
        m = FUNC.match(line)
        if m and not line.rstrip().endswith(";"):
            out.append((i, m.group(1)))
    return out


def owner(funcs, line):
    name = "?"
    for start, f in funcs:
        if start > line:
            break
        name = f
    return name


def parse(rep: str):
    text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                          capture_output=True, text=True, check=True).stdout
    per = collections.defaultdict(lambda: [0.0, 0.0, 0.0])  # (file, func) -> inst, thread inst, samples
    cur, funcs, hdr, launches = None, [], None, 0
    for row in csv.reader(io.StringIO(text)):
        if not row:
            continue
        if row[0] == "File Path":
            cur = Path(row[1])
            funcs = functions_of(cur) if cur.exists() and "paper_2605_20577_b200" in str(cur) else []
            continue
        if row[0] == "Function Name":
            continue
        if row[0] == "Line No":
            hdr = {h: i for i, h in enumerate(row)}
            if cur is not None and cur.name == "rs_abi.cu":
                launches += 1
            continue
        if hdr is None or not row[0].isdigit() or not funcs:
            continue

        def num(k):
            try:
                return float(row[hdr[k]].replace(",", ""))
            except (KeyError, ValueError):
                return 0.0
        f = owner(funcs, int(row[0]))
        acc = per[(cur.name, f)]
        acc[0] += num("Instructions Executed")
        acc[1] += num("Thread Instructions Executed")
        acc[2] += num("Warp Stall Sampling (All Samples)")
    return per, max(launches, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--lanes", type=int, required=True, help="lanes per env (lane group size)")
    ap.add_argument("--epw", type=int, required=True, help="envs per warp")
    ap.add_argument("--out", default="")
    ap.add_argument("--summary", default="", help="also write the bench's ncu summary file")
    ap.add_argument("--batch", type=int)
    ap.add_argument("--rule")
    a = ap.parse_args()
    per, launches = parse(a.rep)
    tot_i = sum(v[0] for v in per.values())
    tot_t = sum(v[1] for v in per.values())

    def stats(keys):
        i = sum(per[k][0] for k in keys)
        t = sum(per[k][1] for k in keys)
        tpi = t / i if i else 0.0
        return {"warp_inst_per_launch": i / launches, "share_of_inst": i / tot_i if tot_i else 0.0,
                "threads_per_inst": tpi, "envs_per_inst": tpi / a.lanes, "env_efficiency": tpi / a.lanes / a.epw}

    funcs = sorted(per, key=lambda k: -per[k][0])
    out = {"report": Path(a.rep).name, "launches": launches, "lanes_per_env": a.lanes, "envs_per_warp": a.epw,
           "kernel": stats(list(per)),
           "regions": {r: dict(stats([k for k in per if k[1] in names]), functions=sorted(
               {k[1] for k in per if k[1] in names})) for r, names in REGIONS.items()},
           "functions": [dict(stats([k]), file=k[0], function=k[1]) for k in funcs[:40]]}
    text = json.dumps(out, indent=1)
    if a.out:
        Path(a.out).write_text(text)
    print(json.dumps({k: out[k] for k in ("kernel", "regions")}, indent=1))
    if a.summary:
        s = json.loads(Path(a.summary).read_text()) if Path(a.summary).exists() else {}
        s.update({"divergence": {"kernel_env_efficiency": out["kernel"]["env_efficiency"],
                                 "claims_env_efficiency": out["regions"]["claims"]["env_efficiency"],
                                 "scoring_env_efficiency": out["regions"]["scoring"]["env_efficiency"],
                                 "envs_per_warp": a.epw, "lanes_per_env": a.lanes,
                                 "definition": "thread instructions / warp instructions / lanes per env / "
                                               "envs per warp, per source region (tools/ncu_regions.py)"}})
        Path(a.summary).write_text(json.dumps(s, indent=1))


if __name__ == "__main__":
    main()
