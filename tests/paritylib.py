"""Shared helpers of the parity tests: projections of records compared
field by field between the CUDA path and the CPU oracle."""

from __future__ import annotations

from paper_2605_20577_b200 import records


def projection(rec) -> dict:
    """Everything a record says about the state, excluding the full event /
    result history (compared through the 64-event window and the last
    result; full histories are compared by the fingerprint tests)."""
    d = records.serialize_state(rec, [], [], None)
    d.pop("events")
    d.pop("results")
    d["internal"] = records.internal_fields(rec)
    d["window"] = records.window_events(rec)
    d["last_result"] = records.result_dict(rec.last_result) if rec.n_results else None
    return d


def diff(a: dict, b: dict, path: str = "") -> list[str]:
    out = []
    for k in sorted(set(a) | set(b)):
        va, vb = a.get(k), b.get(k)
        if isinstance(va, dict) and isinstance(vb, dict):
            out += diff(va, vb, f"{path}{k}.")
        elif va != vb:
            out.append(f"{path}{k}: {str(va)[:200]} != {str(vb)[:200]}")
    return out
