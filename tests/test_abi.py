"""The C-ABI library (no GPU needed): it loads, exports every entry point
declared in include/rinshan.h, its records match the ctypes mirrors, and
its host-built tables reproduce the reference blob."""

from __future__ import annotations

import ctypes as C
import random
import re
from pathlib import Path

from oracle import mjoracle as O
from paper_2605_20577_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "rinshan.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(rs_\w+)\s*\(", text, re.M)))


def test_every_declared_symbol_is_exported():
    L = _lib.lib()
    names = declared()
    assert "rs_step" in names and "rs_rollout" in names and len(names) >= 20
    for name in names:
        assert hasattr(L, name), name
    assert sorted(_lib.SYMBOLS) == names


def test_record_sizes_match_ctypes():
    assert _lib.record_sizes() == _lib.ctypes_record_sizes()


def test_tables_crc_and_geometry():
    L = _lib.lib()
    crc = C.c_uint32()
    assert L.rs_tables_crc(C.byref(crc)) == 0
    assert crc.value == 0x33D1141E  # CRC of the reference's suit-table blob
    v = [C.c_int32() for _ in range(4)]
    L.rs_tables_info(*[C.byref(x) for x in v])
    assert [x.value for x in v] == [70, 25, 95, 84]


def test_factored_standard_shanten_matches_oracle():
    """(class_m, class_p) x (class_s, class_z) pre-merged tables == the
    reference's sequential budget merge (hand/shanten.py:30-63)."""
    L = _lib.lib()
    rnd = random.Random(5)
    out = C.c_int32()
    for _ in range(4000):
        melds = rnd.randrange(5)
        size = rnd.choice([13, 14]) - 3 * melds
        counts = [0] * 34
        while sum(counts) < size:
            k = rnd.randrange(34)
            if counts[k] < 4:
                counts[k] += 1
        codes = [0, 0, 0, 0]
        for i in range(9):
            codes[0] = codes[0] * 5 + counts[i]
            codes[1] = codes[1] * 5 + counts[9 + i]
            codes[2] = codes[2] * 5 + counts[18 + i]
        for i in range(7):
            codes[3] = codes[3] * 5 + counts[27 + i]
        assert L.rs_tables_shanten_std(*codes, melds, C.byref(out)) == 0
        assert out.value == O.lib().orc_shanten_standard((C.c_uint8 * 34)(*counts), melds)


def test_blob_roundtrip_and_corruption_rejected():
    L = _lib.lib()
    size = C.c_int64()
    L.rs_tables_blob(None, 0, C.byref(size))
    buf = (C.c_uint8 * size.value)()
    L.rs_tables_blob(buf, size.value, C.byref(size))
    blob = bytes(buf)
    assert blob == O.tables_blob()  # product builder == oracle restatement, byte for byte
    assert L.rs_tables_load(blob, len(blob)) == 0
    bad = bytearray(blob)
    bad[1000] ^= 1
    assert L.rs_tables_load(bytes(bad), len(bad)) != 0
    assert b"crc" in L.rs_last_error()


def test_create_rejects_bad_config_without_gpu():
    L = _lib.lib()
    from paper_2605_20577_b200 import abi
    h = C.c_void_p()
    cfg = abi.rs_config(rule=7, mode=0, reward_scheme=0, illegal_penalty=-1.0, max_steps=100,
                        kazoe=0, double_yakuman=0, agari_yame=1, renchan_cap=32)
    assert L.rs_create(C.byref(h), 16, C.byref(cfg), 0) != 0
    assert L.rs_state_bytes(None) == 976


def test_python_constants_match_the_header():
    """abi.py's step flags and status codes are the header's #defines"""
    from paper_2605_20577_b200 import abi

    text = (Path(__file__).resolve().parent.parent / "include" / "rinshan.h").read_text()
    defs = {m.group(1): int(m.group(2).strip("()").replace("-2147483647 - 1", str(-2**31)))
            for m in re.finditer(r"#define (RS_(?:STEP|E)_[A-Z_]+) (\(?-?[0-9]+\)?)", text)}
    want = {"RS_STEP_AUTORESET": abi.STEP_AUTORESET, "RS_STEP_OBSERVE": abi.STEP_OBSERVE,
            "RS_STEP_HEURISTIC": abi.STEP_HEURISTIC, "RS_STEP_SIGNAL": abi.STEP_SIGNAL,
            "RS_STEP_RESET_FIRST": abi.STEP_RESET_FIRST, "RS_E_ARG": abi.RS_E_ARG,
            "RS_E_TABLES": abi.RS_E_TABLES, "RS_E_STATE": abi.RS_E_STATE, "RS_E_CORRUPT": abi.RS_E_CORRUPT}
    for name, value in want.items():
        assert defs[name] == value, name
