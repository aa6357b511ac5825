"""Import helper for the Python reference (only present in the build
container at /root/reference; never on the GPU box)."""

from __future__ import annotations

import os
import sys
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")


def available() -> bool:
    return (REF_SRC / "mjsim" / "__init__.py").exists()


def load():
    os.environ.setdefault("MJSIM_TABLE_PATH", "/tmp/mjsim_tables/suit_tables.bin")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    Path(os.environ["MJSIM_TABLE_PATH"]).parent.mkdir(parents=True, exist_ok=True)
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import mjsim  # noqa: F401
    return mjsim
