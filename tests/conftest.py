import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); runs the CUDA path through the C ABI")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_table(name):
    """Parse a golden table: '# ...' comment lines, then rows 'key v1 v2 ...' ('-' = None)."""
    rows = {}
    for line in (GOLDEN / name).read_text().splitlines():
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        rows[float(parts[0])] = [None if p == "-" else float(p) for p in parts[1:]]
    return rows


def rounds_to(value, printed, digits=4):
    """True if `value` rounds to the `digits`-significant-digit number `printed` (half a unit
    in the last printed digit, plus a 1% slack of that unit for the printing's own rounding)."""
    import math
    unit = 10.0 ** (math.floor(math.log10(abs(printed))) - (digits - 1))
    return abs(value - printed) <= 0.51 * unit
