"""Shared pytest configuration.

Markers: ``gpu`` -- needs a B200 (runs on the GPU box: ``pytest -m gpu``);
everything else runs on the CPU-only build container (``-m "not gpu"``).
"""
import os
import sys
from fractions import Fraction
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA B200 device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def read_golden(name):
    """Parse a tests/golden/*.txt fixture: 'KEY v1 v2 ...' lines, values as
    Fractions where possible; repeated keys accumulate rows."""
    out = {}
    for line in (GOLDEN / name).read_text().splitlines():
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        key, *vals = line.split()
        row = []
        for v in vals:
            try:
                row.append(Fraction(v))
            except ValueError:
                row.append(v)
        out.setdefault(key, []).append(row)
    return out
