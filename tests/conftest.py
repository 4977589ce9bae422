"""pytest configuration: the `gpu` marker and shared helpers.

`-m "not gpu"` runs on any host (oracle vs golden vectors, host logic, the
C-ABI surface); `-m gpu` needs a B200 and exercises the CUDA path.
"""

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_sessionstart(session):
    # Build the extension in-tree once per test session (incremental, seconds).
    from paper_1511_04348_b200 import _build

    _build.build()
