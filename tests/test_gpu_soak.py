"""Randomised parity (a short tools/soak.py run): random shapes, block
widths, fields, variants and options; exact mode bitwise = oracle, default
mode within the stated tolerances."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_random_configurations():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "soak.py"), "25", "2026"], capture_output=True,
                       text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failures" in r.stdout, r.stdout[-4000:]
