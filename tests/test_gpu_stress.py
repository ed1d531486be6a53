"""Randomised line-kernel synchronisation stress (scripts/stress_line.py):
random grids, orbital counts, kinds, dtypes, table forms, densities and
non-finite positions; the line kernel must equal the per-position kernel bit
for bit on every case."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [11, 12])
def test_line_kernel_random_cases(seed):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "stress_line.py"), "60", str(seed)],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "all 60 cases bitwise equal" in r.stdout
