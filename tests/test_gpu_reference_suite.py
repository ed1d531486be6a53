"""The reference's own kernel test suite (pkg/tests/test_kernels.py,
unchanged, from baseline/_ref -- scripts/install_reference.sh) run with its
SoA batch drivers kernels.py:357-381 swapped for the GPU ones
(paper_1611_02665_b200.bspb_patch, strict mode): every SoA and tiled
evaluation in that suite runs on the B200 and must match the numba kernels
(AoS evaluations, still numba, bitwise; the f64 oracle within 1e-5)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")),
                    reason="baseline/_ref not installed (scripts/install_reference.sh)")
@pytest.mark.parametrize("mode", ["strict"])
def test_reference_kernel_suite_on_gpu(mode):
    env = dict(os.environ, BSPB_PATCH_MODE=mode)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "run_reference_suite.py")],
                       capture_output=True, text=True, timeout=1200, env=env)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "GPU batch calls served" in r.stdout
    assert "failed" not in r.stdout.splitlines()[-1]
