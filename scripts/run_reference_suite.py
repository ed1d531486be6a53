#!/usr/bin/env python
"""Run the reference's own kernel tests (baseline/_ref/tests, installed by
scripts/install_reference.sh) with bspb.kernels' SoA batch drivers swapped
for the GPU ones (scripts/bspb_gpu_plugin.py).  Exit code = pytest's.

    python scripts/run_reference_suite.py [test files ...]   (default: test_kernels.py)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def main(argv):
    if not os.path.isdir(os.path.join(REF, "bspb")) or not os.path.isdir(os.path.join(REF, "tests")):
        print("baseline/_ref missing: run scripts/install_reference.sh (needs /root/reference)", file=sys.stderr)
        return 2
    files = argv or ["test_kernels.py"]
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(ROOT, "scripts"), ROOT, env.get("PYTHONPATH", "")])
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/bspb_numba_cache")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "bspb_gpu_plugin", "-p", "no:cacheprovider",
           "--rootdir", os.path.join(REF, "tests"), *[os.path.join(REF, "tests", f) for f in files]]
    return subprocess.run(cmd, env=env, cwd=os.path.join(REF, "tests")).returncode


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
