"""pytest plugin: run the reference's own test suite with its SoA batch
drivers replaced by the GPU ones (paper_1611_02665_b200.bspb_patch, strict
mode: bitwise the numba kernels).  Loaded by scripts/run_reference_suite.py;
fails the session if the GPU path never ran."""
import os

MODE = os.environ.get("BSPB_PATCH_MODE", "strict")


def pytest_configure(config):
    import bspb.kernels

    from paper_1611_02665_b200 import bspb_patch

    bspb_patch.install(bspb.kernels, mode=MODE)
    config._bspb_patch = bspb_patch


def pytest_sessionfinish(session, exitstatus):
    bp = session.config._bspb_patch
    calls = dict(bp.CALLS)
    print(f"\n[bspb_gpu_plugin] mode={bp.MODE} GPU batch calls served: {calls}")
    if sum(calls.values()) == 0:
        session.exitstatus = 1
