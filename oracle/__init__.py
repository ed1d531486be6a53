"""CPU oracle for the tricubic B-spline SPO path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package, and only as the checker or
the CPU baseline.  The product package ``paper_1611_02665_b200`` never imports
it and has no CPU fallback.

Two independent restatements of the reference (/root/reference/pkg/src/bspb):

* ``oracle.py`` -- numpy: index mapping (grid.py:109-121), fp32 weights
  (grid.py:124-139), fp64 weights (oracle.py:20-42) and a vectorised
  ``evaluate_f64`` (oracle.py:74-115) for small cases;
* ``spline_oracle.c`` (``liboracle.so`` via ctypes) -- the same mapping and
  weights, the fp32 production kernels (kernels.py:143-247, bitwise) and the
  fp64 oracle with the per-element tolerance scale sum|w*c|.

Parity is PINNED: tests/test_oracle_golden.py checks both restatements
against fixtures generated from the reference itself
(tests/golden/make_golden.py).
"""
from .oracle import *  # noqa: F401,F403
from .oracle import __all__  # noqa: F401
