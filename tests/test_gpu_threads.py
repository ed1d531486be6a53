"""Reentrancy (the reference's nogil kernels): host threads
calling evaluate() at once on their own streams and outputs get the same bits
as sequential calls; errors stay per thread."""
import threading

import numpy as np
import pytest

from paper_1611_02665_b200 import ContractError, DeviceTable, evaluate
from paper_1611_02665_b200.grid import unit_cell_grid

pytestmark = pytest.mark.gpu


def test_concurrent_host_threads():
    import torch

    dt = DeviceTable.random(unit_cell_grid(24), 512, seed=11)
    jobs = [("vgh", 40000), ("vgl", 9000), ("vgh", 700), ("v", 30000)] * 2  # line, TMA and generic paths
    rngs = [np.random.default_rng(i) for i in range(len(jobs))]
    inputs = [r.random((p, 3)) * 2 - 0.5 for r, (_, p) in zip(rngs, jobs)]
    want = [evaluate(dt, k, x) for (k, _), x in zip(jobs, inputs)]
    torch.cuda.synchronize()
    got = [None] * len(jobs)
    errors = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(3):
                    got[i] = evaluate(dt, jobs[i][0], inputs[i])
                if i % 3 == 0:  # an invalid call in the middle: its error is this thread's
                    with pytest.raises(ContractError):
                        evaluate(dt, "vgh", inputs[i], lane_limit=dt.lanes + 1, out=got[i])
            s.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for g, w in zip(got, want):
        assert torch.equal(g, w)
