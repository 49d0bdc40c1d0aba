"""The bitwise path's host inputs prepared in worker processes
(paper_2202_13927_b200/hostprep.py) equal the in-process ones: the
reference's noise streams (rng.reference_noise, rng.py:26-39) and protocol
arrays (compile_protocol of generator.build, simulation.py:500-505)."""

import numpy as np
import pytest

from paper_2202_13927_b200 import hostprep, rng
from paper_2202_13927_b200.population import Patient
from paper_2202_13927_b200.protocol import ThreeMealProtocol, compile_protocol


@pytest.mark.parametrize("pooled", [False, True])
def test_prepared_inputs_equal_the_reference_draws(monkeypatch, pooled):
    monkeypatch.setenv("GLUCOSIM_HOST_WORKERS", "2" if pooled else "1")
    gen, H, ps, n, horizon_s = ThreeMealProtocol(), 2880, 5, 70, 2 * 86400.0
    pts = [Patient(1000 + i, 55.0 + 0.5 * i) for i in range(n)]
    pids = np.array([p.id for p in pts])
    proc, sens = np.ones(n, bool), np.ones(n, bool)
    proc[3], sens[5] = False, False
    block = hostprep.NoiseBlock(n, H, H // ps, shared=pooled)
    try:
        pas, blk = hostprep.prepare(gen, 9, pts, pids, proc, sens, horizon_s, H, H // ps, block=block).result()
        assert blk is block and len(pas) == n
        for i in range(n):
            w, m = rng.reference_noise(9, int(pids[i]), H, ps, bool(proc[i]), bool(sens[i]))
            assert np.array_equal(block.wiener[i], w if w is not None else np.zeros((H, 3))), i
            assert np.array_equal(block.meas[i], m), i
            ref = compile_protocol(gen.build(9, pts[i]), horizon_s)
            for k in ref.__dataclass_fields__:
                assert np.array_equal(getattr(ref, k), getattr(pas[i], k)), (i, k)
    finally:
        block.close()
