"""The host NorthernYearProtocol restatement reproduces the reference's
compiled schedules exactly (golden CSR arrays from the reference)."""

import numpy as np
import pytest

from conftest import golden
from helpers import SimCase

from paper_2202_13927_b200.northern import NorthernYearProtocol
from paper_2202_13927_b200.protocol import compile_protocol, validate_protocol


@pytest.mark.parametrize("name", ["sim_northern_dt30.npz", "sim_northern_dt37p5.npz",
                                  "sim_northern_dt30_8d.npz"])
def test_schedule_equals_reference(name):
    case = SimCase(name)
    gen = NorthernYearProtocol()
    for i, pid in enumerate(case.ids):
        patient = type("P", (), {"id": int(pid), "body_weight_kg": float(case.params[i, 0])})()
        proto = gen.build(case.config.seed, patient)
        assert validate_protocol(proto) == []
        pa = compile_protocol(proto, case.config.horizon_s)
        a, b = case.meal_off[i], case.meal_off[i + 1]
        for k, arr in enumerate((pa.meals_start, pa.meals_end, pa.meals_rate, pa.meals_ann)):
            assert np.array_equal(arr, case.meals[k][a:b])
        a, b = case.ex_off[i], case.ex_off[i + 1]
        for k, arr in enumerate((pa.ex_start, pa.ex_end, pa.ex_hrr, pa.ex_announced)):
            assert np.array_equal(arr, case.ex[k][a:b])


def test_year_counts():
    # Table-1 counts fix 1588 meals and 76 exercise sessions per year
    proto = NorthernYearProtocol().build(5, type("P", (), {"id": 2, "body_weight_kg": 80.0})())
    kinds = [d.kind for d in proto.disturbances]
    assert kinds.count("meal") == 1588 and kinds.count("exercise") == 76
