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


def test_numpy_stream_twin_and_plan_twin():
    """The integer restatement of numpy's SeedSequence / Philox4x64 /
    Generator.shuffle (what csrc/gt_northern.cu runs) equals numpy."""
    import numpy as np
    from paper_2202_13927_b200 import northern, rng
    for seed, key in [(0, (0,)), (12345, (7, 3)), (2**40 + 5, (999_999, 3)), (2**63 + 17, (0,)),
                      (1, ()), (3, (2**33, 1))]:
        ss = np.random.SeedSequence(entropy=seed, spawn_key=key)
        assert list(ss.generate_state(6)) == rng.seed_sequence_state(seed, key, 6)
        t = rng.NumpyPhiloxTwin(seed, key)
        p = np.random.Philox(np.random.SeedSequence(entropy=seed, spawn_key=key))
        assert [t.next_uint64() for _ in range(9)] == [int(v) for v in p.random_raw(9)]
    for trial_seed, pid in [(0, 0), (7, 123), (2**35, 999_999), (42, 2**33 + 1)]:
        d = rng.derive_seed(trial_seed, pid, rng.ROLE_PROTOCOL)
        assert d == rng.derive_seed_twin(trial_seed, pid, rng.ROLE_PROTOCOL)
        assert northern.plan_year_twin(d) == northern.plan_year(d)


def test_northern_year_counts_are_fixed():
    """Every seed yields 1588 meals and 76 exercise sessions per year: the
    fixed stride of the device builder (include/glucosim.h GT_NY_MEALS)."""
    from paper_2202_13927_b200 import northern
    for seed in (0, 1, 99, 2**40 + 7):
        p = northern.compose_year(seed, 70.0)
        kinds = [d.kind for d in p.disturbances]
        assert kinds.count("meal") == 1588 and kinds.count("exercise") == 76
