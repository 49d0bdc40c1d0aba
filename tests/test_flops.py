"""The algorithmic FLOP constants used by the roofline are the reference's
own op counts (tests/golden/flop_counts.json, counted over the reference's
Python source by an op-counting float)."""
import json

from conftest import golden_bytes
from paper_2202_13927_b200 import flops


def test_flop_constants_pinned_to_reference_counts():
    c = json.loads(golden_bytes("flop_counts.json"))
    assert c["drift_typical"] == flops.DRIFT_TYPICAL
    assert c["controller_typical"] == flops.CONTROLLER_TYPICAL
    assert c["diffusion"] == 3
    assert flops.STEP == 119 and flops.TICK == 25
    assert abs(flops.flops_per_patient_week(60.0, 5) - 1.2499e6) < 1e3


def test_structural_zero_counts_pinned():
    """The work left when exercise / glucagon are structurally absent, counted
    by the known-value float over the reference's drift_vec (make_golden.py)."""
    c = json.loads(golden_bytes("flop_counts.json"))
    assert c["drift_typical_noex"] == flops.DRIFT_NOEX
    assert c["drift_typical_nogluc"] == flops.DRIFT_NOGLUC
    assert c["drift_typical_noex_nogluc"] == flops.DRIFT_NOEX_NOGLUC
    assert c["zero_states_noex"] == flops.ZERO_STATES_NOEX
    assert c["zero_states_nogluc"] == flops.ZERO_STATES_NOGLUC
    assert c["zero_states_noex_nogluc"] == flops.ZERO_STATES_NOEX_NOGLUC
    # bench workload: 3-meal generator (no exercise) + pid_pump (no glucagon)
    assert flops.flops_per_step_nontrivial(5, "pid_pump", exercise=False) == 119 - 23 - 10 + 31 / 5
    assert flops.flops_per_step_nontrivial(5, "dual_hormone", exercise=True) == flops.flops_per_step(5)
    assert flops.flops_per_step_nontrivial(5, "dual_hormone", exercise=False) == 119 - 15 - 6 + 25 / 5


def test_pid_controller_op_count():
    """PID_CONTROLLER_TYPICAL = FP64 +,-,*,/ of pid_step_vec on its typical
    branch (no meal bolus), counted with an op-counting float."""
    import numpy as np
    from paper_2202_13927_b200 import pid

    class CF(float):
        n = 0

        def _w(op):
            def f(self, o):
                CF.n += 1
                return CF(getattr(float, op)(self, o))
            return f
        __add__, __radd__ = _w("__add__"), _w("__radd__")
        __sub__, __rsub__ = _w("__sub__"), _w("__rsub__")
        __mul__, __rmul__ = _w("__mul__"), _w("__rmul__")
        __truediv__, __rtruediv__ = _w("__truediv__"), _w("__rtruediv__")

        def __neg__(self):
            return CF(-float(self))

    prof = pid.PIDProfile()
    h = [CF(v) for v in prof.to_vec()]
    c = [CF(v) for v in pid.PIDController(prof, 0.8).initial_state().to_vec()]
    g = np.random.default_rng(1)
    counts = []
    for k in range(300):
        CF.n = 0
        pid.pid_step_vec(c, CF(float(np.clip(g.normal(7, 1.5), 2, 20))), CF(0.0), CF(-1.0), CF(300.0 * k),
                         CF(300.0), h, CF(0.8), [0, 0, 0])
        counts.append(CF.n)
    vals, cnt = np.unique(counts[1:], return_counts=True)
    assert int(vals[np.argmax(cnt)]) == flops.PID_CONTROLLER_TYPICAL
    assert flops.flops_per_step(5, "pid_pump") == 119 + 32 / 5
