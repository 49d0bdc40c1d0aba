"""Hypoglycaemia events and the threshold-tie classifier (CPU).

The reference counts only ticks below 3 mmol/L (analytics.py:129-135);
BASELINE.json north_star asks for hypoglycaemia *event* counts.  The repo's
definition: maximal runs of consecutive ticks with the
statistics' BG below 3.9 (TBR<70) / 3.0 (TBR<54) mmol/L lasting at least
ceil(15 min / dt) ticks.  The golden counts were computed by the numpy twin
from the REFERENCE's own per-tick BG (trace column 1 of _simulate_arrays,
simulation.py:61-64) in tests/golden/make_golden.py.
"""

import numpy as np
import pytest

from helpers import SimCase
import ties

SIMS = [("sim_northern_dt30.npz", 0), ("sim_threemeal_dt60.npz", 0), ("sim_northern_dt37p5.npz", 0),
        ("sim_northern_dt30_8d.npz", 0), ("sim_faults.npz", 0), ("sim_pid_threemeal_dt60.npz", 1),
        ("sim_pid_northern_dt30.npz", 1), ("sim_hypo_threemeal_dt60.npz", 0),
        ("sim_hypo_northern_dt30.npz", 0), ("sim_hypo_pid_threemeal_dt60.npz", 1)]


def test_hypo_twin_known_answers(oracle):
    L = 3
    lo = 3.5
    seq = np.array([lo, lo, lo,            # run of 3 at the start: counts
                    5.0,
                    lo, lo,                # run of 2: too short
                    5.0, 3.9,              # 3.9 itself is not below 3.9
                    lo, 2.9, 2.9, 2.9, lo,  # run of 5 (<3.9) containing a run of 3 (<3.0)
                    5.0,
                    2.0, 2.0, 2.0, 2.0])   # run of 4 at the end: counts for both
    assert oracle.hypo_events(seq, L) == (3, 2)
    assert oracle.hypo_events(seq, 1) == (4, 2)
    assert oracle.hypo_events(seq, 6) == (0, 0)
    assert oracle.hypo_events(np.array([]), L) == (0, 0)
    assert oracle.hypo_events(np.full(10, np.nan), 1) == (0, 0)
    assert oracle.hypo_events(np.full(7, np.nextafter(3.0, 0)), 7) == (1, 1)
    assert oracle.hypo_min_ticks(60.0) == 15 and oracle.hypo_min_ticks(37.5) == 24 and oracle.hypo_min_ticks(30.0) == 30


def test_hypo_fixtures_are_rich():
    """The hypo-rich fixtures exercise both thresholds many times."""
    for name in ("sim_hypo_threemeal_dt60.npz", "sim_hypo_northern_dt30.npz", "sim_hypo_pid_threemeal_dt60.npz"):
        h = SimCase(name).g["hypo"]
        assert h[:, 0].sum() >= 100 and h[:, 1].sum() >= 10, name


@pytest.mark.parametrize("name,controller", SIMS)
def test_oracle_hypo_events_equal_reference_traces(oracle, name, controller):
    """The C oracle's streaming run counter equals the twin applied to the
    reference's own BG trace, for every patient with a steady state."""
    case = SimCase(name)
    g = case.g
    sub = case.subset(case.valid())
    oracle.set_controller(controller)
    try:
        out = oracle.run_batch_injected(sub["params"], sub["x0"], sub["c0"], case.hyper, sub["basal"],
                                        case.sz, case.config.dt_s, case.config.controller_period_s,
                                        sub["meal_off"], sub["meals"], sub["ex_off"], sub["ex"],
                                        sub["wiener"], sub["has_noise"], sub["meas"],
                                        hypo_min=int(g["hypo_min_ticks"]))
    finally:
        oracle.set_controller(0)
    for j, i in enumerate(sub["idx"]):
        assert out["status"][j] == g["status"][i]
        assert tuple(out["hypo_events"][j]) == tuple(g["hypo"][i]), (name, i)
        # integer outputs identical (PID fixtures come from the reference's generic engine)
        assert np.array_equal(out["bg_hist"][j], g["hist"][i]), (name, i)


def test_oracle_trace_hypo_consistent(oracle):
    """The oracle's trace reproduces its own streaming statistics."""
    case = SimCase("sim_hypo_threemeal_dt60.npz")
    sub = case.subset(case.valid())
    mk = ties.case_inputs(case, sub)
    for j in range(3):
        tr, ticks = ties.oracle_trace(oracle, mk(j))
        assert ticks == case.sz["horizon_ticks"]
        hist, _ = ties.trace_hist(tr, ticks)
        assert np.array_equal(hist, case.g["hist"][sub["idx"][j]])
        assert oracle.hypo_events(tr[:, 1], 15) == tuple(case.g["hypo"][sub["idx"][j]])


# ------------------------------------------------------- the classifier itself
def _ref(oracle, name="sim_hypo_threemeal_dt60.npz", controller=0):
    case = SimCase(name)
    sub = case.subset(case.valid())
    pi = ties.case_inputs(case, sub, controller)(0)
    tr, _ = ties.oracle_trace(oracle, pi)
    return pi, tr


def test_classifier_accepts_a_bin_tie(oracle):
    pi, tr = _ref(oracle)
    f = tr.copy()
    k = 1234
    tr[k, 1] = 3.9                       # on the edge: bin 35, range "normo"...
    f[k, 1] = np.nextafter(3.9, 0.0)     # one ulp below: bin 34, range "hypo"
    e = ties.classify(oracle, pi, tr, f, 0)
    assert e.kind == "bin" and e.tick == k and e.detail["edge"] == 3.9 and e.detail["ulps_apart"] == 1


def test_classifier_rejects_a_bin_flip_between_distant_values(oracle):
    pi, tr = _ref(oracle)
    f = tr.copy()
    tr[500, 1], f[500, 1] = 3.95, 3.85
    with pytest.raises(AssertionError, match="not a rounding tie"):
        ties.classify(oracle, pi, tr, f, 0)


def test_classifier_rejects_a_drift(oracle):
    pi, tr = _ref(oracle)
    f = tr.copy()
    f[700:, 1] *= 1 + 1e-7      # same bins at tick 700 unless on an edge: a drift, not a tie
    k = 700 + int(np.flatnonzero(ties._rel(tr[700:, 1], f[700:, 1]) > ties.REL_DRIFT)[0])
    fd = ties.first_divergence(tr, f)
    assert fd["tick"] == k
    with pytest.raises(AssertionError):
        ties.classify(oracle, pi, tr, f, 0)


@pytest.mark.parametrize("controller", [0, 1])
def test_classifier_controller_tie_and_mismatch(oracle, controller):
    name = "sim_hypo_pid_threemeal_dt60.npz" if controller else "sim_hypo_threemeal_dt60.npz"
    pi, tr = _ref(oracle, name, controller)
    ps = pi.sz["period_steps"]
    ys = tr[::ps, 2].copy()
    n = ys.size
    base = ties.replay_controller(oracle, pi, ys, n)
    assert np.array_equal(base, tr[::ps, 5:8])
    # a mismatch: the "fused" run claims a different basal at some tick with the same readings
    f = tr.copy()
    q = 40
    f[q * ps, 5] = tr[q * ps, 5] * 1.5 + 0.1
    with pytest.raises(AssertionError, match="not the reference controller"):
        ties.classify(oracle, pi, tr, f, 0)
    # a tie: bisect the first reading between two values whose decisions
    # differ down to ADJACENT doubles a < b (the reference's own controller is
    # discontinuous there), then let the reference run read a and the "fused"
    # run read b
    def out0(y):
        return ties.replay_controller(oracle, pi, np.array([y]), 1)[0]

    def differ(u, v):
        return bool(np.any(ties._rel(u, v) > 1e-9))

    lo, hi = 1.0, 25.0
    assert differ(out0(lo), out0(hi))
    ilo, ihi = (int(np.array(v).view(np.int64)) for v in (lo, hi))
    olo = out0(lo)
    while ihi - ilo > 1:
        im = (ilo + ihi) // 2
        om = out0(float(np.array(im, np.int64).view(np.float64)))
        if differ(olo, om):
            ihi = im
        else:
            ilo, olo = im, om
    a, b = (float(np.array(v, np.int64).view(np.float64)) for v in (ilo, ihi))
    assert ties.ulps(a, b) == 1
    r, f = tr.copy(), tr.copy()
    for trace, y0 in ((r, a), (f, b)):
        y = ys.copy()
        y[0] = y0
        trace[0, 2] = y0
        trace[::ps, 5:8] = ties.replay_controller(oracle, pi, y, n)
    e = ties.classify(oracle, pi, r, f, 0)
    assert e.kind == "controller" and e.tick == 0, e
