"""PID + pump-quantisation controller (pid.py, BASELINE's controller): the
Python twin is what the reference's own generic engine ran to make the
golden fixtures; the C oracle restates it bit for bit and, closed loop on
the golden inputs, agrees with the reference's _python_block run."""

import numpy as np
import pytest

from helpers import SimCase


def test_pid_oracle_equals_twin(oracle):
    from paper_2202_13927_b200 import pid
    for prof, basal in ((pid.PIDProfile(), 0.8), (pid.PIDProfile(kp=0.4, ki=0.1, integral_max=2.0), 1.7),
                        (pid.PIDProfile(basal_increment_u=0.1, bolus_increment_u=0.5, max_bolus_u=3.0), 0.35)):
        ctl = pid.PIDController(prof, basal)
        st = ctl.initial_state()
        c, h = st.to_vec(), prof.to_vec()
        g = np.random.default_rng(int(basal * 100))
        for k in range(4000):
            y = float(np.clip(6 + 4 * np.sin(k / 9) + g.normal(0, 1.5), 0.5, 30))
            ann = float(g.choice([0.0, 0.0, 0.0, 0.0, 30.0, 75.0, 140.0]))
            st, dec = ctl.step(st, y, ann, -1.0, 300.0 * k, 300.0)
            c, out = oracle.pid_step(c, y, ann, -1.0, 300.0 * k, 300.0, h, basal)
            assert np.array_equal(c, st.vec)
            assert list(out) == [dec.basal_rate_u_per_h, dec.insulin_bolus_u, dec.glucagon_bolus_ug]
            assert dec.basal_rate_u_per_h >= 0 and dec.insulin_bolus_u >= 0
            # pump quantisation: every period's basal volume is a whole number of pulses
            vol = dec.basal_rate_u_per_h * 300.0 / 3600.0
            assert abs(vol / prof.basal_increment_u - round(vol / prof.basal_increment_u)) < 1e-9
            assert abs(dec.insulin_bolus_u / prof.bolus_increment_u
                       - round(dec.insulin_bolus_u / prof.bolus_increment_u)) < 1e-9


def test_pid_initial_state_matches_device_init_layout():
    """gt_controller_init's dual-hormone vector is also the PID's initial state."""
    from paper_2202_13927_b200 import pid
    from paper_2202_13927_b200.controller import ControllerHyperparameters, initial_icr
    prof = pid.PIDProfile()
    v = pid.PIDController(prof, 0.9).initial_state().to_vec()
    assert v[3] == initial_icr(0.9, prof)
    assert np.all(v[[0, 1, 2, 4, 5, 7, 8, 9, 10]] == 0.0) and v[6] == -1e18
    assert prof.to_vec()[17] == prof.icr_min and prof.to_vec()[18] == prof.icr_max
    assert ControllerHyperparameters().to_vec().shape == prof.to_vec().shape


@pytest.mark.parametrize("name", ["sim_pid_threemeal_dt60.npz", "sim_pid_northern_dt30.npz",
                                  "sim_hypo_pid_threemeal_dt60.npz"])
def test_pid_oracle_closed_loop_vs_reference_engine(oracle, name):
    """The golden run is the reference's _python_block (x += f*dt + M @ (sqrt(dt) w),
    simulation.py:290-295), whose operation order differs from simulate_block's
    by ~1e-14; the oracle follows simulate_block.  FP64
    statistics agree to 1e-9; integer counts (histogram, ranges, hypo events)
    are identical -- no threshold tie occurs on these fixtures, so none is allowed."""
    case = SimCase(name)
    g = case.g
    sub = case.subset(case.valid())
    oracle.set_controller(1)
    try:
        out = oracle.run_batch_injected(sub["params"], sub["x0"], sub["c0"], case.hyper, sub["basal"],
                                        case.sz, case.config.dt_s, case.config.controller_period_s,
                                        sub["meal_off"], sub["meals"], sub["ex_off"], sub["ex"],
                                        sub["wiener"], sub["has_noise"], sub["meas"])
    finally:
        oracle.set_controller(0)
    for j, i in enumerate(sub["idx"]):
        assert out["status"][j] == g["status"][i]
        assert np.allclose(out["scal"][j, :3], g["scal"][i], rtol=1e-9, atol=0), (name, i)
        assert np.allclose(out["timeline"][j], g["timeline"][i], rtol=1e-9, atol=0), (name, i)
        assert np.allclose(out["day_dose"][j], g["day_dose"][i], rtol=1e-9, atol=1e-12), (name, i)
        # no threshold tie occurs on these fixtures: every integer count is identical
        assert np.array_equal(out["bg_hist"][j], g["hist"][i]), (name, i)
        assert np.array_equal(out["tir_ticks"][j], g["tir"][i]), (name, i)
        assert np.array_equal(out["hypo_events"][j], g["hypo"][i]), (name, i)
