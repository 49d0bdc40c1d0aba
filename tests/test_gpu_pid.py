"""GPU tests of the PID + pump-quantisation controller (GT_CTRL_PID_PUMP):
parity kernel bitwise vs the C oracle, close to the reference's own
_python_block run of the same controller, fused kernel within 1e-9, and the
trial / study APIs."""

import numpy as np
import pytest

from helpers import SimCase
import ties

pytestmark = pytest.mark.gpu

PID_SIMS = ["sim_pid_threemeal_dt60.npz", "sim_pid_northern_dt30.npz", "sim_hypo_pid_threemeal_dt60.npz"]


@pytest.fixture(scope="module")
def dev():
    import torch
    from paper_2202_13927_b200 import _lib
    assert torch.cuda.is_available()
    _lib.load()
    return torch.device("cuda", 0)


@pytest.mark.parametrize("name", PID_SIMS)
def test_pid_parity_kernel_bitwise_vs_oracle(dev, oracle, name):
    from paper_2202_13927_b200 import engine
    case = SimCase(name)
    sub = case.subset(case.valid())
    b = engine.ParityBatch(sub["params"], sub["x0"], sub["c0"], case.hyper, sub["basal"], sub["meal_off"],
                           sub["meals"], sub["ex_off"], sub["ex"], sub["wiener"], sub["has_noise"], sub["meas"],
                           controller=1)
    out = engine.run_parity(b, case.sz, case.config.dt_s, case.config.controller_period_s, device=dev,
                            record_trace=True)
    oracle.set_controller(1)
    try:
        ref = oracle.run_batch_injected(sub["params"], sub["x0"], sub["c0"], case.hyper, sub["basal"], case.sz,
                                        case.config.dt_s, case.config.controller_period_s, sub["meal_off"],
                                        sub["meals"], sub["ex_off"], sub["ex"], sub["wiener"],
                                        sub["has_noise"], sub["meas"])
    finally:
        oracle.set_controller(0)
    for k in ("status", "ticks", "tir_ticks", "bg_hist", "scal", "day_dose", "timeline", "x_out", "c_out"):
        assert np.array_equal(out[k], ref[k]), k
    # the golden trace columns of the reference's own run (pump-quantised basal / boluses)
    g = case.g
    tr = out["trace"][0]
    if "trace_0" in g.files:
        gt = g["trace_0"]
        assert np.allclose(tr[: gt.shape[0]], gt, rtol=1e-9, atol=1e-12)
    basal_vol = tr[::case.sz["period_steps"], 5] * case.config.controller_period_s / 3600.0
    assert np.allclose(basal_vol / 0.05, np.round(basal_vol / 0.05), atol=1e-9)


def _pid_fused(case, sub, dev, x0=None):
    """The fused pid_pump kernel on a golden case's injected noise (CSR protocol)."""
    import torch
    from paper_2202_13927_b200 import engine, rng
    from paper_2202_13927_b200.protocol import ProtocolArrays, compile_ticks
    n = sub["params"].shape[0]
    D = lambda a, t=torch.float64: engine.dev(a, t, dev)
    tas = []
    for j in range(n):
        a, b = sub["meal_off"][j], sub["meal_off"][j + 1]
        c, d = sub["ex_off"][j], sub["ex_off"][j + 1]
        pa = ProtocolArrays(*(m[a:b] for m in sub["meals"]), *(e[c:d] for e in sub["ex"]))
        tas.append(compile_ticks(pa, case.config.dt_s, case.config.controller_period_s))
    cat = lambda k, dt: np.concatenate([getattr(x, k) for x in tas]).astype(dt)
    nz = lambda a: a if a.size else np.zeros(1, a.dtype)
    csr = {"meal_off": D(sub["meal_off"], torch.int64), "ex_off": D(sub["ex_off"], torch.int64)}
    for k, dt, tdt in (("meal_ks", np.int32, torch.int32), ("meal_ke", np.int32, torch.int32),
                       ("meal_kp", np.int32, torch.int32), ("meal_rate", np.float64, torch.float64),
                       ("meal_ann", np.float64, torch.float64), ("ex_ks", np.int32, torch.int32),
                       ("ex_ke", np.int32, torch.int32), ("ex_hrr", np.float64, torch.float64),
                       ("ex_announced", np.float64, torch.float64)):
        csr[k] = D(nz(cat(k, dt)), tdt)
    csr["ex_start_s"] = D(nz(cat("ex_start", np.float64)))
    inj = {"wiener": D(sub["wiener"].reshape(-1)), "has_noise": D(sub["has_noise"], torch.uint8),
           "meas": D(sub["meas"].reshape(-1))}
    ins = {"params": D(sub["params"]), "x0": D(sub["x0"] if x0 is None else x0), "c0": D(sub["c0"]),
           "hyper": D(case.hyper), "assumed_basal": D(sub["basal"])}
    outs = engine.alloc_fast_outputs(n, int(case.ids[sub["idx"][0]]), case.sz, dev, per_patient_timeline=True)
    engine.launch_fast(ins, outs, case.sz, case.config.dt_s, case.config.controller_period_s, case.config.seed,
                       rng.ROLE_DEVICE_NOISE, max(1, int(np.ceil(900.0 / case.config.dt_s))), dev, csr=csr,
                       injected=inj, controller_code=1)
    return outs


@pytest.mark.parametrize("name", PID_SIMS)
def test_pid_fused_kernel_matches_to_rounding(dev, oracle, name):
    """The fused pid_pump kernel vs the reference's own _python_block run of the
    controller (golden): FP64 statistics to 1e-9, histograms and hypo events
    identical except proven threshold ties (tests/ties.py; the reference side
    of a tie's trace is the oracle, which equals the golden run's integer
    outputs exactly, test_pid.py)."""
    case = SimCase(name)
    g = case.g
    sub = case.subset(case.valid())
    outs = _pid_fused(case, sub, dev)
    st = outs.status.cpu().numpy()
    for j, i in enumerate(sub["idx"]):
        assert st[j] == g["status"][i]
    fused = {"scal": outs.bg_stats.cpu().numpy().T, "hist": outs.bg_hist.cpu().numpy().T,
             "timeline": outs.timeline_pp.cpu().numpy().T, "day_dose": outs.day_dose.cpu().numpy().transpose(2, 0, 1),
             "hypo": outs.hypo_events.cpu().numpy().T}
    refd = {"scal": g["scal"], "hist": g["hist"], "timeline": g["timeline"], "day_dose": g["day_dose"],
            "hypo": g["hypo"]}
    ties.check_patients(oracle, dev, len(sub["idx"]), refd, fused, ties.case_inputs(case, sub, 1), label=name,
                        ref_index=lambda j: sub["idx"][j])


def test_pid_trial_and_arms(dev):
    """run_trial with the PID controller on the fused path; slicing invisible;
    gain-scaled arms ordered sensibly (more gain -> lower mean BG)."""
    from paper_2202_13927_b200 import analytics
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.pid import PIDProfile
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.simulation import run_trial
    from paper_2202_13927_b200.studies import treatment_comparison
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=5 * 86400.0, seed=4, dt_s=60.0)
    pop = generate_population(6, 600, device=dev, on_exhausted="redraw_weight")
    res = run_trial(pop, ThreeMealProtocol(), "pid_pump", PIDProfile(), "hovorka_ext", cfg, noise="philox",
                    device=dev)
    tir = res.metrics["tir"][res.metrics["status"] == 0]
    assert res.accumulator.n_patients >= 590 and 0.5 < tir.mean() < 0.98
    a, b = (FastTrial(0, pop.params_device, pop.basal_device, ThreeMealProtocol(), PIDProfile(), cfg,
                      controller_id="pid_pump", device=dev, n_slices=s) for s in (1, 3))
    for ft in (a, b):
        ft.step()
    ra, rb = (analytics.report_bytes(analytics.build_trial_report(ft.accumulator(), {})) for ft in (a, b))
    assert ra == rb
    base = PIDProfile()
    out = treatment_comparison(800, 1, seed=3, device=dev, controller_id="pid_pump",
                               arms={"x0.5": base.scaled(0.5), "x1": base, "x1.5": base.scaled(1.5)},
                               reference_arm="x1")
    m = {k: v["per_patient"]["mean_bg"]["mean"] for k, v in out["arms"].items()}
    assert m["x0.5"] > m["x1"] > m["x1.5"]


def test_simulate_closed_loop_with_pid_object(dev):
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.pid import PIDController, PIDProfile
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.simulation import simulate_closed_loop
    cfg = SimulationConfig(horizon_s=86400.0, seed=1, dt_s=60.0)
    (pt, ps), = generate_population(2, 1, device=dev, on_exhausted="redraw_weight").entries()
    ctl = PIDController(PIDProfile(), ps.u_basal_u_per_h)
    r = simulate_closed_loop(pt, ps, ThreeMealProtocol().build(cfg.seed, pt), ctl, "hovorka_ext", cfg,
                             record_trace=True, device=dev)
    assert r.status == "ok" and r.trace.shape == (1440, 8)
    vol = r.trace[::5, 5] * 300.0 / 3600.0
    assert np.allclose(vol / 0.05, np.round(vol / 0.05), atol=1e-9)


def test_pid_fused_refuses_nonzero_glucagon_state(dev):
    """pid_pump never doses glucagon, so the fused kernel drops the glucagon
    chain (Z1 = Z2 = 0 from the fasting steady state).  A patient whose x0
    has a glucagon state is refused (GT_STATUS_BAD_INITIAL_STATE, counted as
    aborted), never integrated wrongly; the other patients are unaffected."""
    from paper_2202_13927_b200._lib import GT_STATUS_BAD_INITIAL_STATE
    from paper_2202_13927_b200.layout import IZ1, IZ2
    case = SimCase("sim_pid_threemeal_dt60.npz")
    sub = case.subset(case.valid())
    assert not sub["x0"][:, [IZ1, IZ2]].any()
    ref = _pid_fused(case, sub, dev)
    x0 = sub["x0"].copy()
    x0[0, IZ1] = 1e-3
    x0[1, IZ2] = 1e-3
    out = _pid_fused(case, sub, dev, x0=x0)
    st = out.status.cpu().numpy()
    assert list(st[:2]) == [GT_STATUS_BAD_INITIAL_STATE] * 2
    assert np.array_equal(st[2:], ref.status.cpu().numpy()[2:])
    assert np.array_equal(out.bg_hist.cpu().numpy()[:, 2:], ref.bg_hist.cpu().numpy()[:, 2:])
    assert np.array_equal(out.bg_stats.cpu().numpy()[:, 2:], ref.bg_stats.cpu().numpy()[:, 2:])
