"""GPU parity tests (need a B200): the CUDA path through the C-ABI against
the oracle and the reference's golden vectors."""

import json

import numpy as np
import pytest

from conftest import golden, golden_bytes
from helpers import SimCase
import ties

pytestmark = pytest.mark.gpu

SIMS = ["sim_northern_dt30.npz", "sim_threemeal_dt60.npz", "sim_northern_dt37p5.npz",
        "sim_northern_dt30_8d.npz", "sim_faults.npz", "sim_hypo_threemeal_dt60.npz", "sim_hypo_northern_dt30.npz"]


@pytest.fixture(scope="module")
def dev():
    import torch
    from paper_2202_13927_b200 import _lib
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    _lib.load()
    return torch.device("cuda", 0)


def _parity(case, dev, idx=None, trace=False):
    from paper_2202_13927_b200 import engine
    sub = case.subset(case.valid() if idx is None else idx)
    b = engine.ParityBatch(sub["params"], sub["x0"], sub["c0"], case.hyper, sub["basal"],
                           sub["meal_off"], sub["meals"], sub["ex_off"], sub["ex"], sub["wiener"],
                           sub["has_noise"], sub["meas"])
    return sub, engine.run_parity(b, case.sz, case.config.dt_s, case.config.controller_period_s,
                                  record_trace=trace, device=dev)


def test_steady_state_bitwise(dev):
    from paper_2202_13927_b200 import engine
    g = golden("steady.npz")
    x0, ub, ok = engine.steady_state(g["params"], 6.0, dev)
    assert np.array_equal(x0.cpu().numpy(), g["x0"]) and np.array_equal(ub.cpu().numpy(), g["ub"])
    assert np.all(ok.cpu().numpy() == 0)
    x0, ub, ok = engine.steady_state(g["pert"], 6.0, dev)
    ok = ok.cpu().numpy()
    assert np.array_equal(ok == 0, g["pert_ok"] == 1)
    m = g["pert_ok"] == 1
    assert np.array_equal(x0.cpu().numpy()[m], g["pert_x0"][m])
    assert np.array_equal(ub.cpu().numpy()[m], g["pert_ub"][m])
    _, _, bad = engine.steady_state(g["bad_params"][None, :], 6.0, dev)
    assert int(bad.cpu()[0]) == 2


def test_controller_init_matches_reference(dev):
    from paper_2202_13927_b200 import engine
    case = SimCase("sim_northern_dt30.npz")
    c0 = engine.controller_init(case.hyper, 1.6, case.basal, dev).cpu().numpy()
    assert np.array_equal(c0, case.c0)


@pytest.mark.parametrize("name", SIMS)
def test_parity_kernel_bitwise_vs_reference(dev, name):
    case = SimCase(name)
    g = case.g
    sub, out = _parity(case, dev, trace=True)
    for j, i in enumerate(sub["idx"]):
        assert out["status"][j] == g["status"][i]
        assert out["ticks"][j] == g["ticks"][i]
        assert np.array_equal(out["tir_ticks"][j], g["tir"][i])
        assert np.array_equal(out["bg_hist"][j], g["hist"][i])
        assert np.array_equal(out["scal"][j, :3], g["scal"][i])
        assert np.array_equal(out["day_dose"][j], g["day_dose"][i])
        assert np.array_equal(out["timeline"][j], g["timeline"][i])
        if f"trace_{i}" in g.files:
            tr = g[f"trace_{i}"]
            assert np.array_equal(out["trace"][j][: tr.shape[0]], tr)


@pytest.mark.parametrize("controller", ["dual_hormone", "pid_pump"])
def test_c1_parity_subset_1000_patients_4_weeks(dev, oracle, controller):
    """BASELINE configs[1] correctness subset: the first 1 000 patients of the
    seed-1 device population x 4 weeks at dt 60 s, the reference's own noise
    streams injected, 3-meal schedules.  The parity kernel equals the C oracle
    bit for bit on every output; the fused kernel agrees to relative 1e-9 with
    identical histograms and hypo-event counts except for patients proven
    threshold ties one by one (tests/ties.py)."""
    import torch
    from paper_2202_13927_b200 import engine, rng
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.pid import PIDProfile
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol, compile_protocol
    from paper_2202_13927_b200.simulation import _csr
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=28 * 86400.0, seed=1, dt_s=60.0)
    prof = PIDProfile() if controller == "pid_pump" else ControllerHyperparameters()
    code = 1 if controller == "pid_pump" else 0
    gen = ThreeMealProtocol()
    pop = generate_population(1, 1000, device=dev, on_exhausted="redraw_weight")
    oracle.set_controller(code)
    exc = []
    try:
        for lo in range(0, 1000, 250):
            hi = lo + 250
            ft = FastTrial(lo, pop.params_device[lo:hi].contiguous(), pop.basal_device[lo:hi].contiguous(), gen,
                           prof, cfg, controller_id=controller, device=dev)
            sz = ft.sz
            H, ps = sz["horizon_ticks"], sz["period_steps"]
            params, x0, c0, ub = (t.cpu().numpy() for t in (ft.params, ft.x0, ft.c0, ft.basal))
            pas = [compile_protocol(gen.build(cfg.seed, type("P", (), {"id": lo + i,
                                                                      "body_weight_kg": params[i, 0]})()),
                                    cfg.horizon_s) for i in range(hi - lo)]
            moff, meals, eoff, ex = _csr(pas)
            W = np.zeros((hi - lo, H, 3)); M = np.zeros((hi - lo, H // ps))
            for i in range(hi - lo):
                W[i], M[i] = rng.reference_noise(cfg.seed, lo + i, H, ps, True, True)
            hn = np.ones(hi - lo, np.uint8)
            b = engine.ParityBatch(params, x0, c0, prof.to_vec(), ub, moff, meals, eoff, ex, W, hn, M,
                                   controller=code)
            out = engine.run_parity(b, sz, cfg.dt_s, cfg.controller_period_s, device=dev)
            ref = oracle.run_batch_injected(params, x0, c0, prof.to_vec(), ub, sz, cfg.dt_s,
                                            cfg.controller_period_s, moff, meals, eoff, ex, W, hn, M)
            for k in ("status", "ticks", "tir_ticks", "bg_hist", "scal", "day_dose", "timeline", "x_out", "c_out"):
                assert np.array_equal(out[k], ref[k]), k
            ft.outs = engine.alloc_fast_outputs(hi - lo, lo, sz, dev, per_patient_timeline=True)
            ft.simulate(injected={"wiener": engine.dev(W.reshape(-1), torch.float64, dev),
                                  "has_noise": engine.dev(hn, torch.uint8, dev),
                                  "meas": engine.dev(M.reshape(-1), torch.float64, dev)})
            fused = {"scal": ft.outs.bg_stats.cpu().numpy().T, "hist": ft.outs.bg_hist.cpu().numpy().T,
                     "timeline": ft.outs.timeline_pp.cpu().numpy().T,
                     "day_dose": ft.outs.day_dose.cpu().numpy().transpose(2, 0, 1),
                     "hypo": ft.outs.hypo_events.cpu().numpy().T}
            refd = {"scal": ref["scal"], "hist": ref["bg_hist"], "timeline": ref["timeline"],
                    "day_dose": ref["day_dose"], "hypo": ref["hypo_events"]}
            exc += ties.check_patients(oracle, dev, hi - lo, refd, fused,
                                       ties.inputs_from_arrays(params, x0, c0, ub, prof.to_vec(), moff, meals, eoff,
                                                               ex, W, hn, M, code, sz, cfg.dt_s,
                                                               cfg.controller_period_s, lo),
                                       label=f"C1 {controller} [{lo}, {hi})")
            oracle.set_controller(code)   # (check_patients restores controller 0)
    finally:
        oracle.set_controller(0)
    print(f"C1 {controller}: {len(exc)} proven threshold ties of 1000 patients")


@pytest.mark.parametrize("controller,dt_s,n,days", [("dual_hormone", 60.0, 1000, 28), ("pid_pump", 60.0, 1000, 28),
                                                    ("dual_hormone", 30.0, 500, 14)])
def test_c1_parity_subset_northern_year(dev, oracle, controller, dt_s, n, days):
    """The reference's own configuration at BASELINE configs[1] scale: the
    first 1 000 patients of the seed-1 device population x 4 weeks at dt 60 s
    on the NorthernYear protocol (weight-scaled meals, announced exercise;
    simulation.py:420-453), the schedule planned ON THE DEVICE for the fused
    kernel (gt_northern.cu) and built on the host for the oracle, the
    reference's own noise streams injected.  The parity kernel equals the
    oracle bit for bit on every output; the fused kernel agrees to 1e-9 with
    identical histograms and hypo events except proven threshold ties.
    The third case is the reference's own defaults end to end: its controller,
    its protocol and its default 30 s step (simulation.py:75), 500 x 2 weeks."""
    import torch
    from paper_2202_13927_b200 import engine, rng
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.northern import NorthernYearProtocol
    from paper_2202_13927_b200.pid import PIDProfile
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import compile_protocol
    from paper_2202_13927_b200.simulation import _csr
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=days * 86400.0, seed=1, dt_s=dt_s)
    prof = PIDProfile() if controller == "pid_pump" else ControllerHyperparameters()
    code = 1 if controller == "pid_pump" else 0
    gen = NorthernYearProtocol()
    assert gen.on_device()
    pop = generate_population(1, n, device=dev, on_exhausted="redraw_weight")
    exc, n_ex_sessions, n_hypo = [], 0, 0
    for lo in range(0, n, 250):
        hi = lo + 250
        ft = FastTrial(lo, pop.params_device[lo:hi].contiguous(), pop.basal_device[lo:hi].contiguous(), gen,
                       prof, cfg, controller_id=controller, device=dev)
        sz = ft.sz
        H, ps = sz["horizon_ticks"], sz["period_steps"]
        params, x0, c0, ub = (t.cpu().numpy() for t in (ft.params, ft.x0, ft.c0, ft.basal))
        pas = [compile_protocol(gen.build(cfg.seed, type("P", (), {"id": lo + i, "body_weight_kg": params[i, 0]})()),
                                cfg.horizon_s) for i in range(hi - lo)]
        moff, meals, eoff, ex = _csr(pas)
        n_ex_sessions += int(eoff[-1])
        W = np.zeros((hi - lo, H, 3)); M = np.zeros((hi - lo, H // ps))
        for i in range(hi - lo):
            W[i], M[i] = rng.reference_noise(cfg.seed, lo + i, H, ps, True, True)
        hn = np.ones(hi - lo, np.uint8)
        b = engine.ParityBatch(params, x0, c0, prof.to_vec(), ub, moff, meals, eoff, ex, W, hn, M, controller=code)
        out = engine.run_parity(b, sz, cfg.dt_s, cfg.controller_period_s, device=dev)
        oracle.set_controller(code)
        try:
            ref = oracle.run_batch_injected(params, x0, c0, prof.to_vec(), ub, sz, cfg.dt_s, cfg.controller_period_s,
                                            moff, meals, eoff, ex, W, hn, M)
        finally:
            oracle.set_controller(0)
        for k in ("status", "ticks", "tir_ticks", "bg_hist", "scal", "day_dose", "timeline", "x_out", "c_out"):
            assert np.array_equal(out[k], ref[k]), k
        assert np.all(ref["status"] == 0)
        n_hypo += int(ref["hypo_events"].sum())
        ft.outs = engine.alloc_fast_outputs(hi - lo, lo, sz, dev, per_patient_timeline=True)
        ft.simulate(injected={"wiener": engine.dev(W.reshape(-1), torch.float64, dev),
                              "has_noise": engine.dev(hn, torch.uint8, dev),
                              "meas": engine.dev(M.reshape(-1), torch.float64, dev)})
        fused = {"scal": ft.outs.bg_stats.cpu().numpy().T, "hist": ft.outs.bg_hist.cpu().numpy().T,
                 "timeline": ft.outs.timeline_pp.cpu().numpy().T,
                 "day_dose": ft.outs.day_dose.cpu().numpy().transpose(2, 0, 1),
                 "hypo": ft.outs.hypo_events.cpu().numpy().T}
        refd = {"scal": ref["scal"], "hist": ref["bg_hist"], "timeline": ref["timeline"], "day_dose": ref["day_dose"],
                "hypo": ref["hypo_events"]}
        assert np.array_equal(ft.outs.status.cpu().numpy(), ref["status"])
        exc += ties.check_patients(oracle, dev, hi - lo, refd, fused,
                                   ties.inputs_from_arrays(params, x0, c0, ub, prof.to_vec(), moff, meals, eoff, ex,
                                                           W, hn, M, code, sz, cfg.dt_s, cfg.controller_period_s, lo),
                                   label=f"C1 NorthernYear {controller} dt {dt_s} [{lo}, {hi})")
    assert n_ex_sessions >= n * days // 7   # announced exercise: 76 sessions a year, ~5.5 in 4 weeks
    print(f"C1 NorthernYear {controller} dt {dt_s}: {len(exc)} proven threshold ties of {n} patients; "
          f"{n_ex_sessions} exercise sessions, {n_hypo} hypo events (<3.9) in the reference run")


def test_simulate_closed_loop_api(dev):
    """simulate_closed_loop with the reference's argument types (duck-typed)
    returns the reference's SimulationResult values bit for bit."""
    from paper_2202_13927_b200 import simulate_closed_loop
    from paper_2202_13927_b200.controller import get_controller_factory, ControllerHyperparameters
    from paper_2202_13927_b200.northern import NorthernYearProtocol
    from paper_2202_13927_b200.population import ParameterSet, Patient
    from paper_2202_13927_b200.layout import PARAM_NAMES
    case = SimCase("sim_northern_dt30.npz")
    g = case.g
    for i in (0, 5):
        vals = dict(zip(PARAM_NAMES, case.params[i]))
        patient = Patient(int(case.ids[i]), float(case.params[i, 0]))
        pset = ParameterSet(vals, 0.0)
        proto = NorthernYearProtocol().build(case.config.seed, patient)
        ctl = get_controller_factory("dual_hormone")(ControllerHyperparameters(), float(case.basal[i]))
        res = simulate_closed_loop(patient, pset, proto, ctl, "hovorka_ext", case.config,
                                   record_trace=True, device=dev)
        assert res.status == "ok"
        assert np.array_equal(res.stats.bg_hist, g["hist"][i])
        assert res.stats.sum_bg == g["scal"][i][2]
        if f"trace_{i}" in g.files:
            assert np.array_equal(res.trace, g[f"trace_{i}"])


def _entries_from_population(pop_key_prefix, n):
    from paper_2202_13927_b200.layout import PARAM_NAMES
    from paper_2202_13927_b200.population import ParameterSet, Patient
    g = golden("population.npz")
    P, ub = g[f"{pop_key_prefix}_params"], g[f"{pop_key_prefix}_ubasal"]
    return [(Patient(i, float(P[i, 0])), ParameterSet(dict(zip(PARAM_NAMES, map(float, P[i]))), float(ub[i])))
            for i in range(n)]


@pytest.mark.parametrize("which", ["northern", "threemeal", "faults"])
def test_run_trial_report_bytes_equal_reference(dev, which):
    from paper_2202_13927_b200 import report_bytes, run_trial
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.northern import NorthernYearProtocol
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    prof = ControllerHyperparameters()
    if which == "threemeal":
        entries = _entries_from_population("s0", 64)
        cfg = SimulationConfig(horizon_s=7 * 86400.0, seed=0, dt_s=60.0)
        gen, ref = ThreeMealProtocol(), "report_threemeal_dt60.json"
    else:
        entries = _entries_from_population("s101", 12 if which == "northern" else 4)
        cfg = SimulationConfig(horizon_s=2 * 86400.0, seed=33)
        gen = NorthernYearProtocol()
        ref = "report_northern_dt30.json" if which == "northern" else "report_faults.json"
        if which == "faults":
            entries[2][1].values["tau_cgm"] = -1.0
            entries[3][1].values["EGP0"] = 0.001
    res = run_trial(entries, gen, "dual_hormone", prof, "hovorka_ext", cfg, device=dev)
    assert report_bytes(res.report) == golden_bytes(ref)


def test_worst_trace_reproduces_reference(dev):
    import dataclasses
    from paper_2202_13927_b200 import run_trial
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.northern import NorthernYearProtocol
    g = golden("worst_trace.npz")
    cfg = SimulationConfig(horizon_s=2 * 86400.0, seed=33, store_trace="worst_case_only")
    res = run_trial(_entries_from_population("s101", 4), NorthernYearProtocol(), "dual_hormone",
                    ControllerHyperparameters(), "hovorka_ext", cfg, device=dev)
    assert res.accumulator.worst.patient_id == int(g["worst_id"])
    assert np.array_equal(res.worst_trace, g["trace"])
    assert res.worst_trace[:, 1].min() == res.accumulator.worst.min_bg


def test_unsupported_model_or_controller_raises(dev):
    from paper_2202_13927_b200 import SimulationError, run_trial
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    cfg = SimulationConfig(horizon_s=86400.0, seed=0, dt_s=60.0)
    e = _entries_from_population("s0", 2)
    with pytest.raises(SimulationError):
        run_trial(e, ThreeMealProtocol(), "dual_hormone", ControllerHyperparameters(), "toy", cfg, device=dev)
    with pytest.raises(SimulationError):
        run_trial(e, ThreeMealProtocol(), "pid_mpc", ControllerHyperparameters(), "hovorka_ext", cfg, device=dev)
    with pytest.raises(SimulationError):
        run_trial([], ThreeMealProtocol(), "dual_hormone", ControllerHyperparameters(), "hovorka_ext", cfg, device=dev)


def test_rerun_trial_record_reproduces_reference_report(dev):
    """records.rerun_trial on a record the REFERENCE wrote (storage.py:234-312,
    golden record_rerun.json; NorthernYear with a non-default announcement
    policy) reproduces the reference's report bytes -- both with the
    population passed directly and through a store-like object."""
    from paper_2202_13927_b200 import analytics, records
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.layout import PARAM_NAMES
    from paper_2202_13927_b200.population import ParameterSet, Patient
    rec = records.TrialRecord.from_dict(json.loads(golden_bytes("record_rerun.json")))
    case = SimCase("sim_northern_dt30.npz")       # the same seed-101 cohort
    entries = [(Patient(int(case.ids[i]), float(case.params[i, 0])),
                ParameterSet(values=dict(zip(PARAM_NAMES, (float(v) for v in case.params[i]))),
                             u_basal_u_per_h=float(case.basal[i]))) for i in range(6)]
    prof = ControllerHyperparameters()
    want = golden_bytes("report_rerun.json")
    res = records.rerun_trial(entries, rec, profile=prof, device=dev)
    assert analytics.report_bytes(res.report) == want

    class Store:
        def load_cohort(self, ref):
            assert ref == "pop-a"
            return entries

        def load_profile(self, h):
            assert h == prof.content_hash()
            return prof

    res = records.rerun_trial(Store(), rec, device=dev)
    assert analytics.report_bytes(res.report) == want


def test_c3_arms_parity_subset(dev, oracle):
    """BASELINE configs[3] correctness subset: the four treatment arms (PID gains
    x0.5 / x1 / x1.5 and bolus-only, studies.pid_arms) on 200 shared-parameter
    patients x 2 weeks with the reference's noise streams injected -- the same
    streams in every arm (common random numbers).  Per arm the parity kernel
    equals the C oracle bit for bit and the fused kernel agrees to 1e-9 with
    identical integer outputs except proven threshold ties; the paired per-patient
    TIR differences between arms are therefore the oracle's."""
    import torch
    from paper_2202_13927_b200 import engine, rng
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.pid import PIDProfile
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol, compile_protocol
    from paper_2202_13927_b200.simulation import _csr
    from paper_2202_13927_b200.studies import default_arms
    from paper_2202_13927_b200.trial import FastTrial
    n = 200
    cfg = SimulationConfig(horizon_s=14 * 86400.0, seed=3, dt_s=60.0)
    gen = ThreeMealProtocol()
    pop = generate_population(3, n, device=dev, on_exhausted="redraw_weight")
    arms = default_arms(PIDProfile(), controller_id="pid_pump")
    assert set(arms) == {"pid_x0.5", "pid_x1", "pid_x1.5", "bolus_only"}
    oracle.set_controller(1)
    tir = {}
    try:
        W = M = None
        for name, prof in arms.items():
            ft = FastTrial(0, pop.params_device, pop.basal_device, gen, prof, cfg, controller_id="pid_pump",
                           device=dev)
            sz = ft.sz
            H, ps = sz["horizon_ticks"], sz["period_steps"]
            params, x0, c0, ub = (t.cpu().numpy() for t in (ft.params, ft.x0, ft.c0, ft.basal))
            if W is None:   # one set of streams for every arm
                pas = [compile_protocol(gen.build(cfg.seed, type("P", (), {"id": i, "body_weight_kg": params[i, 0]})()),
                                        cfg.horizon_s) for i in range(n)]
                moff, meals, eoff, ex = _csr(pas)
                W = np.zeros((n, H, 3)); M = np.zeros((n, H // ps))
                for i in range(n):
                    W[i], M[i] = rng.reference_noise(cfg.seed, i, H, ps, True, True)
                hn = np.ones(n, np.uint8)
            b = engine.ParityBatch(params, x0, c0, prof.to_vec(), ub, moff, meals, eoff, ex, W, hn, M, controller=1)
            out = engine.run_parity(b, sz, cfg.dt_s, cfg.controller_period_s, device=dev)
            ref = oracle.run_batch_injected(params, x0, c0, prof.to_vec(), ub, sz, cfg.dt_s, cfg.controller_period_s,
                                            moff, meals, eoff, ex, W, hn, M)
            for k in ("status", "ticks", "tir_ticks", "bg_hist", "scal", "day_dose", "timeline", "x_out", "c_out"):
                assert np.array_equal(out[k], ref[k]), (name, k)
            ft.outs = engine.alloc_fast_outputs(n, 0, sz, dev, per_patient_timeline=True)
            ft.simulate(injected={"wiener": engine.dev(W.reshape(-1), torch.float64, dev),
                                  "has_noise": engine.dev(hn, torch.uint8, dev),
                                  "meas": engine.dev(M.reshape(-1), torch.float64, dev)})
            fused = {"scal": ft.outs.bg_stats.cpu().numpy().T, "hist": ft.outs.bg_hist.cpu().numpy().T,
                     "timeline": ft.outs.timeline_pp.cpu().numpy().T,
                     "day_dose": ft.outs.day_dose.cpu().numpy().transpose(2, 0, 1),
                     "hypo": ft.outs.hypo_events.cpu().numpy().T}
            refd = {"scal": ref["scal"], "hist": ref["bg_hist"], "timeline": ref["timeline"],
                    "day_dose": ref["day_dose"], "hypo": ref["hypo_events"]}
            exc = ties.check_patients(oracle, dev, n, refd, fused,
                                      ties.inputs_from_arrays(params, x0, c0, ub, prof.to_vec(), moff, meals, eoff,
                                                              ex, W, hn, M, 1, sz, cfg.dt_s, cfg.controller_period_s,
                                                              0), label=f"C3 {name}")
            oracle.set_controller(1)   # (check_patients restores controller 0)
            tir[name] = (ref["tir_ticks"][:, 2], {e.patient for e in exc} if exc else set())
    finally:
        oracle.set_controller(0)
    # paired differences against the x1 arm: the oracle's, patient by patient
    base, _ = tir["pid_x1"]
    for name in ("pid_x0.5", "pid_x1.5", "bolus_only"):
        d = tir[name][0] - base
        assert d.shape == (n,) and np.any(d != 0), name


def test_parity_run_trial_pooled_host_inputs_equal_serial(dev, monkeypatch):
    """run_trial(noise="reference") draws the reference's noise streams and
    builds the protocols in a worker-process pool (hostprep) for chunks of
    >= 64 patients; the report bytes equal the in-process path's, chunked
    launches included (PARITY_NOISE_BYTES forced small: 3 chunks)."""
    from paper_2202_13927_b200 import analytics, hostprep, simulation
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    cfg = SimulationConfig(horizon_s=2 * 86400.0, seed=11, dt_s=60.0)
    pop = generate_population(11, 300, device=dev, on_exhausted="redraw_weight").entries()
    per = 8 * (3 * 2880 + 576)
    monkeypatch.setattr(simulation, "PARITY_NOISE_BYTES", 100 * per)
    reports = []
    for w in ("1", "4"):
        monkeypatch.setenv("GLUCOSIM_HOST_WORKERS", w)
        res = simulation.run_trial(pop, ThreeMealProtocol(), "dual_hormone", ControllerHyperparameters(),
                                   "hovorka_ext", cfg, device=dev)
        reports.append(analytics.report_bytes(res.report))
    assert hostprep.workers() == 4
    assert reports[0] == reports[1]
