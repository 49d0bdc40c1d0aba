"""GPU tests of the throughput path: fused integrator, device 3-meal
generator, device reduction, sharding invariance, population sampler."""

import numpy as np
import pytest

from conftest import golden
from helpers import SimCase
import ties

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch
    from paper_2202_13927_b200 import _lib
    assert torch.cuda.is_available()
    _lib.load()
    return torch.device("cuda", 0)


def _t():
    import torch
    return torch


def test_device_meal_generator_bitwise_vs_host_twin(dev):
    from paper_2202_13927_b200 import engine
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    gen = ThreeMealProtocol()
    for seed, pid0 in ((0, 0), (2, 999_990), (2**40 + 3, 17)):
        s, e, c = engine.generate_meals(seed, pid0, 12, 3 * 40, gen.device_spec(), dev)
        for i in range(12):
            hs, he, hc = gen.meals(seed, pid0 + i, 3 * 40)
            assert np.array_equal(s[i], hs) and np.array_equal(e[i], he) and np.array_equal(c[i], hc)


def _inputs(case, sub, dev):
    from paper_2202_13927_b200 import engine
    t = _t()
    n = sub["params"].shape[0]
    return {"params": engine.dev(sub["params"], t.float64, dev), "x0": engine.dev(sub["x0"], t.float64, dev),
            "c0": engine.dev(sub["c0"], t.float64, dev), "hyper": engine.dev(case.hyper, t.float64, dev),
            "assumed_basal": engine.dev(sub["basal"], t.float64, dev)}


def _injected(sub, dev):
    from paper_2202_13927_b200 import engine
    t = _t()
    return {"wiener": engine.dev(sub["wiener"].reshape(-1), t.float64, dev),
            "has_noise": engine.dev(sub["has_noise"], t.uint8, dev),
            "meas": engine.dev(sub["meas"].reshape(-1), t.float64, dev)}


def _csr_ticks(case, sub, dev):
    from paper_2202_13927_b200 import engine
    from paper_2202_13927_b200.protocol import ProtocolArrays, compile_ticks
    t = _t()
    n = sub["params"].shape[0]
    tas = []
    for j in range(n):
        a, b = sub["meal_off"][j], sub["meal_off"][j + 1]
        c, d = sub["ex_off"][j], sub["ex_off"][j + 1]
        pa = ProtocolArrays(*(m[a:b] for m in sub["meals"]), *(e[c:d] for e in sub["ex"]))
        tas.append(compile_ticks(pa, case.config.dt_s, case.config.controller_period_s))
    cat = lambda k, dt: np.concatenate([getattr(x, k) for x in tas]).astype(dt)
    nz = lambda a: a if a.size else np.zeros(1, a.dtype)
    D = lambda a, tdt: engine.dev(nz(a), tdt, dev)
    return {"meal_off": D(sub["meal_off"], t.int64), "meal_ks": D(cat("meal_ks", np.int32), t.int32),
            "meal_ke": D(cat("meal_ke", np.int32), t.int32), "meal_kp": D(cat("meal_kp", np.int32), t.int32),
            "meal_rate": D(cat("meal_rate", np.float64), t.float64),
            "meal_ann": D(cat("meal_ann", np.float64), t.float64), "ex_off": D(sub["ex_off"], t.int64),
            "ex_ks": D(cat("ex_ks", np.int32), t.int32), "ex_ke": D(cat("ex_ke", np.int32), t.int32),
            "ex_start_s": D(cat("ex_start", np.float64), t.float64),
            "ex_hrr": D(cat("ex_hrr", np.float64), t.float64),
            "ex_announced": D(cat("ex_announced", np.float64), t.float64)}


def _run_fast(case, sub, dev, csr=None, meal_spec=None, injected=None, timeline=True):
    from paper_2202_13927_b200 import engine, rng
    n = sub["params"].shape[0]
    outs = engine.alloc_fast_outputs(n, int(case.ids[sub["idx"][0]]), case.sz, dev,
                                     per_patient_timeline=timeline, final_state=True)
    engine.launch_fast(_inputs(case, sub, dev), outs, case.sz, case.config.dt_s,
                       case.config.controller_period_s, case.config.seed, rng.ROLE_DEVICE_NOISE,
                       max(1, int(np.ceil(900 / case.config.dt_s))), dev, meal_spec=meal_spec,
                       csr=csr, injected=injected)
    return outs


def _h(x):
    return x.cpu().numpy()


def _fused_dict(outs):
    """Per-patient fused outputs in the reference's [patient, ...] layout."""
    d = {"scal": _h(outs.bg_stats).T, "hist": _h(outs.bg_hist).T, "day_dose": _h(outs.day_dose).transpose(2, 0, 1),
         "hypo": _h(outs.hypo_events).T}
    if outs.timeline_pp is not None:
        d["timeline"] = _h(outs.timeline_pp).T
    return d


def _golden_dict(g):
    return {"scal": g["scal"], "hist": g["hist"], "timeline": g["timeline"], "day_dose": g["day_dose"],
            "hypo": g["hypo"]}


def test_fast_generator_equals_fast_csr_of_host_twin(dev):
    """Device-generated schedule and host-twin schedule drive the fused
    kernel to bit-identical results."""
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    case = SimCase("sim_threemeal_dt60.npz")
    sub = case.subset(case.valid())
    inj = _injected(sub, dev)
    a = _run_fast(case, sub, dev, csr=_csr_ticks(case, sub, dev), injected=inj)
    b = _run_fast(case, sub, dev, meal_spec=ThreeMealProtocol().device_spec(), injected=inj)
    for k in ("status", "ticks", "bg_hist", "bg_stats", "day_dose", "hypo_events", "timeline_pp", "x_out"):
        assert np.array_equal(_h(getattr(a, k)), _h(getattr(b, k))), k


@pytest.mark.parametrize("name", ["sim_threemeal_dt60.npz", "sim_northern_dt30.npz", "sim_northern_dt30_8d.npz",
                                  "sim_hypo_threemeal_dt60.npz", "sim_hypo_northern_dt30.npz"])
def test_fast_matches_reference_to_rounding(dev, oracle, name):
    """Fused kernel (re-associated FMA arithmetic) vs the reference with the
    reference's injected noise: FP64 statistics agree to relative 1e-9;
    histograms and hypo-event counts (the latter from the reference's own BG
    traces) are identical, except for patients proven threshold ties
    (tests/ties.py: first divergence at a BG within 1e-12 of an edge, or a
    controller decision the reference's own controller flips on readings
    that close)."""
    case = SimCase(name)
    g = case.g
    sub = case.subset(case.valid())
    outs = _run_fast(case, sub, dev, csr=_csr_ticks(case, sub, dev), injected=_injected(sub, dev))
    st = _h(outs.status)
    for j, i in enumerate(sub["idx"]):
        assert st[j] == g["status"][i]
    ties.check_patients(oracle, dev, len(sub["idx"]), _golden_dict(g), _fused_dict(outs),
                        ties.case_inputs(case, sub), label=name, ref_index=lambda j: sub["idx"][j])


def _host_acc_from_fast(outs, case_cfg, sz, pid0):
    from paper_2202_13927_b200.analytics import PatientStats, TrialAccumulator
    acc = TrialAccumulator(case_cfg.dt_s, sz["horizon_ticks"], sz["n_days"], sz["n_grid"], case_cfg.grid_step_s)
    status, hist, st, dd = _h(outs.status), _h(outs.bg_hist), _h(outs.bg_stats), _h(outs.day_dose)
    tl, ev, ticks = _h(outs.timeline_pp), _h(outs.hypo_events), _h(outs.ticks)
    for j in range(outs.n):
        if status[j] != 0:
            acc.add_aborted(pid0 + j)
            continue
        ps = PatientStats(case_cfg.dt_s, sz["horizon_ticks"], sz["n_days"], sz["n_grid"])
        ps.bg_hist = hist[:, j].astype(np.int64)
        c = np.cumsum(ps.bg_hist)
        ps.tir_ticks = np.array([c[25], c[34] - c[25], c[95] - c[34], c[134] - c[95], c[-1] - c[134]], np.int64)
        ps.ticks = int(ticks[j])
        ps.min_bg, ps.max_bg, ps.sum_bg = float(st[0, j]), float(st[1, j]), float(st[2, j])
        ps.timeline_bg = tl[:, j].copy()
        ps.day_dose = dd[:, :, j].copy()
        acc.add_patient(pid0 + j, ps, hypo_events=(int(ev[0, j]), int(ev[1, j])))
    return acc


def _acc_equal(a, b):
    from paper_2202_13927_b200 import analytics
    ra = analytics.report_bytes(analytics.build_trial_report(a, {}))
    rb = analytics.report_bytes(analytics.build_trial_report(b, {}))
    return ra == rb and np.array_equal(a.metric_hist, b.metric_hist) and a.aborted_ids == b.aborted_ids


def _fast_trial(n, pid0, cfg, dev, per_patient_timeline=True, seed_pop=5):
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial
    from paper_2202_13927_b200 import engine
    pop = generate_population(seed_pop, n, pid0=pid0, device=dev, on_exhausted="redraw_weight")
    ft = FastTrial(pid0, pop.params_device, pop.basal_device, ThreeMealProtocol(),
                   ControllerHyperparameters(), cfg, device=dev, per_patient_metrics=True)
    if per_patient_timeline:
        ft.outs = engine.alloc_fast_outputs(ft.n, pid0, ft.sz, dev, per_patient_timeline=True)
    ft.step()
    return ft


def test_device_reduction_equals_host_fold(dev):
    from paper_2202_13927_b200.config import SimulationConfig
    cfg = SimulationConfig(horizon_s=28 * 86400.0, seed=4, dt_s=60.0)
    ft = _fast_trial(1000, 0, cfg, dev)
    dev_acc = ft.accumulator()
    host_acc = _host_acc_from_fast(ft.outs, cfg, ft.sz, 0)
    assert dev_acc.n_patients == host_acc.n_patients == 1000
    assert np.array_equal(dev_acc.tir_hist, host_acc.tir_hist)
    assert np.array_equal(dev_acc.below_min, host_acc.below_min)
    assert np.array_equal(dev_acc.timeline_sum_fp, host_acc.timeline_sum_fp)
    assert dev_acc.dose_sum_fp == host_acc.dose_sum_fp
    assert _acc_equal(dev_acc, host_acc)


def test_sharding_invariance(dev):
    """Two shards (pid ranges) merged == one launch over all patients."""
    from paper_2202_13927_b200.analytics import merge
    from paper_2202_13927_b200.config import SimulationConfig
    cfg = SimulationConfig(horizon_s=7 * 86400.0, seed=9, dt_s=60.0)
    full = _fast_trial(700, 0, cfg, dev, per_patient_timeline=False).accumulator()
    a = _fast_trial(333, 0, cfg, dev, per_patient_timeline=False).accumulator()
    b = _fast_trial(367, 333, cfg, dev, per_patient_timeline=False).accumulator()
    assert _acc_equal(full, merge(a, b))
    assert _acc_equal(full, merge(b, a))


def test_diverged_patients_excluded_exactly(dev):
    """A patient that diverges mid-trial is reported aborted and its warp is
    re-run so no statistic includes it (analytics.py:267-269)."""
    from paper_2202_13927_b200 import engine
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=2 * 86400.0, seed=2, dt_s=60.0)
    pop = generate_population(3, 64, device=dev)
    params = pop.params_device.clone()
    params[5, 4] = -5.0             # ka1 < 0: insulin action grows without bound -> non-finite
    ft = FastTrial(0, params, pop.basal_device, ThreeMealProtocol(), ControllerHyperparameters(), cfg, device=dev)
    ft.outs = engine.alloc_fast_outputs(64, 0, ft.sz, dev, per_patient_timeline=True)
    ft.step()
    acc = ft.accumulator()
    assert acc.aborted_ids == (5,)
    assert acc.n_patients == 63
    host = _host_acc_from_fast(ft.outs, cfg, ft.sz, 0)
    assert _acc_equal(acc, host)


@pytest.mark.parametrize("controller", ["dual_hormone", "pid_pump"])
def test_diverged_rerun_under_sliced_schedule(dev, controller):
    """The diverged-patient re-run under a sliced schedule, whose lane state
    (histogram counters included) is carried between slices through L2
    (evict_last stores, discard after the restore): results and accumulator
    equal the unsliced run's, bit for bit, with 100 patients (4 warps, one
    with padding lanes) and 1, 4 and 7 slices."""
    import torch
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.pid import PIDProfile
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=3 * 86400.0, seed=8, dt_s=60.0)
    pop = generate_population(9, 100, device=dev, on_exhausted="redraw_weight")
    params = pop.params_device.clone()
    params[37, 4] = -5.0             # ka1 < 0: diverges mid-trial
    prof = PIDProfile() if controller == "pid_pump" else ControllerHyperparameters()
    runs = []
    for s in (1, 4, 7):
        ft = FastTrial(0, params, pop.basal_device, ThreeMealProtocol(), prof, cfg, controller_id=controller,
                       device=dev, n_slices=s, per_patient_metrics=True)
        ft.step()
        runs.append((ft, ft.accumulator()))
    ft0, acc0 = runs[0]
    assert acc0.aborted_ids == (37,) and acc0.n_patients == 99
    keep = torch.arange(100, device=dev) != 37  # the aborted lane's float statistics are NaN / discarded
    for ft, acc in runs[1:]:
        assert _acc_equal(acc, acc0)
        for k in ("status", "ticks", "bg_hist", "hypo_events"):
            assert torch.equal(getattr(ft.outs, k), getattr(ft0.outs, k)), k
        for k in ("bg_stats", "day_dose"):
            assert torch.equal(getattr(ft.outs, k)[..., keep], getattr(ft0.outs, k)[..., keep]), k


def test_philox_trial_statistics_match_oracle(dev, oracle):
    """Independent noise streams (device FP32 Box-Muller vs the oracle's
    double Box-Muller) -> population TIR statistics agree within Monte Carlo
    tolerance on the same population and schedules."""
    from paper_2202_13927_b200.config import SimulationConfig, sizes
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    cfg = SimulationConfig(horizon_s=7 * 86400.0, seed=21, dt_s=60.0)
    ft = _fast_trial(512, 0, cfg, dev, per_patient_timeline=False, seed_pop=21)
    m = ft.metrics()
    prof = ControllerHyperparameters()
    params = ft.params.cpu().numpy()
    ref = oracle.run_batch_philox(ThreeMealProtocol(), cfg.seed + 1000, 0, params, ft.x0.cpu().numpy(),
                                  ft.c0.cpu().numpy(), prof.to_vec(), ft.basal.cpu().numpy(), ft.sz,
                                  cfg.dt_s, cfg.controller_period_s)
    H = ft.sz["horizon_ticks"]
    tir_ref = ref["tir_ticks"][:, 2] / H
    tir_dev = m["tir"].astype(np.float64)
    se = np.sqrt(tir_ref.var() / tir_ref.size + tir_dev.var() / tir_dev.size)
    assert abs(tir_ref.mean() - tir_dev.mean()) < 5 * se
    for q in (0.05, 0.25, 0.5, 0.75, 0.95):
        assert abs(np.quantile(tir_ref, q) - np.quantile(tir_dev, q)) < 0.05


@pytest.mark.parametrize("slices", [2, 3, 7])
def test_horizon_slicing_is_invisible(dev, slices):
    """The persistent schedule may cut each patient's horizon into slices
    (state saved/restored between them); results are bit-identical to the
    unsliced run, including a diverged patient's exclusion."""
    from paper_2202_13927_b200 import engine
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=9 * 86400.0, seed=12, dt_s=60.0)
    pop = generate_population(8, 200, device=dev, on_exhausted="redraw_weight")
    params = pop.params_device.clone()
    params[37, 4] = -5.0   # one diverging patient
    runs = []
    for s in (1, slices):
        ft = FastTrial(0, params, pop.basal_device, ThreeMealProtocol(), ControllerHyperparameters(), cfg,
                       device=dev, n_slices=s, per_patient_metrics=True)
        ft.outs = engine.alloc_fast_outputs(ft.n, 0, ft.sz, dev, per_patient_timeline=True, final_state=True)
        ft.step()
        runs.append(ft)
    a, b = runs
    for k in ("status", "ticks", "bg_hist", "bg_stats", "day_dose", "hypo_events", "timeline_pp",
              "timeline_warp", "x_out"):
        # the diverged patient's own (discarded) statistics are NaN in both runs
        assert np.array_equal(_h(getattr(a.outs, k)), _h(getattr(b.outs, k)),
                              equal_nan=getattr(a.outs, k).dtype.is_floating_point), k
    assert _acc_equal(a.accumulator(), b.accumulator())
    assert a.accumulator().aborted_ids == (37,)


def test_fast_worst_trace_reproduces_the_worst_case(dev, tmp_path):
    """store_trace on the fused path: the worst case is re-simulated with the
    per-step trace (same Philox streams and arithmetic), so its minimum BG,
    ticks below 3 mmol/L, histogram and BG sum are reproduced exactly
    (the reference's contract, test_simulation.py:290-306)."""
    import os
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.layout import THRESHOLDS
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.simulation import load_trace, run_trial
    cfg = SimulationConfig(horizon_s=3 * 86400.0, seed=17, dt_s=60.0, store_trace="always")
    pop = generate_population(17, 300, device=dev, on_exhausted="redraw_weight")
    res = run_trial(pop, ThreeMealProtocol(), "dual_hormone", ControllerHyperparameters(), "hovorka_ext", cfg,
                    noise="philox", device=dev, trace_dir=str(tmp_path))
    w = res.accumulator.worst
    tr = res.worst_trace
    H = 3 * 1440
    assert tr.shape == (H, 8)
    bg = tr[:, 1]
    assert bg.min() == w.min_bg and bg.max() == w.max_bg
    assert int((bg < 3.0).sum()) == w.ticks_below_3
    assert np.array_equal(np.bincount(np.searchsorted(THRESHOLDS, bg, side="right"), minlength=247), w.bg_hist)
    assert np.array_equal(tr[:, 0], np.arange(H) * 60.0)
    assert np.all(tr[::5, 5] >= 0) and np.all(np.diff(tr[:, 2])[np.arange(H - 1) % 5 != 4] == 0)
    files = sorted(os.listdir(tmp_path))
    assert len(files) == res.accumulator.n_patients
    again = load_trace(os.path.join(tmp_path, f"patient_{w.patient_id:06d}.npz"))
    assert np.array_equal(again, tr)


def test_run_trial_sharded_world1_equals_single_trial(dev):
    """parallel.run_trial_sharded over NCCL (world size 1 on the one GPU the
    tests have) returns the single-process report and the per-patient arrays."""
    import socket
    import torch.distributed as dist
    from paper_2202_13927_b200 import analytics
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.parallel import run_trial_sharded
    from paper_2202_13927_b200.pid import PIDProfile
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cfg = SimulationConfig(horizon_s=3 * 86400.0, seed=8, dt_s=60.0)
    dist.init_process_group("nccl", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{port}", device_id=dev)
    try:
        rep, acc, met = run_trial_sharded(500, 9, ThreeMealProtocol(), "pid_pump", PIDProfile(), cfg, device=dev,
                                          gather_metrics=True)
    finally:
        dist.destroy_process_group()
    pop = generate_population(9, 500, device=dev, on_exhausted="redraw_weight")
    ft = FastTrial(0, pop.params_device, pop.basal_device, ThreeMealProtocol(), PIDProfile(), cfg, "pid_pump", dev,
                   per_patient_metrics=True)
    ft.step()
    ref = ft.accumulator()
    assert analytics.report_bytes(rep) == analytics.report_bytes(analytics.build_trial_report(ref, {}))
    assert np.array_equal(met["tir"], ft.metrics()["tir"])


def test_validate_parameter_sets(dev):
    """Every sampled set passes the reference's three acceptance rules
    (population.py:262-282); corrupted sets are reported."""
    from paper_2202_13927_b200.layout import PARAM_INDEX
    from paper_2202_13927_b200.population import generate_population, validate_parameter_sets
    pop = generate_population(12, 300, device=dev, on_exhausted="redraw_weight")
    assert all(v == [] for v in validate_parameter_sets(pop.params_device, pop.basal_device, device=dev))
    p = pop.params_device[:4].clone()
    ub = pop.basal_device[:4].clone()
    p[0, PARAM_INDEX["EGP0"]] = -1.0
    p[1, PARAM_INDEX["k12"]] += 10.0
    ub[2] = 0.1
    ub[3] *= 1.01
    v = validate_parameter_sets(p, ub, device=dev)
    assert any("negative" in s for s in v[0]) and any("standard deviation" in s for s in v[1])
    assert any("below" in s for s in v[2]) and any("does not match" in s for s in v[3])


def test_chunked_population_equals_single_launch(dev):
    """run_population_chunked merges per-chunk exact accumulators: same report
    as one launch over all ids (chunk boundaries at ragged sizes)."""
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial, run_population_chunked
    cfg = SimulationConfig(horizon_s=2 * 86400.0, seed=6, dt_s=60.0)
    acc = run_population_chunked(700, 13, ThreeMealProtocol(), ControllerHyperparameters(), cfg, device=dev,
                                 chunk=257)
    pop = generate_population(13, 700, device=dev, on_exhausted="redraw_weight")
    ft = FastTrial(0, pop.params_device, pop.basal_device, ThreeMealProtocol(), ControllerHyperparameters(), cfg,
                   device=dev)
    ft.step()
    assert _acc_equal(acc, ft.accumulator())


@pytest.mark.parametrize("horizon_h,dt_s,grid_s,slices", [(36, 30.0, 1800.0, 1), (36, 30.0, 1800.0, 3),
                                                          (50, 20.0, 3600.0, 2), (25, 60.0, 7200.0, 0),
                                                          (30, 6.0, 3600.0, 2)])   # C4's 0.1-min substep
def test_fused_equals_parity_on_odd_horizons(dev, oracle, horizon_h, dt_s, grid_s, slices):
    """Partial last day, non-hourly grid, other dt, sliced schedules: the fused
    kernel (reference noise injected, CSR schedules) agrees with the reference
    (the oracle; the parity kernel equals it bit for bit) to 1e-9, with
    identical histograms and hypo events apart from proven threshold ties."""
    import torch
    from paper_2202_13927_b200 import engine, rng
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol, compile_protocol, compile_ticks
    from paper_2202_13927_b200.simulation import _csr
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=horizon_h * 3600.0, seed=7, dt_s=dt_s, grid_step_s=grid_s)
    n = 70
    pop = generate_population(21, n, device=dev, on_exhausted="redraw_weight")
    prof, gen = ControllerHyperparameters(), ThreeMealProtocol()
    ft = FastTrial(0, pop.params_device, pop.basal_device, gen, prof, cfg, device=dev, n_slices=slices)
    sz = ft.sz
    H, ps = sz["horizon_ticks"], sz["period_steps"]
    params, x0, c0, ub = (t.cpu().numpy() for t in (ft.params, ft.x0, ft.c0, ft.basal))
    pas = [compile_protocol(gen.build(cfg.seed, type("P", (), {"id": i, "body_weight_kg": params[i, 0]})()),
                            cfg.horizon_s) for i in range(n)]
    moff, meals, eoff, ex = _csr(pas)
    W = np.zeros((n, H, 3)); M = np.zeros((n, H // ps))
    for i in range(n):
        W[i], M[i] = rng.reference_noise(cfg.seed, i, H, ps, True, True)
    hn = np.ones(n, np.uint8)
    par = engine.run_parity(engine.ParityBatch(params, x0, c0, prof.to_vec(), ub, moff, meals, eoff, ex, W, hn, M),
                            sz, cfg.dt_s, cfg.controller_period_s, device=dev)
    ref = oracle.run_batch_injected(params, x0, c0, prof.to_vec(), ub, sz, cfg.dt_s, cfg.controller_period_s,
                                    moff, meals, eoff, ex, W, hn, M)
    ft.outs = engine.alloc_fast_outputs(n, 0, sz, dev, per_patient_timeline=True)
    ft.simulate(injected={"wiener": engine.dev(W.reshape(-1), torch.float64, dev),
                          "has_noise": engine.dev(hn, torch.uint8, dev),
                          "meas": engine.dev(M.reshape(-1), torch.float64, dev)})
    assert ft.outs.timeline_pp.shape[0] == sz["n_grid"] and ft.outs.day_dose.shape[0] == sz["n_days"]
    for k in ("status", "ticks", "tir_ticks", "bg_hist", "scal", "day_dose", "timeline"):
        assert np.array_equal(par[k], ref[k]), k     # parity kernel == oracle (the reference), bitwise
    refd = {"scal": ref["scal"], "hist": ref["bg_hist"], "timeline": ref["timeline"], "day_dose": ref["day_dose"],
            "hypo": ref["hypo_events"]}
    ties.check_patients(oracle, dev, n, refd, _fused_dict(ft.outs),
                        ties.inputs_from_arrays(params, x0, c0, ub, prof.to_vec(), moff, meals, eoff, ex, W, hn, M,
                                                0, sz, cfg.dt_s, cfg.controller_period_s),
                        label=f"odd horizon {horizon_h} h dt {dt_s} grid {grid_s} slices {slices}")


@pytest.mark.parametrize("controller", ["dual_hormone", "pid_pump"])
def test_nonfinite_non_glucose_state_aborts(dev, controller):
    """A non-finite state other than glucose (the sensor Gsc at t = 0) aborts
    the patient, as the reference's per-tick state check does
    (_kernel.py:98-103): the fused kernel checks the state at the horizon's
    last tick (non-finiteness is absorbing) and the BG sum after the last
    step.  The other patients' statistics exclude it exactly."""
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.layout import IGSC
    from paper_2202_13927_b200.pid import PIDProfile
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=86400.0, seed=4, dt_s=60.0)
    pop = generate_population(3, 64, device=dev, on_exhausted="redraw_weight")
    prof = PIDProfile() if controller == "pid_pump" else ControllerHyperparameters()
    ft = FastTrial(0, pop.params_device, pop.basal_device, ThreeMealProtocol(), prof, cfg, controller, dev,
                   per_patient_metrics=True)
    x0 = ft._inputs["x0"].clone()
    x0[7, IGSC] = float("nan")
    ft._inputs["x0"] = x0
    ft.step()
    acc = ft.accumulator()
    assert acc.aborted_ids == (7,)
    assert acc.n_patients == 63
    clean = FastTrial(0, pop.params_device, pop.basal_device, ThreeMealProtocol(), prof, cfg, controller, dev,
                      per_patient_metrics=True)
    clean.step()
    keep = np.arange(64) != 7
    assert np.array_equal(ft.metrics()["tir"][keep], clean.metrics()["tir"][keep])


def test_philox_forms_agree_generator_vs_csr(dev):
    """Under device Philox noise (the per-patient philox_lane form, pinned to
    the plain rounds in test_host.py) the 3-meal generator run and the CSR
    run of its host twin draw the same stream: bit-identical results."""
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    case = SimCase("sim_threemeal_dt60.npz")
    sub = case.subset(case.valid())
    a = _run_fast(case, sub, dev, csr=_csr_ticks(case, sub, dev), injected=None)
    b = _run_fast(case, sub, dev, meal_spec=ThreeMealProtocol().device_spec(), injected=None)
    for k in ("status", "ticks", "bg_hist", "bg_stats", "day_dose", "hypo_events", "timeline_pp", "x_out"):
        assert np.array_equal(_h(getattr(a, k)), _h(getattr(b, k))), k


@pytest.mark.parametrize("name,controller", [("sim_hypo_threemeal_dt60.npz", 0), ("sim_hypo_pid_threemeal_dt60.npz", 1),
                                             ("sim_hypo_northern_dt30.npz", 0)])
def test_tie_classifier_runners_on_device(dev, oracle, name, controller):
    """The classifier's two runners (tests/ties.py) on real patients: the fused
    TRACE run reproduces the fused statistics it stands for, and against the
    reference's trace it has no discrete divergence (so a real tie would be
    located at its first tick)."""
    case = SimCase(name)
    sub = case.subset(case.valid())
    mk = ties.case_inputs(case, sub, controller)
    for j in range(min(4, len(sub["idx"]))):
        pi = mk(j)
        tr_r, ticks = ties.oracle_trace(oracle, pi)
        tr_f, outs = ties.fused_trace(pi, dev)
        hist_f, _ = ties.trace_hist(tr_f, ticks)
        assert np.array_equal(hist_f, _h(outs.bg_hist)[:, 0])
        assert np.array_equal(_h(outs.hypo_events)[:, 0], case.g["hypo"][sub["idx"][j]])
        assert ties.first_divergence(tr_r, tr_f) is None
        assert np.allclose(tr_f[:ticks, 1], tr_r[:ticks, 1], rtol=1e-9, atol=0)


@pytest.mark.parametrize("controller", ["dual_hormone", "pid_pump"])
def test_hypo_runs_across_slices(dev, controller):
    """Hypoglycaemia runs carried across horizon slices (saved lane state):
    an insulin-overdosed population (assumed basal x 2.6) has many events,
    and their counts -- with every other output -- are identical for 1, 5 and
    13 slices."""
    import torch
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.pid import PIDProfile
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=9 * 86400.0, seed=14, dt_s=60.0)
    pop = generate_population(6, 160, device=dev, on_exhausted="redraw_weight")
    prof = PIDProfile() if controller == "pid_pump" else ControllerHyperparameters()
    basal = pop.basal_device * (1.8 if controller == "pid_pump" else 2.6)
    runs = []
    for s in (1, 5, 13):
        ft = FastTrial(0, pop.params_device, basal, ThreeMealProtocol(), prof, cfg, controller_id=controller,
                       device=dev, n_slices=s, per_patient_metrics=True)
        ft.step()
        runs.append(ft)
    h0 = _h(runs[0].outs.hypo_events)
    assert h0[0].sum() >= 100 and h0[1].sum() >= 10, h0.sum(axis=1)
    for ft in runs[1:]:
        for k in ("status", "bg_hist", "bg_stats", "hypo_events", "day_dose"):
            assert torch.equal(getattr(ft.outs, k), getattr(runs[0].outs, k)), k


def test_abort_tick_matches_reference(dev):
    """The fused path's abort tick of a diverging patient is the reference's
    (simulation.py:381: ticks counted before the abort).  The reference's own
    fault fixture (tau_cgm = -1: the sensor state diverges, caught by the
    per-tick state check, _kernel.py:98-103) aborts at tick 1760; the
    throughput launch detects the divergence at the horizon, and the
    abort-tick pass (rerun_diverged = 2) recovers the exact tick."""
    from paper_2202_13927_b200 import engine, rng
    from paper_2202_13927_b200._lib import GT_STATUS_NONFINITE
    case = SimCase("sim_faults.npz")
    g = case.g
    bad = int(np.nonzero(g["status"] == GT_STATUS_NONFINITE)[0][0])
    sub = case.subset(np.arange(case.n) == bad)   # alone: its tau_cgm is a launch constant
    inj = _injected(sub, dev)
    csr = _csr_ticks(case, sub, dev)
    outs = _run_fast(case, sub, dev, csr=csr, injected=inj)
    assert _h(outs.status)[0] == GT_STATUS_NONFINITE
    # lazy detection: the state check at the horizon's last controller tick
    assert _h(outs.ticks)[0] == case.sz["horizon_ticks"] - case.sz["period_steps"]
    for mode in (1, 2):
        engine.launch_fast(_inputs(case, sub, dev), outs, case.sz, case.config.dt_s,
                           case.config.controller_period_s, case.config.seed, rng.ROLE_DEVICE_NOISE,
                           max(1, int(np.ceil(900 / case.config.dt_s))), dev, csr=csr, injected=inj,
                           rerun_diverged=mode)
    assert _h(outs.status)[0] == GT_STATUS_NONFINITE
    assert int(_h(outs.ticks)[0]) == int(g["ticks"][bad]) == 1760


@pytest.mark.parametrize("controller", ["dual_hormone", "pid_pump"])
def test_fast_trial_abort_tick_is_exact(dev, controller):
    """FastTrial.step() ends with the abort-tick pass: a diverging patient's
    ticks is the first tick whose state or BG is non-finite (the traced
    re-simulation, which checks every tick and step as the reference does,
    agrees, and its BG column is finite before it), every other patient's
    outputs are untouched by the pass."""
    from paper_2202_13927_b200._lib import GT_STATUS_NONFINITE
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.pid import PIDProfile
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=2 * 86400.0, seed=2, dt_s=60.0)
    pop = generate_population(3, 64, device=dev, on_exhausted="redraw_weight")
    params = pop.params_device.clone()
    params[5, 4] = -5.0             # ka1 < 0: diverges mid-trial
    prof = PIDProfile() if controller == "pid_pump" else ControllerHyperparameters()
    ft = FastTrial(0, params, pop.basal_device, ThreeMealProtocol(), prof, cfg, controller, dev,
                   per_patient_metrics=True)
    ft.simulate()
    ft.simulate(rerun_diverged=1)
    before = {k: _h(getattr(ft.outs, k)).copy() for k in ("status", "ticks", "bg_hist", "bg_stats", "day_dose",
                                                            "hypo_events", "timeline_warp")}
    ft.simulate(rerun_diverged=2)
    st, ticks = _h(ft.outs.status), _h(ft.outs.ticks)
    H = ft.sz["horizon_ticks"]
    assert st[5] == GT_STATUS_NONFINITE and 0 < ticks[5] < H
    keep = np.arange(64) != 5
    for k, v in before.items():
        now = _h(getattr(ft.outs, k))
        if k in ("status", "ticks"):
            assert np.array_equal(now[keep], v[keep]), k
        else:
            assert np.array_equal(now, v, equal_nan=True), k
    _s, tt, tr = ft.trace_range(5, 6)
    assert _s[0] == GT_STATUS_NONFINITE and tt[0] == ticks[5]
    assert np.all(np.isfinite(tr[0, : ticks[5], 1]))
