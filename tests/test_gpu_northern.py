"""GPU tests of the on-device NorthernYearProtocol builder
(csrc/gt_northern.cu): bit-identical to the host path
generator.build -> compile_protocol -> compile_ticks, and a fused trial on
the device-built schedule equals one on the host-built CSR."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch
    from paper_2202_13927_b200 import _lib
    assert torch.cuda.is_available()
    _lib.load()
    return torch.device("cuda", 0)


class _P:
    def __init__(self, pid, w):
        self.id, self.body_weight_kg = pid, w


@pytest.mark.parametrize("days,dt_s,trial_seed,pid0", [(364, 60.0, 5, 0), (28, 30.0, 2**40 + 3, 77_777),
                                                       (9, 60.0, 0, 2**33 - 5)])
def test_device_northern_csr_equals_host_compile(dev, days, dt_s, trial_seed, pid0):
    import torch
    from paper_2202_13927_b200 import engine, northern
    from paper_2202_13927_b200.protocol import compile_protocol, compile_ticks
    n = 40
    rs = np.random.default_rng(days)
    params = np.zeros((n, 30))
    params[:, 0] = rs.uniform(30.0, 120.0, n)
    horizon = days * 86400.0
    csr = engine.northern_csr(engine.dev(params, torch.float64, dev), pid0, trial_seed, dt_s, 300.0, horizon,
                              dev, week_days=True)
    h = {k: v.cpu().numpy() for k, v in csr.items()}
    gen = northern.NorthernYearProtocol()
    for i in range(n):
        pid = pid0 + i
        pa = compile_protocol(gen.build(trial_seed, _P(pid, float(params[i, 0]))), horizon)
        ta = compile_ticks(pa, dt_s, 300.0)
        nm, ne = ta.meal_ks.size, ta.ex_ks.size
        assert h["n_meals"][i] == nm and h["n_ex"][i] == ne
        m0, e0 = i * 1588, i * 76
        for k in ("meal_ks", "meal_ke", "meal_kp", "meal_rate", "meal_ann"):
            assert np.array_equal(h[k][m0:m0 + nm], getattr(ta, k)), k
        assert np.all(h["meal_ks"][m0 + nm:m0 + 1588] == np.iinfo(np.int32).max)
        for k, hk in (("ex_ks", "ex_ks"), ("ex_ke", "ex_ke"), ("ex_start_s", "ex_start"), ("ex_hrr", "ex_hrr"),
                      ("ex_announced", "ex_announced")):
            assert np.array_equal(h[k][e0:e0 + ne], getattr(ta, hk)), k
        from paper_2202_13927_b200 import rng
        _, plan = northern.plan_year(rng.derive_seed(trial_seed, pid, rng.ROLE_PROTOCOL))
        codes = northern.week_day_codes(plan)
        assert [int(c) & 0xFFFF for c in h["week_days"][:, i]] == codes


def test_fused_trial_on_device_northern_equals_host_csr(dev):
    """Same schedule whether compiled on the host or planned on the device:
    the fused trial's report is byte-identical."""
    from paper_2202_13927_b200 import analytics
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.northern import NorthernYearProtocol
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=10 * 86400.0, seed=3, dt_s=60.0)
    pop = generate_population(4, 96, device=dev, on_exhausted="redraw_weight")

    class HostOnly(NorthernYearProtocol):
        def on_device(self):
            return False

    accs = []
    for gen in (NorthernYearProtocol(), HostOnly()):
        ft = FastTrial(0, pop.params_device, pop.basal_device, gen, ControllerHyperparameters(), cfg,
                       device=dev, per_patient_metrics=True)
        ft.step()
        accs.append(ft.accumulator())
    ra, rb = (analytics.report_bytes(analytics.build_trial_report(a, {})) for a in accs)
    assert ra == rb and np.array_equal(accs[0].metric_hist, accs[1].metric_hist)


@pytest.mark.parametrize("frac,lo,hi", [(0.3, 0.8, 1.2), (0.0, 0.9, 0.9), (1.0, 1.0, 1.0), (0.05, 1.0, 1.5)])
def test_device_announcement_policy_equals_host(dev, frac, lo, hi):
    """The announcement policy (protocol.py:373-394) applied on the device
    from the reference's own stream(trial_seed, pid, ROLE_ANNOUNCEMENT):
    announced carbs of every meal equal the host path (numpy Generator)."""
    import torch
    from paper_2202_13927_b200 import engine, northern
    from paper_2202_13927_b200.protocol import compile_protocol, compile_ticks
    n, days, dt_s, trial_seed, pid0 = 24, 364, 60.0, 11, 500
    rs = np.random.default_rng(3)
    params = np.zeros((n, 30))
    params[:, 0] = rs.uniform(30.0, 120.0, n)
    pol = northern.AnnouncementPolicy(fraction_unannounced=frac, misannouncement_factor_range=(lo, hi))
    gen = northern.NorthernYearProtocol(announcement=pol)
    assert gen.on_device()
    csr = engine.northern_csr(engine.dev(params, torch.float64, dev), pid0, trial_seed, dt_s, 300.0,
                              days * 86400.0, dev, announcement=pol)
    ann = csr["meal_ann"].cpu().numpy()
    for i in range(n):
        pa = compile_protocol(gen.build(trial_seed, _P(pid0 + i, float(params[i, 0]))), days * 86400.0)
        ta = compile_ticks(pa, dt_s, 300.0)
        m0 = i * 1588
        assert np.array_equal(ann[m0:m0 + ta.meal_ann.size], ta.meal_ann), i
    if frac == 1.0:
        assert not ann.any()


def test_fused_trial_with_announcement_policy_on_device(dev):
    """A fused trial under a non-default policy planned on the device equals
    the one on the host-compiled schedule, report bytes included."""
    from paper_2202_13927_b200 import analytics
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.northern import AnnouncementPolicy, NorthernYearProtocol
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=9 * 86400.0, seed=6, dt_s=60.0)
    pop = generate_population(4, 64, device=dev, on_exhausted="redraw_weight")
    pol = AnnouncementPolicy(fraction_unannounced=0.25, misannouncement_factor_range=(0.7, 1.3))

    class HostOnly(NorthernYearProtocol):
        def on_device(self):
            return False

    accs = []
    for gen in (NorthernYearProtocol(announcement=pol), HostOnly(announcement=pol)):
        ft = FastTrial(0, pop.params_device, pop.basal_device, gen, ControllerHyperparameters(), cfg,
                       device=dev, per_patient_metrics=True)
        ft.step()
        accs.append(ft.accumulator())
    ra, rb = (analytics.report_bytes(analytics.build_trial_report(a, {})) for a in accs)
    assert ra == rb
