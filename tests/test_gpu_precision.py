"""GPU tests of the precision / step study path (BASELINE configs[4]):
Brownian aggregation (a dt step driven by the sum of the dt/agg fine
increments, i.e. the same Philox path as a run at dt/agg) and the FP32
integrator (controller and statistics stay FP64)."""

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


@pytest.fixture(scope="module")
def pop(dev):
    from paper_2202_13927_b200.population import generate_population
    return generate_population(31, 2048, device=dev, on_exhausted="redraw_weight")


def _run(pop, dev, dt_s, agg=1, fp32=False, days=7, seed=5):
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=days * 86400.0, seed=seed, dt_s=dt_s)
    ft = FastTrial(0, pop.params_device, pop.basal_device, ThreeMealProtocol(), ControllerHyperparameters(),
                   cfg, device=dev, per_patient_metrics=True, noise_agg=agg, fp32=fp32)
    ft.step()
    m = ft.metrics()
    ok = m["status"] == 0
    mean_bg = ft.outs.bg_stats[2].cpu().numpy() / ft.outs.ticks.cpu().numpy()
    return ft, m, ok, mean_bg


def test_noise_agg_one_is_the_default_path(pop, dev):
    _, a, _, bga = _run(pop, dev, 60.0, agg=1, days=2)
    ft, b, _, bgb = _run(pop, dev, 60.0, days=2)
    assert np.array_equal(bga, bgb) and np.array_equal(a["tir"], b["tir"])


def test_aggregated_step_shares_the_fine_brownian_path(pop, dev):
    """dt=60 s driven by agg=10 fine increments tracks the dt=6 s run on the
    same Philox path far more closely than a dt=60 s run on an independent
    path does (strong, pathwise agreement), and the population metrics agree."""
    _, m_c, ok_c, bg_c = _run(pop, dev, 60.0, agg=10)
    _, m_f, ok_f, bg_f = _run(pop, dev, 6.0, agg=1)
    _, m_i, ok_i, bg_i = _run(pop, dev, 60.0, agg=1)
    ok = ok_c & ok_f & ok_i
    assert ok.mean() > 0.99
    d_shared = np.median(np.abs(bg_c[ok] - bg_f[ok]))
    d_indep = np.median(np.abs(bg_i[ok] - bg_f[ok]))
    assert d_shared < 0.3 * d_indep, (d_shared, d_indep)
    tir_c, tir_f = m_c["tir"][ok].astype(np.float64), m_f["tir"][ok].astype(np.float64)
    assert abs(tir_c.mean() - tir_f.mean()) < 0.01
    assert np.corrcoef(bg_c[ok], bg_f[ok])[0, 1] > 0.99


def test_fp32_integrator_deviation_is_small(pop, dev):
    """Same streams, FP32 vs FP64 integrator: per-patient and population
    metrics deviate at the level BASELINE configs[4] reports."""
    _, m64, ok64, bg64 = _run(pop, dev, 60.0)
    _, m32, ok32, bg32 = _run(pop, dev, 60.0, fp32=True)
    ok = ok64 & ok32
    assert np.array_equal(ok64, ok32)
    rel = np.abs(bg32[ok] - bg64[ok]) / bg64[ok]
    assert np.median(rel) < 1e-3, np.median(rel)
    assert np.quantile(rel, 0.99) < 2e-2
    for k in ("tir", "tbr70", "tbr54", "tar180", "tar250"):
        a, b = m64[k][ok].astype(np.float64), m32[k][ok].astype(np.float64)
        assert abs(a.mean() - b.mean()) < 2e-3, k


def test_fp32_agg_combination_runs(pop, dev):
    _, m, ok, bg = _run(pop, dev, 60.0, agg=4, fp32=True, days=2)
    _, m2, ok2, bg2 = _run(pop, dev, 60.0, agg=4, days=2)
    assert np.array_equal(ok, ok2)
    assert np.median(np.abs(bg - bg2)[ok] / bg2[ok]) < 1e-3


def test_unsupported_combinations_fail_loudly(pop, dev):
    from paper_2202_13927_b200._lib import GlucosimError
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.northern import NorthernYearProtocol
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=1 * 86400.0, seed=1, dt_s=60.0)
    params, basal = pop.params_device[:64].contiguous(), pop.basal_device[:64].contiguous()
    ft = FastTrial(0, params, basal, NorthernYearProtocol(), ControllerHyperparameters(), cfg,
                   device=dev, fp32=True)
    with pytest.raises(GlucosimError, match="FP32"):
        ft.simulate()
    ft = FastTrial(0, params, basal, NorthernYearProtocol(), ControllerHyperparameters(), cfg,
                   device=dev, noise_agg=0)
    with pytest.raises(GlucosimError, match="noise_agg"):
        ft.simulate()
