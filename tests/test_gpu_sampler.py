"""GPU tests of the population sampler (csrc/gt_sampler.cu): bit for bit
equal to the oracle's C twin, and distributed like the reference's own
generate_population (population.py:217-259; golden seed-7 n-4000 draw)."""

import numpy as np
import pytest

import sampler_checks

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch
    from paper_2202_13927_b200 import _lib
    assert torch.cuda.is_available()
    _lib.load()
    return torch.device("cuda", 0)


@pytest.mark.parametrize("seed,pid0,n", [(1, 0, 3000), (7, 123_456, 2000), (2**40 + 9, 0, 777)])
def test_device_sampler_bitwise_vs_oracle_twin(dev, oracle, seed, pid0, n):
    from paper_2202_13927_b200 import engine
    from paper_2202_13927_b200.layout import PARAM_INDEX, PARAM_NAMES
    from paper_2202_13927_b200.tables import default_parameter_table
    table = default_parameter_table()
    d = engine.sample_population(seed, n, table, pid0=pid0, device=dev, max_weight_redraws=16)
    o = oracle.sample_patients(table, seed, pid0, n, PARAM_INDEX, PARAM_NAMES, max_weight_redraws=16)
    for k in ("params", "x0", "u_basal", "attempts", "status", "reject_counts"):
        assert np.array_equal(d[k].cpu().numpy(), o[k]), k


def test_device_sampler_bitwise_vs_oracle_twin_on_edited_table(dev, oracle):
    """The cheap rules are decided on the uniform key with flip points found on
    the device (gt_sampler.cu key_rules_kernel); tables whose normal entries
    reject far more often (F01 sd x3: a value is negative below z = -1.47),
    have a zero sd (no variability, the 1-SD rule never fires) or a wide sd
    still give the sequential twin's populations and counters bit for bit."""
    import dataclasses
    from paper_2202_13927_b200 import engine
    from paper_2202_13927_b200.layout import PARAM_INDEX, PARAM_NAMES
    from paper_2202_13927_b200.tables import default_parameter_table
    table = default_parameter_table()
    s = dict(table.sampled)
    s["F01"] = dataclasses.replace(s["F01"], sd=3 * s["F01"].sd)
    s["EGP0"] = dataclasses.replace(s["EGP0"], sd=0.0)
    s["ka2"] = dataclasses.replace(s["ka2"], sd=0.5 * s["ka2"].mean)
    table = dataclasses.replace(table, sampled=s)
    d = engine.sample_population(3, 3000, table, device=dev, max_attempts=2000, max_weight_redraws=2)
    o = oracle.sample_patients(table, 3, 0, 3000, PARAM_INDEX, PARAM_NAMES, max_attempts=2000, max_weight_redraws=2)
    for k in ("params", "x0", "u_basal", "attempts", "status", "reject_counts"):
        assert np.array_equal(d[k].cpu().numpy(), o[k]), k
    assert int(o["reject_counts"][0]) > 0   # the negative-value rule fired


def test_device_sampler_distribution_matches_reference(dev):
    from paper_2202_13927_b200.population import generate_population
    pop = generate_population(2, 4000, device=dev, on_exhausted="redraw_weight")
    assert pop.n_weight_redraws == 0
    rc = (pop.stats.rejected_negative, pop.stats.rejected_outside_sd, pop.stats.rejected_no_steady_state,
          pop.stats.rejected_basal)
    rep, z = sampler_checks.check_against_reference(pop.params_device.cpu().numpy(), pop.basal_device.cpu().numpy(),
                                                     pop.stats.attempts, rc)
    print({k: round(v, 4) for k, v in rep.items()}, {k: round(float(v), 2) for k, v in z.items()})


@pytest.mark.parametrize("n", [100_000, 1_000_000])
def test_weight_redraw_counts_at_scale(dev, n):
    """How many patients redraw_weight touches: about
    1.7e-4 of the population (a body weight below ~30 kg)."""
    from paper_2202_13927_b200.population import generate_population
    pop = generate_population(1, n, device=dev, on_exhausted="redraw_weight")
    r = pop.n_weight_redraws
    print(f"n = {n}: {r} patients with a redrawn body weight ({r / n:.2e})")
    assert 0 < r < 5e-4 * n


@pytest.mark.parametrize("max_attempts,n", [(10_000, 100_000), (500, 20_000), (129, 4000)])
def test_straggler_path_bitwise(dev, oracle, max_attempts, n):
    """Patients still unaccepted after 384 attempts of one body weight are
    finished by the block-parallel straggler kernel; small budgets also force
    budget exhaustion, weight redraws and the failure path (the latest
    survivor's values).  The device equals the sequential C twin bit for bit
    either way, rejection counters and per-patient attempt totals included."""
    from paper_2202_13927_b200 import engine
    from paper_2202_13927_b200.layout import PARAM_INDEX, PARAM_NAMES
    from paper_2202_13927_b200.tables import default_parameter_table
    table = default_parameter_table()
    for redraws in (0, 3):
        d = engine.sample_population(2, n, table, device=dev, max_attempts=max_attempts,
                                     max_weight_redraws=redraws)
        o = oracle.sample_patients(table, 2, 0, n, PARAM_INDEX, PARAM_NAMES, max_attempts=max_attempts,
                                   max_weight_redraws=redraws)
        for k in ("params", "x0", "u_basal", "attempts", "status", "reject_counts"):
            assert np.array_equal(d[k].cpu().numpy(), o[k]), (k, max_attempts, redraws)
        if max_attempts > 384:
            assert int((o["attempts"] > 384).sum()) > 0       # the straggler kernel ran
        if max_attempts == 129 and redraws == 0:
            assert int((o["status"] != 0).sum()) > 0          # the failure path ran


def test_sampler_steady_states_reused_by_the_trial(dev):
    """FastTrial(x0=population.x0_device) skips the staging solve: the
    sampler's steady states are the same solve at the same target BG, so the
    trial's outputs are bit-identical."""
    import torch
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.pid import PIDProfile
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial
    cfg = SimulationConfig(horizon_s=3 * 86400.0, seed=5, dt_s=60.0)
    pop = generate_population(5, 300, device=dev, on_exhausted="redraw_weight")
    runs = []
    for x0 in (None, pop.x0_device):
        ft = FastTrial(0, pop.params_device, pop.basal_device, ThreeMealProtocol(), PIDProfile(), cfg,
                       controller_id="pid_pump", device=dev, per_patient_metrics=True, x0=x0)
        ft.step()
        runs.append(ft)
    assert torch.equal(runs[0].x0, runs[1].x0)
    for k in ("status", "bg_hist", "bg_stats", "hypo_events", "day_dose"):
        assert torch.equal(getattr(runs[0].outs, k), getattr(runs[1].outs, k)), k
