"""BASELINE configs[1] at its full size (100 000 patients x 4 weeks, dt 60 s,
seed 1, PID + pump quantisation, 3-meal generator, device-sampled
population) through the fused path, checked by size-independent properties:
the oracle cannot run this size in seconds, so these tests pin what must hold
for any correct run of it.

* determinism: a repeat launch is bit-identical;
* sharding: two pid-range shards give the single launch's per-patient outputs
  bit for bit, and their merged accumulators its report bytes (the 8-GPU
  layout, parallel.shard_range);
* slicing: the unsliced horizon equals the persistent sliced schedule;
* per patient: the 247 histogram bins sum to the horizon, the five glycaemic
  ranges partition it (analytics.py:21-23 bounds), min <= mean <= max BG, and a
  hypoglycaemia event needs at least hypo_min_ticks ticks below its threshold;
* the device reduction equals the host fold of the per-patient outputs
  (analytics.py:150-265), report bytes included.
"""

import numpy as np
import pytest

from test_gpu_fast import _acc_equal, _h, _host_acc_from_fast

pytestmark = pytest.mark.gpu

N, WEEKS, SEED = 100_000, 4, 1
PER_PATIENT = ("status", "ticks", "bg_hist", "bg_stats", "day_dose", "hypo_events")


@pytest.fixture(scope="module")
def dev():
    import torch
    from paper_2202_13927_b200 import _lib
    assert torch.cuda.is_available()
    _lib.load()
    return torch.device("cuda", 0)


@pytest.fixture(scope="module")
def setup(dev):
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.population import generate_population
    cfg = SimulationConfig(horizon_s=WEEKS * 7 * 86400.0, seed=SEED, dt_s=60.0)
    pop = generate_population(SEED, N, device=dev, on_exhausted="redraw_weight")
    return cfg, pop


def _run(setup, dev, lo=0, hi=N, n_slices=0, timeline=False):
    from paper_2202_13927_b200 import engine
    from paper_2202_13927_b200.pid import PIDProfile
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial
    cfg, pop = setup
    ft = FastTrial(lo, pop.params_device[lo:hi], pop.basal_device[lo:hi], ThreeMealProtocol(), PIDProfile(), cfg,
                   controller_id="pid_pump", device=dev, per_patient_metrics=True, n_slices=n_slices,
                   x0=pop.x0_device[lo:hi])
    if timeline:
        ft.outs = engine.alloc_fast_outputs(ft.n, lo, ft.sz, dev, per_patient_timeline=True)
    ft.step()
    return ft


def test_full_size_repeat_is_bit_identical(setup, dev):
    a, b = _run(setup, dev), _run(setup, dev)
    for k in PER_PATIENT:
        assert np.array_equal(_h(getattr(a.outs, k)), _h(getattr(b.outs, k))), k
    assert _acc_equal(a.accumulator(), b.accumulator())


def test_full_size_two_shards_equal_one_launch(setup, dev):
    from paper_2202_13927_b200.analytics import merge
    from paper_2202_13927_b200.parallel import shard_range
    full = _run(setup, dev)
    parts = [_run(setup, dev, *shard_range(N, r, 2)) for r in range(2)]
    assert parts[0].n + parts[1].n == N
    for k in PER_PATIENT:
        cat = np.concatenate([_h(getattr(p.outs, k)) for p in parts], axis=-1)
        assert np.array_equal(cat, _h(getattr(full.outs, k))), k
    assert _acc_equal(full.accumulator(), merge(parts[0].accumulator(), parts[1].accumulator()))


def test_full_size_unsliced_equals_sliced_schedule(setup, dev):
    a, b = _run(setup, dev, n_slices=1), _run(setup, dev)
    for k in PER_PATIENT:
        assert np.array_equal(_h(getattr(a.outs, k)), _h(getattr(b.outs, k))), k


def test_full_size_per_patient_invariants_and_host_fold(setup, dev):
    cfg, _ = setup
    ft = _run(setup, dev, timeline=True)
    H = ft.sz["horizon_ticks"]
    status, hist, st = _h(ft.outs.status), _h(ft.outs.bg_hist).astype(np.int64), _h(ft.outs.bg_stats)
    ev, ticks = _h(ft.outs.hypo_events), _h(ft.outs.ticks)
    ok = status == 0
    assert ok.sum() >= N - 10          # the bench population: (next to) no aborted patient
    assert np.all(ticks[ok] == H)
    assert np.all(hist[:, ok].sum(axis=0) == H)
    c = np.cumsum(hist[:, ok], axis=0)
    ranges = np.stack([c[25], c[34] - c[25], c[95] - c[34], c[134] - c[95], c[-1] - c[134]])
    assert np.all(ranges >= 0) and np.all(ranges.sum(axis=0) == H)
    mean = st[2, ok] / H
    assert np.all(st[0, ok] <= mean) and np.all(mean <= st[1, ok])
    # an event is a run of >= hypo_min_ticks ticks below 3.9 (3.0) mmol/L
    L = ft.hypo_min_ticks
    assert np.all(ev[0, ok] * L <= c[34]) and np.all(ev[1, ok] * L <= c[25])
    assert int(ev[0, ok].sum()) > 0
    dev_acc = ft.accumulator()
    host_acc = _host_acc_from_fast(ft.outs, cfg, ft.sz, 0)
    assert dev_acc.n_patients == host_acc.n_patients == int(ok.sum())
    assert _acc_equal(dev_acc, host_acc)
