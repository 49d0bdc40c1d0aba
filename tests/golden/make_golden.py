"""Generate the golden fixtures from the REAL reference package.

Run in the build container, where the reference is importable:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src:/root/repo \
        python tests/golden/make_golden.py

Every fixture is produced by calling the reference's own public functions
(no restatement here).  The reference does not exist on the GPU box, so the
fixtures are committed; numpy / scipy / numba versions are recorded in
``versions.json`` because numpy Generator streams are not version-guaranteed.
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
REPO = os.path.dirname(os.path.dirname(HERE))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

import numba  # noqa: E402
import scipy  # noqa: E402

from glucotrial import analytics, hovorka  # noqa: E402
from glucotrial.controller import DualHormoneController, controller_step_vec, load_profile  # noqa: E402
from glucotrial.physiology import get_model  # noqa: E402
from glucotrial.population import ParameterSet, generate_population  # noqa: E402
from glucotrial.protocol import Disturbance, Protocol  # noqa: E402
from glucotrial.rng import ROLE_MEASUREMENT_NOISE, ROLE_PROCESS_NOISE, stream  # noqa: E402
from glucotrial.simulation import (NorthernYearProtocol, SimulationConfig, _simulate_arrays,  # noqa: E402
                                   compile_protocol, run_trial)
from glucotrial.storage import report_bytes  # noqa: E402

from paper_2202_13927_b200.protocol import ThreeMealProtocol  # noqa: E402  (BASELINE generator plug-in)

sys.path.insert(0, os.path.join(REPO, "oracle"))
import oracle as _oracle  # noqa: E402  (numpy twin of the hypo-event count, applied to the reference's BG)

DAY = 86400.0


def _save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays)


def population_fixture():
    out = {}
    for seed, n in ((0, 64), (101, 12)):
        entries, stats = generate_population(seed=seed, n=n)
        out[f"s{seed}_weights"] = np.array([p.body_weight_kg for p, _ in entries])
        out[f"s{seed}_params"] = np.stack([hovorka.pack_params(ps.values) for _, ps in entries])
        out[f"s{seed}_ubasal"] = np.array([ps.u_basal_u_per_h for _, ps in entries])
        out[f"s{seed}_stats"] = np.array([stats.attempts, stats.accepted, stats.rejected_negative,
                                          stats.rejected_outside_sd, stats.rejected_basal,
                                          stats.rejected_no_steady_state])
    _save("population.npz", **out)
    return out


def population_4000_fixture():
    """A large reference population for distribution parity of the device
    sampler: generate_population(seed=7, n=4000) (population.py:303-341).
    Seeds 5 and 6 raise PopulationError at this size (a body weight below
    ~30 kg admits no parameter set); seed 7 succeeds.  Stored:
    body weights, the 14 sampled parameters (table order), u_basal and the
    SamplingStats counters."""
    from glucotrial.population import load_parameter_table
    entries, stats = generate_population(seed=7, n=4000, workers=os.cpu_count() or 1)
    table = load_parameter_table()
    names = list(table.sampled)
    _save("population_s7_n4000.npz",
          weights=np.array([p.body_weight_kg for p, _ in entries]),
          sampled=np.array([[ps.values[k] for k in names] for _, ps in entries]),
          names=np.array(names), ubasal=np.array([ps.u_basal_u_per_h for _, ps in entries]),
          stats=np.array([stats.attempts, stats.accepted, stats.rejected_negative, stats.rejected_outside_sd,
                          stats.rejected_basal, stats.rejected_no_steady_state]))


def steady_fixture(pop):
    params = pop["s0_params"].copy()
    x0 = np.zeros((params.shape[0], 16))
    ub = np.zeros(params.shape[0])
    for i, p in enumerate(params):
        x0[i], ub[i] = hovorka.steady_state(p, 6.0)
    # random perturbations: exercise the bracket / brentq branches broadly
    rng = np.random.default_rng(7)
    pert = np.repeat(params[:16], 8, axis=0) * rng.uniform(0.7, 1.3, size=(128, 30))
    pert[:, 27:] = params[0, 27:]
    px0 = np.zeros((128, 16))
    pub = np.zeros(128)
    pok = np.zeros(128, dtype=np.int8)
    for i, p in enumerate(pert):
        try:
            px0[i], pub[i] = hovorka.steady_state(p, 6.0)
            pok[i] = 1
        except hovorka.SteadyStateError:
            pok[i] = 0
    bad = params[0].copy()
    bad[hovorka.PEGP0] = 0.001
    try:
        hovorka.steady_state(bad, 6.0)
        bad_ok = 1
    except hovorka.SteadyStateError:
        bad_ok = 0
    _save("steady.npz", params=params, x0=x0, ub=ub, pert=pert, pert_x0=px0, pert_ub=pub,
          pert_ok=pok, bad_params=bad, bad_ok=np.array(bad_ok))


def drift_fixture(pop):
    rng = np.random.default_rng(11)
    n = 400
    X = np.zeros((n, 16))
    X[:, 0] = rng.uniform(5, 250, n); X[:, 1] = rng.uniform(0, 150, n)
    X[:, 2] = rng.uniform(0, 500, n); X[:, 3] = rng.uniform(0, 500, n)
    X[:, 4] = rng.uniform(0, 60, n); X[:, 5] = rng.uniform(0, 0.2, n)
    X[:, 6] = rng.uniform(0, 0.1, n); X[:, 7] = rng.uniform(0, 1.5, n)
    X[:, 8] = rng.uniform(0, 400, n); X[:, 9] = rng.uniform(0, 400, n)
    X[:, 10] = rng.uniform(1, 25, n); X[:, 11] = rng.uniform(0, 100, n)
    X[:, 12] = rng.uniform(0, 50, n); X[:, 13] = rng.uniform(0, 1, n)
    X[:, 14] = rng.uniform(0, 1, n); X[:, 15] = rng.uniform(0, 0.5, n)
    U = np.stack([rng.uniform(0, 50, n), rng.uniform(0, 400, n), rng.uniform(0, 40, n)], 1)
    Dd = np.stack([rng.uniform(0, 8, n), rng.uniform(0, 1, n)], 1)
    P = pop["s0_params"][rng.integers(0, 64, n)]
    OUT = np.zeros((n, 16))
    for i in range(n):
        hovorka.drift_vec(0.0, X[i], U[i], Dd[i], P[i], OUT[i])
    _save("drift.npz", X=X, U=U, D=Dd, P=P, OUT=OUT)


def controller_fixture():
    prof = load_profile()
    ctl = DualHormoneController(prof, 0.7)
    hyper = ctl.hyper_vec
    g = stream(99, 0)
    c = ctl.initial_state().to_vec()
    rows = []
    t, phase = 0.0, -1.0
    for k in range(3000):
        y = float(np.clip(6.0 + 4.0 * np.sin(k / 11.0) + g.normal(0, 1.2), 0.5, 30.0))
        ann = float(g.choice([0.0, 0.0, 0.0, 0.0, 30.0, 75.0]))
        if phase < 0 and g.random() < 0.03:
            phase = 0.0
        elif phase >= 0:
            phase += 300.0
            if phase > 2700.0:
                phase = -1.0
        c_before = c.copy()
        out = np.zeros(3)
        controller_step_vec(c, y, ann, phase, t, 300.0, hyper, 0.7, out)
        rows.append(np.concatenate([c_before, [y, ann, phase, t], out, c]))
        t += 300.0
    _save("controller.npz", rows=np.array(rows), hyper=hyper, basal=np.array(0.7),
          icr_initial_factor=np.array(prof.icr_initial_factor),
          profile_hash=np.array(prof.content_hash()))


class _P:
    def __init__(self, pid, w):
        self.id, self.body_weight_kg = pid, w


def sim_fixture(name, entries, generator, cfg, trace_for=(0, 1), extra_params=None, make_ctl=None,
                prof=None):
    prof = prof or load_profile()
    make_ctl = make_ctl or (lambda basal: DualHormoneController(prof, basal))
    model = get_model("hovorka_ext")
    rec = {"ids": [], "params": [], "x0": [], "c0": [], "basal": [], "status": [], "ticks": [],
           "tir": [], "hist": [], "scal": [], "day_dose": [], "timeline": [], "meal_off": [0],
           "ex_off": [0], "noise_sha": [], "hypo": []}
    hmin = _oracle.hypo_min_ticks(cfg.dt_s)
    meals, ex = [[], [], [], []], [[], [], [], []]
    traces = {}
    for j, (patient, pset) in enumerate(entries):
        values = dict(pset.values)
        if extra_params and patient.id in extra_params:
            values.update(extra_params[patient.id])
        p = hovorka.pack_params(values)
        ctl = make_ctl(pset.u_basal_u_per_h)
        pa = compile_protocol(generator.build(cfg.seed, patient), cfg.horizon_s)
        try:
            x0, _ = hovorka.steady_state(p, cfg.initial_bg_mmol_per_l)
        except hovorka.SteadyStateError:
            x0 = np.full(16, np.nan)
        res = None
        if np.isfinite(x0).all():
            res = _simulate_arrays(patient.id, values, pa, ctl, model, cfg, True)
        H = cfg.horizon_ticks
        w = stream(cfg.seed, patient.id, ROLE_PROCESS_NOISE).standard_normal((H, 3))
        m = stream(cfg.seed, patient.id, ROLE_MEASUREMENT_NOISE).standard_normal(H // cfg.period_steps)
        rec["noise_sha"].append(hashlib.sha256(w.tobytes() + m.tobytes()).hexdigest())
        rec["ids"].append(patient.id)
        rec["params"].append(p)
        rec["x0"].append(x0)
        rec["c0"].append(ctl.initial_state().to_vec())
        rec["basal"].append(ctl.assumed_basal_u_per_h)
        for k, arr in enumerate((pa.meals_start, pa.meals_end, pa.meals_rate, pa.meals_ann)):
            meals[k].append(arr)
        for k, arr in enumerate((pa.ex_start, pa.ex_end, pa.ex_hrr, pa.ex_announced)):
            ex[k].append(arr)
        rec["meal_off"].append(rec["meal_off"][-1] + pa.meals_start.size)
        rec["ex_off"].append(rec["ex_off"][-1] + pa.ex_start.size)
        if res is None:
            rec["status"].append(2); rec["ticks"].append(0)
            rec["tir"].append(np.zeros(5, np.int64)); rec["hist"].append(np.zeros(247, np.int64))
            rec["scal"].append(np.zeros(3)); rec["day_dose"].append(np.zeros((cfg.n_days, 3)))
            rec["timeline"].append(np.zeros(cfg.n_grid))
            rec["hypo"].append((0, 0))
            continue
        st = res.stats
        rec["status"].append(0 if res.status == "ok" else 1)
        rec["ticks"].append(st.ticks)
        rec["tir"].append(st.tir_ticks); rec["hist"].append(st.bg_hist)
        rec["scal"].append([st.min_bg, st.max_bg, st.sum_bg])
        rec["day_dose"].append(st.day_dose); rec["timeline"].append(st.timeline_bg)
        # hypo events of the reference's own per-tick BG (trace column 1), up to the abort tick
        rec["hypo"].append(_oracle.hypo_events(res.trace[:st.ticks, 1], hmin))
        if j in trace_for:
            traces[f"trace_{j}"] = res.trace
    arrays = {k: np.array(v) for k, v in rec.items()}
    for k, nm in enumerate(("meals_start", "meals_end", "meals_rate", "meals_ann")):
        arrays[nm] = np.concatenate(meals[k]) if meals[k] else np.zeros(0)
    for k, nm in enumerate(("ex_start", "ex_end", "ex_hrr", "ex_announced")):
        arrays[nm] = np.concatenate(ex[k]) if ex[k] else np.zeros(0)
    arrays["hypo"] = arrays["hypo"].astype(np.int32).reshape(-1, 2)
    arrays["hypo_min_ticks"] = np.array(hmin)
    arrays["hyper"] = prof.to_vec()
    arrays["config"] = np.array([cfg.horizon_s, cfg.seed, cfg.dt_s, cfg.controller_period_s,
                                 cfg.grid_step_s, cfg.initial_bg_mmol_per_l])
    arrays.update(traces)
    _save(name, **arrays)


def trial_fixture(name, entries, generator, cfg, workers=1):
    prof = load_profile()
    res = run_trial(entries, generator, "dual_hormone", prof, "hovorka_ext", cfg, workers=workers)
    with open(os.path.join(HERE, name), "wb") as fh:
        fh.write(report_bytes(res.report))
    return res


class _CF(float):
    """Float that counts +, -, *, / (the survey's Appendix-B method)."""
    n = 0

    def _w(op):
        def f(self, o):
            _CF.n += 1
            return _CF(getattr(float, op)(self, o))
        return f
    __add__, __radd__ = _w("__add__"), _w("__radd__")
    __sub__, __rsub__ = _w("__sub__"), _w("__rsub__")
    __mul__, __rmul__ = _w("__mul__"), _w("__rmul__")
    __truediv__, __rtruediv__ = _w("__truediv__"), _w("__rtruediv__")

    def __neg__(self):
        return _CF(-float(self))


class _KF(float):
    """Float that tracks STRUCTURAL zeros / ones (k = 0.0 / 1.0 / None): an
    op whose result is fixed by a known operand (x + 0, x * 1, x * 0, 0 / x,
    0 - 0 ...) is trivial -- the fused kernel compiles it out -- every other
    +, -, *, / is counted.  Used to count the algorithmic work that remains
    when a workload structurally has no exercise (E = 0, HRR = 0) or no
    glucagon (Z = 0, u[2] = 0)."""
    n = 0

    def __new__(cls, v, k=None):
        o = float.__new__(cls, v)
        o.k = k
        return o

    @staticmethod
    def _k(o):
        if isinstance(o, _KF):
            return o.k
        return float(o) if float(o) in (0.0, 1.0) else None   # literal constants of the source

    def _op(op):
        def f(self, o):
            a, b = (self, o) if not op.startswith("__r") else (o, self)
            ka, kb = _KF._k(a), _KF._k(b)
            name = op.replace("__r", "__", 1) if op.startswith("__r") else op
            v = getattr(float, name)(float(a), float(b))
            k = None
            trivial = False
            if name == "__add__":
                if ka == 0.0 or kb == 0.0:
                    trivial, k = True, (kb if ka == 0.0 else ka)
            elif name == "__sub__":
                if kb == 0.0:
                    trivial, k = True, ka
                elif ka == 0.0 and kb is not None:
                    trivial, k = True, -kb
            elif name == "__mul__":
                if ka == 0.0 or kb == 0.0:
                    trivial, k = True, 0.0
                elif ka == 1.0 or kb == 1.0:
                    trivial, k = True, (kb if ka == 1.0 else ka)
            elif name == "__truediv__":
                if ka == 0.0:
                    trivial, k = True, 0.0
            if not trivial:
                _KF.n += 1
            return _KF(v, k)
        return f
    __add__, __radd__ = _op("__add__"), _op("__radd__")
    __sub__, __rsub__ = _op("__sub__"), _op("__rsub__")
    __mul__, __rmul__ = _op("__mul__"), _op("__rmul__")
    __truediv__, __rtruediv__ = _op("__truediv__"), _op("__rtruediv__")

    def __neg__(self):
        return _KF(-float(self), None if self.k is None else -self.k)


def _structural_counts(p, x):
    """Non-trivial drift ops and structurally-zero derivatives with exercise
    and/or glucagon absent (typical branch state x)."""
    from glucotrial.hovorka import IE1, IE2, IE3, IZ1, IZ2
    res = {}
    for label, zero_x, zero_u, zero_d in (("noex", (IE1, IE2, IE3), (), (1,)),
                                          ("nogluc", (IZ1, IZ2), (2,), ()),
                                          ("noex_nogluc", (IE1, IE2, IE3, IZ1, IZ2), (2,), (1,))):
        xx = np.array([_KF(0.0, 0.0) if k in zero_x else _KF(v) for k, v in enumerate(x)], dtype=object)
        uu = np.array([_KF(0.0, 0.0) if k in zero_u else _KF(v) for k, v in enumerate([10.0, 0.0, 0.0])],
                      dtype=object)
        dd = np.array([_KF(0.0, 0.0) if k in zero_d else _KF(v) for k, v in enumerate([0.0, 0.0])], dtype=object)
        out = np.empty(16, dtype=object)
        _KF.n = 0
        hovorka.drift_vec.py_func(_KF(0.0), xx, uu, dd, np.array([_KF(v) for v in p], dtype=object), out)
        res[f"drift_typical_{label}"] = _KF.n
        # Euler updates x += f * dt (2 ops) vanish for states held at a known 0
        res[f"zero_states_{label}"] = sum(1 for k in range(16) if _KF._k(out[k]) == 0.0 and k in zero_x)
    return res


def flop_fixture():
    """Op counts of drift_vec / diffusion_diag / controller_step_vec over the
    reference's own Python source (.py_func), on golden-like states."""
    from glucotrial._kernel import simulate_block  # noqa: F401
    pop = np.load(os.path.join(HERE, "population.npz"))
    p = pop["s0_params"][0]
    x, _ = hovorka.steady_state(p, 6.0)
    obj = lambda a: np.array([_CF(v) for v in a], dtype=object)
    counts = {}
    for label, bgscale in (("typical", 1.0), ("renal", 2.0), ("hypo", 0.6)):
        xx = x.copy()
        xx[hovorka.IQ1] *= bgscale
        out = np.empty(16, dtype=object)
        _CF.n = 0
        hovorka.drift_vec.py_func(_CF(0.0), obj(xx), obj([10.0, 0.0, 0.0]), obj([0.0, 0.0]), obj(p), out)
        counts[f"drift_{label}"] = _CF.n
    _CF.n = 0
    hovorka.diffusion_diag.py_func(_CF(0.0), obj(x), obj([0, 0, 0]), obj([0, 0]), obj(p), np.empty(3, dtype=object))
    counts["diffusion"] = _CF.n
    prof = load_profile()
    ctl = DualHormoneController(prof, 0.8)
    hyper = obj(ctl.hyper_vec)
    ctrl_counts = []
    g = np.random.default_rng(3)
    c = obj(ctl.initial_state().to_vec())
    for k in range(2000):
        out = np.empty(3, dtype=object)
        _CF.n = 0
        controller_step_vec.py_func(c, _CF(float(np.clip(g.normal(7, 1.5), 2, 20))),
                                    _CF(0.0 if k % 50 else 60.0), _CF(-1.0), _CF(300.0 * k),
                                    _CF(300.0), hyper, _CF(0.8), out)
        ctrl_counts.append(_CF.n)
    vals, cnt = np.unique(ctrl_counts, return_counts=True)
    counts["controller_typical"] = int(vals[np.argmax(cnt)])
    counts["controller_min"], counts["controller_max"] = int(min(ctrl_counts)), int(max(ctrl_counts))
    counts.update(_structural_counts(p, x))
    with open(os.path.join(HERE, "flop_counts.json"), "w") as fh:
        json.dump(counts, fh, indent=1, sort_keys=True)


def pid_fixtures():
    """The BASELINE PID + pump-quantisation controller (paper_2202_13927_b200/pid.py)
    registered in the REFERENCE's controller registry and run by the reference's
    own generic engine (_python_block, simulation.py:199-298)."""
    from glucotrial.controller import register_controller as ref_register
    from paper_2202_13927_b200.pid import PIDController, PIDProfile
    try:
        ref_register("pid_pump", lambda profile, basal: PIDController(profile, basal))
    except ValueError:
        pass
    prof = PIDProfile()
    e0, _ = generate_population(seed=0, n=64)
    e101, _ = generate_population(seed=101, n=12)
    tm = ThreeMealProtocol()
    cfg_tm = SimulationConfig(horizon_s=3 * DAY, seed=0, dt_s=60.0)
    sim_fixture("sim_pid_threemeal_dt60.npz", e0[:8], tm, cfg_tm, prof=prof,
                make_ctl=lambda basal: PIDController(prof, basal))
    cfg_ny = SimulationConfig(horizon_s=2 * DAY, seed=33)
    sim_fixture("sim_pid_northern_dt30.npz", e101[:4], NorthernYearProtocol(), cfg_ny, prof=prof,
                make_ctl=lambda basal: PIDController(prof, basal))


def hypo_fixtures():
    """Hypoglycaemia-rich closed loops (the bench's short fixtures have almost
    no events): the controllers are told an assumed basal rate scaled up, as
    run_trial's basal_scale does (simulation.py:502), so insulin is overdosed
    and BG repeatedly crosses 3.9 and 3.0 mmol/L.  Event counts come from the
    reference's own BG traces (sim_fixture)."""
    from paper_2202_13927_b200.pid import PIDController, PIDProfile
    prof = load_profile()
    e0, _ = generate_population(seed=0, n=64)
    e101, _ = generate_population(seed=101, n=12)
    cfg_tm = SimulationConfig(horizon_s=7 * DAY, seed=0, dt_s=60.0)
    sim_fixture("sim_hypo_threemeal_dt60.npz", e0[:16], ThreeMealProtocol(), cfg_tm, trace_for=(),
                make_ctl=lambda basal: DualHormoneController(prof, 2.8 * basal))
    cfg_ny = SimulationConfig(horizon_s=7 * DAY, seed=8, dt_s=30.0)
    sim_fixture("sim_hypo_northern_dt30.npz", e101[:8], NorthernYearProtocol(), cfg_ny, trace_for=(),
                make_ctl=lambda basal: DualHormoneController(prof, 2.4 * basal))
    pp = PIDProfile()
    cfg_pid = SimulationConfig(horizon_s=4 * DAY, seed=4, dt_s=60.0)
    sim_fixture("sim_hypo_pid_threemeal_dt60.npz", e0[16:28], ThreeMealProtocol(), cfg_pid, trace_for=(),
                prof=pp, make_ctl=lambda basal: PIDController(pp, 1.8 * basal))


def record_fixture():
    """The reference's own record round trip (storage.py:234-312; its test
    test_storage.py:181-199) on a cohort of 6, a 2-day NorthernYear trial with a
    NON-default announcement policy: the record, and the report its rerun
    reproduces.  The product's records.rerun_trial must give the same bytes."""
    import tempfile
    from glucotrial.protocol import AnnouncementPolicy as RefPolicy
    from glucotrial.storage import Store, TrialRecord, rerun_trial as ref_rerun
    e101, _ = generate_population(seed=101, n=12)
    prof = load_profile()
    cfg = SimulationConfig(horizon_s=2 * DAY, seed=21)
    gen = NorthernYearProtocol(announcement=RefPolicy(fraction_unannounced=0.2,
                                                      misannouncement_factor_range=(0.8, 1.2)))
    with tempfile.TemporaryDirectory() as d:
        store = Store(d)
        store.save_cohort("pop-a", e101[:6])
        res = run_trial(e101[:6], gen, "dual_hormone", prof, "hovorka_ext", cfg, workers=1, basal_scale=1.0,
                        run_meta={"trial_id": "trial-x", "population_ref": "pop-a"})
        h = store.save_profile(prof)
        rec = TrialRecord.create(trial_id="trial-x", seed=cfg.seed, model_id="hovorka_ext",
                                 controller_id="dual_hormone", profile_hash=h, population_ref="pop-a",
                                 protocol_generator=gen.describe(), basal_scale=1.0, config=cfg.to_dict())
        fresh = ref_rerun(store, rec)
        assert report_bytes(fresh.report) == report_bytes(res.report)
    d = rec.to_dict()
    d["created_at"] = "2026-01-01T00:00:00+00:00"   # fixed for a reproducible fixture
    with open(os.path.join(HERE, "record_rerun.json"), "w") as fh:
        json.dump(d, fh, indent=1, sort_keys=True)
    with open(os.path.join(HERE, "report_rerun.json"), "wb") as fh:
        fh.write(report_bytes(res.report))


def main():
    if "--only-pid" in sys.argv:
        pid_fixtures()
        return
    if "--only-hypo" in sys.argv:
        hypo_fixtures()
        return
    if "--only-pop4k" in sys.argv:
        population_4000_fixture()
        return
    if "--only-record" in sys.argv:
        record_fixture()
        return
    if "--only-flops" in sys.argv:
        flop_fixture()
        return
    pop = population_fixture()
    population_4000_fixture()
    record_fixture()
    flop_fixture()
    steady_fixture(pop)
    drift_fixture(pop)
    controller_fixture()
    e101, _ = generate_population(seed=101, n=12)
    e0, _ = generate_population(seed=0, n=64)
    nyp = NorthernYearProtocol()
    tm = ThreeMealProtocol()
    cfg_ny = SimulationConfig(horizon_s=2 * DAY, seed=33)                       # dt 30 (default)
    cfg_tm = SimulationConfig(horizon_s=7 * DAY, seed=0, dt_s=60.0)              # BASELINE configs[0] shape
    cfg_odd = SimulationConfig(horizon_s=DAY, seed=5, dt_s=37.5, grid_step_s=3600.0)
    cfg_long = SimulationConfig(horizon_s=8 * DAY, seed=3, dt_s=60.0)           # > 1 block (20160 ticks at dt 30)
    sim_fixture("sim_northern_dt30.npz", e101, nyp, cfg_ny)
    sim_fixture("sim_threemeal_dt60.npz", e0[:32], tm, cfg_tm)
    sim_fixture("sim_northern_dt37p5.npz", e101[:4], nyp, cfg_odd)
    sim_fixture("sim_northern_dt30_8d.npz", e101[:3], nyp, dataclasses.replace(cfg_long, dt_s=30.0))
    # fault injection (test_simulation.py:271-288): diverging sensor, no steady state
    faults = {e101[2][0].id: {"tau_cgm": -1.0}, e101[3][0].id: {"EGP0": 0.001}}
    sim_fixture("sim_faults.npz", e101[:4], nyp, cfg_ny, extra_params=faults)
    trial_fixture("report_northern_dt30.json", e101, nyp, cfg_ny)
    trial_fixture("report_threemeal_dt60.json", e0, tm, cfg_tm)
    faulty = [(p, ParameterSet(values=dict(ps.values), u_basal_u_per_h=ps.u_basal_u_per_h))
              for p, ps in e101[:4]]
    faulty[2][1].values["tau_cgm"] = -1.0
    faulty[3][1].values["EGP0"] = 0.001
    trial_fixture("report_faults.json", faulty, nyp, cfg_ny)
    worst_cfg = dataclasses.replace(cfg_ny, store_trace="worst_case_only")
    res = run_trial(e101[:4], nyp, "dual_hormone", load_profile(), "hovorka_ext", worst_cfg)
    _save("worst_trace.npz", trace=res.worst_trace, worst_id=np.array(res.accumulator.worst.patient_id))
    pid_fixtures()
    hypo_fixtures()
    # one empty-protocol day, no noise: fixed point (test_simulation.py:133-144)
    with open(os.path.join(HERE, "versions.json"), "w") as fh:
        json.dump({"numpy": np.__version__, "scipy": scipy.__version__, "numba": numba.__version__,
                   "reference": "glucotrial 0.1.0 (/root/reference/pkg)"}, fh, indent=1)


if __name__ == "__main__":
    main()
