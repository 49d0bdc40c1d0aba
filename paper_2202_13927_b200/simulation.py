"""Drop-in trial API on the B200 engine.

``simulate_closed_loop`` and ``run_trial`` keep the reference signatures,
argument meaning, return types and error behaviour (simulation.py:394-413,
551-628 of the reference) and run every patient on device:

* ``noise="reference"`` (default): the reference's own per-patient noise
  streams (rng.py:26-39) are drawn on the host and injected into the
  bitwise parity kernel — reports are byte-identical to the reference's;
* ``noise="philox"``: the fused fast integrator with on-device Philox
  noise (and the on-device 3-meal generator when the protocol generator is
  a ``ThreeMealProtocol``), reduced on device — statistically equivalent,
  the throughput path.

Unsupported model/controller pairs raise ``SimulationError`` exactly as the
reference's ``engine="fast"`` gate does (simulation.py:301-311); there is no
CPU fallback.  ``workers`` is accepted for signature compatibility: all
patients of a call run on the device.
"""

from __future__ import annotations

import math
import itertools
import operator
import os
import time
from dataclasses import dataclass

import numpy as np

from . import analytics, engine, rng
from ._lib import GT_STATUS_NO_STEADY_STATE, GT_STATUS_NONFINITE, GT_STATUS_OK
from .analytics import PatientStats, TrialAccumulator
from .config import SimulationConfig, SimulationError, sizes
from .controller import device_code, hyper_vector, icr_initial_factor
from .layout import N_CSTATE, PARAM_NAMES, PR, PSIGEGP, PSIGGUT, TRACE_COLUMNS
from .protocol import ThreeMealProtocol, compile_protocol, compile_ticks, validate_protocol

MODEL_ID = "hovorka_ext"
PARITY_CHUNK_MAX = 4096   # patients per parity launch at most
PARITY_NOISE_BYTES = 1 << 30   # injected-noise bytes per parity launch (host shared memory + device)


class SteadyStateError(RuntimeError):
    """No basal rate holds the target BG (hovorka.py:69-70)."""


@dataclass
class SimulationResult:
    patient_id: int
    status: str
    stats: PatientStats
    min_bg: float
    trace: np.ndarray | None = None


@dataclass
class TrialResult:
    report: dict
    accumulator: TrialAccumulator
    worst_trace: np.ndarray | None
    wall_s: float
    n_patients: int
    metrics: dict | None = None      # BASELINE per-patient metric arrays (philox path)


def _model_id(model) -> str:
    return model if isinstance(model, str) else getattr(model, "model_id", None)


def _check_model(model) -> None:
    if _model_id(model) != MODEL_ID:
        raise SimulationError(
            f"the B200 engine implements the {MODEL_ID} model only (got {_model_id(model)!r})")


def pack_params(values: dict) -> np.ndarray:
    missing = [n for n in PARAM_NAMES if n not in values]
    if missing:
        raise ValueError(f"missing parameters: {missing}")
    return np.array([float(values[n]) for n in PARAM_NAMES])


_PARAM_GETTER = operator.itemgetter(*PARAM_NAMES)


def pack_params_many(values_seq) -> np.ndarray:
    """pack_params over a sequence of parameter maps -> [n, 30] float64 (one
    C-level item lookup per map; the same values and the same error)."""
    seq = list(values_seq)
    try:
        flat = np.fromiter(itertools.chain.from_iterable(map(_PARAM_GETTER, seq)), dtype=np.float64,
                           count=len(seq) * len(PARAM_NAMES))
    except KeyError:
        for v in seq:
            pack_params(v)   # raises the reference-shaped ValueError
        raise
    return flat.reshape(len(seq), len(PARAM_NAMES))


def _controller_inputs(controller):
    """(hyper[30], assumed basal, c0[11] or None, device code) from a reference
    DualHormoneController, a PIDController (pid.py) or a DeviceController."""
    if hasattr(controller, "initial_state") and hasattr(controller, "hyper_vec"):
        name = type(controller).__name__
        if name == "DualHormoneController":
            code = device_code("dual_hormone")
        elif name == "PIDController":
            code = device_code("pid_pump")
        else:
            raise SimulationError(f"controller {name!r} has no device implementation")
        c0 = np.asarray(controller.initial_state().to_vec(), dtype=np.float64)
        return np.asarray(controller.hyper_vec, np.float64), float(controller.assumed_basal_u_per_h), c0, code
    if hasattr(controller, "code") and hasattr(controller, "profile"):
        code = device_code(controller.controller_id)
        return hyper_vector(controller.profile), float(controller.assumed_basal_u_per_h), None, code
    raise SimulationError("controller has no device implementation")


def _noise_flags(p: np.ndarray):
    return bool(p[PSIGEGP] > 0.0 or p[PSIGGUT] > 0.0), bool(p[PR] > 0.0)


def _csr(pas: list):
    """Concatenate per-patient ProtocolArrays into CSR arrays."""
    moff = np.zeros(len(pas) + 1, dtype=np.int64)
    eoff = np.zeros(len(pas) + 1, dtype=np.int64)
    for i, pa in enumerate(pas):
        moff[i + 1] = moff[i] + pa.meals_start.size
        eoff[i + 1] = eoff[i] + pa.ex_start.size
    cat = lambda name: (np.concatenate([getattr(pa, name) for pa in pas]).astype(np.float64)
                        if pas else np.zeros(0))
    meals = tuple(cat(k) for k in ("meals_start", "meals_end", "meals_rate", "meals_ann"))
    ex = tuple(cat(k) for k in ("ex_start", "ex_end", "ex_hrr", "ex_announced"))
    return moff, meals, eoff, ex


def _stats_from_parity(out: dict, i: int, config, sz) -> PatientStats:
    st = PatientStats(dt_s=config.dt_s, horizon_ticks=sz["horizon_ticks"], n_days=sz["n_days"],
                      n_grid=sz["n_grid"])
    st.tir_ticks = out["tir_ticks"][i].copy()
    st.bg_hist = out["bg_hist"][i].copy()
    st.timeline_bg = out["timeline"][i].copy()
    st.day_dose = out["day_dose"][i].copy()
    st.ticks = int(out["ticks"][i])
    st.min_bg = float(out["scal"][i, 0])
    st.max_bg = float(out["scal"][i, 1])
    st.sum_bg = float(out["scal"][i, 2])
    return st


def _parity_run(items, config, hyper, device, record_trace=False, controller=0, noise=None, fetch=True):
    """items: list of (pid, p[30], x0[16], c0[11], basal, ProtocolArrays);
    noise: (wiener [n,H,3], meas [n,H/ps], has_noise [n]) already drawn
    (hostprep), else drawn here from the reference's streams."""
    sz = sizes(config)
    H, ps = sz["horizon_ticks"], sz["period_steps"]
    n = len(items)
    if noise is not None:
        wiener, meas, has_noise = noise
    else:
        wiener = np.zeros((n, H, 3))
        meas = np.zeros((n, H // ps))
        has_noise = np.zeros(n, dtype=np.uint8)
        for i, (pid, p, *_rest) in enumerate(items):
            proc, sens = _noise_flags(p)
            w, m = rng.reference_noise(config.seed, pid, H, ps, proc, sens)
            if w is not None:
                wiener[i] = w
            has_noise[i] = proc
            meas[i] = m
    moff, meals, eoff, ex = _csr([it[5] for it in items])
    batch = engine.ParityBatch(
        params=np.stack([it[1] for it in items]), x0=np.stack([it[2] for it in items]),
        c0=np.stack([it[3] for it in items]), hyper=hyper,
        assumed_basal=np.array([it[4] for it in items], dtype=np.float64),
        meal_off=moff, meals=meals, ex_off=eoff, ex=ex, wiener=wiener, has_noise=has_noise,
        meas=meas, controller=int(controller))
    return engine.run_parity(batch, sz, config.dt_s, config.controller_period_s,
                             record_trace=record_trace, device=device, fetch=fetch), sz


def simulate_closed_loop(patient, parameter_set, protocol, controller, model,
                         config, record_trace: bool | None = None,
                         validate: bool = True, device=None) -> SimulationResult:
    """One patient, closed loop, bitwise parity kernel with the reference's
    noise streams (simulation.py:394-413)."""
    _check_model(model)
    if validate:
        v = validate_protocol(protocol)
        if v:
            raise SimulationError(f"invalid protocol: {v[:3]}")
    if record_trace is None:
        record_trace = config.store_trace == "always"
    hyper, basal, c0, code = _controller_inputs(controller)
    p = pack_params(parameter_set.values)
    x0, _ub, ok = engine.steady_state(p[None, :], config.initial_bg_mmol_per_l, device)
    if int(ok.cpu()[0]) != GT_STATUS_OK:
        raise SteadyStateError("no positive basal rate holds the target BG")
    x0 = x0.cpu().numpy()[0]
    if c0 is None:
        c0 = engine.controller_init(hyper, icr_initial_factor(controller.profile), [basal], device).cpu().numpy()[0]
    pa = compile_protocol(protocol, config.horizon_s)
    out, sz = _parity_run([(int(patient.id), p, x0, c0, basal, pa)], config, hyper, device, record_trace, code)
    st = _stats_from_parity(out, 0, config, sz)
    status = "ok" if int(out["status"][0]) == GT_STATUS_OK else "nonfinite"
    trace = out["trace"][0][:st.ticks] if record_trace else None
    return SimulationResult(patient_id=int(patient.id), status=status, stats=st,
                            min_bg=st.min_bg, trace=trace)


# ------------------------------------------------------------------ trials
def _empty_acc(config) -> TrialAccumulator:
    sz = sizes(config)
    return TrialAccumulator(dt_s=config.dt_s, horizon_ticks=sz["horizon_ticks"], n_days=sz["n_days"],
                            n_grid=sz["n_grid"], grid_step_s=config.grid_step_s)


def _population_arrays(population, basal_scale):
    ids = np.array([int(pt.id) for pt, _ in population], dtype=np.int64)
    params = pack_params_many([ps.values for _, ps in population])
    basal = np.array([ps.u_basal_u_per_h for _, ps in population], dtype=np.float64) * basal_scale
    return ids, params, basal


def _meta(config, population_n, model_id, controller_id, profile, basal_scale, generator, run_meta):
    meta = {
        "seed": config.seed, "n_patients": population_n, "model": model_id,
        "controller": controller_id,
        "profile_hash": profile.content_hash() if hasattr(profile, "content_hash") else None,
        "basal_scale": basal_scale, "protocol": generator.describe(), "config": config.to_dict(),
    }
    if run_meta:
        meta.update(run_meta)
    return meta


def run_trial(population, protocol_generator, controller_id: str, profile, model_id: str,
              config, workers: int = 1, basal_scale: float = 1.0, run_meta: dict | None = None,
              trace_dir: str | None = None, progress=None, *, noise: str = "reference",
              device=None, hypo_min_s: float = 900.0) -> TrialResult:
    """Simulate every patient and build the report (simulation.py:551-628)."""
    if population is None or len(population) == 0:
        raise SimulationError("population must be nonempty")
    if workers < 1:
        raise SimulationError("workers must be >= 1")
    _check_model(model_id)
    code = device_code(controller_id) if controller_id in _known_ids() else None
    if code is None:
        raise SimulationError(f"controller {controller_id!r} has no device implementation")
    if config.store_trace == "always" and trace_dir is not None:
        os.makedirs(trace_dir, exist_ok=True)
    if noise == "reference":
        return _run_trial_parity(population, protocol_generator, controller_id, profile, model_id,
                                 config, basal_scale, run_meta, trace_dir, progress, device)
    if noise == "philox":
        from .trial import run_trial_fast
        return run_trial_fast(population, protocol_generator, controller_id, profile, model_id,
                              config, basal_scale=basal_scale, run_meta=run_meta, progress=progress,
                              device=device, hypo_min_s=hypo_min_s, trace_dir=trace_dir)
    raise SimulationError("noise must be 'reference' or 'philox'")


def _known_ids():
    from .controller import _REGISTRY
    return _REGISTRY


def _parity_chunk(sz) -> int:
    """Patients per parity launch: the injected reference noise (~24 B per
    patient-step) is bounded to PARITY_NOISE_BYTES per chunk."""
    per = 8 * (3 * sz["horizon_ticks"] + sz["horizon_ticks"] // sz["period_steps"])
    return int(max(32, min(PARITY_CHUNK_MAX, PARITY_NOISE_BYTES // per)))


def _run_trial_parity(population, generator, controller_id, profile, model_id, config,
                      basal_scale, run_meta, trace_dir, progress, device) -> TrialResult:
    from . import hostprep
    t0 = time.perf_counter()
    ids, params, basal = _population_arrays(population, basal_scale)
    hyper = hyper_vector(profile)
    code = device_code(controller_id)
    x0_d, _ub, ok_d = engine.steady_state(params, config.initial_bg_mmol_per_l, device)
    c0 = engine.controller_init(hyper, icr_initial_factor(profile), basal, device).cpu().numpy()
    x0, ok = x0_d.cpu().numpy(), ok_d.cpu().numpy()
    acc = _empty_acc(config)
    record = config.store_trace == "always"
    sz = sizes(config)
    H, ps = sz["horizon_ticks"], sz["period_steps"]
    flags = np.array([_noise_flags(params[i]) for i in range(len(population))], dtype=bool).reshape(-1, 2)
    # the patients to simulate, in order; the others are aborted at staging
    run = [i for i in range(len(population)) if ok[i] == GT_STATUS_OK]
    chunk = _parity_chunk(sz)
    spans = [run[lo:lo + chunk] for lo in range(0, len(run), chunk)]

    # two page-locked noise blocks, alternated: the workers fill one while the
    # device reads the other
    nb = min(chunk, len(run))
    use_pool = nb >= 64 and hostprep.pool() is not None
    blocks = []

    def start(c):
        # host inputs of chunk c (protocols + the reference's noise streams),
        # in the worker pool while the previous chunk runs on the device
        idx = spans[c]
        return hostprep.prepare(generator, config.seed, [population[i][0] for i in idx], ids[idx],
                                flags[idx, 0], flags[idx, 1], config.horizon_s, H, H // ps,
                                block=blocks[c % 2])

    for i in range(len(population)):   # no steady state: aborted at staging (ids kept sorted)
        if ok[i] != GT_STATUS_OK:
            acc.add_aborted(int(ids[i]))
    done = 0
    tm = ({"setup": time.perf_counter() - t0, "prep_wait": 0.0, "device": 0.0, "fold": 0.0}
          if os.environ.get("GLUCOSIM_PARITY_TIMING") else None)
    def fold(idx, out_d):
        out = engine.fetch_parity(out_d)
        for j, i in enumerate(idx):
            if int(out["status"][j]) != GT_STATUS_OK:
                acc.add_aborted(int(ids[i]))
                continue
            acc.add_patient(int(ids[i]), _stats_from_parity(out, j, config, sz))
            if record and trace_dir is not None:
                save_trace(os.path.join(trace_dir, f"patient_{int(ids[i]):06d}.npz"), out["trace"][j])
        if progress:
            progress(idx[-1] + 1, len(population))
        return idx[-1] + 1

    nxt, pending = None, None
    hostprep.LOCK.acquire()
    try:
        blocks = hostprep.blocks(nb, H, H // ps, use_pool, count=min(2, len(spans))) if spans else []
        nxt = start(0) if spans else None
        for c, idx in enumerate(spans):
            ta = time.perf_counter()
            pas, block = nxt.result()
            # the other block's chunk (c - 1) is done on the device: refill it now,
            # while this chunk runs
            nxt = start(c + 1) if c + 1 < len(spans) else None
            tb = time.perf_counter()
            m = len(idx)
            items = [(int(ids[i]), params[i], x0[i], c0[i], basal[i], pa) for i, pa in zip(idx, pas)]
            # launched without waiting (its inputs are copied before the call returns):
            # the previous chunk is folded on the host while this one runs
            out_d, _sz = _parity_run(items, config, hyper, device, record_trace=record, controller=code,
                                     noise=(block.wiener[:m], block.meas[:m], flags[idx, 0].astype(np.uint8)),
                                     fetch=False)
            tc = time.perf_counter()
            if tm is not None:
                tm["prep_wait"] += tb - ta
                tm["device"] += tc - tb
            if pending is not None:
                done = fold(*pending)
            pending = (idx, out_d)
            if tm is not None:
                tm["fold"] += time.perf_counter() - tc
        if pending is not None:
            td = time.perf_counter()
            done = fold(*pending)
            pending = None
            if tm is not None:
                tm["fold"] += time.perf_counter() - td
    finally:
        if nxt is not None:
            try:
                nxt.result()   # let in-flight workers finish with the block before it goes
            except Exception:
                pass
        hostprep.LOCK.release()
    if tm is not None:
        print(f"parity run_trial: {len(spans)} chunks of <= {chunk}; " +
              ", ".join(f"{k} {v:.3f} s" for k, v in tm.items()), flush=True)
    if progress and done < len(population):
        progress(len(population), len(population))
    wall_s = time.perf_counter() - t0
    if acc.n_patients == 0:
        raise SimulationError("all simulations diverged; nothing to report")
    meta = _meta(config, len(population), model_id, controller_id, profile, basal_scale, generator, run_meta)
    report = analytics.build_trial_report(acc, meta)
    worst_trace = None
    if config.store_trace in ("worst_case_only", "always") and acc.worst is not None:
        wi = int(np.nonzero(ids == acc.worst.patient_id)[0][0])
        pa = compile_protocol(generator.build(config.seed, population[wi][0]), config.horizon_s)
        out, sz = _parity_run([(int(ids[wi]), params[wi], x0[wi], c0[wi], basal[wi], pa)],
                              config, hyper, device, record_trace=True, controller=code)
        worst_trace = out["trace"][0][: int(out["ticks"][0])]
    return TrialResult(report=report, accumulator=acc, worst_trace=worst_trace, wall_s=wall_s,
                       n_patients=len(population))


def save_trace(path: str, trace: np.ndarray) -> None:
    np.savez_compressed(path, columns=np.array(TRACE_COLUMNS), trace=trace)


def load_trace(path: str) -> np.ndarray:
    with np.load(path) as data:
        if tuple(data["columns"]) != TRACE_COLUMNS:
            raise SimulationError(f"unexpected trace columns in {path}")
        return data["trace"]
