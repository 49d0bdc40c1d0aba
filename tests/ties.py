"""Threshold-tie classifier (TEST INFRASTRUCTURE ONLY).

The fused kernel re-associates the model arithmetic, so its
trajectories differ from the reference's in the last bits.  Those bits are
invisible unless a value lands within rounding of a discontinuity: a
histogram / range edge (analytics.py:21-27, searchsorted at _kernel.py:142-143)
or a controller comparison (controller.py:343-458, pid.py).  Then one
patient's integer counts flip and, after a controller flip, its trajectory
moves on.  Such a patient is not allowed as a bare count ("ties <= N"): every
exception must be *proven* a tie, patient by patient:

1. trace the patient through the reference (the C oracle, bitwise equal to
   the reference's simulate_block) and through the fused kernel's TRACE
   variant on identical inputs, and find the first tick where the two runs
   differ discretely (histogram bin, range, controller output) or drift
   apart beyond 1e-9;
2. at that tick the difference must be explained by rounding alone:
   * BIN: the two BG values are within ``REL_TIE`` of each other and a
     histogram threshold or range bound lies between them;
   * CONTROLLER: the CGM readings of every controller tick so far agree to
     ``REL_TIE``, and replaying the reference's own controller (the oracle,
     bitwise equal to controller_step_vec / the PID twin) on the FUSED
     readings reproduces the fused outputs exactly -- i.e. the reference
     itself maps inputs that far apart to the two different decisions.
Anything else (a continuous drift beyond 1e-9 first, a controller output the
reference would not produce from the fused readings, a bin flip between far
apart values) is a failure.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

THRESHOLDS = np.array([(5 + i) / 10.0 for i in range(246)])   # analytics.py:27
RANGE_BOUNDS = np.array([3.0, 3.9, 10.0, 13.9])                # analytics.py:21-23
EDGES = np.union1d(THRESHOLDS, RANGE_BOUNDS)
REL_TIE = 1e-12     # "within rounding": ~4500 ulp, far below any physiological scale
REL_DRIFT = 1e-9    # north_star's trajectory tolerance
CTL_ATOL = 1e-12    # U/h, U, ug: a controller output this close is the same decision.  Outputs computed
                    # from a cancellation (filt - setpoint, a clamp near 0) differ by ~1e-14 in absolute
                    # terms between runs 1e-15 apart, which a purely relative test would call a divergence


@dataclass
class PatientInputs:
    """Everything one closed-loop run needs (numpy, reference layouts)."""
    params: np.ndarray        # [30]
    x0: np.ndarray            # [16]
    c0: np.ndarray            # [11]
    basal: float              # assumed basal (U/h)
    hyper: np.ndarray         # [30]
    meals: tuple              # (start, end, rate, ann) seconds / g/min / g
    ex: tuple                 # (start, end, hrr, announced)
    wiener: np.ndarray        # [H, 3]
    has_noise: int
    meas: np.ndarray          # [H / period_steps]
    controller: int           # 0 dual_hormone, 1 pid_pump
    sz: dict
    dt_s: float
    period_s: float
    pid: int = 0


@dataclass
class Exception_:
    patient: int
    kind: str                 # "bin" | "controller"
    tick: int
    detail: dict = field(default_factory=dict)

    def __str__(self):
        d = ", ".join(f"{k}={v}" for k, v in self.detail.items())
        return f"patient {self.patient}: {self.kind} tie at tick {self.tick} ({d})"


def ulps(a: float, b: float) -> int:
    """Distance in units of the last place between two finite doubles."""
    ia = np.array(a, np.float64).view(np.int64)
    ib = np.array(b, np.float64).view(np.int64)
    return int(abs(int(ia) - int(ib)))


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    den = np.maximum(np.abs(a), np.abs(b))
    with np.errstate(invalid="ignore", divide="ignore"):
        r = np.where(den > 0, np.abs(a - b) / den, 0.0)
    return r


def announced_and_phase(pi: PatientInputs, t: float):
    """_kernel.py:105-117 restated: announced carbs of meals starting in
    [t, t + period) summed in schedule order from 0.0, and the exercise phase
    of an announced active session (else -1)."""
    ms, me, mr, ma = pi.meals
    announced = 0.0
    for j in range(ms.size):
        if t <= ms[j] < t + pi.period_s:
            announced += ma[j]
    es, ee, eh, ea = pi.ex
    phase = -1.0
    for j in range(es.size):
        if ee[j] > t:            # first session not yet ended (ex_ptr)
            if es[j] <= t and ea[j] != 0.0:
                phase = t - es[j]
            break
    return announced, phase


def replay_controller(oracle, pi: PatientInputs, ys, n_ticks: int):
    """The reference's controller (oracle, bitwise) on the readings ys[0:n];
    returns outputs [n, 3] (basal U/h, bolus U, glucagon ug)."""
    step = oracle.pid_step if pi.controller == 1 else oracle.controller_step
    c = np.array(pi.c0, np.float64)
    out = np.zeros((n_ticks, 3))
    for q in range(n_ticks):
        t = q * pi.period_s
        ann, ph = announced_and_phase(pi, t)
        c, o = step(c, float(ys[q]), ann, ph, t, pi.period_s, pi.hyper, float(pi.basal))
        out[q] = o
    return out


def first_divergence(tr_ref: np.ndarray, tr_fast: np.ndarray):
    """First tick where the runs differ: a histogram bin / range, a controller
    output (trace columns 5-7), or BG beyond REL_DRIFT.  None if identical."""
    bg_r, bg_f = tr_ref[:, 1], tr_fast[:, 1]
    bin_r = np.searchsorted(THRESHOLDS, bg_r, side="right")
    bin_f = np.searchsorted(THRESHOLDS, bg_f, side="right")
    rng_r = np.searchsorted(RANGE_BOUNDS, bg_r, side="right")
    rng_f = np.searchsorted(RANGE_BOUNDS, bg_f, side="right")
    dc = np.abs(tr_ref[:, 5:8] - tr_fast[:, 5:8])
    ctl = np.any(dc > REL_TIE * np.maximum(np.abs(tr_ref[:, 5:8]), np.abs(tr_fast[:, 5:8])) + CTL_ATOL, axis=1)
    drift = _rel(bg_r, bg_f) > REL_DRIFT
    flag = (bin_r != bin_f) | (rng_r != rng_f) | ctl | drift
    k = np.flatnonzero(flag)
    if k.size == 0:
        return None
    k = int(k[0])
    return {"tick": k, "bin": bool(bin_r[k] != bin_f[k] or rng_r[k] != rng_f[k]), "ctl": bool(ctl[k]),
            "drift": bool(drift[k])}


def classify(oracle, pi: PatientInputs, tr_ref: np.ndarray, tr_fast: np.ndarray, patient: int):
    """Prove the first divergence of one patient a threshold tie, or raise."""
    fd = first_divergence(tr_ref, tr_fast)
    if fd is None:
        raise AssertionError(f"patient {patient}: outputs differ but the traces never diverge")
    k = fd["tick"]
    if fd["ctl"]:
        ps = pi.sz["period_steps"]
        if k % ps:
            raise AssertionError(f"patient {patient}: controller output differs off a controller tick ({k})")
        q = k // ps
        y_r, y_f = tr_ref[: k + 1: ps, 2], tr_fast[: k + 1: ps, 2]
        dy = float(np.max(_rel(y_r, y_f)))
        if dy > REL_TIE:
            raise AssertionError(f"patient {patient}: CGM readings differ by {dy:.3g} before the "
                                 f"controller divergence at tick {k}")
        rep_r = replay_controller(oracle, pi, y_r, q + 1)
        rep_f = replay_controller(oracle, pi, y_f, q + 1)
        ref_out = tr_ref[: k + 1: ps, 5:8]
        fast_out = tr_fast[: k + 1: ps, 5:8]
        # the oracle replay of the reference readings is the reference run itself
        assert np.array_equal(rep_r, ref_out), f"patient {patient}: controller replay broken"
        if not np.allclose(rep_f, fast_out, rtol=REL_TIE, atol=CTL_ATOL):
            raise AssertionError(f"patient {patient}: fused controller output at tick {k} "
                                 f"{fast_out[-1]} is not the reference controller's on the same readings "
                                 f"{rep_f[-1]}")
        return Exception_(patient, "controller", k, {"max_rel_dy": f"{dy:.2g}",
                                                     "ref": tuple(ref_out[-1]), "fused": tuple(fast_out[-1])})
    if fd["bin"]:
        a, b = float(tr_ref[k, 1]), float(tr_fast[k, 1])
        lo, hi = min(a, b), max(a, b)
        edge = EDGES[(EDGES >= lo) & (EDGES <= hi)]
        if edge.size == 0 or _rel(a, b) > REL_TIE:
            raise AssertionError(f"patient {patient}: bin flip at tick {k} between {a!r} and {b!r} "
                                 "is not a rounding tie")
        return Exception_(patient, "bin", k, {"edge": float(edge[0]), "bg_ref": a, "bg_fused": b,
                                              "ulps_apart": ulps(a, b)})
    raise AssertionError(f"patient {patient}: BG drifts beyond {REL_DRIFT} at tick {k} without a "
                         "discrete cause")


def trace_hist(tr: np.ndarray, ticks: int):
    """The statistics a trace implies: histogram [247], range ticks [5]."""
    bg = tr[:ticks, 1]
    hist = np.bincount(np.searchsorted(THRESHOLDS, bg, side="right"), minlength=247)
    tir = np.bincount(np.searchsorted(RANGE_BOUNDS, bg, side="right"), minlength=5)
    return hist, tir


def same_patient(ref: dict, fused: dict, j: int, i: int | None = None) -> bool:
    """Fused patient j vs reference patient i (default j): FP64 statistics to
    1e-9, integer counts (histogram, hypo events) identical.
    Both dicts: scal [n, >=3] (min, max, sum), hist [n, 247], timeline [n, g]
    (optional), day_dose [n, d, 3] (optional), hypo [n, 2] (optional)."""
    i = j if i is None else i
    ok = np.allclose(fused["scal"][j][:3], ref["scal"][i][:3], rtol=REL_DRIFT, atol=0)
    ok &= np.array_equal(fused["hist"][j], ref["hist"][i])
    if "timeline" in ref and "timeline" in fused:
        ok &= np.allclose(fused["timeline"][j], ref["timeline"][i], rtol=REL_DRIFT, atol=0)
    if "day_dose" in ref and "day_dose" in fused:
        ok &= np.allclose(fused["day_dose"][j], ref["day_dose"][i], rtol=REL_DRIFT, atol=1e-12)
    if "hypo" in ref and "hypo" in fused:
        ok &= np.array_equal(fused["hypo"][j], ref["hypo"][i])
    return bool(ok)


# ------------------------------------------------------------------ runners
def oracle_trace(oracle, pi: PatientInputs):
    """The reference run of one patient (C oracle, bitwise) with its trace."""
    oracle.set_controller(pi.controller)
    try:
        out = oracle.run_batch_injected(
            pi.params[None], pi.x0[None], pi.c0[None], pi.hyper, np.array([pi.basal]), pi.sz, pi.dt_s,
            pi.period_s, np.array([0, pi.meals[0].size]), pi.meals, np.array([0, pi.ex[0].size]), pi.ex,
            pi.wiener[None], np.array([pi.has_noise], np.uint8), pi.meas[None], trace=True)
    finally:
        oracle.set_controller(0)
    return out["trace"][0], int(out["ticks"][0])


def fused_trace(pi: PatientInputs, dev):
    """The same patient through the fused kernel's TRACE variant (CSR protocol,
    injected noise): same arithmetic as the benchmarked instance."""
    import torch
    from paper_2202_13927_b200 import engine, rng
    from paper_2202_13927_b200.protocol import ProtocolArrays, compile_ticks
    D = lambda a, t=torch.float64: engine.dev(np.ascontiguousarray(a), t, dev)
    ta = compile_ticks(ProtocolArrays(*pi.meals, *pi.ex), pi.dt_s, pi.period_s)
    nz = lambda a: a if a.size else np.zeros(1, a.dtype)
    csr = {"meal_off": D(np.array([0, ta.meal_ks.size]), torch.int64),
           "ex_off": D(np.array([0, ta.ex_ks.size]), torch.int64)}
    for k, dt, tdt in (("meal_ks", np.int32, torch.int32), ("meal_ke", np.int32, torch.int32),
                       ("meal_kp", np.int32, torch.int32), ("meal_rate", np.float64, torch.float64),
                       ("meal_ann", np.float64, torch.float64), ("ex_ks", np.int32, torch.int32),
                       ("ex_ke", np.int32, torch.int32), ("ex_hrr", np.float64, torch.float64),
                       ("ex_announced", np.float64, torch.float64)):
        csr[k] = D(nz(getattr(ta, k).astype(dt)), tdt)
    csr["ex_start_s"] = D(nz(ta.ex_start.astype(np.float64)))
    inj = {"wiener": D(pi.wiener.reshape(-1)), "has_noise": D(np.array([pi.has_noise], np.uint8), torch.uint8),
           "meas": D(pi.meas.reshape(-1))}
    ins = {"params": D(pi.params[None]), "x0": D(pi.x0[None]), "c0": D(pi.c0[None]), "hyper": D(pi.hyper),
           "assumed_basal": D(np.array([pi.basal]))}
    H = pi.sz["horizon_ticks"]
    outs = engine.alloc_fast_outputs(1, pi.pid, pi.sz, dev, per_patient_timeline=True)
    tr = engine.empty((1, H, 8), torch.float64, dev)
    engine.launch_fast(ins, outs, pi.sz, pi.dt_s, pi.period_s, 0, rng.ROLE_DEVICE_NOISE,
                       max(1, int(np.ceil(900.0 / pi.dt_s))), dev, csr=csr, injected=inj,
                       controller_code=pi.controller, trace=tr)
    return tr.cpu().numpy()[0], outs


def check_patients(oracle, dev, n: int, ref: dict, fused: dict, inputs, label: str = "", ref_index=None):
    """Every patient j < n equals the reference (same_patient) or is a proven
    threshold tie (classify).  ``inputs(j)`` -> PatientInputs; ``ref_index(j)``
    maps to the reference's row (default j).  Returns the exception list
    (printed, so the test log carries it)."""
    exc = []
    for j in range(n):
        i = j if ref_index is None else ref_index(j)
        if same_patient(ref, fused, j, i):
            continue
        pi = inputs(j)
        tr_r, ticks_r = oracle_trace(oracle, pi)
        tr_f, outs = fused_trace(pi, dev)
        # the traced fused run is the run whose statistics are being compared
        hist_f, _ = trace_hist(tr_f, ticks_r)
        assert np.array_equal(hist_f, fused["hist"][j]), f"{label} patient {j}: traced fused run differs"
        e = classify(oracle, pi, tr_r, tr_f, j)
        exc.append(e)
    for e in exc:
        print(f"[{label}] {e}")
    print(f"[{label}] {len(exc)} proven threshold ties of {n} patients")
    return exc


def inputs_from_arrays(params, x0, c0, basal, hyper, meal_off, meals, ex_off, ex, wiener, has_noise, meas,
                       controller, sz, dt_s, period_s, pid0=0):
    """PatientInputs factory over batched arrays (reference CSR layouts)."""
    def make(j):
        a, b = int(meal_off[j]), int(meal_off[j + 1])
        c, d = int(ex_off[j]), int(ex_off[j + 1])
        return PatientInputs(
            params=np.asarray(params[j], np.float64), x0=np.asarray(x0[j], np.float64),
            c0=np.asarray(c0[j], np.float64), basal=float(basal[j]), hyper=np.asarray(hyper, np.float64),
            meals=tuple(np.asarray(m[a:b], np.float64) for m in meals),
            ex=tuple(np.asarray(e[c:d], np.float64) for e in ex),
            wiener=np.asarray(wiener[j], np.float64), has_noise=int(has_noise[j]),
            meas=np.asarray(meas[j], np.float64), controller=int(controller), sz=sz, dt_s=float(dt_s),
            period_s=float(period_s), pid=int(pid0) + j)
    return make


def case_inputs(case, sub, controller=0):
    """PatientInputs factory over a golden SimCase subset (tests/helpers.py)."""
    return inputs_from_arrays(sub["params"], sub["x0"], sub["c0"], sub["basal"], case.hyper, sub["meal_off"],
                              sub["meals"], sub["ex_off"], sub["ex"], sub["wiener"], sub["has_noise"],
                              sub["meas"], controller, case.sz, case.config.dt_s,
                              case.config.controller_period_s, int(case.ids[sub["idx"][0]]))
