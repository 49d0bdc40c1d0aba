"""Device engine: buffers, launches and result transfer around libglucosim.

PyTorch provides device memory and streams only; all compute runs in the
hand-written kernels behind the C-ABI (_lib.py).  There is no CPU path:
without a CUDA device or the built library every call raises.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import (FastArgs, MealGen, ParityArgs, ReduceArgs, SamplerArgs, check)
from .layout import N_BG_BINS, N_CSTATE, N_PARAMS, N_STATES, N_THRESHOLDS, TIR_BINS

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_device(device=None):
    t = torch()
    if not t.cuda.is_available():
        raise _lib.GlucosimError("no CUDA device: the glucosim engine has no CPU fallback")
    _lib.load()
    if device is None:
        device = t.device("cuda", t.cuda.current_device())
    return t.device(device)


class nvtx:
    """NVTX range around a host-side phase (sampler, schedule planning,
    integrator, exclusion re-run, reduction, read-back), visible in Nsight
    Systems / ncu --nvtx timelines.  A no-op without a CUDA build of torch."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        try:
            torch().cuda.nvtx.range_push(self.name)
            self._on = True
        except Exception:
            self._on = False
        return self

    def __exit__(self, *exc):
        if self._on:
            torch().cuda.nvtx.range_pop()
        return False


def ptr(x) -> C.c_void_p:
    return C.c_void_p(0 if x is None else x.data_ptr())


def stream_ptr(device) -> C.c_void_p:
    return C.c_void_p(torch().cuda.current_stream(device).cuda_stream)


def dev(a, dtype, device):
    t = torch()
    arr = np.ascontiguousarray(a)
    tt = t.from_numpy(arr)
    if dtype is not None:
        tt = tt.to(dtype)
    return tt.to(device, non_blocking=False)


def empty(shape, dtype, device):
    return torch().empty(shape, dtype=dtype, device=device)


# ----------------------------------------------------------- steady state
def steady_state(params: np.ndarray, target_bg: float, device=None):
    """Batched hovorka.steady_state on device -> (x0 [n,16], u_basal [n], ok [n])."""
    device = require_device(device)
    t = torch()
    n = params.shape[0]
    p = params.contiguous() if hasattr(params, "data_ptr") else dev(params.astype(np.float64), t.float64, device)
    x0 = empty((n, N_STATES), t.float64, device)
    ub = empty((n,), t.float64, device)
    st = empty((n,), t.int32, device)
    check(_lib.load().gt_steady_state(n, ptr(p), float(target_bg), ptr(x0), ptr(ub), ptr(st),
                                      stream_ptr(device)), "gt_steady_state")
    return x0, ub, st


def controller_init(hyper: np.ndarray, icr_factor: float, basal, device=None):
    device = require_device(device)
    t = torch()
    basal_t = basal if hasattr(basal, "data_ptr") else dev(np.asarray(basal, np.float64), t.float64, device)
    n = basal_t.shape[0]
    h = dev(np.asarray(hyper, np.float64), t.float64, device)
    c0 = empty((n, N_CSTATE), t.float64, device)
    check(_lib.load().gt_controller_init(n, ptr(h), float(icr_factor), ptr(basal_t), ptr(c0),
                                         stream_ptr(device)), "gt_controller_init")
    return c0


# ------------------------------------------------------------ parity path
@dataclass
class ParityBatch:
    """Host inputs of the parity kernel (see include/glucosim.h gt_parity_args)."""
    params: np.ndarray        # [n,30]
    x0: np.ndarray            # [n,16]
    c0: np.ndarray            # [n,11]
    hyper: np.ndarray         # [30]
    assumed_basal: np.ndarray # [n]
    meal_off: np.ndarray      # [n+1] int64
    meals: tuple              # 4 x float64 [total]
    ex_off: np.ndarray
    ex: tuple
    wiener: np.ndarray        # [n,H,3]
    has_noise: np.ndarray     # [n] uint8
    meas: np.ndarray          # [n,H/ps]
    active: np.ndarray | None = None
    controller: int = 0       # GT_CTRL_*


def run_parity(batch: ParityBatch, sz: dict, dt_s: float, period_s: float,
               record_trace: bool = False, device=None, fetch: bool = True) -> dict:
    """Run the bitwise-parity integrator; returns numpy per-patient outputs
    (fetch=False: the device tensors, still being computed on the current
    stream -- ``fetch_parity`` reads them; the inputs are stream-ordered, so
    their memory is reused only after the launch)."""
    device = require_device(device)
    t = torch()
    n = batch.params.shape[0]
    H, nd, ng = sz["horizon_ticks"], sz["n_days"], sz["n_grid"]
    f64, i64 = t.float64, t.int64
    D = lambda a, dt=f64: dev(a, dt, device)
    nz1 = lambda a: a if a.size else np.zeros(1)
    ins = {
        "params": D(batch.params), "x0": D(batch.x0), "c0": D(batch.c0), "hyper": D(batch.hyper),
        "assumed_basal": D(batch.assumed_basal),
        "active": D(batch.active.astype(np.int32), t.int32) if batch.active is not None else None,
        "meal_off": D(batch.meal_off, i64), "ex_off": D(batch.ex_off, i64),
        "meals": [D(nz1(m)) for m in batch.meals], "ex": [D(nz1(e)) for e in batch.ex],
        "wiener": D(nz1(batch.wiener.reshape(-1))), "has_noise": D(batch.has_noise.astype(np.uint8), t.uint8),
        "meas": D(nz1(batch.meas.reshape(-1))),
    }
    out = {
        "status": empty((n,), t.int32, device), "ticks": empty((n,), i64, device),
        "tir_ticks": empty((n, 5), i64, device), "bg_hist": empty((n, N_BG_BINS), i64, device),
        "scal": empty((n, 4), f64, device), "day_dose": empty((n, nd, 3), f64, device),
        "timeline": empty((n, ng), f64, device), "x_out": empty((n, N_STATES), f64, device),
        "c_out": empty((n, N_CSTATE), f64, device),
        "trace": empty((n, H, 8), f64, device) if record_trace else None,
    }
    a = ParityArgs()
    a.n, a.dt_s, a.period_s = n, float(dt_s), float(period_s)
    a.period_steps, a.horizon_ticks, a.grid_step_ticks = sz["period_steps"], H, sz["grid_step_ticks"]
    a.n_days, a.n_grid, a.block_ticks = nd, ng, sz["block_ticks"]
    a.controller = int(batch.controller)
    for k in ("params", "x0", "c0", "hyper", "assumed_basal", "active", "meal_off", "ex_off",
              "wiener", "has_noise", "meas"):
        setattr(a, k, ptr(ins[k]))
    a.meals_start, a.meals_end, a.meals_rate, a.meals_ann = (ptr(m) for m in ins["meals"])
    a.ex_start, a.ex_end, a.ex_hrr, a.ex_announced = (ptr(e) for e in ins["ex"])
    for k, v in out.items():
        setattr(a, k, ptr(v))
    check(_lib.load().gt_simulate_parity(C.byref(a), stream_ptr(device)), "gt_simulate_parity")
    return fetch_parity(out) if fetch else out


def fetch_parity(out: dict) -> dict:
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in out.items()}


# -------------------------------------------------------------- fast path
def meal_gen_struct(spec: dict | None) -> MealGen:
    g = MealGen()
    if spec:
        for j in range(3):
            g.clock_s[j] = spec["clock_s"][j]
            g.mean_g[j] = spec["mean_g"][j]
        g.sd_g, g.jitter_s, g.duration_s, g.role = (spec["sd_g"], spec["jitter_s"],
                                                     spec["duration_s"], spec["role"])
    return g


@dataclass
class FastOutputs:
    """Device-resident per-patient outputs of the fused integrator (SoA)."""
    n: int
    pid0: int
    status: object
    ticks: object
    bg_hist: object       # [247, n] int32
    bg_stats: object      # [3, n]
    day_dose: object      # [n_days, 3, n]
    hypo_events: object   # [2, n]
    timeline_warp: object # [n_grid, n_warps, 3]
    timeline_pp: object = None
    x_out: object = None
    scratch: object = None  # uint8 [gt_fast_scratch_bytes(n)]: the persistent schedule's workspace


def alloc_fast_outputs(n: int, pid0: int, sz: dict, device, per_patient_timeline=False,
                       final_state=False) -> FastOutputs:
    t = torch()
    nw = (n + 31) // 32
    return FastOutputs(
        n=n, pid0=pid0,
        status=empty((n,), t.int32, device), ticks=empty((n,), t.int64, device),
        bg_hist=empty((N_BG_BINS, n), t.int32, device), bg_stats=empty((3, n), t.float64, device),
        day_dose=empty((sz["n_days"], 3, n), t.float64, device),
        hypo_events=empty((2, n), t.int32, device),
        timeline_warp=empty((sz["n_grid"], nw, 3), t.int64, device),
        timeline_pp=empty((sz["n_grid"], n), t.float64, device) if per_patient_timeline else None,
        x_out=empty((N_STATES, n), t.float64, device) if final_state else None,
        scratch=empty((int(_lib.load().gt_fast_scratch_bytes(n)),), t.uint8, device),
    )


def launch_fast(inputs: dict, outs: FastOutputs, sz: dict, dt_s: float, period_s: float,
                seed: int, noise_role: int, hypo_min_ticks: int, device,
                meal_spec: dict | None = None, csr: dict | None = None,
                injected: dict | None = None, controller_code: int = 0, fixed=None,
                rerun_diverged: bool = False, n_slices: int = 0, noise_agg: int = 1,
                fp32: bool = False, trace=None) -> None:
    """Enqueue the fused integrator on the current stream (no sync).
    ``fixed``: the launch-uniform values of the non-sampled parameters
    (p[30] order); defaults to row 0 of ``inputs['params']`` after checking
    every row agrees (see :func:`uniform_fixed`)."""
    from ._lib import GT_NOISE_INJECTED, GT_NOISE_PHILOX, GT_PROTO_CSR, GT_PROTO_THREE_MEAL
    if fixed is None:
        fixed = uniform_fixed(inputs["params"])
    a = FastArgs()
    for k in range(N_PARAMS):
        a.fixed[k] = float(fixed[k])
    a.n, a.pid0, a.seed = outs.n, outs.pid0, int(seed) & 0xFFFFFFFFFFFFFFFF
    a.proto_kind = GT_PROTO_THREE_MEAL if csr is None else GT_PROTO_CSR
    a.noise_kind = GT_NOISE_PHILOX if injected is None else GT_NOISE_INJECTED
    a.controller = controller_code
    a.n_slices = int(n_slices)
    a.noise_agg = int(noise_agg)
    a.precision = 1 if fp32 else 0
    a.dt_s, a.period_s = float(dt_s), float(period_s)
    a.period_steps, a.horizon_ticks, a.grid_step_ticks = (sz["period_steps"], sz["horizon_ticks"],
                                                          sz["grid_step_ticks"])
    a.n_days, a.n_grid, a.hypo_min_ticks = sz["n_days"], sz["n_grid"], int(hypo_min_ticks)
    a.noise_role = noise_role
    a.rerun_diverged = int(rerun_diverged)   # 0 off, 1 exclusion re-run, 2 abort-tick pass
    for k in ("params", "x0", "c0", "assumed_basal", "active"):
        setattr(a, k, ptr(inputs.get(k)))
    # hyperparameters by value (the kernel's parameter bank): the host copy
    # when the caller has one, else read back once from the device tensor
    hy = inputs.get("hyper_host")
    if hy is None:
        hy = inputs["hyper"]
        hy = hy.detach().cpu().numpy() if hasattr(hy, "detach") else np.asarray(hy)
    for k in range(len(a.hyper)):
        a.hyper[k] = float(hy[k])
    a.meal_gen = meal_gen_struct(meal_spec)
    if csr is not None:
        for k in ("meal_off", "meal_ks", "meal_ke", "meal_kp", "meal_rate", "meal_ann", "ex_off",
                  "ex_ks", "ex_ke", "ex_start_s", "ex_hrr", "ex_announced"):
            setattr(a, k, ptr(csr[k]))
    if injected is not None:
        a.wiener, a.has_noise, a.meas = ptr(injected["wiener"]), ptr(injected["has_noise"]), ptr(injected["meas"])
    a.status, a.ticks, a.bg_hist, a.bg_stats = ptr(outs.status), ptr(outs.ticks), ptr(outs.bg_hist), ptr(outs.bg_stats)
    a.day_dose, a.hypo_events, a.timeline_warp = ptr(outs.day_dose), ptr(outs.hypo_events), ptr(outs.timeline_warp)
    a.timeline_pp, a.x_out = ptr(outs.timeline_pp), ptr(outs.x_out)
    if outs.scratch is not None:
        a.scratch, a.scratch_bytes = ptr(outs.scratch), outs.scratch.numel()
    a.trace = ptr(trace)   # [n, horizon_ticks, 8] float64 or None
    check(_lib.load().gt_simulate_fast(C.byref(a), stream_ptr(device)), "gt_simulate_fast")


def northern_csr(params, pid0: int, trial_seed: int, dt_s: float, period_s: float, horizon_s: float,
                 device, week_days: bool = False, announcement=None) -> dict:
    """Device NorthernYearProtocol in the fused kernel's CSR layout (fixed
    stride GT_NY_MEALS / GT_NY_EX per patient; see include/glucosim.h).
    Returns the CSR dict of FastTrial plus ``n_meals`` / ``n_ex`` (events
    before the horizon) and optionally ``week_days`` [52, n] uint16."""
    from ._lib import GT_NY_EX, GT_NY_MEALS, NorthernArgs
    t = torch()
    n = int(params.shape[0])
    i32, f64 = t.int32, t.float64
    out = {
        "meal_ks": empty((n * GT_NY_MEALS,), i32, device), "meal_ke": empty((n * GT_NY_MEALS,), i32, device),
        "meal_kp": empty((n * GT_NY_MEALS,), i32, device), "meal_rate": empty((n * GT_NY_MEALS,), f64, device),
        "meal_ann": empty((n * GT_NY_MEALS,), f64, device),
        "ex_ks": empty((n * GT_NY_EX,), i32, device), "ex_ke": empty((n * GT_NY_EX,), i32, device),
        "ex_start_s": empty((n * GT_NY_EX,), f64, device), "ex_hrr": empty((n * GT_NY_EX,), f64, device),
        "ex_announced": empty((n * GT_NY_EX,), f64, device),
        "n_meals": empty((n,), i32, device), "n_ex": empty((n,), i32, device),
        "meal_off": t.arange(n + 1, dtype=t.int64, device=device) * GT_NY_MEALS,
        "ex_off": t.arange(n + 1, dtype=t.int64, device=device) * GT_NY_EX,
    }
    if week_days:
        out["week_days"] = empty((52, n), t.int16, device)
    a = NorthernArgs()
    a.n, a.pid0, a.trial_seed = n, int(pid0), int(trial_seed) & 0xFFFFFFFFFFFFFFFF
    a.dt_s, a.period_s, a.horizon_s = float(dt_s), float(period_s), float(horizon_s)
    a.params = ptr(params.contiguous())
    for k in ("meal_ks", "meal_ke", "meal_kp", "meal_rate", "meal_ann", "ex_ks", "ex_ke", "ex_start_s",
              "ex_hrr", "ex_announced", "n_meals", "n_ex"):
        setattr(a, k, ptr(out[k]))
    a.week_days = ptr(out.get("week_days"))
    frac, (lo, hi) = (0.0, (1.0, 1.0)) if announcement is None else (
        float(announcement.fraction_unannounced), tuple(float(v) for v in announcement.misannouncement_factor_range))
    a.fraction_unannounced, a.factor_lo, a.factor_hi = frac, lo, hi
    check(_lib.load().gt_northern_protocol(C.byref(a), stream_ptr(device)), "gt_northern_protocol")
    return out


def noise_normals(n: int, pid0: int, seed: int, role: int, k0: int, n_ticks: int, device):
    """The fused kernel's noise stream as a [n, n_ticks, 4] float32 tensor."""
    t = torch()
    out = empty((n, n_ticks, 4), t.float32, device)
    check(_lib.load().gt_noise_normals(n, pid0, int(seed) & 0xFFFFFFFFFFFFFFFF, role, k0, n_ticks, ptr(out),
                                       stream_ptr(device)), "gt_noise_normals")
    return out


FIXED_PARAM_INDEX = tuple(range(_lib.GT_FIXED_FIRST, 30))   # AG .. R: the table's fixed block (hovorka.py:53-55)


def stage_fast(params, ss_status=None, want_active: bool = True):
    """One device pass (gt_stage_fast): the fused kernel's launch constants
    and active mask.  Returns (fixed [30] numpy = row 0 of ``params``, active
    int32 device tensor or None); raises unless every patient shares the
    fixed parameters (hovorka_distributions.yaml: 'identical for every
    generated patient'), which the fused kernel folds into launch constants.
    active[i] = ss_status[i] == GT_STATUS_OK (all ones without ss_status)."""
    t = torch()
    device = params.device
    n = int(params.shape[0])
    p = params.contiguous()
    active = empty((n,), t.int32, device) if want_active else None
    fixed_d = empty((30,), t.float64, device)
    flag_d = empty((1,), t.int32, device)
    check(_lib.load().gt_stage_fast(n, ptr(p), ptr(ss_status), ptr(active), ptr(fixed_d), ptr(flag_d),
                                    stream_ptr(device)), "gt_stage_fast")
    fixed_h = t.empty((30,), dtype=t.float64, pin_memory=True)
    flag_h = t.empty((1,), dtype=t.int32, pin_memory=True)
    fixed_h.copy_(fixed_d, non_blocking=True)
    flag_h.copy_(flag_d, non_blocking=True)
    t.cuda.current_stream(device).synchronize()
    if int(flag_h[0]) != 0:
        raise _lib.GlucosimError("the fused path needs fixed parameters shared by all patients; "
                                 "use the parity path (noise='reference') for per-patient overrides")
    return fixed_h.numpy().astype(np.float64), active


def uniform_fixed(params) -> np.ndarray:
    """Row 0 of the parameter matrix after verifying on the device that every
    patient shares the fixed parameters (see :func:`stage_fast`)."""
    return stage_fast(params, want_active=False)[0]


@dataclass
class ReduceOutputs:
    counts: object
    tir_ticks_total: object
    tir_hist: object
    bg_hist_total: object
    below_min: object
    below_max: object
    minmax_bg_bits: object
    timeline: object
    dose_hist: object
    dose_sum_fp: object
    worst: object
    metric_hist: object
    metrics: dict | None = None
    scratch: object = None  # uint8 [GT_REDUCE_SCRATCH_BYTES]


def alloc_reduce_outputs(n: int, sz: dict, device, per_patient_metrics=False) -> ReduceOutputs:
    t = torch()
    i64 = t.int64
    return ReduceOutputs(
        counts=empty((6,), i64, device), tir_ticks_total=empty((5,), i64, device),
        tir_hist=empty((5, TIR_BINS + 1), i64, device), bg_hist_total=empty((N_BG_BINS,), i64, device),
        below_min=empty((N_THRESHOLDS,), i64, device), below_max=empty((N_THRESHOLDS,), i64, device),
        minmax_bg_bits=empty((2,), i64, device), timeline=empty((3, sz["n_grid"]), i64, device),
        dose_hist=empty((3, 201), i64, device), dose_sum_fp=empty((6,), i64, device),
        worst=empty((4,), i64, device), metric_hist=empty((7, TIR_BINS + 1), i64, device),
        metrics={k: empty((n,), t.float32, device) for k in ("tir", "tbr70", "tbr54", "tar180", "tar250")}
        if per_patient_metrics else None,
        scratch=empty((_lib.GT_REDUCE_SCRATCH_BYTES,), t.uint8, device),
    )


def launch_reduce(outs: FastOutputs, red: ReduceOutputs, sz: dict, dt_s: float, device) -> None:
    a = ReduceArgs()
    a.n, a.pid0, a.horizon_ticks, a.n_days, a.n_grid = outs.n, outs.pid0, sz["horizon_ticks"], sz["n_days"], sz["n_grid"]
    a.n_warps, a.dt_s = (outs.n + 31) // 32, float(dt_s)
    a.status, a.ticks, a.bg_hist, a.bg_stats = ptr(outs.status), ptr(outs.ticks), ptr(outs.bg_hist), ptr(outs.bg_stats)
    a.day_dose, a.hypo_events, a.timeline_warp = ptr(outs.day_dose), ptr(outs.hypo_events), ptr(outs.timeline_warp)
    for k in ("counts", "tir_ticks_total", "tir_hist", "bg_hist_total", "below_min", "below_max",
              "minmax_bg_bits", "timeline", "dose_hist", "dose_sum_fp", "worst", "metric_hist"):
        setattr(a, k, ptr(getattr(red, k)))
    if red.metrics is not None:
        a.metric_tir, a.metric_tbr70, a.metric_tbr54 = (ptr(red.metrics[k]) for k in ("tir", "tbr70", "tbr54"))
        a.metric_tar180, a.metric_tar250 = ptr(red.metrics["tar180"]), ptr(red.metrics["tar250"])
    if red.scratch is not None:
        a.scratch, a.scratch_bytes = ptr(red.scratch), red.scratch.numel()
    check(_lib.load().gt_reduce_trial(C.byref(a), stream_ptr(device)), "gt_reduce_trial")


def ordered_bits_to_double(b: int) -> float:
    b = int(b)
    if b < 0:
        b ^= 0x7FFFFFFFFFFFFFFF
    return float(np.array([b], dtype=np.int64).view(np.float64)[0])


# ------------------------------------------------------ population sampler
def sample_population(seed: int, n: int, table, pid0: int = 0, target_bg: float = 6.0,
                      device=None, max_attempts: int = 10_000, weight=(74.0, 13.0),
                      min_basal: float = 0.4, max_weight_redraws: int = 0):
    """Device rejection sampler -> dict of device tensors."""
    from .layout import PARAM_INDEX, PARAM_NAMES
    device = require_device(device)
    t = torch()
    a = SamplerArgs()
    a.n, a.pid0, a.seed = n, pid0, int(seed) & 0xFFFFFFFFFFFFFFFF
    names = list(table.sampled)
    if len(names) > 16:
        raise ValueError("at most 16 sampled parameters")
    a.n_sampled, a.max_attempts = len(names), max_attempts
    a.max_weight_redraws = int(max_weight_redraws)
    a.target_bg, a.min_basal_uh = float(target_bg), float(min_basal)
    a.weight_mean, a.weight_sd = float(weight[0]), float(weight[1])
    for j, name in enumerate(names):
        spec = table.sampled[name]
        a.kind[j] = 0 if spec.kind == "normal" else 1
        a.param_index[j] = PARAM_INDEX[name]
        a.a[j], a.b[j] = ((spec.mean, spec.sd) if spec.kind == "normal" else (spec.log_mu, spec.log_sigma))
    for k, name in enumerate(PARAM_NAMES):
        a.fixed_params[k] = float(table.fixed.get(name, 0.0))
    out = {
        "params": empty((n, N_PARAMS), t.float64, device), "x0": empty((n, N_STATES), t.float64, device),
        "u_basal": empty((n,), t.float64, device), "attempts": empty((n,), t.int32, device),
        "status": empty((n,), t.int32, device), "reject_counts": t.zeros((4,), dtype=t.int64, device=device),
    }
    a.params, a.x0, a.u_basal_uh = ptr(out["params"]), ptr(out["x0"]), ptr(out["u_basal"])
    a.attempts, a.status, a.reject_counts = ptr(out["attempts"]), ptr(out["status"]), ptr(out["reject_counts"])
    check(_lib.load().gt_sample_population(C.byref(a), stream_ptr(device)), "gt_sample_population")
    return out


def generate_meals(seed: int, pid0: int, n: int, n_meals: int, spec: dict, device=None):
    device = require_device(device)
    t = torch()
    s = empty((n, n_meals), t.float64, device)
    e = empty((n, n_meals), t.float64, device)
    g = empty((n, n_meals), t.float64, device)
    mg = meal_gen_struct(spec)
    check(_lib.load().gt_generate_meals(n, pid0, int(seed) & 0xFFFFFFFFFFFFFFFF, C.byref(mg), n_meals,
                                        ptr(s), ptr(e), ptr(g), stream_ptr(device)), "gt_generate_meals")
    return s.cpu().numpy(), e.cpu().numpy(), g.cpu().numpy()
