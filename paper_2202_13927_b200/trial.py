"""Fast trial path: fused integrator + device reduction (+ optional sharding).

``FastTrial`` stages a shard of patients on one device once (parameters,
steady states, controller states, protocol source) and runs
simulate -> reduce on a CUDA stream; ``accumulator()`` converts the exact
device fields into a ``TrialAccumulator``.  Patients whose simulation
diverges are excluded exactly as the reference does (analytics.py:267-269):
warps that contained one are re-run with the diverged lanes masked, so the
per-warp timeline partials never include them.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import analytics, engine, rng
from ._lib import (GT_STATUS_BAD_INITIAL_STATE, GT_STATUS_EXCLUDED, GT_STATUS_NO_STEADY_STATE, GT_STATUS_NONFINITE,
                   GT_STATUS_OK)
from .analytics import TrialAccumulator, WorstCase
from .config import SimulationError, sizes
from .controller import device_code, hyper_vector, icr_initial_factor
from .layout import DOSE_SIGNALS, N_BG_BINS, N_THRESHOLDS
from .protocol import ThreeMealProtocol, compile_protocol, compile_ticks


@dataclass
class ShardInputs:
    pid0: int
    n: int
    params: object       # device [n,30]
    basal: object        # device [n]


def population_to_device(population, basal_scale: float, device):
    """(pid0, params[n,30] device, basal[n] device) from a list of
    (patient, parameter_set) or a DevicePopulation."""
    t = engine.torch()
    if hasattr(population, "params_device"):
        return population.pid0, population.params_device, population.basal_device * basal_scale
    from .simulation import pack_params_many
    ids = np.array([int(pt.id) for pt, _ in population], dtype=np.int64)
    if ids.size and not np.array_equal(ids, ids[0] + np.arange(ids.size)):
        raise SimulationError("the fused path keys RNG streams by contiguous patient ids")
    params = pack_params_many([ps.values for _, ps in population])
    basal = np.array([ps.u_basal_u_per_h for _, ps in population], dtype=np.float64) * basal_scale
    return int(ids[0]), engine.dev(params, t.float64, device), engine.dev(basal, t.float64, device)


class FastTrial:
    def __init__(self, pid0, params, basal, generator, profile, config, controller_id="dual_hormone",
                 device=None, hypo_min_s: float = 900.0, per_patient_metrics: bool = False,
                 seed: int | None = None, n_slices: int = 0, noise_agg: int = 1,
                 fp32: bool = False, x0=None):
        self.n_slices = int(n_slices)   # 0 = chosen by the launcher
        # BASELINE configs[4]: each step's Brownian increment aggregated from
        # noise_agg fine Philox increments (the path a dt/noise_agg run draws),
        # and the FP32 integrator (controller and statistics stay FP64)
        self.noise_agg, self.fp32 = int(noise_agg), bool(fp32)
        self.device = engine.require_device(device)
        t = engine.torch()
        self.config = config
        self.sz = sizes(config)
        self.pid0 = int(pid0)
        self.n = int(params.shape[0])
        self.seed = int(config.seed if seed is None else seed)
        self.controller_id = controller_id
        self.code = device_code(controller_id)
        self.profile = profile
        self.hyper = hyper_vector(profile)
        self.params, self.basal = params, basal
        self.hypo_min_ticks = max(1, int(np.ceil(hypo_min_s / config.dt_s)))
        self.generator = generator
        with t.cuda.device(self.device):
            if x0 is not None:
                # the sampler's own steady states (same solve, same target BG): every
                # sampled patient has one, so nothing is aborted at staging
                self.x0 = x0
                self.ss_status = None
            else:
                self.x0, _ub, self.ss_status = engine.steady_state(params, config.initial_bg_mmol_per_l, self.device)
            self.c0 = engine.controller_init(self.hyper, icr_initial_factor(profile), basal, self.device)
            self.hyper_d = engine.dev(self.hyper, t.float64, self.device)
            # launch constants (fixed block verified uniform) and the active mask, one device pass
            self.fixed, self.active = engine.stage_fast(params, self.ss_status)
            self.meal_spec, self.csr = None, None
            if isinstance(generator, ThreeMealProtocol):
                self.meal_spec = generator.device_spec()
            else:
                self.csr = self._build_csr(generator)
            self.outs = engine.alloc_fast_outputs(self.n, self.pid0, self.sz, self.device)
            self.red = engine.alloc_reduce_outputs(self.n, self.sz, self.device, per_patient_metrics)
        self._inputs = {"params": self.params, "x0": self.x0, "c0": self.c0, "hyper": self.hyper_d,
                        "hyper_host": np.asarray(self.hyper, np.float64),
                        "assumed_basal": self.basal, "active": self.active}

    def _build_csr(self, generator):
        t = engine.torch()
        cfg = self.config
        from .northern import NorthernYearProtocol
        if isinstance(generator, NorthernYearProtocol) and generator.on_device():
            # planned on the device from the reference's own keyed stream
            csr = engine.northern_csr(self.params, self.pid0, cfg.seed, cfg.dt_s, cfg.controller_period_s,
                                      cfg.horizon_s, self.device, announcement=generator.announcement)
            if bool((csr["n_meals"] < 0).any()):
                raise SimulationError("NorthernYear week plan failed (no admissible day order)")
            return csr

        class _P:  # minimal patient for generator.build
            def __init__(self, pid, w):
                self.id, self.body_weight_kg = pid, w
        w = self.params[:, 0].cpu().numpy()
        tas = []
        for i in range(self.n):
            pa = compile_protocol(generator.build(cfg.seed, _P(self.pid0 + i, float(w[i]))), cfg.horizon_s)
            tas.append(compile_ticks(pa, cfg.dt_s, cfg.controller_period_s))
        moff = np.zeros(self.n + 1, np.int64)
        eoff = np.zeros(self.n + 1, np.int64)
        for i, ta in enumerate(tas):
            moff[i + 1] = moff[i] + ta.meal_ks.size
            eoff[i + 1] = eoff[i] + ta.ex_ks.size
        cat = lambda k, dt: np.concatenate([getattr(ta, k) for ta in tas]).astype(dt) if tas else np.zeros(0, dt)
        nz = lambda a: a if a.size else np.zeros(1, a.dtype)
        D = lambda a, tdt: engine.dev(nz(a), tdt, self.device)
        return {
            "meal_off": D(moff, t.int64), "meal_ks": D(cat("meal_ks", np.int32), t.int32),
            "meal_ke": D(cat("meal_ke", np.int32), t.int32), "meal_kp": D(cat("meal_kp", np.int32), t.int32),
            "meal_rate": D(cat("meal_rate", np.float64), t.float64), "meal_ann": D(cat("meal_ann", np.float64), t.float64),
            "ex_off": D(eoff, t.int64), "ex_ks": D(cat("ex_ks", np.int32), t.int32),
            "ex_ke": D(cat("ex_ke", np.int32), t.int32), "ex_start_s": D(cat("ex_start", np.float64), t.float64),
            "ex_hrr": D(cat("ex_hrr", np.float64), t.float64),
            "ex_announced": D(cat("ex_announced", np.float64), t.float64),
        }

    # ------------------------------------------------------------- running
    def simulate(self, active=None, injected=None, rerun_diverged=0):
        """Enqueue the fused integrator (current stream, no sync).
        rerun_diverged: 0 the full run, 1 the exclusion re-run, 2 the
        abort-tick pass (see ``_rerun_if_diverged``)."""
        inputs = dict(self._inputs)
        if active is not None:
            inputs["active"] = active
        name = {0: "gt.fused_integrator", 1: "gt.exclusion_rerun", 2: "gt.abort_tick_pass"}[int(rerun_diverged)]
        with engine.nvtx(name):
            self._launch(inputs, injected, rerun_diverged)

    def _launch(self, inputs, injected, rerun_diverged):
        engine.launch_fast(inputs, self.outs, self.sz, self.config.dt_s,
                           self.config.controller_period_s, self.seed, rng.ROLE_DEVICE_NOISE,
                           self.hypo_min_ticks, self.device, meal_spec=self.meal_spec, csr=self.csr,
                           injected=injected, controller_code=self.code, fixed=self.fixed,
                           rerun_diverged=rerun_diverged,
                           # the re-run passes skip whole warps: one unit per warp (a slice of
                           # a warp waits for the previous one anyway, and slicing is
                           # bit-invisible), so a pass with nothing to do is one check per warp
                           n_slices=1 if rerun_diverged else self.n_slices,
                           noise_agg=self.noise_agg, fp32=self.fp32)

    def trace_range(self, lo: int, hi: int):
        """Re-simulate patients [lo, hi) of this shard with the per-step trace
        (the 8 columns of simulation.py:61-64).  Same streams and arithmetic as
        ``simulate``, so every statistic of a traced patient is reproduced
        exactly.  Returns numpy (status [m], ticks [m], trace [m, H, 8])."""
        t = engine.torch()
        sub = FastTrial(self.pid0 + lo, self.params[lo:hi].contiguous(), self.basal[lo:hi].contiguous(),
                        self.generator, self.profile, self.config, self.controller_id, self.device,
                        hypo_min_s=self.hypo_min_ticks * self.config.dt_s, seed=self.seed,
                        noise_agg=self.noise_agg, fp32=self.fp32)
        tr = engine.empty((sub.n, self.sz["horizon_ticks"], 8), t.float64, self.device)
        engine.launch_fast(sub._inputs, sub.outs, sub.sz, self.config.dt_s, self.config.controller_period_s,
                           sub.seed, rng.ROLE_DEVICE_NOISE, sub.hypo_min_ticks, self.device,
                           meal_spec=sub.meal_spec, csr=sub.csr, controller_code=sub.code, fixed=sub.fixed,
                           noise_agg=sub.noise_agg, fp32=sub.fp32, trace=tr)
        return sub.outs.status.cpu().numpy(), sub.outs.ticks.cpu().numpy(), tr.cpu().numpy()

    def worst_trace(self, acc: TrialAccumulator):
        """Trace of the accumulator's worst case (simulation.py:619-624), or None."""
        if acc.worst is None:
            return None
        i = acc.worst.patient_id - self.pid0
        if not 0 <= i < self.n:
            return None
        _st, ticks, tr = self.trace_range(i, i + 1)
        return tr[0, : int(ticks[0])]

    def reduce(self):
        with engine.nvtx("gt.reduction"):
            self._reduce()

    def _reduce(self):
        engine.launch_reduce(self.outs, self.red, self.sz, self.config.dt_s, self.device)

    def step(self):
        """One full pass: simulate + (exclusion re-run if needed) + reduce."""
        self.simulate()
        self._rerun_if_diverged()
        self.reduce()

    def _rerun_if_diverged(self, injected=None):
        """Device-side: warps that hold a diverged patient re-simulate with it
        masked (deterministic streams); all other warps exit at once.  Then
        the abort-tick pass runs the diverged lanes alone with the reference's
        per-tick state and per-step BG checks, so their ``ticks`` is the
        reference's abort tick (simulation.py:381) rather than the horizon
        (the throughput launch detects divergence at the horizon only).  No
        host synchronisation; both passes exit at once when nothing diverged."""
        self.simulate(injected=injected, rerun_diverged=1)
        self.simulate(injected=injected, rerun_diverged=2)

    # ----------------------------------------------------------- readback
    def _fetch(self, *xs):
        """D2H of several device tensors: pinned, stream-ordered copies and one
        synchronisation (instead of one per tensor)."""
        t = engine.torch()
        hosts = []
        for x in xs:
            if x.device.type == "cpu":
                hosts.append(x)
                continue
            h = t.empty(x.shape, dtype=x.dtype, pin_memory=True)
            h.copy_(x, non_blocking=True)
            hosts.append(h)
        if any(x.device.type != "cpu" for x in xs):
            t.cuda.current_stream(self.device).synchronize()
        return [h.numpy() for h in hosts]

    def _ss_status_or_ok(self):
        if self.ss_status is not None:
            return self.ss_status
        return engine.torch().zeros((self.n,), dtype=engine.torch().int32)   # host: every patient has one

    def accumulator(self) -> TrialAccumulator:
        cfg, sz, red = self.config, self.sz, self.red
        acc = TrialAccumulator(dt_s=cfg.dt_s, horizon_ticks=sz["horizon_ticks"], n_days=sz["n_days"],
                               n_grid=sz["n_grid"], grid_step_s=cfg.grid_step_s)
        (counts, status, ss, tir_total, tir_hist, bg_total, below_min, below_max, mm, tl, dh, dsum, mhist,
         w) = self._fetch(red.counts, self.outs.status, self._ss_status_or_ok(), red.tir_ticks_total, red.tir_hist,
                          red.bg_hist_total, red.below_min, red.below_max, red.minmax_bg_bits, red.timeline,
                          red.dose_hist, red.dose_sum_fp, red.metric_hist, red.worst)
        acc.n_patients = int(counts[0])
        aborted = np.nonzero((status == GT_STATUS_NONFINITE) | (status == GT_STATUS_BAD_INITIAL_STATE)
                             | (ss == GT_STATUS_NO_STEADY_STATE))[0]
        acc.n_aborted = int(aborted.size)
        acc.aborted_ids = tuple(int(self.pid0 + i) for i in aborted)
        acc.sum_bg_fp = (int(counts[4]) << 64) + (int(counts[2]) & 0xFFFFFFFFFFFFFFFF)
        acc.n_patient_days = int(counts[3])
        acc.tir_ticks_total = tir_total.astype(np.int64)
        acc.tir_hist = tir_hist.astype(np.int64)
        acc.bg_hist_total = bg_total.astype(np.int64)
        acc.below_min = below_min.astype(np.int64)
        acc.below_max = below_max.astype(np.int64)
        acc.min_bg = engine.ordered_bits_to_double(mm[0]) if acc.n_patients else np.inf
        acc.max_bg = engine.ordered_bits_to_double(mm[1]) if acc.n_patients else -np.inf
        acc.timeline_sum_fp, acc.timeline_min_fp, acc.timeline_max_fp = (tl[0].copy(), tl[1].copy(), tl[2].copy())
        acc.dose_hist = {s: dh[k].astype(np.int64) for k, s in enumerate(DOSE_SIGNALS)}
        acc.dose_sum_fp = [(int(dsum[3 + k]) << 64) + (int(dsum[k]) & 0xFFFFFFFFFFFFFFFF) for k in range(3)]
        acc.metric_hist = mhist.astype(np.int64)
        if int(w[3]):
            i = int(w[2]) - self.pid0
            hist, wmax, wticks = self._fetch(self.outs.bg_hist[:, i].contiguous(), self.outs.bg_stats[1, i:i + 1],
                                             self.outs.ticks[i:i + 1])
            hist = hist.astype(np.int64)
            cum = np.cumsum(hist)
            tir = np.array([cum[25], cum[34] - cum[25], cum[95] - cum[34], cum[134] - cum[95],
                            cum[-1] - cum[134]], dtype=np.int64)
            acc.worst = WorstCase(patient_id=int(w[2]), min_bg=engine.ordered_bits_to_double(w[0]),
                                  max_bg=float(wmax[0]), ticks_below_3=int(w[1]),
                                  ticks=int(wticks[0]), tir_ticks=tir, bg_hist=hist)
        return acc

    def metrics_device(self) -> dict | None:
        """Per-patient metric arrays as device tensors (shard order): the five
        range fractions, the two hypo-event counts and the status."""
        if self.red.metrics is None:
            return None
        out = dict(self.red.metrics)
        out["hypo_events_lt70"], out["hypo_events_lt54"] = self.outs.hypo_events[0], self.outs.hypo_events[1]
        out["status"] = self.outs.status
        return out

    def metrics(self) -> dict | None:
        if self.red.metrics is None:
            return None
        keys = list(self.red.metrics)
        vals = self._fetch(*[self.red.metrics[k] for k in keys], self.outs.hypo_events[0], self.outs.hypo_events[1],
                           self.outs.status)
        out = dict(zip(keys, vals[:len(keys)]))
        out["hypo_events_lt70"], out["hypo_events_lt54"], out["status"] = vals[len(keys):]
        return out


def run_trial_fast(population, generator, controller_id, profile, model_id, config, *,
                   basal_scale=1.0, run_meta=None, progress=None, device=None,
                   hypo_min_s=900.0, per_patient_metrics=True, trace_dir=None):
    """Fused-path ``run_trial`` (simulation.py:551-628 semantics): one staged
    shard, device reduction, report; ``store_trace`` policies by traced
    re-simulation (same streams, so the worst case's statistics are exact)."""
    import os
    from .simulation import TrialResult, _meta, save_trace
    t0 = time.perf_counter()
    device = engine.require_device(device)
    pid0, params, basal = population_to_device(population, basal_scale, device)
    ft = FastTrial(pid0, params, basal, generator, profile, config, controller_id, device,
                   hypo_min_s=hypo_min_s, per_patient_metrics=per_patient_metrics)
    ft.step()
    acc = ft.accumulator()
    wall_s = time.perf_counter() - t0
    if progress:
        progress(ft.n, ft.n)
    if acc.n_patients == 0:
        raise SimulationError("all simulations diverged; nothing to report")
    meta = _meta(config, ft.n, model_id, controller_id, profile, basal_scale, generator, run_meta)
    report = analytics.build_trial_report(acc, meta)
    worst_trace = None
    if config.store_trace in ("worst_case_only", "always"):
        worst_trace = ft.worst_trace(acc)
    if config.store_trace == "always" and trace_dir is not None:
        os.makedirs(trace_dir, exist_ok=True)
        chunk = max(1, int(2**31 // (ft.sz["horizon_ticks"] * 64)))   # <= 2 GiB of trace per launch
        for lo in range(0, ft.n, chunk):
            hi = min(ft.n, lo + chunk)
            st, ticks, tr = ft.trace_range(lo, hi)
            for j in range(hi - lo):
                if int(st[j]) == GT_STATUS_OK:
                    save_trace(os.path.join(trace_dir, f"patient_{pid0 + lo + j:06d}.npz"), tr[j, : int(ticks[j])])
    return TrialResult(report=report, accumulator=acc, worst_trace=worst_trace, wall_s=wall_s,
                       n_patients=ft.n, metrics=ft.metrics())


def run_population_arrays(params_host, basal_host, generator, profile, config, *, pid0=0,
                          controller_id="dual_hormone", device=None, hypo_min_s=900.0):
    """Public array API of the fused path (host buffers in, host results out):
    H2D of the per-patient parameter rows and basal rates, steady state,
    controller set-up, fused simulation, device reduction, D2H of the exact
    accumulator fields and the per-patient metric arrays.
    Returns ``(TrialAccumulator, metrics dict)``."""
    t = engine.torch()
    device = engine.require_device(device)
    p = params_host if hasattr(params_host, "data_ptr") else t.from_numpy(np.ascontiguousarray(params_host))
    b = basal_host if hasattr(basal_host, "data_ptr") else t.from_numpy(np.ascontiguousarray(basal_host))
    p_d = p.to(device, non_blocking=True)
    b_d = b.to(device, non_blocking=True)
    ft = FastTrial(pid0, p_d, b_d, generator, profile, config, controller_id, device,
                   hypo_min_s=hypo_min_s, per_patient_metrics=True)
    ft.step()
    return ft.accumulator(), ft.metrics()


def fast_bytes_per_patient(config) -> int:
    """Device bytes one patient occupies in a FastTrial (outputs, inputs,
    scratch; the NorthernYear CSR adds ~47 KB per patient on top)."""
    sz = sizes(config)
    return int(8 * (30 + 16 + 11 + 4) + 4 * 247 + 8 * 3 + 8 * 3 * sz["n_days"] + 4 * 2 + 8 + 4
               + 24 * sz["n_grid"] / 32 + 404 + 4 * 5 + 64)


def run_population_chunked(n: int, population_seed: int, generator, profile, config, *, pid0: int = 0,
                           controller_id: str = "dual_hormone", device=None, chunk: int | None = None,
                           hypo_min_s: float = 900.0, memory_fraction: float = 0.5) -> TrialAccumulator:
    """Simulate global ids [pid0, pid0 + n) on one device in chunks sized to fit
    ``memory_fraction`` of its free memory (or ``chunk`` patients), sampling
    each chunk on the device and merging the exact accumulators.  Results
    equal a single launch over all ids (pid-keyed streams, exact merge)."""
    from .analytics import merge
    from .population import generate_population
    t = engine.torch()
    device = engine.require_device(device)
    if chunk is None:
        free, _total = t.cuda.mem_get_info(device)
        chunk = max(1024, int(free * memory_fraction / fast_bytes_per_patient(config)))
    acc = None
    for lo in range(pid0, pid0 + n, chunk):
        m = min(chunk, pid0 + n - lo)
        pop = generate_population(population_seed, m, pid0=lo, device=device, on_exhausted="redraw_weight")
        ft = FastTrial(lo, pop.params_device, pop.basal_device, generator, profile, config, controller_id, device,
                       hypo_min_s=hypo_min_s)
        ft.step()
        part = ft.accumulator()
        acc = part if acc is None else merge(acc, part)
        del ft, pop
    return acc
