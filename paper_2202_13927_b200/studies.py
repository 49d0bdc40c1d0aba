"""Population studies on the fused path (BASELINE configs[3] and configs[4]).

``treatment_comparison``: several controller profiles run on ONE shared
population with common random numbers.  Every stream is keyed by
(seed, patient id, role) only (rng.py:1-10 in the reference; the device
Philox counters here), so each arm sees the same meals, process noise and
sensor noise.  The output holds each arm's population report quantiles and
the paired per-patient differences against a reference arm.

``precision_study``: one population run as FP64 at dt, FP64 at dt/agg, and
FP32 at dt on the same Philox path.  The dt run draws each step's Brownian
increment as the sum of the agg fine increments.  The output holds each
variant's throughput and the deviation of its metrics from the FP64 runs.

Both run on one device.  For N devices, shard the population with
``parallel.shard_range`` and merge the accumulators with
``parallel.allreduce_accumulator``; the paired differences are per patient
and need no exchange.
"""

from __future__ import annotations

import numpy as np

from . import analytics, engine
from .config import SimulationConfig
from .controller import ControllerHyperparameters
from .protocol import ThreeMealProtocol

METRICS = ("tir", "tbr70", "tbr54", "tar180", "tar250", "hypo_events_lt70", "hypo_events_lt54")
Q = (0.05, 0.25, 0.5, 0.75, 0.95)


def default_arms(base=None, controller_id: str = "dual_hormone") -> dict:
    """BASELINE configs[3] arms: gains x0.5 / x1 / x1.5 and bolus-only.

    * ``pid_pump`` (pid.py, the BASELINE's PID): kp, ki, kd scaled together;
      bolus-only = all three 0, i.e. the pump-quantised assumed basal plus
      meal boluses.
    * ``dual_hormone`` (the reference's controller): its basal law is a PD on
      the filtered CGM (controller.py:449-457), so the gains are basal_kp and
      basal_kd; bolus-only sets both to 0."""
    if controller_id == "pid_pump":
        from .pid import PIDProfile
        base = base or PIDProfile()
        return {"pid_x0.5": base.scaled(0.5), "pid_x1": base, "pid_x1.5": base.scaled(1.5),
                "bolus_only": base.scaled(0.0)}
    base = base or ControllerHyperparameters()
    return {"pd_x0.5": base.scaled(0.5, 0.5), "pd_x1": base, "pd_x1.5": base.scaled(1.5, 1.5),
            "bolus_only": base.scaled(0.0, 0.0)}


def _timed_step(ft):
    """One trial pass (simulate + exclusion re-run + reduce), device-timed."""
    t = engine.torch()
    st = t.cuda.current_stream(ft.device)
    ev = [t.cuda.Event(enable_timing=True) for _ in range(3)]
    t.cuda.synchronize(ft.device)
    ev[0].record(st)
    ft.simulate()
    ev[1].record(st)
    ft._rerun_if_diverged()
    ft.reduce()
    ev[2].record(st)
    t.cuda.synchronize(ft.device)
    return ev[0].elapsed_time(ev[1]), ev[0].elapsed_time(ev[2])


def _trial(pop, profile, cfg, device, generator=None, controller_id="dual_hormone", **kw):
    from .trial import FastTrial
    return FastTrial(pop.pid0, pop.params_device, pop.basal_device, generator or ThreeMealProtocol(),
                     profile, cfg, controller_id=controller_id, device=device, per_patient_metrics=True, **kw)


def _per_patient(ft) -> dict:
    m = ft.metrics()
    out = {k: m[k].astype(np.float64) for k in METRICS}
    out["ok"] = m["status"] == 0
    out["mean_bg"] = ft.outs.bg_stats[2].cpu().numpy() / np.maximum(ft.outs.ticks.cpu().numpy(), 1)
    return out


def _dist(x: np.ndarray) -> dict:
    if x.size == 0:
        return {"n": 0}
    return {"n": int(x.size), "mean": float(x.mean()), "sd": float(x.std(ddof=1)) if x.size > 1 else 0.0,
            "se": float(x.std(ddof=1) / np.sqrt(x.size)) if x.size > 1 else 0.0,
            **{f"p{int(round(100 * q))}": float(np.quantile(x, q)) for q in Q}}


def treatment_comparison(n: int, weeks: int, seed: int, device=None, arms: dict | None = None,
                         reference_arm: str | None = None, dt_s: float = 60.0, pid0: int = 0,
                         population_seed: int | None = None, generator=None,
                         controller_id: str = "dual_hormone") -> dict:
    """BASELINE configs[3]: ``arms`` (name -> profile) x one shared population
    under common random numbers.  Returns per-arm report quantiles, per-arm
    per-patient metric distributions, and paired differences (arm minus
    ``reference_arm``) over the patients that finished in both arms."""
    from .population import generate_population
    device = engine.require_device(device)
    arms = arms or default_arms(controller_id=controller_id)
    if reference_arm is None:
        reference_arm = "pid_x1" if controller_id == "pid_pump" else "pd_x1"
    if reference_arm not in arms:
        raise ValueError(f"reference arm {reference_arm!r} is not among {sorted(arms)}")
    cfg = SimulationConfig(horizon_s=weeks * 7 * 86400.0, seed=seed, dt_s=dt_s)
    pop = generate_population(seed if population_seed is None else population_seed, n, pid0=pid0,
                              device=device, on_exhausted="redraw_weight")
    per, out = {}, {"config": {"patients": n, "weeks": weeks, "seed": seed, "dt_s": dt_s,
                               "controller": controller_id,
                               "crn": "streams keyed by (seed, patient id, role)"}, "arms": {}}
    for name, prof in arms.items():
        ft = _trial(pop, prof, cfg, device, generator, controller_id)
        sim_ms, step_ms = _timed_step(ft)
        acc = ft.accumulator()
        per[name] = _per_patient(ft)
        out["arms"][name] = {
            "gains": ({"kp": prof.kp, "ki": prof.ki, "kd": prof.kd} if controller_id == "pid_pump"
                      else {"basal_kp": prof.basal_kp, "basal_kd": prof.basal_kd}),
            "n_patients": acc.n_patients,
            "n_aborted": acc.n_aborted, "sim_ms": sim_ms, "step_ms": step_ms,
            "patient_weeks_per_s": n * weeks / (step_ms / 1000.0),
            "quantiles": analytics.metric_quantiles(acc),
            "per_patient": {k: _dist(per[name][k][per[name]["ok"]]) for k in METRICS + ("mean_bg",)},
        }
        del ft
    ref = per[reference_arm]
    out["paired_differences"] = {}
    for name in arms:
        if name == reference_arm:
            continue
        ok = per[name]["ok"] & ref["ok"]
        out["paired_differences"][f"{name} - {reference_arm}"] = {
            k: _dist(per[name][k][ok] - ref[k][ok]) for k in METRICS + ("mean_bg",)}
    return out


def precision_study(n: int, weeks: int, seed: int, device=None, agg: int = 10, dt_s: float = 60.0,
                    pid0: int = 0, profile=None, generator=None, controller_id: str = "dual_hormone") -> dict:
    """BASELINE configs[4]: FP64 at dt, FP64 at dt/agg, FP32 at dt on one
    population.  Variants:

    * ``fp64_dt`` / ``fp32_dt`` run on the production streams (one Philox
      draw per step), so FP32 is compared pathwise with FP64;
    * ``fp64_dt_agg`` and ``fp64_fine`` share one Brownian path: the fine run
      draws at dt/agg and the coarse run sums agg fine increments per step.
      Their difference is the time-discretisation error alone.

    Returns each variant's throughput and the per-patient metric deviations."""
    from .population import generate_population
    device = engine.require_device(device)
    if profile is None:
        if controller_id == "pid_pump":
            from .pid import PIDProfile
            profile = PIDProfile()
        else:
            profile = ControllerHyperparameters()
    pop = generate_population(seed, n, pid0=pid0, device=device, on_exhausted="redraw_weight")
    fine = dt_s / agg
    variants = {
        "fp64_dt": (dt_s, 1, False), "fp32_dt": (dt_s, 1, True),
        "fp64_dt_agg": (dt_s, agg, False), "fp32_dt_agg": (dt_s, agg, True), "fp64_fine": (fine, 1, False),
    }
    per, out = {}, {"config": {"patients": n, "weeks": weeks, "seed": seed, "dt_s": dt_s, "agg": agg,
                               "fine_dt_s": fine}, "variants": {}}
    for name, (dt, a, fp32) in variants.items():
        cfg = SimulationConfig(horizon_s=weeks * 7 * 86400.0, seed=seed, dt_s=dt)
        ft = _trial(pop, profile, cfg, device, generator, controller_id, noise_agg=a, fp32=fp32)
        _timed_step(ft)                       # warm-up (module load, allocator)
        sim_ms, step_ms = _timed_step(ft)
        acc = ft.accumulator()
        per[name] = _per_patient(ft)
        out["variants"][name] = {
            "dt_s": dt, "noise_agg": a, "integrator": "fp32" if fp32 else "fp64",
            "n_patients": acc.n_patients, "n_aborted": acc.n_aborted, "sim_ms": sim_ms, "step_ms": step_ms,
            "patient_weeks_per_s": n * weeks / (step_ms / 1000.0),
            "quantiles": analytics.metric_quantiles(acc),
        }
        del ft

    def dev(a, b):
        ok = per[a]["ok"] & per[b]["ok"]
        d = {k: _dist(np.abs(per[a][k][ok] - per[b][k][ok])) for k in METRICS}
        rel = np.abs(per[a]["mean_bg"][ok] - per[b]["mean_bg"][ok]) / per[b]["mean_bg"][ok]
        d["mean_bg_rel"] = _dist(rel)
        d["population_mean_shift"] = {k: float(per[a][k][ok].mean() - per[b][k][ok].mean()) for k in METRICS}
        return d

    out["deviation"] = {
        "fp32_dt vs fp64_dt (same streams)": dev("fp32_dt", "fp64_dt"),
        "fp32_dt_agg vs fp64_dt_agg (same streams)": dev("fp32_dt_agg", "fp64_dt_agg"),
        "fp64_dt_agg vs fp64_fine (same Brownian path)": dev("fp64_dt_agg", "fp64_fine"),
        "fp32_dt_agg vs fp64_fine (same Brownian path)": dev("fp32_dt_agg", "fp64_fine"),
    }
    return out
