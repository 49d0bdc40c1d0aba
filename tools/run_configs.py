"""Run BASELINE.json configs[0..4] on one GPU and write one JSON summary.

  C0  1 000 x 7 d, seed 0 (the reference's CPU-runnable case; bench.py times
      the CPU path).
  C1  the first 1 000 patients of seed 1 x 4 weeks (the bitwise parity check on
      this subset is tests/test_gpu_parity.py::test_c1_parity_subset_...).
  C2  1 000 000 x 52 w, seed 2, on one GPU: device sampler, fused
      integrator, device reduction, histograms and 5/25/50/75/95 %
      quantiles.  On N GPUs each rank runs 1/N of the ids
      (bench.py --workload trial1m --gpus N spawns the N ranks).
  C3  4 controller arms x 250 000 shared patients x 12 w under common random
      numbers; paired differences (studies.treatment_comparison).
  C4  precision / step study, 250 000 x 12 w (studies.precision_study).

usage: python tools/run_configs.py [--only C0,C2] [--out gpurun_out/configs.json] [--scale 1.0]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


CTRL = "pid_pump"   # BASELINE's controller; --controller dual_hormone for the reference's


def _prof():
    """(profile, device code) of the configured controller."""
    if CTRL == "pid_pump":
        from paper_2202_13927_b200.pid import PIDProfile
        return PIDProfile(), 1
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    return ControllerHyperparameters(), 0


def _sync():
    import torch
    torch.cuda.synchronize()


def c0(dev, scale):
    """BASELINE configs[0] on the GPU (its CPU timing is bench.py's cpu_baseline leg)."""
    from paper_2202_13927_b200 import analytics, flops
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.studies import _timed_step, _trial
    n, days = max(32, int(1000 * scale)), 7
    cfg = SimulationConfig(horizon_s=days * 86400.0, seed=0, dt_s=60.0)
    (prof, _code), gen = _prof(), ThreeMealProtocol()
    t0 = time.perf_counter()
    pop = generate_population(0, n, device=dev, on_exhausted="redraw_weight")
    _sync()
    sampler_s = time.perf_counter() - t0
    ft = _trial(pop, prof, cfg, dev, controller_id=CTRL)
    _timed_step(ft)
    sim_ms, step_ms = _timed_step(ft)
    acc = ft.accumulator()
    pw = n * days / 7.0
    return {"patients": n, "days": days, "sampler_s": sampler_s, "sim_ms": sim_ms, "step_ms": step_ms,
            "gpu_patient_weeks_per_s": pw / (step_ms / 1000.0),
            "flops_per_step": flops.flops_per_step(ft.sz["period_steps"], CTRL),
            "quantiles": analytics.metric_quantiles(acc)}


def c1(dev, scale):
    """BASELINE configs[1] correctness subset: the bitwise oracle comparison at
    the full 1 000 x 4 weeks is tests/test_gpu_parity.py::test_c1_parity_subset_...;
    here the fused kernel (device Philox) is timed on the same subset."""
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.studies import _timed_step, _trial
    n, weeks = max(32, int(1000 * scale)), 4
    cfg = SimulationConfig(horizon_s=weeks * 7 * 86400.0, seed=1, dt_s=60.0)
    pop = generate_population(1, n, device=dev, on_exhausted="redraw_weight")
    ft = _trial(pop, _prof()[0], cfg, dev, ThreeMealProtocol(), controller_id=CTRL)
    _timed_step(ft)
    sim_ms, step_ms = _timed_step(ft)
    return {"patients": n, "weeks": weeks, "sim_ms": sim_ms, "step_ms": step_ms,
            "parity_check": "tests/test_gpu_parity.py::test_c1_parity_subset_1000_patients_4_weeks"}


def c2(dev, scale):
    import torch
    from paper_2202_13927_b200 import analytics
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.studies import _timed_step, _trial
    n, weeks = int(1_000_000 * scale), 52
    cfg = SimulationConfig(horizon_s=weeks * 7 * 86400.0, seed=2, dt_s=60.0)
    t0 = time.perf_counter()
    pop = generate_population(2, n, device=dev, on_exhausted="redraw_weight")
    _sync()
    sampler_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    ft = _trial(pop, _prof()[0], cfg, dev, controller_id=CTRL)
    _sync()
    setup_s = time.perf_counter() - t0
    sim_ms, step_ms = _timed_step(ft)
    t0 = time.perf_counter()
    acc = ft.accumulator()
    readback_s = time.perf_counter() - t0
    rep = analytics.build_trial_report(acc, {})
    return {"patients": n, "weeks": weeks, "sampler_s": sampler_s, "setup_s": setup_s, "sim_ms": sim_ms,
            "step_ms": step_ms, "readback_s": readback_s,
            "patient_weeks_per_s": n * weeks / (step_ms / 1000.0),
            "wall_s_total": sampler_s + setup_s + step_ms / 1000.0 + readback_s,
            "n_patients": acc.n_patients, "n_aborted": acc.n_aborted,
            "peak_mem_gb": torch.cuda.max_memory_allocated(dev) / 1e9,
            "quantiles": analytics.metric_quantiles(acc), "tir_report": rep.get("tir")}


def c2n(dev, scale):
    """C2 scale with the reference's own lifestyle protocol (NorthernYear,
    planned on the device) instead of the BASELINE 3-meal generator."""
    import torch
    from paper_2202_13927_b200 import analytics
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.northern import NorthernYearProtocol
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.studies import _timed_step, _trial
    n, weeks = int(1_000_000 * scale), 52
    cfg = SimulationConfig(horizon_s=weeks * 7 * 86400.0, seed=2, dt_s=60.0)
    pop = generate_population(2, n, device=dev, on_exhausted="redraw_weight")
    _sync()
    t0 = time.perf_counter()
    ft = _trial(pop, _prof()[0], cfg, dev, NorthernYearProtocol(), controller_id=CTRL)
    _sync()
    setup_s = time.perf_counter() - t0
    sim_ms, step_ms = _timed_step(ft)
    acc = ft.accumulator()
    return {"patients": n, "weeks": weeks, "protocol": "northern_year (device-planned)",
            "setup_s_incl_protocol_build": setup_s, "sim_ms": sim_ms, "step_ms": step_ms,
            "patient_weeks_per_s": n * weeks / (step_ms / 1000.0), "n_patients": acc.n_patients,
            "n_aborted": acc.n_aborted, "peak_mem_gb": torch.cuda.max_memory_allocated(dev) / 1e9,
            "quantiles": analytics.metric_quantiles(acc)}


def c3(dev, scale):
    from paper_2202_13927_b200.studies import treatment_comparison
    return treatment_comparison(max(1000, int(250_000 * scale)), 12, seed=3, device=dev, controller_id=CTRL)


def _peaks():
    """Measured DFMA / FFMA peaks (tools/fp64_peak.cu, profiles/fp64_peak_r01.jsonl)."""
    best = {"dfma": 0.0, "ffma": 0.0}
    for line in open(os.path.join(ROOT, "profiles", "fp64_peak_r01.jsonl")):
        d = json.loads(line)
        if d.get("kernel") in best:
            best[d["kernel"]] = max(best[d["kernel"]], d["tflops"])
    return best


def c4(dev, scale):
    from paper_2202_13927_b200 import flops
    from paper_2202_13927_b200.studies import precision_study
    n, weeks = max(1000, int(250_000 * scale)), 12
    out = precision_study(n, weeks, seed=4, device=dev, controller_id=CTRL)
    peaks = _peaks()
    for name, v in out["variants"].items():
        ps = int(round(300.0 / v["dt_s"]))
        steps = n * weeks * 7 * 86400.0 / v["dt_s"]
        tf = flops.flops_per_step(ps, CTRL) * steps / (v["sim_ms"] / 1000.0) / 1e12
        peak = peaks["ffma"] if v["integrator"] == "fp32" else peaks["dfma"]
        v["roofline"] = {"achieved_tflops": tf, "peak_tflops": peak, "frac": tf / peak,
                         "peak": "measured FFMA" if v["integrator"] == "fp32" else "measured DFMA",
                         "note": "algorithmic flops of the reference (flops.py); the FP32 variant keeps the "
                                 "controller and statistics in FP64"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C0,C1,C2,C2N,C3,C4")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "configs.json"))
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--controller", default="pid_pump", choices=["pid_pump", "dual_hormone"])
    args = ap.parse_args()
    global CTRL
    CTRL = args.controller
    import torch
    dev = torch.device("cuda", 0)
    from paper_2202_13927_b200 import _lib
    _lib.load()
    out = {"device": torch.cuda.get_device_name(dev), "scale": args.scale, "controller": CTRL}
    fns = {"C0": c0, "C1": c1, "C2": c2, "C2N": c2n, "C3": c3, "C4": c4}
    for name in args.only.split(","):
        t0 = time.perf_counter()
        out[name] = fns[name](dev, args.scale)
        out[name]["runner_wall_s"] = time.perf_counter() - t0
        print(name, "done", f"{out[name]['runner_wall_s']:.1f}s", flush=True)
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1, default=float)
    print(json.dumps({k: (v if not isinstance(v, dict) else "...") for k, v in out.items()}))


if __name__ == "__main__":
    main()
