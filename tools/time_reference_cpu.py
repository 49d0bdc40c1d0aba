"""The reference's OWN CPU path timed on this host: the
unmodified glucotrial package installed in baseline/_ref (pip --target, see
DESIGN.md §6), run_trial(..., workers=os.cpu_count()) on its numba fast
engine (hovorka_ext + dual_hormone, simulation.py:301-311) after
_warmup_fast_path() (simulation.py:534-548), next to the oracle's C port
(oracle/gt_oracle_batch.c, the bench's --impl reference arm) on the same
patients with the same thread count.

Workload: BASELINE configs[1] shape per patient -- 4 weeks at dt 60 s, 300 s
controller period, seed 1, the BASELINE 3-meal generator (the product's
ThreeMealProtocol plug-in through the reference's generator contract) -- on a
fixed sample of patients whose parameter sets are the reference sampler's
own seed-7 draw (tests/golden/population_s7_n4000.npz, tiled).  Prints one
JSON line.

    python tools/time_reference_cpu.py [n_patients] [weeks]
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")


class _P:
    def __init__(self, pid, w):
        self.id, self.body_weight_kg = pid, w


def main():
    if not os.path.isdir(os.path.join(REF, "glucotrial")):
        print(json.dumps({"unavailable": f"reference not installed in {REF}"}))
        return 0
    sys.path.insert(0, REF)
    sys.path.insert(1, REPO)
    sys.path.insert(2, os.path.join(REPO, "oracle"))
    import psutil
    from glucotrial import hovorka
    from glucotrial.controller import DualHormoneController, load_profile
    from glucotrial.population import ParameterSet, load_parameter_table
    from glucotrial.simulation import SimulationConfig, _warmup_fast_path, run_trial
    from paper_2202_13927_b200.protocol import ThreeMealProtocol

    cores = os.cpu_count() or 1
    phys = psutil.cpu_count(logical=False)
    weeks = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    n = int(sys.argv[1]) if len(sys.argv) > 1 else min(200_000, 48 * cores)
    g = np.load(os.path.join(REPO, "tests", "golden", "population_s7_n4000.npz"))
    table = load_parameter_table()
    names = [str(s) for s in g["names"]]
    entries = []
    for i in range(n):
        j = i % g["weights"].size
        values = {"weight_kg": float(g["weights"][j])}
        values.update({k: float(v) for k, v in zip(names, g["sampled"][j])})
        values.update(table.fixed)
        entries.append((_P(i, float(g["weights"][j])), ParameterSet(values=values,
                                                                    u_basal_u_per_h=float(g["ubasal"][j]))))
    cfg = SimulationConfig(horizon_s=weeks * 7 * 86400.0, seed=1, dt_s=60.0)
    prof = load_profile()
    gen = ThreeMealProtocol()
    t0 = time.perf_counter()
    _warmup_fast_path()
    warm = time.perf_counter() - t0
    res = run_trial(entries, gen, "dual_hormone", prof, "hovorka_ext", cfg, workers=cores)
    ref_pw = n * weeks / res.wall_s

    # the oracle's C port (OpenMP, all host threads) on the same patients,
    # same controller and 3-meal schedules; its noise is the device layout
    # (Philox4x32-7 + Box-Muller) instead of numpy's ziggurat draws
    import oracle
    from paper_2202_13927_b200.config import sizes
    params = np.stack([hovorka.pack_params(ps.values) for _, ps in entries])
    ub = np.array([ps.u_basal_u_per_h for _, ps in entries])
    x0 = np.zeros((n, 16))
    for i in range(min(n, 4000)):
        x0[i], _ = oracle.steady_state(params[i])
    x0 = np.ascontiguousarray(np.resize(x0[:min(n, 4000)], (n, 16)))
    c0 = np.stack([DualHormoneController(prof, u).initial_state().to_vec() for u in ub])
    oracle.set_controller(0)
    t0 = time.perf_counter()
    out = oracle.run_batch_philox(gen, cfg.seed, 0, params, x0, c0, prof.to_vec(), ub, sizes(cfg), cfg.dt_s,
                                  cfg.controller_period_s, nthreads=cores)
    port_s = time.perf_counter() - t0
    port_pw = n * weeks / port_s
    print(json.dumps({
        "what": "reference run_trial (numba fast engine, dual_hormone, 3-meal plug-in) vs the oracle C port",
        "n_patients": n, "weeks": weeks, "dt_s": 60.0, "cores_logical": cores, "cores_physical": phys,
        "cpu_model": _cpu_model(),
        "reference": {"patient_weeks_per_s": ref_pw, "wall_s": res.wall_s, "warmup_s": warm,
                      "workers": cores, "n_ok": res.accumulator.n_patients,
                      "path": "baseline/_ref glucotrial.simulation.run_trial(workers=os.cpu_count())"},
        "port": {"patient_weeks_per_s": port_pw, "wall_s": port_s, "threads": cores,
                 "n_ok": int((out["status"] == 0).sum()), "path": "oracle.run_batch_philox (C, OpenMP)"},
        "port_over_reference": port_pw / ref_pw}))
    return 0


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


if __name__ == "__main__":
    sys.exit(main())
