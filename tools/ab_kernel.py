"""A/B timing of the fused kernel alone (CUDA events on the launch stream,
median of reps after a warm-up) for prebuilt library variants.

    GLUCOSIM_LIB=build_vX/libglucosim.so python tools/ab_kernel.py [label]

Prints one JSON line per workload: BASELINE configs[1] shape (100k x 4 w,
dt 60 s) with pid_pump / dual_hormone on the 3-meal generator, and pid_pump
/ dual_hormone on the device-planned NorthernYear protocol."""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import numpy as np
    import torch
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.northern import NorthernYearProtocol
    from paper_2202_13927_b200.pid import PIDProfile
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial
    label = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("GLUCOSIM_LIB", "default")
    only = set(sys.argv[2].split(",")) if len(sys.argv) > 2 else None
    dev = torch.device("cuda", 0)
    n, weeks = 100_000, 4
    cfg = SimulationConfig(horizon_s=weeks * 7 * 86400.0, seed=1, dt_s=60.0)
    pop = generate_population(1, n, device=dev, on_exhausted="redraw_weight")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for proto in ("three_meal", "northern"):
        for ctrl in ("pid_pump", "dual_hormone"):
            name = f"{proto}/{ctrl}"
            if only and name not in only:
                continue
            gen = NorthernYearProtocol() if proto == "northern" else ThreeMealProtocol()
            prof = PIDProfile() if ctrl == "pid_pump" else ControllerHyperparameters()
            ft = FastTrial(0, pop.params_device, pop.basal_device, gen, prof, cfg, controller_id=ctrl, device=dev)
            for _ in range(2):
                ft.simulate()
            ms = []
            st = torch.cuda.current_stream(dev)
            for _ in range(7):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                ft.simulate()
                e1.record(st)
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            print(json.dumps({"variant": label, "workload": name, "ms_median": float(np.median(ms)),
                              "ms_min": float(np.min(ms)), "pw_per_s": n * weeks / (np.median(ms) / 1e3)}),
                  flush=True)
            del ft


if __name__ == "__main__":
    main()
