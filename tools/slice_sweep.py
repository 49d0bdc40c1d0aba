"""Fused-kernel time vs the persistent schedule's slice count (CUDA events,
median of 5 after an L2 flush), BASELINE configs[1] shape.
    python tools/slice_sweep.py [controller] [protocol] [slices,...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


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
    ctrl = sys.argv[1] if len(sys.argv) > 1 else "pid_pump"
    proto = sys.argv[2] if len(sys.argv) > 2 else "three_meal"
    slices = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "0,1,4,9,13,19,25,33,45,60").split(",")]
    dev = torch.device("cuda", 0)
    n, weeks = 100_000, 4
    cfg = SimulationConfig(horizon_s=weeks * 7 * 86400.0, seed=1, dt_s=60.0)
    pop = generate_population(1, n, device=dev, on_exhausted="redraw_weight")
    gen = NorthernYearProtocol() if proto == "northern" else ThreeMealProtocol()
    prof = PIDProfile() if ctrl == "pid_pump" else ControllerHyperparameters()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for s in slices:
        ft = FastTrial(0, pop.params_device, pop.basal_device, gen, prof, cfg, controller_id=ctrl, device=dev,
                       n_slices=s)
        ft.simulate()
        ms = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ft.simulate()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        print(json.dumps({"controller": ctrl, "protocol": proto, "n_slices": s, "ms_median": float(np.median(ms))}),
              flush=True)
        del ft


if __name__ == "__main__":
    main()
