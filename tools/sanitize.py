"""Small closed-loop runs for compute-sanitizer (memcheck / racecheck /
synccheck): the sliced persistent schedule at n = 33 (one full warp plus a
one-lane warp with 31 padding lanes, 4 slices, a diverged patient so the
exclusion re-run executes), the device reduction, the sampler's warp queue
and the NorthernYear planner.

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.northern import NorthernYearProtocol
    from paper_2202_13927_b200.pid import PIDProfile
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial
    dev = torch.device("cuda", 0)
    cfg = SimulationConfig(horizon_s=86400.0, seed=1, dt_s=60.0)
    pop = generate_population(3, 33, device=dev, on_exhausted="redraw_weight")
    params = pop.params_device.clone()
    params[5, 4] = -5.0      # ka1 < 0: this patient diverges -> exclusion re-run
    for gen, prof, ctl in ((ThreeMealProtocol(), PIDProfile(), "pid_pump"),
                           (ThreeMealProtocol(), ControllerHyperparameters(), "dual_hormone"),
                           (NorthernYearProtocol(), ControllerHyperparameters(), "dual_hormone")):
        ft = FastTrial(0, params, pop.basal_device, gen, prof, cfg, controller_id=ctl, device=dev,
                       per_patient_metrics=True, n_slices=4)
        ft.step()
        acc = ft.accumulator()
        torch.cuda.synchronize()
        print(ctl, type(gen).__name__, "n_patients", acc.n_patients, "aborted", acc.aborted_ids, flush=True)
    print("done", flush=True)


if __name__ == "__main__":
    main()
