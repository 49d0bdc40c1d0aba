"""Profiling driver: stage a FastTrial and run simulate+reduce a few times.

    python tools/prof_fast.py [n_patients] [weeks] [reps] [three_meal|northern] [dual_hormone|pid_pump] [dt_s] [n_slices]
"""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

from paper_2202_13927_b200.config import SimulationConfig  # noqa: E402
from paper_2202_13927_b200.controller import ControllerHyperparameters  # noqa: E402
from paper_2202_13927_b200.population import generate_population  # noqa: E402
from paper_2202_13927_b200.protocol import ThreeMealProtocol  # noqa: E402
from paper_2202_13927_b200.trial import FastTrial  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
weeks = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
proto = sys.argv[4] if len(sys.argv) > 4 else "three_meal"
ctrl = sys.argv[5] if len(sys.argv) > 5 else "dual_hormone"
dt_s = float(sys.argv[6]) if len(sys.argv) > 6 else 60.0
n_slices = int(sys.argv[7]) if len(sys.argv) > 7 else 0
dev = torch.device("cuda", 0)
cfg = SimulationConfig(horizon_s=weeks * 7 * 86400.0, seed=1, dt_s=dt_s)
pop = generate_population(1, n, device=dev, on_exhausted="redraw_weight")
if proto == "northern":
    from paper_2202_13927_b200.northern import NorthernYearProtocol
    gen = NorthernYearProtocol()
else:
    gen = ThreeMealProtocol()
if ctrl == "pid_pump":
    from paper_2202_13927_b200.pid import PIDProfile
    prof = PIDProfile()
else:
    prof = ControllerHyperparameters()
ft = FastTrial(0, pop.params_device, pop.basal_device, gen, prof, cfg, controller_id=ctrl, device=dev,
               n_slices=n_slices)
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ft.step()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    from paper_2202_13927_b200 import flops
    tf = flops.flops_per_step(ft.sz["period_steps"], ctrl) * n * ft.sz["horizon_ticks"] / dt / 1e12
    print(f"rep {r}: {dt * 1000:.2f} ms  {n * weeks / dt:.4g} patient-weeks/s  {tf:.2f} TFLOP/s (wall, incl. reduce)",
          flush=True)
