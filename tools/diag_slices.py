"""Developer diagnostic: fused kernel with 1 vs k horizon slices."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO]

import torch  # noqa: E402
from paper_2202_13927_b200 import engine  # noqa: E402
from paper_2202_13927_b200.config import SimulationConfig  # noqa: E402
from paper_2202_13927_b200.controller import ControllerHyperparameters  # noqa: E402
from paper_2202_13927_b200.population import generate_population  # noqa: E402
from paper_2202_13927_b200.protocol import ThreeMealProtocol  # noqa: E402
from paper_2202_13927_b200.trial import FastTrial  # noqa: E402

dev = torch.device("cuda", 0)
cfg = SimulationConfig(horizon_s=9 * 86400.0, seed=12, dt_s=60.0)
pop = generate_population(8, 200, device=dev, on_exhausted="redraw_weight")
params = pop.params_device.clone()
bad = len(sys.argv) > 1 and sys.argv[1] == "bad"
if bad:
    params[37, 4] = -5.0
runs = []
for s in (1, 2, 3):
    ft = FastTrial(0, params, pop.basal_device, ThreeMealProtocol(), ControllerHyperparameters(), cfg,
                   device=dev, n_slices=s)
    ft.outs = engine.alloc_fast_outputs(ft.n, 0, ft.sz, dev, per_patient_timeline=True, final_state=True)
    ft.simulate()
    torch.cuda.synchronize()
    runs.append(ft)
for r in runs[1:]:
    for k in ("status", "ticks", "bg_hist", "bg_stats", "day_dose", "hypo_events", "timeline_pp",
              "timeline_warp", "x_out"):
        x = getattr(runs[0].outs, k).cpu().numpy().astype(np.float64)
        y = getattr(r.outs, k).cpu().numpy().astype(np.float64)
        d = np.abs(x - y)
        if d.max() > 0:
            w = np.argwhere(d > 0)
            print(r.n_slices, k, "max", d.max(), "n", len(w), "first", w[:6].tolist())
print("done")
