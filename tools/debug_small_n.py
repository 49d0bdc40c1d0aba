import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2202_13927_b200.config import SimulationConfig
from paper_2202_13927_b200.controller import ControllerHyperparameters
from paper_2202_13927_b200.population import generate_population
from paper_2202_13927_b200.protocol import ThreeMealProtocol
from paper_2202_13927_b200.trial import FastTrial
dev = torch.device("cuda", 0)
cfg = SimulationConfig(horizon_s=86400.0, seed=1, dt_s=60.0)
pop = generate_population(3, 33, device=dev, on_exhausted="redraw_weight")
for n in [int(a) for a in sys.argv[1:]]:
    ft = FastTrial(0, pop.params_device[:n].contiguous(), pop.basal_device[:n].contiguous(), ThreeMealProtocol(),
                   ControllerHyperparameters(), cfg, device=dev, per_patient_metrics=True,
                   n_slices=int(os.environ.get('NS', '0')))
    ft.simulate(); torch.cuda.synchronize(); print(n, "simulate ok", flush=True)
    ft._rerun_if_diverged(); torch.cuda.synchronize(); print(n, "rerun ok", flush=True)
    ft.reduce(); torch.cuda.synchronize(); print(n, "reduce ok", flush=True)
    print(n, ft.metrics()["tir"][:3], flush=True)
