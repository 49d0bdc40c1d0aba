"""Phase timing of the end-to-end array API (trial.run_population_arrays):
H2D, staging (steady state, controller set-up, output allocation), step,
readback.  python tools/e2e_breakdown.py [n] [weeks] [reps]"""
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
from paper_2202_13927_b200.trial import FastTrial, run_population_arrays  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
weeks = int(sys.argv[2]) if len(sys.argv) > 2 else 4
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dev = torch.device("cuda", 0)
cfg = SimulationConfig(horizon_s=weeks * 7 * 86400.0, seed=1, dt_s=60.0)
pop = generate_population(1, n, device=dev, on_exhausted="redraw_weight")
ph = pop.params_device.cpu().pin_memory()
bh = pop.basal_device.cpu().pin_memory()
prof, gen = ControllerHyperparameters(), ThreeMealProtocol()


def now():
    torch.cuda.synchronize()
    return time.perf_counter()


for r in range(reps):
    t0 = now()
    p_d = ph.to(dev, non_blocking=True)
    b_d = bh.to(dev, non_blocking=True)
    t1 = now()
    ft = FastTrial(0, p_d, b_d, gen, prof, cfg, device=dev, per_patient_metrics=True)
    t2 = now()
    ft.step()
    t3 = now()
    acc = ft.accumulator()
    t4 = now()
    m = ft.metrics()
    t5 = now()
    tot = t5 - t0
    print(f"rep {r}: h2d {1e3*(t1-t0):.1f} stage {1e3*(t2-t1):.1f} step {1e3*(t3-t2):.1f} "
          f"acc {1e3*(t4-t3):.1f} metrics {1e3*(t5-t4):.1f} total {1e3*tot:.1f} ms", flush=True)
    del ft
import subprocess  # noqa: E402
for r in range(reps):
    t0 = now()
    run_population_arrays(ph, bh, gen, prof, cfg, device=dev)
    t1 = now()
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks_throttle_reasons.active,power.draw",
                          "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    print(f"api rep {r}: {1e3*(t1-t0):.1f} ms  [{clk}]", flush=True)

# device-side phase timing of repeated steps on one staged trial
ft = FastTrial(0, pop.params_device, pop.basal_device, gen, prof, cfg, device=dev, per_patient_metrics=True)
st = torch.cuda.current_stream(dev)
rows = []
for r in range(3 * reps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(st)
    ft.simulate()
    ev[1].record(st)
    ft._rerun_if_diverged()
    ev[2].record(st)
    ft.reduce()
    ev[3].record(st)
    torch.cuda.synchronize()
    rows.append([ev[i].elapsed_time(ev[i + 1]) for i in range(3)])
for r in rows:
    print("device ms: simulate %.2f rerun %.2f reduce %.2f" % tuple(r))
