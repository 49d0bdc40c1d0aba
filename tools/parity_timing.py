"""Phase timing of the bitwise parity path (run_trial(noise="reference")):
host protocol build, host reference-noise draw, parity kernel.
    python tools/parity_timing.py [n] [weeks]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2202_13927_b200 import engine, rng
    from paper_2202_13927_b200.config import SimulationConfig, sizes
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol, compile_protocol
    from paper_2202_13927_b200.simulation import _csr, run_trial
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    weeks = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    dev = torch.device("cuda", 0)
    cfg = SimulationConfig(horizon_s=weeks * 7 * 86400.0, seed=1, dt_s=60.0)
    pop = generate_population(1, n, device=dev, on_exhausted="redraw_weight")
    entries = pop.entries()
    gen, prof = ThreeMealProtocol(), ControllerHyperparameters()
    sz = sizes(cfg)
    H, ps = sz["horizon_ticks"], sz["period_steps"]
    t0 = time.perf_counter()
    pas = [compile_protocol(gen.build(cfg.seed, pt), cfg.horizon_s) for pt, _ in entries]
    t1 = time.perf_counter()
    for i in range(n):
        rng.reference_noise(cfg.seed, i, H, ps, True, True)
    t2 = time.perf_counter()
    res = run_trial(entries, gen, "dual_hormone", prof, "hovorka_ext", cfg, device=dev)
    t3 = time.perf_counter()
    print(f"first call (worker pool start-up included): {t3 - t2:.2f} s", flush=True)
    t2 = time.perf_counter()
    res = run_trial(entries, gen, "dual_hormone", prof, "hovorka_ext", cfg, device=dev)
    t3 = time.perf_counter()
    print(f"n {n} weeks {weeks}: protocol {1e3 * (t1 - t0) / n:.2f} ms/patient, noise {1e3 * (t2 - t1) / n:.2f} "
          f"ms/patient, run_trial(noise='reference') {t3 - t2:.2f} s = {n * weeks / (t3 - t2):.0f} patient-weeks/s "
          f"(wall_s {res.wall_s:.2f})", flush=True)




def kernel_only(n=1024, weeks=4):
    """The parity kernel alone on n patients (reference noise injected)."""
    import numpy as np
    import torch
    from paper_2202_13927_b200 import engine, rng
    from paper_2202_13927_b200.config import SimulationConfig, sizes
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol, compile_protocol
    from paper_2202_13927_b200.simulation import _csr
    from paper_2202_13927_b200.trial import FastTrial
    dev = torch.device("cuda", 0)
    cfg = SimulationConfig(horizon_s=weeks * 7 * 86400.0, seed=1, dt_s=60.0)
    pop = generate_population(1, n, device=dev, on_exhausted="redraw_weight")
    prof, gen = ControllerHyperparameters(), ThreeMealProtocol()
    ft = FastTrial(0, pop.params_device, pop.basal_device, gen, prof, cfg, device=dev)
    sz = ft.sz
    H, ps = sz["horizon_ticks"], sz["period_steps"]
    params, x0, c0, ub = (t.cpu().numpy() for t in (ft.params, ft.x0, ft.c0, ft.basal))
    pas = [compile_protocol(gen.build(cfg.seed, pt), cfg.horizon_s) for pt, _ in pop.entries()]
    moff, meals, eoff, ex = _csr(pas)
    W = np.zeros((n, H, 3)); M = np.zeros((n, H // ps))
    hn = np.ones(n, np.uint8)
    b = engine.ParityBatch(params, x0, c0, prof.to_vec(), ub, moff, meals, eoff, ex, W, hn, M)
    for r in range(2):
        t0 = time.perf_counter()
        engine.run_parity(b, sz, cfg.dt_s, cfg.controller_period_s, device=dev)
        print(f"parity kernel + copies, {n} patients x {weeks} w: {time.perf_counter() - t0:.3f} s", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 3 and sys.argv[3] == "kernel":
        kernel_only(int(sys.argv[1]), int(sys.argv[2]))
    else:
        main()
