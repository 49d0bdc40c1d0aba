"""Device population sampler timing (CUDA events, after a warm-up) at 1e5
and 1e6 patients, seed 1 / 2, redraw_weight; one JSON line per size."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2202_13927_b200.population import generate_population
    dev = torch.device("cuda", 0)
    generate_population(1, 10_000, device=dev, on_exhausted="redraw_weight")
    for n, seed in ((100_000, 1), (1_000_000, 2), (125_000, 2)):
        ms = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            pop = generate_population(seed, n, device=dev, on_exhausted="redraw_weight")
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        st = pop.stats
        print(json.dumps({"n": n, "seed": seed, "ms": min(ms), "ms_all": ms, "attempts": st.attempts,
                          "acceptance": st.accepted / st.attempts, "weight_redraws": pop.n_weight_redraws}))


if __name__ == "__main__":
    main()
