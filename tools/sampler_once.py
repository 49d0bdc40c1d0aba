"""One device-sampler call per size (for ncu launch lists): 125k seed 2, 1M seed 2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2202_13927_b200.population import generate_population
    dev = torch.device("cuda", 0)
    for n, seed in ((125_000, 2), (1_000_000, 2)):
        generate_population(seed, n, device=dev, on_exhausted="redraw_weight")
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
