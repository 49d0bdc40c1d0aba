"""Developer diagnostic: fused kernel, device 3-meal generator vs CSR of the
host twin schedule, same injected noise — print per-field differences."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "tests"), os.path.join(REPO, "oracle")]

import torch  # noqa: E402
from helpers import SimCase  # noqa: E402
import test_gpu_fast as T  # noqa: E402
from paper_2202_13927_b200.protocol import ThreeMealProtocol  # noqa: E402

dev = torch.device("cuda", 0)
case = SimCase("sim_threemeal_dt60.npz")
sub = case.subset(case.valid())
inj = T._injected(sub, dev)
a = T._run_fast(case, sub, dev, csr=T._csr_ticks(case, sub, dev), injected=inj)
b = T._run_fast(case, sub, dev, meal_spec=ThreeMealProtocol().device_spec(), injected=inj)
for k in ("status", "ticks", "bg_hist", "bg_stats", "day_dose", "hypo_events", "timeline_pp", "x_out"):
    x, y = T._h(getattr(a, k)).astype(np.float64), T._h(getattr(b, k)).astype(np.float64)
    d = np.abs(x - y)
    print(k, "max abs diff", d.max(), "n diff", int((d > 0).sum()), "where", np.argwhere(d > 0)[:5].tolist())
