"""Diagnostics: fused kernel vs reference golden (per-field errors) and
sampler failure inspection.  Developer tool, not part of the product."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "tests"), os.path.join(REPO, "oracle")]

import torch  # noqa: E402
from helpers import SimCase  # noqa: E402
import test_gpu_fast as T  # noqa: E402

dev = torch.device("cuda", 0)
for name in ("sim_threemeal_dt60.npz", "sim_northern_dt30.npz"):
    case = SimCase(name)
    g = case.g
    sub = case.subset(case.valid())
    outs = T._run_fast(case, sub, dev, csr=T._csr_ticks(case, sub, dev), injected=T._injected(sub, dev))
    st, hist, dd, tl = (T._h(outs.bg_stats), T._h(outs.bg_hist), T._h(outs.day_dose), T._h(outs.timeline_pp))
    for j, i in enumerate(sub["idx"][:6]):
        rs = g["scal"][i]
        rel = lambda a, b: float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))
        print(name, j, "status", T._h(outs.status)[j], g["status"][i],
              "sum", rel(st[2, j], rs[2]), "min", rel(st[0, j], rs[0]), "max", rel(st[1, j], rs[1]),
              "tl", rel(tl[:, j], g["timeline"][i]), "dd", rel(dd[:, :, j], g["day_dose"][i]),
              "hist_diff", int(np.abs(hist[:, j] - g["hist"][i]).sum()), "ticks", T._h(outs.ticks)[j])
        print("   dd dev", dd[:2, :, j].ravel(), "\n   dd ref", g["day_dose"][i][:2].ravel())

from paper_2202_13927_b200 import engine  # noqa: E402
from paper_2202_13927_b200.tables import default_parameter_table  # noqa: E402
out = engine.sample_population(1, 3000, default_parameter_table(), device=dev)
st = out["status"].cpu().numpy()
bad = np.nonzero(st)[0]
print("sampler failures", bad[:10], "weights", out["params"][bad[:10], 0].cpu().numpy(),
      "attempts", out["attempts"][bad[:10]].cpu().numpy(), "rejects", out["reject_counts"].cpu().numpy())
ok = st == 0
print("weights ok stats", out["params"][:, 0].cpu().numpy()[ok].mean(), out["params"][:, 0].cpu().numpy()[ok].std())
