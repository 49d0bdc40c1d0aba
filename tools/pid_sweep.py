"""Sweep PID defaults (treatment_comparison arms on one CRN population)."""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2202_13927_b200.pid import PIDProfile  # noqa: E402
from paper_2202_13927_b200.studies import treatment_comparison  # noqa: E402

dev = torch.device("cuda", 0)
arms = {}
for sp, kp, ki, kd, fmax in itertools.product((6.0, 6.5, 7.0), (0.05, 0.1, 0.15), (0.0, 0.005, 0.02),
                                              (1.0, 3.0), (2.0, 3.0)):
    arms[f"sp{sp}_kp{kp}_ki{ki}_kd{kd}_f{fmax}"] = PIDProfile(setpoint=sp, kp=kp, ki=ki, kd=kd, factor_max=fmax)
arms["default"] = PIDProfile()
out = treatment_comparison(20000, 4, seed=11, device=dev, controller_id="pid_pump", arms=arms,
                           reference_arm="default")
rows = []
for name, v in out["arms"].items():
    pp = v["per_patient"]
    rows.append((name, pp["tir"]["mean"], pp["tbr70"]["mean"], pp["tbr54"]["mean"], pp["tar180"]["mean"],
                 pp["tar250"]["mean"]))
rows.sort(key=lambda r: -(r[1] - 3 * r[2]))
for r in rows[:25]:
    print("%-40s tir %.3f tbr70 %.3f tbr54 %.4f tar180 %.3f tar250 %.3f" % r)
print([r for r in rows if r[0] == "default"])
