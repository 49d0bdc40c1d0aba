"""Distribution-parity checks of a sampled population against the
reference's own generate_population(seed=7, n=4000) (tests/golden/
population_s7_n4000.npz, made by make_golden.py).  TEST INFRASTRUCTURE."""

from __future__ import annotations

import numpy as np

from conftest import golden

KS_P_MIN = 1e-3
Z_99 = 2.576


def two_proportion_z(k1, n1, k2, n2):
    p = (k1 + k2) / (n1 + n2)
    return (k1 / n1 - k2 / n2) / np.sqrt(p * (1 - p) * (1 / n1 + 1 / n2))


def check_against_reference(params, u_basal, attempts, reject_counts):
    """params [n, 30] (packed order), u_basal [n], attempts = total attempts,
    reject_counts = (negative, outside 1 SD, no steady state, basal).
    Two-sample KS per sampled parameter, the body weight and u_basal
    (p > 1e-3), and the acceptance and per-reason rejection rates per attempt
    within the 99 % two-proportion bound of the reference's."""
    from scipy import stats
    from paper_2202_13927_b200.layout import PARAM_INDEX
    g = golden("population_s7_n4000.npz")
    report = {}
    for j, name in enumerate(g["names"]):
        report[str(name)] = stats.ks_2samp(params[:, PARAM_INDEX[str(name)]], g["sampled"][:, j]).pvalue
    report["weight_kg"] = stats.ks_2samp(params[:, 0], g["weights"]).pvalue
    report["u_basal"] = stats.ks_2samp(u_basal, g["ubasal"]).pvalue
    bad = {k: v for k, v in report.items() if v <= KS_P_MIN}
    assert not bad, f"KS p-values at or below {KS_P_MIN}: {bad}"
    st = g["stats"]   # attempts, accepted, negative, outside_sd, basal, no_steady_state
    n = params.shape[0]
    z = {"accepted": two_proportion_z(n, attempts, st[1], st[0]),
         "negative": two_proportion_z(reject_counts[0], attempts, st[2], st[0]),
         "outside_sd": two_proportion_z(reject_counts[1], attempts, st[3], st[0]),
         "basal": two_proportion_z(reject_counts[3], attempts, st[4], st[0])}
    bad = {k: v for k, v in z.items() if abs(v) >= Z_99}
    assert not bad, f"rates outside the 99 % bound: {bad}"
    assert reject_counts[2] == 0 and st[5] == 0   # no steady-state failures in either sampler's range
    return report, z
