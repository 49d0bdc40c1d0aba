"""Pin the C oracle against golden vectors produced by the real reference.

CPU only.  A failure here means the oracle (the checker for every GPU
parity test) no longer restates the reference bit for bit.
"""

import hashlib
import json

import numpy as np
import pytest

from conftest import golden, golden_bytes
from helpers import SimCase


def test_versions_recorded():
    v = json.loads(golden_bytes("versions.json"))
    assert {"numpy", "scipy", "numba", "reference"} <= set(v)


def test_drift_bitwise(oracle):
    g = golden("drift.npz")
    for i in range(g["X"].shape[0]):
        out = oracle.drift(g["X"][i], g["U"][i], g["D"][i], g["P"][i])
        assert np.array_equal(out, g["OUT"][i]), i


def test_controller_bitwise(oracle):
    g = golden("controller.npz")
    rows = g["rows"]
    hyper, basal = g["hyper"], float(g["basal"])
    c = rows[0, :11].copy()
    for r in rows:
        assert np.array_equal(c, r[:11])
        y, ann, phase, t = r[11:15]
        c, out = oracle.controller_step(c, y, ann, phase, t, 300.0, hyper, basal)
        assert np.array_equal(out, r[15:18])
        assert np.array_equal(c, r[18:29])


def test_steady_state_bitwise(oracle):
    g = golden("steady.npz")
    for i in range(g["params"].shape[0]):
        x, ub = oracle.steady_state(g["params"][i])
        assert np.array_equal(x, g["x0"][i]) and ub == g["ub"][i]
    for i in range(g["pert"].shape[0]):
        x, ub = oracle.steady_state(g["pert"][i])
        if g["pert_ok"][i]:
            assert np.array_equal(x, g["pert_x0"][i]) and ub == g["pert_ub"][i], i
        else:
            assert x is None
    assert int(g["bad_ok"]) == 0 and oracle.steady_state(g["bad_params"])[0] is None


def test_py_floordiv_semantics(oracle):
    rng = np.random.default_rng(0)
    for w in (86400.0, 0.5, 10.0):
        for v in np.concatenate([rng.uniform(0, 1e6, 2000), np.arange(0, 2e6, 37.5)[:2000]]):
            assert oracle.py_floordiv(float(v), w) == float(v) // w


@pytest.mark.parametrize("name", ["sim_northern_dt30.npz", "sim_threemeal_dt60.npz",
                                  "sim_northern_dt37p5.npz", "sim_northern_dt30_8d.npz",
                                  "sim_faults.npz"])
def test_simulation_bitwise(oracle, name):
    case = SimCase(name)
    g = case.g
    for i, pid in enumerate(case.ids):
        W, hn, M = case.noise()
        h = hashlib.sha256(W[i].tobytes() + M[i].tobytes()).hexdigest()
        assert h == str(g["noise_sha"][i]), "numpy reference stream changed"
    sub = case.subset(case.valid())
    out = oracle.run_batch_injected(sub["params"], sub["x0"], sub["c0"], case.hyper, sub["basal"],
                                    case.sz, case.config.dt_s, case.config.controller_period_s,
                                    sub["meal_off"], sub["meals"], sub["ex_off"], sub["ex"],
                                    sub["wiener"], sub["has_noise"], sub["meas"])
    for j, i in enumerate(sub["idx"]):
        assert out["status"][j] == g["status"][i]
        assert out["ticks"][j] == g["ticks"][i]
        assert np.array_equal(out["tir_ticks"][j], g["tir"][i])
        assert np.array_equal(out["bg_hist"][j], g["hist"][i])
        assert np.array_equal(out["scal"][j, :3], g["scal"][i])
        assert np.array_equal(out["day_dose"][j], g["day_dose"][i])
        assert np.array_equal(out["timeline"][j], g["timeline"][i])
