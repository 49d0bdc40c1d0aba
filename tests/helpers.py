"""Shared test plumbing: rebuild simulation inputs from the golden fixtures."""

from __future__ import annotations

import numpy as np

from paper_2202_13927_b200 import rng
from paper_2202_13927_b200.config import SimulationConfig, sizes
from paper_2202_13927_b200.layout import PR, PSIGEGP, PSIGGUT

from conftest import golden


class SimCase:
    """Inputs + reference outputs of one golden simulation fixture."""

    def __init__(self, name):
        g = golden(name)
        self.g = g
        h, seed, dt, period, grid, bg0 = g["config"]
        self.config = SimulationConfig(horizon_s=float(h), seed=int(seed), dt_s=float(dt),
                                       controller_period_s=float(period), grid_step_s=float(grid),
                                       initial_bg_mmol_per_l=float(bg0))
        self.sz = sizes(self.config)
        self.ids = g["ids"].astype(np.int64)
        self.n = self.ids.size
        self.params = g["params"]
        self.x0 = g["x0"]
        self.c0 = g["c0"]
        self.basal = g["basal"]
        self.hyper = g["hyper"]
        self.meal_off = g["meal_off"].astype(np.int64)
        self.ex_off = g["ex_off"].astype(np.int64)
        self.meals = tuple(g[k] for k in ("meals_start", "meals_end", "meals_rate", "meals_ann"))
        self.ex = tuple(g[k] for k in ("ex_start", "ex_end", "ex_hrr", "ex_announced"))
        self.status = g["status"]
        self._noise = None

    def noise(self):
        """The reference's own streams (rng.py:26-39), as the reference draws them."""
        if self._noise is None:
            H, ps = self.sz["horizon_ticks"], self.sz["period_steps"]
            W = np.zeros((self.n, H, 3))
            M = np.zeros((self.n, H // ps))
            hn = np.zeros(self.n, dtype=np.uint8)
            for i, pid in enumerate(self.ids):
                p = self.params[i]
                proc = bool(p[PSIGEGP] > 0 or p[PSIGGUT] > 0)
                w, m = rng.reference_noise(self.config.seed, int(pid), H, ps, proc, bool(p[PR] > 0))
                if w is not None:
                    W[i] = w
                M[i] = m
                hn[i] = proc
            self._noise = (W, hn, M)
        return self._noise

    def valid(self):
        """Patients with a steady state (status != 2)."""
        return self.status != 2

    def subset(self, mask):
        """CSR/params restricted to mask (returns dict of arrays)."""
        idx = np.nonzero(mask)[0]
        W, hn, M = self.noise()
        mo, eo = [0], [0]
        meals = [[], [], [], []]
        ex = [[], [], [], []]
        for i in idx:
            a, b = self.meal_off[i], self.meal_off[i + 1]
            for k in range(4):
                meals[k].append(self.meals[k][a:b])
            mo.append(mo[-1] + (b - a))
            a, b = self.ex_off[i], self.ex_off[i + 1]
            for k in range(4):
                ex[k].append(self.ex[k][a:b])
            eo.append(eo[-1] + (b - a))
        cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0)
        return dict(idx=idx, params=self.params[idx], x0=self.x0[idx], c0=self.c0[idx],
                    basal=self.basal[idx], meal_off=np.array(mo, np.int64),
                    meals=tuple(cat(m) for m in meals), ex_off=np.array(eo, np.int64),
                    ex=tuple(cat(e) for e in ex), wiener=W[idx], has_noise=hn[idx], meas=M[idx])
