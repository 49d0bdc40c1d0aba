"""Virtual populations.

``generate_population`` runs the device rejection sampler (csrc/gt_sampler.cu,
BASELINE north_star subsystem 1): same parameter distributions and
acceptance rules as the reference (population.py:207-259), counter-based
device streams keyed by (seed, patient id).  The result stays on device
(``DevicePopulation``) and feeds the fused trial path directly; ``entries()``
materialises reference-style ``(Patient, ParameterSet)`` pairs.
Populations produced by the reference's own sampler are accepted everywhere
a population is expected.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import engine, rng, tables
from .layout import PARAM_NAMES


class PopulationError(RuntimeError):
    pass


@dataclass(slots=True)
class Patient:
    """Minimal patient record: the simulation uses id and body weight only
    (population.py:42-58); names/dates/places carry no simulation semantics."""
    id: int
    body_weight_kg: float


@dataclass(slots=True)
class ParameterSet:
    values: dict
    u_basal_u_per_h: float


@dataclass
class SamplingStats:
    attempts: int = 0
    accepted: int = 0
    rejected_negative: int = 0
    rejected_outside_sd: int = 0
    rejected_basal: int = 0
    rejected_no_steady_state: int = 0

    @property
    def acceptance_rate(self) -> float:
        return self.accepted / self.attempts if self.attempts else 0.0


class DevicePopulation:
    """A device-resident population shard (ids pid0 .. pid0+n-1)."""

    def __init__(self, pid0, params_device, basal_device, x0_device, stats: SamplingStats,
                 attempts_device=None, max_attempts: int = tables.MAX_ATTEMPTS, target_bg: float = 6.0):
        self.pid0 = int(pid0)
        self.params_device = params_device
        self.basal_device = basal_device
        self.x0_device = x0_device
        self.stats = stats
        self.attempts_device = attempts_device   # per patient, redraw rounds included
        self.max_attempts = int(max_attempts)
        self.target_bg = float(target_bg)   # the steady state x0_device was solved at

    @property
    def n_weight_redraws(self) -> int:
        """Patients whose body weight was redrawn (each redraw follows a whole
        exhausted attempt budget; on_exhausted="redraw_weight")."""
        if self.attempts_device is None:
            return 0
        return int((self.attempts_device >= self.max_attempts).sum().item())

    def __len__(self):
        return int(self.params_device.shape[0])

    def entries(self):
        p = self.params_device.cpu().numpy()
        ub = self.basal_device.cpu().numpy()
        out = []
        for i in range(len(self)):
            vals = {name: float(p[i, k]) for k, name in enumerate(PARAM_NAMES)}
            out.append((Patient(self.pid0 + i, vals["weight_kg"]), ParameterSet(vals, float(ub[i]))))
        return out


def generate_population(seed: int, n: int, table=None, target_bg: float = 6.0, pid0: int = 0,
                        device=None, max_attempts: int = tables.MAX_ATTEMPTS,
                        on_exhausted: str = "raise") -> DevicePopulation:
    """``on_exhausted="raise"`` keeps the reference's contract (PopulationError
    when a patient exhausts the attempt budget, population.py:257-259).  Very
    low body weights (< ~30 kg, 3.4e-4 of N(74,13)) admit no parameter set with
    u_basal >= 0.4 U/h, so populations of 1e5+ patients hit that error with
    near certainty; ``"redraw_weight"`` redraws such a patient's weight
    (up to 16 times) instead — the body-weight distribution conditioned on
    feasibility."""
    if on_exhausted not in ("raise", "redraw_weight"):
        raise ValueError("on_exhausted must be 'raise' or 'redraw_weight'")
    if n < 1:
        raise PopulationError("population size must be >= 1")
    table = table or tables.default_parameter_table()
    with engine.nvtx("gt.population_sampler"):
        out = engine.sample_population(seed, n, table, pid0=pid0, target_bg=target_bg, device=device,
                                       max_attempts=max_attempts,
                                       weight=(tables.WEIGHT_MEAN_KG, tables.WEIGHT_SD_KG),
                                       min_basal=tables.MIN_BASAL_U_PER_H,
                                       max_weight_redraws=16 if on_exhausted == "redraw_weight" else 0)
    status = out["status"]
    if bool((status != 0).any()):
        bad = int(np.nonzero(status.cpu().numpy())[0][0]) + pid0
        raise PopulationError(f"no acceptable parameter set for patient {bad} in {max_attempts} attempts")
    rc = out["reject_counts"].cpu().numpy()
    attempts = int(out["attempts"].sum().item())
    st = SamplingStats(attempts=attempts, accepted=n, rejected_negative=int(rc[0]),
                       rejected_outside_sd=int(rc[1]), rejected_no_steady_state=int(rc[2]),
                       rejected_basal=int(rc[3]))
    return DevicePopulation(pid0, out["params"], out["u_basal"], out["x0"], st, out["attempts"], max_attempts,
                            target_bg)


def validate_parameter_sets(params, u_basal, table=None, target_bg: float = 6.0, device=None) -> list:
    """Batched ``validate_parameter_set`` (population.py:262-282): the three
    acceptance rules re-checked for every row of ``params`` [n, 30] with its
    stored basal rate; the steady state is re-solved on the device.  Returns
    one list of violation strings per patient (empty = valid)."""
    import math
    from .layout import PARAM_INDEX
    table = table or tables.default_parameter_table()
    p = params.detach().cpu().numpy() if hasattr(params, "detach") else np.asarray(params, np.float64)
    ub = u_basal.detach().cpu().numpy() if hasattr(u_basal, "detach") else np.asarray(u_basal, np.float64)
    x0, ub_solved, st = engine.steady_state(np.ascontiguousarray(p, np.float64), target_bg, device)
    ub_solved, st = ub_solved.cpu().numpy(), st.cpu().numpy()
    out = []
    for i in range(p.shape[0]):
        v = []
        for k, name in enumerate(PARAM_NAMES):
            if p[i, k] < 0.0:
                v.append(f"{name} is negative")
        for name, spec in table.sampled.items():
            if spec.kind == "normal" and abs(p[i, PARAM_INDEX[name]] - spec.mean) > spec.sd:
                v.append(f"{name} outside one standard deviation")
        if ub[i] < tables.MIN_BASAL_U_PER_H:
            v.append(f"u_basal {ub[i]:.3f} U/h below {tables.MIN_BASAL_U_PER_H}")
        if st[i] != 0:
            v.append("steady state failed")
        elif not math.isclose(float(ub_solved[i]), float(ub[i]), rel_tol=1e-9, abs_tol=1e-12):
            v.append("stored u_basal does not match the steady-state solve")
        out.append(v)
    return out
