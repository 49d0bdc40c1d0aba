"""Default model data: parameter distributions, demographics, controller profile.

Values are the bundled defaults of the reference package
(data/hovorka_distributions.yaml:17-81, data/demographics.yaml:5-8,
data/controller_default.yaml:6-38).  Files in the reference's YAML schemas
can be loaded instead with :func:`load_parameter_table`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import yaml


@dataclass(frozen=True)
class DistributionSpec:
    """One sampled parameter (hovorka.py:246-263): normal(mean, sd) or
    lognormal given by arithmetic mean and coefficient of variation."""

    name: str
    kind: str
    mean: float
    sd: float = 0.0
    cv: float = 0.0

    @property
    def log_sigma(self) -> float:
        return math.sqrt(math.log(1.0 + self.cv ** 2))

    @property
    def log_mu(self) -> float:
        return math.log(self.mean) - 0.5 * math.log(1.0 + self.cv ** 2)


@dataclass(frozen=True)
class ParameterTable:
    model_id: str
    sampled: dict   # name -> DistributionSpec, in draw order
    fixed: dict     # name -> float


_SAMPLED = (
    ("EGP0", "normal", 0.0161, 0.0021, 0.0),
    ("F01", "normal", 0.0097, 0.0022, 0.0),
    ("k12", "normal", 0.0649, 0.0185, 0.0),
    ("ka1", "normal", 0.0055, 0.0031, 0.0),
    ("ka2", "normal", 0.0683, 0.0411, 0.0),
    ("ka3", "normal", 0.0304, 0.0090, 0.0),
    ("SIT", "lognormal", 51.2e-4, 0.0, 0.32),
    ("SID", "lognormal", 8.2e-4, 0.0, 0.35),
    ("SIE", "lognormal", 520.0e-4, 0.0, 0.30),
    ("ke", "lognormal", 0.138, 0.0, 0.15),
    ("VI", "lognormal", 0.12, 0.0, 0.12),
    ("VG", "lognormal", 0.16, 0.0, 0.12),
    ("tmaxI", "lognormal", 55.0, 0.0, 0.20),
    ("tmaxG", "lognormal", 40.0, 0.0, 0.20),
)
_FIXED = {
    "AG": 0.8, "tau_cgm": 10.0, "R": 0.0625, "t_gluc": 19.0, "ke_gluc": 0.12,
    "V_gluc": 0.25, "S_gluc": 1.6e-2, "tau_hr": 5.0, "tau_ex": 15.0, "tau_late": 120.0,
    "a_late": 5.0e-3, "q_ex": 1.5, "s_ex": 0.5, "sigma_egp": 3.0e-3, "sigma_gut": 0.03,
}

# body weight N(74, 13) kg redrawn until positive (demographics.yaml:6)
WEIGHT_MEAN_KG = 74.0
WEIGHT_SD_KG = 13.0
MIN_BASAL_U_PER_H = 0.4   # population.py:31
MAX_ATTEMPTS = 10_000      # population.py:32


def default_parameter_table() -> ParameterTable:
    sampled = {n: DistributionSpec(n, k, m, sd, cv) for n, k, m, sd, cv in _SAMPLED}
    return ParameterTable("hovorka_ext", sampled, dict(_FIXED))


def load_parameter_table(path: str | None = None) -> ParameterTable:
    """Parse a table in the reference schema
    ``glucotrial/parameter-distributions/1`` (or return the default)."""
    if path is None:
        return default_parameter_table()
    with open(path) as fh:
        raw = yaml.safe_load(fh)
    if raw.get("schema") != "glucotrial/parameter-distributions/1":
        raise ValueError(f"unsupported distribution schema: {raw.get('schema')!r}")
    sampled = {}
    for name, e in raw["sampled"].items():
        if e["kind"] not in ("normal", "lognormal"):
            raise ValueError(f"parameter {name!r}: unknown kind {e['kind']!r}")
        sampled[name] = DistributionSpec(name, e["kind"], float(e["mean"]),
                                         float(e.get("sd", 0.0)), float(e.get("cv", 0.0)))
    fixed = {n: float(e["value"]) for n, e in raw["fixed"].items()}
    return ParameterTable(raw["model"], sampled, fixed)


def nominal_values(weight_kg: float, table: ParameterTable | None = None) -> dict:
    """Parameter map at distribution means (hovorka.py:318-325)."""
    table = table or default_parameter_table()
    v = {"weight_kg": float(weight_kg)}
    v.update({n: s.mean for n, s in table.sampled.items()})
    v.update(table.fixed)
    return v
