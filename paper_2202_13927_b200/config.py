"""Simulation configuration: same fields, validation and derived sizes as
the reference's ``SimulationConfig`` (simulation.py:71-130), so a config
object from either package drives either engine."""

from __future__ import annotations

import math
from dataclasses import dataclass

STORE_TRACE_MODES = ("never", "worst_case_only", "always")
CHUNK_PATIENTS = 32            # simulation.py:56 (reduction structure of the reference)
BLOCK_TARGET_STEPS = 20160     # simulation.py:59


class SimulationError(RuntimeError):
    """Invalid simulation configuration or unsupported model/controller."""


@dataclass(frozen=True)
class SimulationConfig:
    horizon_s: float
    seed: int
    dt_s: float = 30.0
    controller_period_s: float = 300.0
    store_trace: str = "never"
    initial_bg_mmol_per_l: float = 6.0
    grid_step_s: float = 3600.0
    engine: str = "auto"

    def __post_init__(self):
        if self.dt_s <= 0:
            raise SimulationError("dt must be positive")
        checks = (("controller period", self.controller_period_s, self.dt_s),
                  ("horizon", self.horizon_s, self.controller_period_s),
                  ("grid step", self.grid_step_s, self.dt_s))
        for what, value, base in checks:
            ratio = value / base
            if value <= 0 or abs(ratio - round(ratio)) > 1e-9:
                raise SimulationError(f"{what} must be a positive integer multiple of its base step")
        if self.store_trace not in STORE_TRACE_MODES:
            raise SimulationError(f"store_trace must be one of {STORE_TRACE_MODES}")
        if self.engine not in ("auto", "fast", "python"):
            raise SimulationError("engine must be auto, fast or python")
        if self.initial_bg_mmol_per_l <= 0:
            raise SimulationError("initial BG must be positive")

    @property
    def horizon_ticks(self) -> int:
        return int(round(self.horizon_s / self.dt_s))

    @property
    def period_steps(self) -> int:
        return int(round(self.controller_period_s / self.dt_s))

    @property
    def grid_step_ticks(self) -> int:
        return int(round(self.grid_step_s / self.dt_s))

    @property
    def n_grid(self) -> int:
        return -(-self.horizon_ticks // self.grid_step_ticks)

    @property
    def n_days(self) -> int:
        return max(1, math.ceil(self.horizon_s / 86400.0))

    def to_dict(self) -> dict:
        return {
            "horizon_s": self.horizon_s, "seed": self.seed, "dt_s": self.dt_s,
            "controller_period_s": self.controller_period_s, "store_trace": self.store_trace,
            "initial_bg_mmol_per_l": self.initial_bg_mmol_per_l,
            "grid_step_s": self.grid_step_s, "engine": self.engine,
        }


def sizes(config) -> dict:
    """Derived integer sizes of any config object with the reference fields."""
    H = int(round(config.horizon_s / config.dt_s))
    ps = int(round(config.controller_period_s / config.dt_s))
    gs = int(round(config.grid_step_s / config.dt_s))
    block = ps * max(1, BLOCK_TARGET_STEPS // ps)
    return {
        "horizon_ticks": H, "period_steps": ps, "grid_step_ticks": gs,
        "n_grid": -(-H // gs), "n_days": max(1, math.ceil(config.horizon_s / 86400.0)),
        "block_ticks": block,
    }
