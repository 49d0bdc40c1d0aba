"""Disturbance protocols and protocol generators.

* ``Disturbance`` / ``Protocol`` carry the reference's fields
  (protocol.py:64-164), so protocols from either package interoperate.
* ``compile_protocol`` restates simulation.py:142-168; ``compile_ticks``
  converts the compiled arrays to the integer tick form the fused kernel
  walks.
* ``ThreeMealProtocol`` is the BASELINE configs[0] disturbance generator
  (3 meals/day, carbs ~ N(50/70/80 g, 10 g) clipped at 0, meal-time jitter
  ~ U(±30 min)).  It follows the reference's generator plug-in contract
  (``build(trial_seed, patient) -> Protocol`` and ``describe()``,
  simulation.py:431-466); its schedule is a pure function of
  (trial seed, patient id, meal index), generated bit-identically on the
  host (this file) and on device (gt_common.cuh gen_meal).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import rng

DAY_S = 86400.0


@dataclass(slots=True)
class Disturbance:
    kind: str                 # "meal" | "exercise"
    start_s: float
    end_s: float
    magnitude: float          # g CHO (meal) or heart-rate-reserve fraction (exercise)
    announced: bool = True
    announced_magnitude: float | None = None

    def __post_init__(self):
        if self.announced_magnitude is None:
            self.announced_magnitude = self.magnitude

    def to_dict(self) -> dict:
        return {"kind": self.kind, "start_s": self.start_s, "end_s": self.end_s,
                "magnitude": self.magnitude, "announced": self.announced,
                "announced_magnitude": self.announced_magnitude}


@dataclass(slots=True)
class Protocol:
    id: str
    horizon_s: float
    disturbances: list


@dataclass(frozen=True)
class ProtocolArrays:
    meals_start: np.ndarray
    meals_end: np.ndarray
    meals_rate: np.ndarray
    meals_ann: np.ndarray
    ex_start: np.ndarray
    ex_end: np.ndarray
    ex_hrr: np.ndarray
    ex_announced: np.ndarray


def compile_protocol(protocol, horizon_s: float) -> ProtocolArrays:
    """Flat event arrays of the events starting before the horizon
    (simulation.py:156-168); works on any object with ``disturbances``."""
    meals = [d for d in protocol.disturbances if d.kind == "meal" and d.start_s < horizon_s]
    ex = [d for d in protocol.disturbances if d.kind == "exercise" and d.start_s < horizon_s]
    f = lambda xs: np.array(xs, dtype=np.float64)
    return ProtocolArrays(
        meals_start=f([m.start_s for m in meals]),
        meals_end=f([m.end_s for m in meals]),
        meals_rate=f([m.magnitude / ((m.end_s - m.start_s) / 60.0) for m in meals]),
        meals_ann=f([m.announced_magnitude if m.announced else 0.0 for m in meals]),
        ex_start=f([e.start_s for e in ex]),
        ex_end=f([e.end_s for e in ex]),
        ex_hrr=f([e.magnitude for e in ex]),
        ex_announced=f([1.0 if e.announced else 0.0 for e in ex]),
    )


def validate_protocol(protocol) -> list:
    """Invariant violations (protocol.py:397-426); empty list = valid."""
    out = []
    if protocol.horizon_s < 0:
        out.append("horizon is negative")
    prev_start = -np.inf
    end_of = {"meal": -np.inf, "exercise": -np.inf}
    idx_of = {"meal": None, "exercise": None}
    for i, d in enumerate(protocol.disturbances):
        tag = f"disturbance[{i}] ({d.kind} @ {d.start_s:g}s)"
        if d.kind not in end_of:
            out.append(f"{tag}: unknown kind")
            continue
        if not d.start_s < d.end_s:
            out.append(f"{tag}: start must be before end")
        if d.magnitude < 0:
            out.append(f"{tag}: negative magnitude")
        if d.announced_magnitude is None or d.announced_magnitude < 0:
            out.append(f"{tag}: negative announced magnitude")
        if d.start_s < 0 or d.end_s > protocol.horizon_s:
            out.append(f"{tag}: outside [0, horizon]")
        if d.start_s < prev_start:
            out.append(f"{tag}: disturbances not time-ordered")
        prev_start = d.start_s
        if d.start_s < end_of[d.kind]:
            out.append(f"{tag}: overlaps disturbance[{idx_of[d.kind]}] of same kind")
        if d.end_s > end_of[d.kind]:
            end_of[d.kind] = d.end_s
            idx_of[d.kind] = i
    return out


@dataclass(frozen=True)
class TickArrays:
    """Protocol arrays in integer ticks for the fused kernel."""
    meal_ks: np.ndarray   # first tick with t >= start
    meal_ke: np.ndarray   # first tick with t >= end
    meal_kp: np.ndarray   # controller period containing start
    meal_rate: np.ndarray
    meal_ann: np.ndarray
    ex_ks: np.ndarray
    ex_ke: np.ndarray
    ex_start: np.ndarray
    ex_hrr: np.ndarray
    ex_announced: np.ndarray


def compile_ticks(pa: ProtocolArrays, dt_s: float, period_s: float) -> TickArrays:
    """Exact tick form of the pointer walk of _kernel.py:85-117 for integer-
    second times: active while ks <= k < ke; announced at period kp."""
    def ticks(t):
        q = np.ceil(np.asarray(t) / dt_s)
        if not np.all(q * dt_s - np.asarray(t) < dt_s):
            raise ValueError("protocol times not representable on the tick grid")
        return q.astype(np.int32)
    for arr in (pa.meals_start, pa.meals_end, pa.ex_start, pa.ex_end):
        if arr.size and not np.all(arr == np.floor(arr)):
            raise ValueError("fused kernel requires whole-second protocol times")
    return TickArrays(
        meal_ks=ticks(pa.meals_start), meal_ke=ticks(pa.meals_end),
        meal_kp=np.floor(pa.meals_start / period_s).astype(np.int32),
        meal_rate=pa.meals_rate.astype(np.float64), meal_ann=pa.meals_ann.astype(np.float64),
        ex_ks=ticks(pa.ex_start), ex_ke=ticks(pa.ex_end), ex_start=pa.ex_start.astype(np.float64),
        ex_hrr=pa.ex_hrr.astype(np.float64), ex_announced=pa.ex_announced.astype(np.float64),
    )


@dataclass(frozen=True)
class ThreeMealProtocol:
    """BASELINE 3-meal disturbance generator.

    Meal ``m = 3*day + slot`` of patient ``pid`` draws one Philox4x32-10
    block (key = trial seed, counter = (m, pid, ROLE_MEALS, m >> 32)):
    word 0 -> integer jitter in [-jitter_s, jitter_s] seconds; words 1-2 ->
    52-bit uniform -> Acklam inverse normal -> carbs = mean + sd*z, clipped
    at 0 ("truncated at 0").  Meals last ``duration_s`` and are announced.
    """

    clock_s: tuple = (7 * 3600.0, 12 * 3600.0, 18 * 3600.0)
    mean_g: tuple = (50.0, 70.0, 80.0)
    sd_g: float = 10.0
    jitter_s: int = 1800
    duration_s: int = 900
    days: int = 364
    role: int = rng.ROLE_MEALS

    def __post_init__(self):
        if len(self.clock_s) != 3 or len(self.mean_g) != 3:
            raise ValueError("three meal slots required")
        if self.jitter_s < 0 or self.duration_s <= 0:
            raise ValueError("bad jitter/duration")
        # meals stay time-ordered and non-overlapping within and across days
        c = sorted(self.clock_s)
        if list(c) != list(self.clock_s):
            raise ValueError("meal clock times must be increasing")
        span = 2 * self.jitter_s + self.duration_s
        if c[0] - self.jitter_s < 0 or c[2] + self.jitter_s + self.duration_s > DAY_S:
            raise ValueError("jittered meals must stay within the day")
        if c[1] - c[0] < span or c[2] - c[1] < span:
            raise ValueError("jittered meals would overlap")

    def meals(self, trial_seed: int, pid: int, n_meals: int):
        """(start_s, end_s, carbs_g) arrays of meals 0..n_meals-1."""
        m = np.arange(n_meals, dtype=np.uint64)
        r = rng.philox4x32_10(rng.philox_counters(m, pid, self.role), trial_seed)
        day = (m // np.uint64(3)).astype(np.int64)
        slot = (m % np.uint64(3)).astype(np.int64)
        span = np.uint64(2 * self.jitter_s + 1)
        jit = ((r[:, 0].astype(np.uint64) * span) >> np.uint64(32)).astype(np.int64) - self.jitter_s
        clock = np.asarray(self.clock_s, dtype=np.float64)[slot]
        mean = np.asarray(self.mean_g, dtype=np.float64)[slot]
        start = (day.astype(np.float64) * 86400.0 + clock) + jit.astype(np.float64)
        z = rng.det_inv_norm(rng.u52(r[:, 1], r[:, 2]))
        carbs = mean + float(self.sd_g) * z
        carbs = np.where(carbs < 0.0, 0.0, carbs)
        return start, start + float(self.duration_s), carbs

    def build(self, trial_seed: int, patient) -> Protocol:
        start, end, carbs = self.meals(trial_seed, int(patient.id), 3 * self.days)
        dist = [Disturbance("meal", float(s), float(e), float(g), True, float(g))
                for s, e, g in zip(start, end, carbs)]
        return Protocol(id=f"three-meal/seed={trial_seed}/pid={patient.id}",
                        horizon_s=self.days * DAY_S, disturbances=dist)

    def describe(self) -> dict:
        return {"kind": "three_meal", "clock_s": list(self.clock_s), "mean_g": list(self.mean_g),
                "sd_g": self.sd_g, "jitter_s": self.jitter_s, "duration_s": self.duration_s,
                "days": self.days}

    @classmethod
    def from_spec(cls, spec: dict) -> "ThreeMealProtocol":
        """Inverse of describe() (trial records, records.generator_from_spec)."""
        return cls(clock_s=tuple(spec["clock_s"]), mean_g=tuple(spec["mean_g"]), sd_g=spec["sd_g"],
                   jitter_s=spec["jitter_s"], duration_s=spec["duration_s"], days=spec["days"])

    def device_spec(self) -> dict:
        return {"clock_s": tuple(float(c) for c in self.clock_s),
                "mean_g": tuple(float(m) for m in self.mean_g), "sd_g": float(self.sd_g),
                "jitter_s": int(self.jitter_s), "duration_s": int(self.duration_s),
                "role": int(self.role)}


@dataclass(frozen=True)
class FixedProtocol:
    """The same explicit protocol for every patient (simulation.py:456-466)."""

    protocol: Protocol

    def build(self, trial_seed: int, patient):
        return self.protocol

    def describe(self) -> dict:
        return {"kind": "fixed", "protocol_id": self.protocol.id}
