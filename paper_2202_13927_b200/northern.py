"""The reference's lifestyle protocol generator, restated for the host.

``NorthernYearProtocol`` builds the 52-week schedule of the reference
(simulation.py:420-453 -> protocol.py:191-394): four seasons of 13 weeks
shuffled from the season composition table, each week's day multiset
shuffled (an active day never next to a late night), basis days from the
transcribed templates, weight-scaled meals, optional announcement policy.
It draws through the same keyed numpy streams in the same order
(derive_seed / stream, rng.py:26-48), so schedules equal the reference's
exactly (tests/test_northern.py against the golden CSR arrays).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

from . import rng
from .protocol import DAY_S, Disturbance, Protocol

DAY_TYPES = ("standard", "active", "movie_night", "late_night")
WEEK_TYPES = ("standard", "active", "vacation")
SEASON_NAMES = ("winter", "spring", "summer", "autumn")
MEAL_CHO_PER_KG = {"large": 1.29, "medium": 0.86, "small": 0.57, "snack": 0.29}
WEEK_COMPOSITIONS = {
    "standard": {"standard": 4, "active": 1, "movie_night": 1, "late_night": 1},
    "active": {"standard": 3, "active": 3, "movie_night": 1, "late_night": 0},
    "vacation": {"standard": 5, "active": 0, "movie_night": 0, "late_night": 2},
}
SEASON_COMPOSITIONS = {
    "winter": {"standard": 6, "active": 4, "vacation": 3},
    "spring": {"standard": 6, "active": 6, "vacation": 1},
    "summer": {"standard": 7, "active": 3, "vacation": 3},
    "autumn": {"standard": 9, "active": 3, "vacation": 1},
}
SEASON_CLASS_OF = {"winter": "winter_autumn", "autumn": "winter_autumn",
                   "spring": "summer_spring", "summer": "summer_spring"}
WEEK_S = 7 * DAY_S
YEAR_WEEKS = 52

# basis-day templates (data/basis_days.yaml): clock "HH:MM" and meal class
_STANDARD = {
    "winter_autumn": (("07:30", "medium"), ("12:00", "medium"), ("15:30", "snack"), ("18:30", "large")),
    "summer_spring": (("07:30", "medium"), ("10:00", "snack"), ("12:00", "medium"), ("18:30", "medium")),
}
_EXTRA_MEALS = {"movie_night": (("21:30", "snack"),), "late_night": (("22:00", "snack"), ("23:30", "snack"))}
_EXERCISE = ("17:00", 45.0, 0.5)   # start, duration (min), HRR fraction
_MEAL_DURATION_S = 15 * 60.0


def _clock(s: str) -> float:
    hh, mm = s.split(":")
    return float(int(hh) * 3600 + int(mm) * 60)


def basis_days() -> dict:
    out = {}
    for sc, base in _STANDARD.items():
        for day_type in DAY_TYPES:
            ev = [("meal", _clock(t), c) for t, c in base]
            if day_type == "active":
                ev.append(("exercise", _clock(_EXERCISE[0]), _EXERCISE[1] * 60.0, _EXERCISE[2]))
            for t, c in _EXTRA_MEALS.get(day_type, ()):
                ev.append(("meal", _clock(t), c))
            ev.sort(key=lambda e: e[1])
            out[(day_type, sc)] = ev
    return out


_BASIS = basis_days()


def _bad_adjacency(days) -> bool:
    return any({a, b} == {"active", "late_night"} for a, b in zip(days, days[1:]))


def _plan_week(week_type, g):
    counts = WEEK_COMPOSITIONS[week_type]
    days = [d for d in DAY_TYPES for _ in range(counts.get(d, 0))]
    constrained = counts.get("active", 0) > 0 and counts.get("late_night", 0) > 0
    for _ in range(1000):
        g.shuffle(days)
        if not constrained or not _bad_adjacency(days):
            return list(days)
    raise ValueError(f"could not order week {week_type!r}")


def plan_year_twin(seed: int):
    """plan_year through the integer restatement of numpy's stream
    (rng.NumpyPhiloxTwin) -- the algorithm csrc/gt_northern.cu runs."""
    g = rng.NumpyPhiloxTwin(seed, (0,))
    weeks, days = [], []
    for season in SEASON_NAMES:
        counts = SEASON_COMPOSITIONS[season]
        wk = [w for w in WEEK_TYPES for _ in range(counts.get(w, 0))]
        g.shuffle(wk)
        for w in wk:
            weeks.append(w)
            days.append(_plan_week(w, g))
    return weeks, days


def week_day_codes(days) -> list:
    """2-bit day-type codes per week (the device builder's week_days)."""
    return [sum(DAY_TYPES.index(d) << (2 * i) for i, d in enumerate(wk)) for wk in days]


def plan_year(seed: int):
    g = rng.stream(seed, 0)
    weeks, days = [], []
    for season in SEASON_NAMES:
        counts = SEASON_COMPOSITIONS[season]
        wk = [w for w in WEEK_TYPES for _ in range(counts.get(w, 0))]
        g.shuffle(wk)
        for w in wk:
            weeks.append(w)
            days.append(_plan_week(w, g))
    return weeks, days


def compose_year(seed: int, body_weight_kg: float) -> Protocol:
    if body_weight_kg <= 0:
        raise ValueError("body weight must be positive")
    _, days = plan_year(seed)
    out = []
    for wi in range(YEAR_WEEKS):
        sc = SEASON_CLASS_OF[SEASON_NAMES[wi // 13]]
        for di, day_type in enumerate(days[wi]):
            offset = wi * WEEK_S + di * DAY_S
            for ev in _BASIS[(day_type, sc)]:
                start = offset + ev[1]
                if ev[0] == "meal":
                    out.append(Disturbance("meal", start, start + _MEAL_DURATION_S,
                                           MEAL_CHO_PER_KG[ev[2]] * body_weight_kg))
                else:
                    out.append(Disturbance("exercise", start, start + ev[2], ev[3]))
    return Protocol(id=f"northern-year/seed={seed}/bw={body_weight_kg:g}",
                    horizon_s=YEAR_WEEKS * WEEK_S, disturbances=out)


@dataclass
class AnnouncementPolicy:
    fraction_unannounced: float = 0.0
    misannouncement_factor_range: tuple = (1.0, 1.0)


def apply_announcement_policy(protocol: Protocol, policy: AnnouncementPolicy, g) -> Protocol:
    lo, hi = policy.misannouncement_factor_range
    out = []
    for d in protocol.disturbances:
        if d.kind != "meal":
            out.append(replace(d))
        elif g.random() < policy.fraction_unannounced:
            out.append(replace(d, announced=False, announced_magnitude=0.0))
        else:
            f = lo if lo == hi else g.uniform(lo, hi)
            out.append(replace(d, announced=True, announced_magnitude=d.magnitude * f))
    return Protocol(id=protocol.id, horizon_s=protocol.horizon_s, disturbances=out)


@dataclass(frozen=True)
class NorthernYearProtocol:
    announcement: AnnouncementPolicy = field(default_factory=AnnouncementPolicy)
    basis_days_path: str | None = None

    def build(self, trial_seed: int, patient) -> Protocol:
        if self.basis_days_path is not None:
            raise NotImplementedError("custom basis-day files: use the reference generator object")
        proto = compose_year(rng.derive_seed(trial_seed, patient.id, rng.ROLE_PROTOCOL),
                             patient.body_weight_kg)
        pol = self.announcement
        if pol.fraction_unannounced > 0.0 or tuple(pol.misannouncement_factor_range) != (1.0, 1.0):
            proto = apply_announcement_policy(proto, pol, rng.stream(trial_seed, patient.id,
                                                                     rng.ROLE_ANNOUNCEMENT))
        return proto

    def on_device(self) -> bool:
        """The device builder (csrc/gt_northern.cu) covers the bundled basis
        days with any announcement policy (drawn from the reference's own
        stream(trial_seed, pid, ROLE_ANNOUNCEMENT))."""
        return self.basis_days_path is None

    def describe(self) -> dict:
        return {"kind": "northern_year",
                "fraction_unannounced": self.announcement.fraction_unannounced,
                "misannouncement_factor_range": list(self.announcement.misannouncement_factor_range),
                "basis_days_path": self.basis_days_path}
