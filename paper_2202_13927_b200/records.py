"""Trial records, byte-identical re-runs and population queries on the device
engine.

Mirrors the reference's record plumbing (storage.py:229-358) without its
file-backed store, which is out of scope:

* ``TrialRecord`` has the reference's fields and schema
  (``glucotrial/trial-record/1``, storage.py:234-281), so a record written by
  the reference round-trips through ``from_dict`` / ``to_dict``.
* ``rerun_trial(store_or_population, record, ...)`` re-executes a recorded
  trial (storage.py:284-312) through this package's ``run_trial``.  Given a
  store-like object (``load_cohort`` / ``load_profile``, e.g. the reference's
  ``Store``) it loads the cohort and profile the record names, as the
  reference does; given the population and profile directly it skips the
  store.  With ``noise="reference"`` the report is byte-identical to the
  reference's own run of the same record.
* ``PopulationFilter`` / ``query_population`` restate storage.py:318-358; the
  predicates read only the attributes they need, so they also work on the
  device population's (id, body weight) patients for the weight bounds.
"""

from __future__ import annotations

import datetime
from dataclasses import dataclass, field

SCHEMA_TRIAL_RECORD = "glucotrial/trial-record/1"   # storage.py:35
ENGINE_VERSION = "glucotrial 0.1.0 / paper_2202_13927_b200 (B200 engine)"


class RecordError(RuntimeError):
    pass


@dataclass(frozen=True)
class TrialRecord:
    """Everything needed to re-run a trial bit-identically (storage.py:234-281)."""

    trial_id: str
    created_at: str
    seed: int
    model_id: str
    controller_id: str
    profile_hash: str
    population_ref: str
    protocol_generator: dict
    basal_scale: float
    config: dict
    workers_hint: int = 1
    engine_version: str = ""

    @classmethod
    def create(cls, trial_id, seed, model_id, controller_id, profile_hash, population_ref, protocol_generator,
               basal_scale, config, workers_hint=1):
        return cls(trial_id=trial_id,
                   created_at=datetime.datetime.now(datetime.timezone.utc).isoformat(),
                   seed=seed, model_id=model_id, controller_id=controller_id, profile_hash=profile_hash,
                   population_ref=population_ref, protocol_generator=dict(protocol_generator),
                   basal_scale=basal_scale, config=dict(config), workers_hint=workers_hint,
                   engine_version=ENGINE_VERSION)

    def to_dict(self) -> dict:
        return {"schema": SCHEMA_TRIAL_RECORD, **self.__dict__}

    @classmethod
    def from_dict(cls, d: dict) -> "TrialRecord":
        if d.get("schema") != SCHEMA_TRIAL_RECORD:
            raise RecordError(f"unsupported trial record schema: {d.get('schema')!r}")
        return cls(**{k: v for k, v in d.items() if k != "schema"})


def generator_from_spec(spec: dict):
    """Rebuild a protocol generator from its ``describe()`` dict: the
    reference's NorthernYear kind (storage.py:296-306) and this package's
    BASELINE 3-meal generator."""
    kind = spec.get("kind")
    if kind == "northern_year":
        from .northern import AnnouncementPolicy, NorthernYearProtocol
        return NorthernYearProtocol(
            announcement=AnnouncementPolicy(
                fraction_unannounced=spec["fraction_unannounced"],
                misannouncement_factor_range=tuple(spec["misannouncement_factor_range"])),
            basis_days_path=spec.get("basis_days_path"))
    if kind == "three_meal":
        from .protocol import ThreeMealProtocol
        return ThreeMealProtocol.from_spec(spec)
    raise RecordError(f"cannot rebuild protocol generator of kind {kind!r}")


def rerun_trial(store_or_population, record: TrialRecord, workers: int = 1, *, profile=None,
                noise: str = "reference", device=None):
    """Re-execute a recorded trial (storage.py:284-312) on the device engine.

    ``store_or_population``: a store with ``load_cohort(ref)`` and
    ``load_profile(hash)`` (the reference's ``Store`` works), or the population
    itself, in which case ``profile`` must be given.  Returns the fresh
    TrialResult; under ``noise="reference"`` its report equals the recorded
    trial's byte for byte."""
    from .config import SimulationConfig
    from .simulation import run_trial
    if hasattr(store_or_population, "load_cohort"):
        population = store_or_population.load_cohort(record.population_ref)
        profile = store_or_population.load_profile(record.profile_hash)
    else:
        population = store_or_population
        if profile is None:
            raise RecordError("rerun_trial without a store needs the profile")
    if hasattr(profile, "content_hash") and profile.content_hash() != record.profile_hash:
        raise RecordError("profile does not match the record's profile_hash")
    generator = generator_from_spec(record.protocol_generator)
    config = SimulationConfig(**record.config)
    return run_trial(population, generator, record.controller_id, profile, record.model_id, config,
                     workers=workers, basal_scale=record.basal_scale,
                     run_meta={"trial_id": record.trial_id, "population_ref": record.population_ref},
                     noise=noise, device=device)


@dataclass(frozen=True)
class PopulationFilter:
    """Conjunctive demographic predicates; None disables one (storage.py:318-346)."""

    sex: str | None = None
    min_weight_kg: float | None = None
    max_weight_kg: float | None = None
    min_height_cm: float | None = None
    max_height_cm: float | None = None
    min_age_years: float | None = None
    max_age_years: float | None = None
    as_of: datetime.date = field(default=datetime.date(2026, 1, 1))

    def matches(self, patient) -> bool:
        if self.sex is not None and patient.sex != self.sex:
            return False
        if self.min_weight_kg is not None and patient.body_weight_kg < self.min_weight_kg:
            return False
        if self.max_weight_kg is not None and patient.body_weight_kg > self.max_weight_kg:
            return False
        if self.min_height_cm is not None and patient.height_cm < self.min_height_cm:
            return False
        if self.max_height_cm is not None and patient.height_cm > self.max_height_cm:
            return False
        if self.min_age_years is not None or self.max_age_years is not None:
            age = patient.age_years(self.as_of)
            if self.min_age_years is not None and age < self.min_age_years:
                return False
            if self.max_age_years is not None and age > self.max_age_years:
                return False
        return True


def query_population(entries, flt: PopulationFilter):
    """Filter patients (or (Patient, ParameterSet) pairs) by demographics (storage.py:349-357)."""
    out = []
    for entry in entries:
        patient = entry[0] if isinstance(entry, tuple) else entry
        if flt.matches(patient):
            out.append(entry)
    return out
