"""Trial records, population queries (CPU) -- records.py restating
storage.py:234-358 without the file-backed store."""

import datetime
import json

import pytest

from paper_2202_13927_b200 import records
from paper_2202_13927_b200.northern import AnnouncementPolicy, NorthernYearProtocol
from paper_2202_13927_b200.protocol import ThreeMealProtocol


def test_record_round_trip_and_schema():
    r = records.TrialRecord.create("t1", 33, "hovorka_ext", "dual_hormone", "abc", "cohort-1",
                                   NorthernYearProtocol().describe(), 1.0, {"horizon_s": 86400.0, "seed": 33})
    d = json.loads(json.dumps(r.to_dict()))
    assert d["schema"] == "glucotrial/trial-record/1"
    assert records.TrialRecord.from_dict(d) == r
    with pytest.raises(records.RecordError):
        records.TrialRecord.from_dict({**d, "schema": "glucotrial/trial-record/0"})


def test_reference_written_record_loads():
    """A record dict in the reference's layout (storage.py:273-281) loads."""
    d = {"schema": "glucotrial/trial-record/1", "trial_id": "x", "created_at": "2026-01-01T00:00:00+00:00",
         "seed": 1, "model_id": "hovorka_ext", "controller_id": "dual_hormone", "profile_hash": "h",
         "population_ref": "p", "protocol_generator": {"kind": "northern_year", "fraction_unannounced": 0.1,
                                                      "misannouncement_factor_range": [0.8, 1.2],
                                                      "basis_days_path": None},
         "basal_scale": 1.0, "config": {}, "workers_hint": 4, "engine_version": "0.1.0"}
    r = records.TrialRecord.from_dict(d)
    g = records.generator_from_spec(r.protocol_generator)
    assert isinstance(g, NorthernYearProtocol)
    assert g.announcement == AnnouncementPolicy(0.1, (0.8, 1.2))
    assert g.describe() == d["protocol_generator"]


def test_three_meal_spec_round_trip():
    g = ThreeMealProtocol(mean_g=(40.0, 60.0, 90.0), days=30)
    assert records.generator_from_spec(g.describe()) == g
    with pytest.raises(records.RecordError):
        records.generator_from_spec({"kind": "fixed"})


class _Pt:
    def __init__(self, pid, w, sex=None, height=None, dob=None):
        self.id, self.body_weight_kg, self.sex, self.height_cm, self.dob = pid, w, sex, height, dob

    def age_years(self, as_of):
        return (as_of - self.dob).days / 365.25


def test_population_filter():
    pts = [_Pt(0, 50.0, "female", 160.0, datetime.date(1990, 1, 1)),
           _Pt(1, 80.0, "male", 180.0, datetime.date(1960, 1, 1)),
           _Pt(2, 95.0, "male", 175.0, datetime.date(2000, 6, 1))]
    q = records.query_population
    assert [p.id for p in q(pts, records.PopulationFilter(min_weight_kg=60.0))] == [1, 2]
    assert [p.id for p in q(pts, records.PopulationFilter(sex="male", max_age_years=40.0))] == [2]
    assert [e[0].id for e in q([(p, None) for p in pts], records.PopulationFilter(max_height_cm=176.0))] == [0, 2]
    # the device population's (id, weight) patients work for the weight bounds
    assert len(q([_Pt(5, 70.0)], records.PopulationFilter(min_weight_kg=60.0, max_weight_kg=75.0))) == 1


def test_golden_record_profile_hash_matches_default_profile():
    from conftest import golden_bytes
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    rec = records.TrialRecord.from_dict(json.loads(golden_bytes("record_rerun.json")))
    assert rec.profile_hash == ControllerHyperparameters().content_hash()
