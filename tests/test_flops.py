"""The algorithmic FLOP constants used by the roofline are the reference's
own op counts (tests/golden/flop_counts.json, counted over the reference's
Python source by an op-counting float)."""
import json

from conftest import golden_bytes
from paper_2202_13927_b200 import flops


def test_flop_constants_pinned_to_reference_counts():
    c = json.loads(golden_bytes("flop_counts.json"))
    assert c["drift_typical"] == flops.DRIFT_TYPICAL
    assert c["controller_typical"] == flops.CONTROLLER_TYPICAL
    assert c["diffusion"] == 3
    assert flops.STEP == 119 and flops.TICK == 25
    assert abs(flops.flops_per_patient_week(60.0, 5) - 1.2499e6) < 1e3
