"""PID basal controller with pump quantisation (BASELINE configs[0..2]).

The reference ships one controller, ``dual_hormone``, whose basal law is a PD
on the filtered CGM (controller.py:449-457); PID is a non-goal of its SPEC
(SURVEY.md §8.0).  This module defines the BASELINE's "PID controller at
5-min interval with pump quantisation" as a plug-in for the reference's
controller contract (``factory(profile, assumed_basal_u_per_h)`` ->
``initial_state()`` / ``step(state, y, announced_g, exercise_phase_s, t_s,
period_s)``, controller.py:466-527), so the reference's own generic engine
(``_python_block``, simulation.py:199-298) runs it.  That run is the golden
reference for the device implementations (parity kernel, fused kernel, C
oracle), which restate ``pid_step_vec`` operation by operation.

Law, once per controller period P (all in IEEE double, this order):

* filtered CGM  f = (1-a)*f + a*y          (first call: f = y; as dual_hormone)
* error e = f - setpoint;  trend = f - f_prev
* integral I = clip(I + e*P_h, -I_max, I_max)      (P_h = P / 3600)
* factor = clip(1 + kp*e + ki*I + kd*trend, 0, factor_max)
* pump: volume v = assumed_basal*factor*P_h + carry;
  pulses = max(floor(v / q_basal), 0); delivered = pulses*q_basal;
  carry = v - delivered; basal rate = delivered / P_h
* meal bolus for announced carbs: floor(min(g/ICR, max_bolus) / q_bolus)*q_bolus
* no glucagon; exercise is ignored.

The state uses the dual-hormone vector layout (controller.py:40-41), so the
device's ``gt_controller_init`` builds both controllers' initial states:
CFILT/CPREV = filtered CGM, CICR = ICR (500 rule), CSUSPEND_UNTIL = pump
carry (U), CWINEND = integral (mmol/L h), CINIT = initialised.
"""

from __future__ import annotations

import hashlib
import json
import math
from dataclasses import asdict, dataclass

import numpy as np

from .layout import CFILT, CICR, CINIT, CPREV, CSUSPEND_UNTIL, CWINEND, N_CSTATE

# hyper-vector slots (the remaining slots are 0; 17/18 are ICR min/max, shared
# with the dual-hormone layout so the initial-ICR rule reads them)
PF, PSP, PKP, PKI, PKD, PFMAX, PIMAX, PQB, PQBOL, PMAXBOL = range(10)
PICRMIN, PICRMAX = 17, 18


@dataclass(frozen=True)
class PIDProfile:
    # defaults: the best TIR - 3*TBR70 of a 108-point grid over setpoint, kp,
    # ki, kd, factor_max (tools/pid_sweep.py, 20k patients x 4 weeks, CRN):
    # TIR 84.8 %, TBR<70 1.0 %, TBR<54 0.02 %, TAR>250 2.5 %
    filter_coeff: float = 0.35
    setpoint: float = 6.5
    kp: float = 0.05            # basal factor per mmol/L
    ki: float = 0.02            # basal factor per mmol/L * h
    kd: float = 3.0             # basal factor per mmol/L change per period
    factor_max: float = 2.0
    integral_max: float = 20.0  # mmol/L * h
    basal_increment_u: float = 0.05
    bolus_increment_u: float = 0.05
    max_bolus_u: float = 25.0
    icr_initial_factor: float = 1.6
    icr_min: float = 2.0
    icr_max: float = 50.0

    def __post_init__(self):
        if not 0.0 < self.filter_coeff <= 1.0:
            raise ValueError("filter_coeff must be in (0, 1]")
        if self.basal_increment_u <= 0 or self.bolus_increment_u <= 0:
            raise ValueError("pump increments must be positive")
        if self.factor_max < 0 or self.integral_max < 0 or self.max_bolus_u < 0:
            raise ValueError("limits must be nonnegative")
        if not 0 < self.icr_min <= self.icr_max:
            raise ValueError("need 0 < icr_min <= icr_max")

    def to_vec(self) -> np.ndarray:
        v = np.zeros(30)
        v[PF], v[PSP], v[PKP], v[PKI], v[PKD] = (self.filter_coeff, self.setpoint, self.kp, self.ki,
                                                 self.kd)
        v[PFMAX], v[PIMAX], v[PQB], v[PQBOL] = (self.factor_max, self.integral_max, self.basal_increment_u,
                                                self.bolus_increment_u)
        v[PMAXBOL], v[PICRMIN], v[PICRMAX] = self.max_bolus_u, self.icr_min, self.icr_max
        return v

    def to_dict(self) -> dict:
        return {"controller": "pid_pump", **asdict(self)}

    def content_hash(self) -> str:
        blob = json.dumps(self.to_dict(), sort_keys=True).encode()
        return hashlib.sha256(blob).hexdigest()[:16]

    def scaled(self, gain_scale: float) -> "PIDProfile":
        """Treatment arm: kp, ki and kd scaled together (BASELINE configs[3])."""
        from dataclasses import replace
        return replace(self, kp=self.kp * gain_scale, ki=self.ki * gain_scale, kd=self.kd * gain_scale)


def pid_step_vec(c, y: float, announced_cho_g: float, exercise_phase_s: float, t_s: float,
                 period_s: float, hyper, assumed_basal_uh: float, out) -> None:
    """One controller update on the state vector ``c`` (in place); writes
    (basal U/h, bolus U, glucagon ug) to ``out``.  The device kernels and the
    C oracle restate this line by line."""
    a = hyper[PF]
    if c[CINIT] == 0.0:
        c[CFILT] = y
        c[CPREV] = y
        c[CINIT] = 1.0
    else:
        c[CPREV] = c[CFILT]
        c[CFILT] = (1.0 - a) * c[CFILT] + a * y
    filt = c[CFILT]
    e = filt - hyper[PSP]
    trend = filt - c[CPREV]
    ph = period_s / 3600.0
    integ = c[CWINEND] + e * ph
    imax = hyper[PIMAX]
    if integ > imax:
        integ = imax
    if integ < -imax:
        integ = -imax
    c[CWINEND] = integ
    factor = 1.0 + hyper[PKP] * e + hyper[PKI] * integ + hyper[PKD] * trend
    if factor < 0.0:
        factor = 0.0
    if factor > hyper[PFMAX]:
        factor = hyper[PFMAX]
    vol = assumed_basal_uh * factor * ph + c[CSUSPEND_UNTIL]
    q = hyper[PQB]
    pulses = float(math.floor(vol / q))
    if pulses < 0.0:
        pulses = 0.0
    delivered = pulses * q
    c[CSUSPEND_UNTIL] = vol - delivered
    out[0] = delivered / ph
    out[1] = 0.0
    if announced_cho_g > 0.0:
        b = announced_cho_g / c[CICR]
        if b > hyper[PMAXBOL]:
            b = hyper[PMAXBOL]
        qb = hyper[PQBOL]
        out[1] = float(math.floor(b / qb)) * qb
    out[2] = 0.0


@dataclass(frozen=True)
class PIDDecision:
    basal_rate_u_per_h: float
    insulin_bolus_u: float
    glucagon_bolus_ug: float


@dataclass
class PIDState:
    vec: np.ndarray

    def to_vec(self) -> np.ndarray:
        return self.vec.copy()


class PIDController:
    """Reference-contract controller object (controller.py:466-487 shape)."""

    controller_id = "pid_pump"

    def __init__(self, profile: PIDProfile, assumed_basal_u_per_h: float):
        self.profile = profile
        self.assumed_basal_u_per_h = float(assumed_basal_u_per_h)
        self.hyper_vec = profile.to_vec()

    def initial_state(self) -> PIDState:
        from .controller import initial_icr
        v = np.zeros(N_CSTATE)
        v[6] = -1e18   # CLASTGLUC: the dual-hormone initial value (unused by PID)
        v[CICR] = initial_icr(self.assumed_basal_u_per_h, self.profile)
        return PIDState(v)

    def step(self, state: PIDState, y_k: float, announced_cho_g: float, exercise_phase_s: float,
             t_s: float, period_s: float):
        c = state.vec.copy()
        out = [0.0, 0.0, 0.0]
        pid_step_vec(c, float(y_k), float(announced_cho_g), float(exercise_phase_s), float(t_s),
                     float(period_s), self.hyper_vec, self.assumed_basal_u_per_h, out)
        return PIDState(c), PIDDecision(out[0], out[1], out[2])
