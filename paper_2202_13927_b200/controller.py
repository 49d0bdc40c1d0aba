"""Controller profiles and the device controller registry.

``ControllerHyperparameters`` keeps the reference profile's fields, defaults,
validation, packing order and content hash (controller.py:55-180) so report
metadata is byte-identical; profile objects from the reference package are
accepted anywhere a profile is expected (duck-typed on ``to_vec``).

Controllers themselves run on device: ``register_controller`` maps a
controller id to a device controller code (include/glucosim.h GT_CTRL_*),
mirroring the reference registry (controller.py:506-527).  There is no host
fallback; an id without a device implementation raises.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass, field, fields

import numpy as np
import yaml

from . import layout
from ._lib import GT_CTRL_DUAL_HORMONE, GT_CTRL_PID_PUMP


class ProfileError(ValueError):
    pass


@dataclass(frozen=True)
class ExerciseOverrides:
    setpoint: float = 8.0
    basal_factor: float = 0.5
    gluc_threshold: float = 5.5
    microbolus_ug: float = 50.0


@dataclass(frozen=True)
class ControllerHyperparameters:
    filter_coeff: float = 0.35
    setpoint: float = 6.0
    gluc_threshold: float = 4.5
    mode_hysteresis: float = 0.5
    predict_horizon_min: float = 30.0
    basal_kp: float = 0.15
    basal_kd: float = 3.0
    basal_factor_max: float = 2.0
    superbolus_bg: float = 9.0
    superbolus_fraction: float = 0.5
    suspend_min: float = 90.0
    microbolus_ug: float = 40.0
    microbolus_lockout_min: float = 15.0
    microbolus_falling_trend: float = 0.0
    cf_per_icr: float = 0.3
    icr_initial_factor: float = 1.6
    icr_step: float = 0.05
    icr_step_up: float = 0.06
    icr_min: float = 2.0
    icr_max: float = 50.0
    meal_window_min: float = 240.0
    excursion_hi: float = 7.0
    undershoot_bg: float = 4.7
    max_bolus_u: float = 25.0
    max_glucagon_ug: float = 200.0
    exercise_bolus_ug: float = 100.0
    exercise_bolus_bg: float = 7.0
    exercise: ExerciseOverrides = field(default_factory=ExerciseOverrides)

    def __post_init__(self):
        if not 0.0 < self.filter_coeff <= 1.0:
            raise ProfileError("filter_coeff must be in (0, 1]")
        if not self.gluc_threshold < self.setpoint:
            raise ProfileError("glucagon-mode threshold must be below the setpoint")

    def to_vec(self) -> np.ndarray:
        out = []
        for name in layout.HYPER_FIELDS:
            obj = self
            for part in name.split("."):
                obj = getattr(obj, part)
            out.append(float(obj))
        return np.array(out, dtype=np.float64)

    def to_dict(self) -> dict:
        d = {"schema": "glucotrial/controller-profile/1", "controller": "dual_hormone"}
        for f in fields(self):
            if f.name == "exercise":
                ex = self.exercise
                d["exercise"] = {"setpoint": ex.setpoint, "basal_factor": ex.basal_factor,
                                 "gluc_threshold": ex.gluc_threshold,
                                 "microbolus_ug": ex.microbolus_ug}
            else:
                d[f.name] = getattr(self, f.name)
        return d

    def content_hash(self) -> str:
        blob = json.dumps(self.to_dict(), sort_keys=True).encode()
        return hashlib.sha256(blob).hexdigest()[:16]

    def scaled(self, kp_scale: float = 1.0, kd_scale: float = 1.0) -> "ControllerHyperparameters":
        """Treatment-arm variant with scaled basal PD gains (BASELINE configs[3])."""
        from dataclasses import replace
        return replace(self, basal_kp=self.basal_kp * kp_scale, basal_kd=self.basal_kd * kd_scale)


def load_profile(path: str | None = None) -> ControllerHyperparameters:
    """Profile in the reference schema ``glucotrial/controller-profile/1``."""
    if path is None:
        return ControllerHyperparameters()
    with open(path) as fh:
        raw = yaml.safe_load(fh)
    if raw.get("schema") != "glucotrial/controller-profile/1":
        raise ProfileError(f"unsupported profile schema: {raw.get('schema')!r}")
    if raw.get("controller") != "dual_hormone":
        raise ProfileError(f"profile is for controller {raw.get('controller')!r}")
    kw = {k: float(v) for k, v in raw.items() if k not in ("schema", "controller", "exercise")}
    known = {f.name for f in fields(ControllerHyperparameters)}
    if set(kw) - known:
        raise ProfileError(f"unknown profile fields: {sorted(set(kw) - known)}")
    kw["exercise"] = ExerciseOverrides(**{k: float(v) for k, v in raw.get("exercise", {}).items()})
    return ControllerHyperparameters(**kw)


def hyper_vector(profile) -> np.ndarray:
    return np.ascontiguousarray(profile.to_vec(), dtype=np.float64)


def icr_initial_factor(profile) -> float:
    return float(profile.icr_initial_factor)


def initial_icr(u_basal_u_per_h: float, profile) -> float:
    """500-rule initial insulin-to-carb ratio (controller.py:241-250)."""
    tdd = u_basal_u_per_h * 24.0 / 0.47
    icr = 500.0 / tdd * profile.icr_initial_factor
    return float(np.clip(icr, profile.icr_min, profile.icr_max))


@dataclass(frozen=True)
class DeviceController:
    """A controller the fused kernels implement: id, device code, profile."""
    controller_id: str
    code: int
    profile: object
    assumed_basal_u_per_h: float

    @property
    def hyper_vec(self) -> np.ndarray:
        return hyper_vector(self.profile)


_REGISTRY: dict = {}


def register_controller(controller_id: str, device_code: int) -> None:
    if controller_id in _REGISTRY:
        raise ValueError(f"controller id already registered: {controller_id!r}")
    _REGISTRY[controller_id] = device_code


def device_code(controller_id: str) -> int:
    try:
        return _REGISTRY[controller_id]
    except KeyError:
        raise KeyError(f"unknown controller {controller_id!r}; registered: {sorted(_REGISTRY)}") from None


def get_controller_factory(controller_id: str):
    code = device_code(controller_id)
    return lambda profile, basal: DeviceController(controller_id, code, profile, float(basal))


register_controller("dual_hormone", GT_CTRL_DUAL_HORMONE)
register_controller("pid_pump", GT_CTRL_PID_PUMP)   # pid.py: PIDProfile / PIDController
