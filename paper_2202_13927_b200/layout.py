"""Packed-vector layouts shared with the kernels (include/glucosim.h).

Restates the reference conventions so packed vectors are interchangeable:
states and parameters (hovorka.py:38-62), controller hyperparameters and
state (controller.py:31-42), statistics constants (analytics.py:21-42).
"""

from __future__ import annotations

import numpy as np

STATE_NAMES = (
    "Q1_mmol", "Q2_mmol", "S1_mU", "S2_mU", "I_mU_per_L",
    "x1_per_min", "x2_per_min", "x3", "D1_mmol", "D2_mmol",
    "G_sensor_mmol_per_L", "Z1_ug", "Z2_ug", "E_hrr", "E_uptake", "E_late",
)
(IQ1, IQ2, IS1, IS2, II, IX1, IX2, IX3, ID1, ID2, IGSC, IZ1, IZ2, IE1, IE2, IE3) = range(16)
N_STATES = 16
N_WIENER = 3

PARAM_NAMES = (
    "weight_kg", "EGP0", "F01", "k12", "ka1", "ka2", "ka3", "SIT", "SID",
    "SIE", "ke", "VI", "VG", "tmaxI", "tmaxG", "AG", "tau_cgm", "t_gluc",
    "ke_gluc", "V_gluc", "S_gluc", "tau_hr", "tau_ex", "tau_late", "a_late",
    "q_ex", "s_ex", "sigma_egp", "sigma_gut", "R",
)
PARAM_INDEX = {name: i for i, name in enumerate(PARAM_NAMES)}
N_PARAMS = 30
PW, PSIGEGP, PSIGGUT, PR = 0, 27, 28, 29

# controller hyperparameter vector order (controller.py:100-132)
HYPER_FIELDS = (
    "filter_coeff", "setpoint", "gluc_threshold", "mode_hysteresis", "predict_horizon_min",
    "basal_kp", "basal_kd", "basal_factor_max", "superbolus_bg", "superbolus_fraction",
    "suspend_min", "microbolus_ug", "microbolus_lockout_min", "microbolus_falling_trend",
    "cf_per_icr", "icr_step", "icr_step_up", "icr_min", "icr_max", "meal_window_min",
    "excursion_hi", "undershoot_bg", "max_bolus_u", "max_glucagon_ug", "exercise_bolus_ug",
    "exercise_bolus_bg", "exercise.setpoint", "exercise.basal_factor",
    "exercise.gluc_threshold", "exercise.microbolus_ug",
)
N_HYPER = 30
N_CSTATE = 11
(CFILT, CPREV, CMODE, CICR, CSUSPEND_UNTIL, CEXBOLUSDONE, CLASTGLUC, CWINEND,
 CWINPEAK, CWINMIN, CINIT) = range(11)

# statistics (analytics.py:21-42)
RANGE_NAMES = ("severe_hypo", "hypo", "normo", "hyper", "severe_hyper")
RANGE_BOUNDS = np.array([3.0, 3.9, 10.0, 13.9])
N_THRESHOLDS = 246
THRESHOLDS = np.array([(5 + i) / 10 for i in range(N_THRESHOLDS)])
N_BG_BINS = N_THRESHOLDS + 1
IDX_3_MMOL = 25
TIR_BINS = 200
DOSE_SIGNALS = ("basal_u", "bolus_u", "glucagon_ug")
DOSE_BIN_WIDTH = {"basal_u": 0.5, "bolus_u": 0.5, "glucagon_ug": 10.0}
DOSE_BIN_COUNT = {"basal_u": 200, "bolus_u": 200, "glucagon_ug": 200}
FP_SCALE = 2**24
SCHEMA_REPORT = "glucotrial/trial-report/1"

TRACE_COLUMNS = (
    "t_s", "bg_mmol_per_l", "cgm_mmol_per_l", "cho_g_per_min", "hrr",
    "basal_u_per_h", "bolus_u", "glucagon_ug",
)

# BASELINE metric names over the five ranges: mg/dL labels of
# the mmol/L bounds used bit-for-bit.
METRIC_NAMES = ("tir_70_180", "tbr_lt70", "tbr_lt54", "tar_gt180", "tar_gt250",
                "hypo_events_lt70", "hypo_events_lt54")
