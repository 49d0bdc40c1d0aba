"""Algorithmic FP64 work of the hot path, counted from the reference code.

A "flop" is one FP64 add, subtract, multiply or divide of the reference's
arithmetic (compares / min / max count 0).  Per integration step
(_kernel.py:79-177): 2 (t = t0 + i*dt) + 1 (bg) + 1 (sum_bg) + 1
(t // 86400) + 1 (day basal) + drift_vec (69 on the typical branch,
hovorka.py:76-136) + diffusion_diag 3 + 16 x (x += f*dt) 32 + 3 x
(x += sig*sqrt(dt)*w) 9 = 119.  Per controller tick: controller_step_vec
15 (typical) + y 2 + u conversions 7 + announcement horizon 1 = 25.
tests/golden/flop_counts.json holds the drift/controller counts measured by
an op-counting float over the reference's own functions (make_golden.py);
tests/test_flops.py pins these constants to it.  The BASELINE's PID
controller (pid.py, run by the reference's generic engine) takes 22 on its
typical branch (no meal bolus), counted the same way over pid_step_vec.
"""

DRIFT_TYPICAL = 69
CONTROLLER_TYPICAL = 15
STEP_OTHER = 2 + 1 + 1 + 1 + 1 + 3 + 32 + 9
STEP = STEP_OTHER + DRIFT_TYPICAL            # 119
TICK = CONTROLLER_TYPICAL + 2 + 7 + 1        # 25
PID_CONTROLLER_TYPICAL = 22
PID_TICK = PID_CONTROLLER_TYPICAL + 2 + 7 + 1   # 32


# Structurally-zero work, counted (not hand-typed) by a known-value float over
# the reference's drift_vec (tests/golden/flop_counts.json, make_golden.py
# _structural_counts): an op whose result a known 0 / 1 operand fixes is
# trivial.  A workload without exercise sessions (the 3-meal generator) keeps
# E1..E3 = 0 and HRR = 0 for the whole horizon; the pid_pump controller never
# doses glucagon, so Z1 = Z2 = 0 and u[2] = 0.  The fused kernel compiles those
# terms out (gt_fast.cu: HAS_EX, CTRL == GT_CTRL_PID_PUMP), so the roofline
# also reports the fraction on the work that remains ("nontrivial").
DRIFT_NOEX, DRIFT_NOGLUC, DRIFT_NOEX_NOGLUC = 54, 60, 46
ZERO_STATES_NOEX, ZERO_STATES_NOGLUC, ZERO_STATES_NOEX_NOGLUC = 3, 2, 5
TICK_TRIVIAL_NOGLUC = 1      # glucagon_ug / (period / 60) with glucagon 0 (_kernel.py:129)


def flops_per_step_nontrivial(period_steps: int, controller: str = "dual_hormone",
                              exercise: bool = False) -> float:
    """flops_per_step minus the structurally-zero terms of the workload."""
    gluc = controller != "pid_pump"
    drift, zs = {(True, True): (DRIFT_TYPICAL, 0), (False, True): (DRIFT_NOEX, ZERO_STATES_NOEX),
                 (True, False): (DRIFT_NOGLUC, ZERO_STATES_NOGLUC),
                 (False, False): (DRIFT_NOEX_NOGLUC, ZERO_STATES_NOEX_NOGLUC)}[(bool(exercise), gluc)]
    step = STEP_OTHER + drift - 2 * zs
    tick = TICK if gluc else PID_TICK - TICK_TRIVIAL_NOGLUC
    return step + tick / period_steps


def flops_per_step(period_steps: int, controller: str = "dual_hormone") -> float:
    return STEP + (PID_TICK if controller == "pid_pump" else TICK) / period_steps


def flops_per_patient_week(dt_s: float, period_steps: int, controller: str = "dual_hormone") -> float:
    return flops_per_step(period_steps, controller) * 604800.0 / dt_s
