"""ctypes binding of libglucosim.so (include/glucosim.h).

The shared library is built in-tree by ``__graft_entry__.build()`` /
``make -C paper_2202_13927_b200/csrc``.  There is no fallback: if the library
is missing or no CUDA device is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libglucosim.so")

GT_REDUCE_SCRATCH_BYTES = 65536
GT_STATUS_OK = 0
GT_STATUS_NONFINITE = 1
GT_STATUS_NO_STEADY_STATE = 2
GT_STATUS_EXCLUDED = 3
GT_STATUS_BAD_INITIAL_STATE = 4
GT_FIXED_FIRST = 15

GT_PROTO_CSR = 0
GT_PROTO_THREE_MEAL = 1
GT_NOISE_INJECTED = 0
GT_NOISE_PHILOX = 1
GT_CTRL_DUAL_HORMONE = 0
GT_CTRL_PID_PUMP = 1

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
U32 = C.c_uint32
U64 = C.c_uint64
D = C.c_double


class MealGen(C.Structure):
    _fields_ = [
        ("clock_s", D * 3), ("mean_g", D * 3), ("sd_g", D),
        ("jitter_s", I32), ("duration_s", I32), ("role", U32), ("pad", I32),
    ]


class ParityArgs(C.Structure):
    _fields_ = [
        ("n", I64), ("dt_s", D), ("period_s", D),
        ("period_steps", I64), ("horizon_ticks", I64), ("grid_step_ticks", I64),
        ("n_days", I64), ("n_grid", I64), ("block_ticks", I64),
        ("params", P), ("x0", P), ("c0", P), ("hyper", P), ("assumed_basal", P), ("active", P),
        ("meal_off", P), ("meals_start", P), ("meals_end", P), ("meals_rate", P), ("meals_ann", P),
        ("ex_off", P), ("ex_start", P), ("ex_end", P), ("ex_hrr", P), ("ex_announced", P),
        ("wiener", P), ("has_noise", P), ("meas", P),
        ("status", P), ("ticks", P), ("tir_ticks", P), ("bg_hist", P), ("scal", P),
        ("day_dose", P), ("timeline", P), ("x_out", P), ("c_out", P), ("trace", P),
        ("controller", I32), ("pad", I32),
    ]


class FastArgs(C.Structure):
    _fields_ = [
        ("n", I64), ("pid0", I64), ("seed", U64),
        ("proto_kind", I32), ("noise_kind", I32), ("controller", I32),
        ("n_slices", I32),
        ("dt_s", D), ("period_s", D),
        ("period_steps", I64), ("horizon_ticks", I64), ("grid_step_ticks", I64),
        ("n_days", I64), ("n_grid", I64), ("hypo_min_ticks", I64),
        ("noise_role", U32), ("rerun_diverged", I32), ("fixed", D * 30),
        ("params", P), ("x0", P), ("c0", P), ("hyper", D * 30), ("assumed_basal", P), ("active", P),
        ("meal_gen", MealGen),
        ("meal_off", P), ("meal_ks", P), ("meal_ke", P), ("meal_kp", P),
        ("meal_rate", P), ("meal_ann", P),
        ("ex_off", P), ("ex_ks", P), ("ex_ke", P),
        ("ex_start_s", P), ("ex_hrr", P), ("ex_announced", P),
        ("wiener", P), ("has_noise", P), ("meas", P),
        ("status", P), ("ticks", P), ("bg_hist", P), ("bg_stats", P), ("day_dose", P),
        ("hypo_events", P), ("timeline_pp", P), ("timeline_warp", P), ("x_out", P),
        ("noise_agg", I32), ("precision", I32), ("scratch", P), ("scratch_bytes", I64),
        ("trace", P),
    ]


class ReduceArgs(C.Structure):
    _fields_ = [
        ("n", I64), ("pid0", I64), ("horizon_ticks", I64), ("n_days", I64), ("n_grid", I64),
        ("n_warps", I64), ("dt_s", D),
        ("status", P), ("ticks", P), ("bg_hist", P), ("bg_stats", P), ("day_dose", P),
        ("hypo_events", P), ("timeline_warp", P),
        ("counts", P), ("tir_ticks_total", P), ("tir_hist", P), ("bg_hist_total", P),
        ("below_min", P), ("below_max", P), ("minmax_bg_bits", P), ("timeline", P),
        ("dose_hist", P), ("dose_sum_fp", P), ("worst", P),
        ("metric_tir", P), ("metric_tbr70", P), ("metric_tbr54", P), ("metric_tar180", P),
        ("metric_tar250", P), ("metric_hist", P), ("scratch", P), ("scratch_bytes", I64),
    ]


class SamplerArgs(C.Structure):
    _fields_ = [
        ("n", I64), ("pid0", I64), ("seed", U64), ("n_sampled", I32), ("max_attempts", I32),
        ("target_bg", D), ("min_basal_uh", D), ("weight_mean", D), ("weight_sd", D),
        ("kind", I32 * 16), ("param_index", I32 * 16), ("a", D * 16), ("b", D * 16),
        ("fixed_params", D * 30),
        ("params", P), ("x0", P), ("u_basal_uh", P), ("attempts", P), ("status", P),
        ("reject_counts", P), ("max_weight_redraws", I32), ("pad", I32),
    ]


GT_NY_MEALS = 1588
GT_NY_EX = 76


class NorthernArgs(C.Structure):
    _fields_ = [
        ("n", I64), ("pid0", I64), ("trial_seed", U64), ("dt_s", D), ("period_s", D), ("horizon_s", D),
        ("params", P), ("meal_ks", P), ("meal_ke", P), ("meal_kp", P), ("meal_rate", P), ("meal_ann", P),
        ("ex_ks", P), ("ex_ke", P), ("ex_start_s", P), ("ex_hrr", P), ("ex_announced", P),
        ("n_meals", P), ("n_ex", P), ("fraction_unannounced", D), ("factor_lo", D), ("factor_hi", D),
        ("week_days", P),
    ]


# (name, restype, argtypes) of every symbol include/glucosim.h declares
SIGNATURES = [
    ("gt_abi_version", C.c_int, []),
    ("gt_last_error", C.c_int, [C.c_char_p, I64]),
    ("gt_device_sm_count", C.c_int, [C.c_int]),
    ("gt_steady_state", C.c_int, [I64, P, D, P, P, P, P]),
    ("gt_controller_init", C.c_int, [I64, P, D, P, P, P]),
    ("gt_stage_fast", C.c_int, [I64, P, P, P, P, P, P]),
    ("gt_simulate_parity", C.c_int, [C.POINTER(ParityArgs), P]),
    ("gt_simulate_fast", C.c_int, [C.POINTER(FastArgs), P]),
    ("gt_fast_num_warps", I64, [I64]),
    ("gt_fast_scratch_bytes", I64, [I64]),
    ("gt_noise_normals", C.c_int, [I64, I64, U64, U32, I64, I64, P, P]),
    ("gt_reduce_trial", C.c_int, [C.POINTER(ReduceArgs), P]),
    ("gt_sample_population", C.c_int, [C.POINTER(SamplerArgs), P]),
    ("gt_generate_meals", C.c_int, [I64, I64, U64, C.POINTER(MealGen), I64, P, P, P, P]),
    ("gt_northern_protocol", C.c_int, [C.POINTER(NorthernArgs), P]),
]


class GlucosimError(RuntimeError):
    """Raised when a libglucosim entry point reports an error."""


_lib = None


def load(path: str | None = None):
    """Load (once) and return the ctypes handle; raises if the .so is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or os.environ.get("GLUCOSIM_LIB") or LIB_PATH
    if not os.path.exists(p):
        raise GlucosimError(
            f"libglucosim.so not built ({p}); run __graft_entry__.build() or "
            "`make -C paper_2202_13927_b200/csrc`"
        )
    lib = C.CDLL(p)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.gt_abi_version() != 4:   # include/glucosim.h GT_ABI_VERSION
        raise GlucosimError("libglucosim ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


def last_error() -> str:
    lib = load()
    buf = C.create_string_buffer(1024)
    lib.gt_last_error(buf, 1024)
    return buf.value.decode(errors="replace")


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise GlucosimError(f"{what} failed (rc={rc}): {last_error()}")
