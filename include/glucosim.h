/*
 * glucosim.h — C-ABI of the B200-native closed-loop Monte Carlo hot path
 * (paper_2202_13927_b200/csrc → libglucosim.so).
 *
 * Plain pointers and sizes only; no torch / C++ types.  All array pointers are
 * DEVICE pointers unless the name ends in `_host`.  `stream` is a cudaStream_t
 * passed as void* (NULL = legacy default stream).  Every entry point returns
 * 0 on success and a negative GT_E* code on error (message via gt_last_error);
 * nothing throws across the ABI.  Per-patient outcomes are status codes:
 * GT_STATUS_OK / GT_STATUS_NONFINITE / GT_STATUS_NO_STEADY_STATE.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/glucotrial).
 */
#ifndef GLUCOSIM_H
#define GLUCOSIM_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define GT_ABI_VERSION 4  /* 2: gt_fast_args.hyper by value; 3: dose_sum_fp [6] (128-bit); 4: gt_stage_fast */

/* layouts — hovorka.py:38-55, controller.py:32-41, analytics.py:21-37 */
#define GT_N_STATES 16
#define GT_N_PARAMS 30
#define GT_N_HYPER 30
#define GT_N_CSTATE 11
#define GT_N_RANGES 5
#define GT_N_THRESHOLDS 246
#define GT_N_BG_BINS 247
#define GT_TIR_BINS 200
#define GT_DOSE_BINS 200
#define GT_N_SCAL 4

/* per-patient status — _kernel.py:22-23 plus the SteadyStateError outcome
 * (simulation.py:507-510) */
#define GT_STATUS_OK 0
#define GT_STATUS_NONFINITE 1
#define GT_STATUS_NO_STEADY_STATE 2
#define GT_STATUS_EXCLUDED 3 /* masked out by the caller (e.g. padding) */
/* fused kernel, pid_pump: x0's glucagon states Z1/Z2 are not 0.  That
 * controller never doses glucagon, so from the fasting steady state (which
 * simulation.py:317-319 always starts from, Z1 = Z2 = 0) the glucagon chain
 * stays exactly 0 and the kernel drops it; any other x0 is refused per
 * patient (counted as aborted), never integrated wrongly. */
#define GT_STATUS_BAD_INITIAL_STATE 4

/* error codes */
#define GT_OK 0
#define GT_EINVAL -1
#define GT_ECUDA -2
#define GT_EUNSUPPORTED -3

/* protocol sources for the fast integrator */
#define GT_PROTO_CSR 0        /* compiled protocol arrays (simulation.py:142-168) */
#define GT_PROTO_THREE_MEAL 1 /* on-device 3-meal generator (BASELINE configs[0]) */

/* noise sources */
#define GT_NOISE_INJECTED 0 /* reference streams drawn on the host (rng.py:26-39) */
#define GT_NOISE_PHILOX 1   /* on-device counter-based Philox4x32-7: fixed key
                               (0xA4093822, 0x299F31D0), counter (pid, tick,
                               seed_lo, seed_hi ^ role << 24); 4 FP32 Box-Muller
                               normals per tick (3 Wiener, 1 CGM) */

/* controllers (device registry; mirrors controller.py:506-527) */
#define GT_CTRL_DUAL_HORMONE 0
#define GT_CTRL_PID_PUMP 1      /* PID basal + pump quantisation (pid.py; BASELINE's controller) */

/* ------------------------------------------------------------------ info */
int gt_abi_version(void);
/* copies the last error message of the calling thread into buf (NUL-terminated) */
int gt_last_error(char *buf, int64_t len);
int gt_device_sm_count(int device);

/* --------------------------------------------------------- steady state */
/* Replaces hovorka.steady_state (hovorka.py:201-243) incl. the scipy brentq
 * solve (hovorka.py:222-225), batched over n parameter vectors.
 * params [n][30] -> x0 [n][16], u_basal_uh [n], status [n]
 * (GT_STATUS_OK or GT_STATUS_NO_STEADY_STATE).  Bitwise identical to the
 * reference (IEEE order, no contraction). */
int gt_steady_state(int64_t n, const double *params, double target_bg, double *x0,
                    double *u_basal_uh, int32_t *status, void *stream);

/* ----------------------------------------------------- controller setup */
/* Replaces DualHormoneController.__init__ + initial_state().to_vec()
 * (controller.py:466-475, 241-250, 197-210): c0 [n][11] from the uniform
 * hyper [30] (device), the profile's icr_initial_factor (not part of the
 * packed hyper vector, controller.py:100-132) and assumed basal [n] (U/h). */
int gt_controller_init(int64_t n, const double *hyper, double icr_initial_factor,
                       const double *assumed_basal_uh,
                       double *c0, void *stream);

/* ------------------------------------------------ fused-path staging */
/* The fused kernel's launch-time inputs in one device pass (the reference
 * runs hovorka.steady_state per patient and then simulates only patients
 * with one, simulation.py:320-323, analytics.py:267-269):
 *   active[i] = (ss_status == NULL || ss_status[i] == GT_STATUS_OK)
 *   fixed[0..29] = params[0][0..29], and *mismatch = 1 when any patient's
 *   fixed block params[i][GT_FIXED_FIRST..29] differs from row 0 (NaN counts
 *   as a difference): the fused kernel folds that block into launch constants
 *   (gt_fast_args.fixed), so the caller must reject such a population.
 * All outputs are device pointers; active may be NULL. */
#define GT_FIXED_FIRST 15
int gt_stage_fast(int64_t n, const double *params, const int32_t *ss_status, int32_t *active,
                  double *fixed, int32_t *mismatch, void *stream);

/* ------------------------------------------------ parity-mode integrator */
/* Batched restatement of _simulate_arrays' fast-engine loop
 * (simulation.py:314-391) over simulate_block (_kernel.py:38-182): one
 * thread per patient, IEEE operation order, no FMA contraction; with the
 * reference's own noise injected it is bitwise identical to the reference.
 * Inputs are per-patient AoS rows; protocol is CSR (offsets [n+1]). */
typedef struct gt_parity_args {
    int64_t n;
    /* config (SimulationConfig, simulation.py:71-118) */
    double dt_s, period_s;
    int64_t period_steps, horizon_ticks, grid_step_ticks, n_days, n_grid, block_ticks;
    /* inputs */
    const double *params;        /* [n][30] */
    const double *x0;            /* [n][16] */
    const double *c0;            /* [n][11] */
    const double *hyper;         /* [30] uniform */
    const double *assumed_basal; /* [n] U/h */
    const int32_t *active;       /* [n] 0 = skip (status EXCLUDED); NULL = all */
    const int64_t *meal_off;     /* [n+1] */
    const double *meals_start, *meals_end, *meals_rate, *meals_ann;
    const int64_t *ex_off; /* [n+1] */
    const double *ex_start, *ex_end, *ex_hrr, *ex_announced;
    const double *wiener;     /* [n][horizon][3] (rows ignored where !has_noise) */
    const uint8_t *has_noise; /* [n] noise_active(p) (_kernel.py:33-35) */
    const double *meas;       /* [n][horizon/period_steps] */
    /* outputs */
    int32_t *status;    /* [n] */
    int64_t *ticks;     /* [n] accounted ticks */
    int64_t *tir_ticks; /* [n][5] */
    int64_t *bg_hist;   /* [n][247] */
    double *scal;       /* [n][4] min, max, sum, last_y */
    double *day_dose;   /* [n][n_days][3] (basal rate sum, bolus U, glucagon ug) */
    double *timeline;   /* [n][n_grid] */
    double *x_out;      /* [n][16] or NULL */
    double *c_out;      /* [n][11] or NULL */
    double *trace;      /* [n][horizon][8] or NULL (simulation.py:61-64) */
    int32_t controller; /* GT_CTRL_* (hyper/c0 in that controller's layout) */
    int32_t pad;
} gt_parity_args;
int gt_simulate_parity(const gt_parity_args *a, void *stream);

/* -------------------------------------------------- fast fused integrator */
/* The throughput path (BASELINE north_star subsystem 3): one thread per
 * patient keeps SDE state, controller state, Philox noise and metric
 * accumulators on chip for the whole horizon; HBM sees parameters in and
 * metrics out.  Same model/controller/statistics as the parity path with FMA
 * contraction and per-patient reciprocals (agreement to rounding; see
 * DESIGN.md §4 for the documented threshold ties).  Patient `i` has global id
 * pid0 + i (all RNG keys use the global id: results independent of sharding). */
typedef struct gt_meal_gen {
    double clock_s[3]; /* nominal meal clock times */
    double mean_g[3];  /* carbs mean per meal */
    double sd_g;       /* carbs SD */
    int32_t jitter_s;  /* uniform jitter half-width (integer seconds) */
    int32_t duration_s;
    uint32_t role;     /* RNG role of the meal stream */
    int32_t pad;
} gt_meal_gen;

typedef struct gt_fast_args {
    int64_t n, pid0;
    uint64_t seed;
    int32_t proto_kind, noise_kind, controller;
    /* horizon slices of the persistent schedule (0 = chosen from the SM count;
     * results are identical for any value) */
    int32_t n_slices;
    double dt_s, period_s;
    int64_t period_steps, horizon_ticks, grid_step_ticks, n_days, n_grid, hypo_min_ticks;
    uint32_t noise_role;
    /* 1 = re-run only the warps that contain a lane whose `status` (an output
     * of a previous launch over the same arrays) is GT_STATUS_NONFINITE, with
     * those lanes masked: rewrites the other lanes' outputs and the warps'
     * timeline partials so no statistic includes a diverged patient
     * (analytics.py:267-269); warps without one exit at once.
     * 2 = abort-tick pass, after the re-run: only those lanes run, with the
     * reference's per-tick state and per-step BG checks (_kernel.py:98-103,
     * 139-141), and only their `ticks` (the reference's abort tick,
     * simulation.py:381) and `status` are written.  Takes no trace. */
    int32_t rerun_diverged;
    /* Values of the non-sampled ("fixed", hovorka_distributions.yaml:46-81)
     * parameters shared by every patient of the launch, in p[30] order; the
     * fused kernel folds them into launch constants (kernel-parameter bank)
     * and ignores those columns of `params`.  Entries of sampled parameters
     * (and weight) are ignored. */
    double fixed[30];
    const double *params;        /* [n][30] */
    const double *x0;            /* [n][16] */
    const double *c0;            /* [n][11] */
    /* controller hyperparameters [30] (controller.py:100-132 packing), by
     * VALUE: the fused kernel reads them from its parameter bank (the parity
     * path's gt_parity_args.hyper is a device pointer) */
    double hyper[30];
    const double *assumed_basal; /* [n] */
    const int32_t *active;       /* [n] or NULL */
    gt_meal_gen meal_gen;        /* GT_PROTO_THREE_MEAL */
    /* GT_PROTO_CSR, tick-compiled */
    const int64_t *meal_off;
    const int32_t *meal_ks, *meal_ke, *meal_kp; /* activation / end tick, announce period */
    const double *meal_rate, *meal_ann;
    const int64_t *ex_off;
    const int32_t *ex_ks, *ex_ke;
    const double *ex_start_s, *ex_hrr, *ex_announced;
    /* GT_NOISE_INJECTED */
    const double *wiener; const uint8_t *has_noise; const double *meas;
    /* outputs: per patient, structure-of-arrays [field][n] */
    int32_t *status;        /* [n] */
    int64_t *ticks;         /* [n] */
    int32_t *bg_hist;       /* [247][n] */
    double *bg_stats;       /* [3][n] min, max, sum */
    double *day_dose;       /* [n_days][3][n] */
    int32_t *hypo_events;   /* [2][n] runs <3.9 and <3.0 mmol/L of >= hypo_min_ticks */
    double *timeline_pp;    /* [n_grid][n] or NULL */
    int64_t *timeline_warp; /* [n_grid][n_warps][3] per-warp sum/min/max (2^24 fixed point) */
    double *x_out;          /* [16][n] or NULL */
    /* Brownian aggregation (BASELINE configs[4]): with noise_agg = m > 1 each
     * step's Wiener normals are sum_{j<m} Z(m*k + j) / sqrt(m) of the fine
     * Philox stream, so a run at dt sees the same Brownian path as a run at
     * dt/m with noise_agg = 1 (the CGM normal is the fine tick's, as well).
     * precision: 0 = FP64 integrator, 1 = FP32 integrator (controller and
     * statistics stay FP64). */
    int32_t noise_agg, precision;
    /* caller-owned device scratch for the persistent schedule (claim counter,
     * per-warp slice flags, lane state saved between horizon slices), at
     * least gt_fast_scratch_bytes(n) bytes, 16-byte aligned; it is reused
     * stream-ordered by every launch.  NULL: the library allocates and frees
     * it stream-ordered per launch (cudaMallocAsync). */
    void *scratch;
    int64_t scratch_bytes;
    /* optional per-step trace, [n][horizon_ticks][8] = the parity kernel's
     * columns (t, bg, last CGM reading, meal g/min, exercise HRR, basal U/h,
     * bolus U, glucagon ug); NULL = off.  A traced launch runs unsliced. */
    double *trace;
} gt_fast_args;
int gt_simulate_fast(const gt_fast_args *a, void *stream);
/* The fused kernel's Philox noise, materialised for inspection / tests:
 * out[n][n_ticks][4] = the 4 FP32 normals of ticks k0..k0+n_ticks-1 of
 * patients pid0..pid0+n-1 (lanes 0-2 Wiener increments, 3 CGM noise), drawn by
 * the same device code as gt_simulate_fast with noise_agg = 1. */
int gt_noise_normals(int64_t n, int64_t pid0, uint64_t seed, uint32_t role, int64_t k0,
                     int64_t n_ticks, float *out, void *stream);
int64_t gt_fast_num_warps(int64_t n);
int64_t gt_fast_scratch_bytes(int64_t n);

/* --------------------------------------------------- population reduction */
/* Replaces TrialAccumulator.add_patient / merge (analytics.py:234-302) for a
 * whole shard on device: exact int64 sums, min/max, fixed-point (2^24) sums
 * with numpy rint, numpy pairwise summation of daily doses, dose histograms,
 * TIR histograms and the worst-case candidate.  Inputs are the fast
 * integrator's SoA outputs. */
typedef struct gt_reduce_args {
    int64_t n, pid0, horizon_ticks, n_days, n_grid, n_warps;
    double dt_s;
    const int32_t *status;
    const int64_t *ticks;
    const int32_t *bg_hist;   /* [247][n] */
    const double *bg_stats;   /* [3][n] */
    const double *day_dose;   /* [n_days][3][n] */
    const int32_t *hypo_events; /* [2][n] */
    const int64_t *timeline_warp; /* [n_grid][n_warps][3] */
    /* outputs (int64 exact; zero/identity-initialised by the call) */
    int64_t *counts;          /* [6] n_ok, n_aborted, sum_bg_fp (low 64 bits, unsigned),
                                 n_patient_days, sum_bg_fp carry (high 64 bits), reserved */
    int64_t *tir_ticks_total; /* [5] */
    int64_t *tir_hist;        /* [5][201] */
    int64_t *bg_hist_total;   /* [247] */
    int64_t *below_min;       /* [246] */
    int64_t *below_max;       /* [246] */
    int64_t *minmax_bg_bits;  /* [2] order-preserving int64 of min_bg / max_bg */
    int64_t *timeline;        /* [3][n_grid] sum, min, max */
    int64_t *dose_hist;       /* [3][201] */
    int64_t *dose_sum_fp;     /* [6] low 64 bits (unsigned) of the 3 fixed-point dose
                                 sums, then their 3 carry words (high 64 bits) */
    int64_t *worst;           /* [4] key_bits(min_bg), ticks_below_3, pid, found */
    /* per-patient metric arrays (optional, NULL to skip): [n] each */
    float *metric_tir;        /* fraction 3.9-10 */
    float *metric_tbr70, *metric_tbr54, *metric_tar180, *metric_tar250;
    int64_t *metric_hist;     /* [7][201] population histograms of the 5 range
                                 fractions + 2 hypo-event counts (clamped) */
    /* caller-owned device scratch (per-block worst-case candidates), at least
     * GT_REDUCE_SCRATCH_BYTES; NULL: allocated stream-ordered per call */
    void *scratch;
    int64_t scratch_bytes;
} gt_reduce_args;
#define GT_REDUCE_SCRATCH_BYTES 65536
int gt_reduce_trial(const gt_reduce_args *a, void *stream);

/* ------------------------------------------------------ population sampler */
/* Replaces population.sample_parameter_set's rejection loop
 * (population.py:207-259) and the body-weight draw of sample_patient
 * (population.py:156-173) with on-device counter-based RNG: same
 * distributions and acceptance rules (nonnegative, normals within 1 SD,
 * steady state exists, u_basal >= 0.4 U/h), different streams. */
typedef struct gt_sampler_args {
    int64_t n, pid0;
    uint64_t seed;
    int32_t n_sampled, max_attempts;
    double target_bg, min_basal_uh;
    double weight_mean, weight_sd;
    int32_t kind[16];      /* 0 normal, 1 lognormal, per sampled parameter */
    int32_t param_index[16]; /* destination index in the packed p[30] */
    double a[16], b[16];   /* normal: mean, sd; lognormal: log_mu, log_sigma */
    double fixed_params[30]; /* values of the non-sampled parameters */
    double *params;        /* [n][30] out */
    double *x0;            /* [n][16] out */
    double *u_basal_uh;    /* [n] out */
    int32_t *attempts;     /* [n] out */
    int32_t *status;       /* [n] out: 0 ok, 1 budget exhausted */
    int64_t *reject_counts; /* [4] negative, outside_sd, no_steady_state, basal (atomic) */
    /* 0 = reference semantics (budget exhausted -> status 1, PopulationError
     * on the host).  k > 0: redraw the body weight up to k times when a
     * weight admits no accepted parameter set within max_attempts (very low
     * weights cannot reach u_basal >= 0.4 U/h). */
    int32_t max_weight_redraws, pad;
} gt_sampler_args;
int gt_sample_population(const gt_sampler_args *a, void *stream);

/* -------------------------------------------------- disturbance generator */
/* Materialises the on-device 3-meal schedule of patients pid0..pid0+n-1 for
 * meals 0..n_meals-1 (export / parity of the generator itself). */
int gt_generate_meals(int64_t n, int64_t pid0, uint64_t seed, const gt_meal_gen *gen,
                      int64_t n_meals, double *start_s, double *end_s, double *carbs_g,
                      void *stream);

/* ------------------------------------------- NorthernYear protocol builder */
/* The reference's NorthernYearProtocol (simulation.py:420-453 ->
 * protocol.py:191-394, default announcement policy) for patients
 * pid0..pid0+n-1, planned on the device from the reference's own keyed numpy
 * stream (derive_seed(trial_seed, pid, 3) -> Philox4x64) and written in the
 * fused kernel's tick-compiled CSR layout at a fixed stride: patient i owns
 * records [i*GT_NY_MEALS, (i+1)*GT_NY_MEALS) and [i*GT_NY_EX, (i+1)*GT_NY_EX).
 * Events starting at or after horizon_s are inert (ticks INT_MAX).  Replaces
 * the host path generator.build -> compile_protocol -> compile_ticks. */
#define GT_NY_MEALS 1588
#define GT_NY_EX 76
typedef struct {
    int64_t n, pid0;
    uint64_t trial_seed;
    double dt_s, period_s, horizon_s;
    const double *params;           /* [n][30]; body weight = p[0] */
    int32_t *meal_ks, *meal_ke, *meal_kp;
    double *meal_rate, *meal_ann;   /* [n][GT_NY_MEALS] */
    int32_t *ex_ks, *ex_ke;
    double *ex_start_s, *ex_hrr, *ex_announced;  /* [n][GT_NY_EX] */
    int32_t *n_meals, *n_ex;        /* optional [n]: events before the horizon
                                       (n_meals = -1: week plan failed) */
    /* announcement policy (protocol.py:373-394, NorthernYearProtocol.announcement):
     * each meal of the year is left unannounced with probability
     * fraction_unannounced, else announced at magnitude x U(factor_lo,
     * factor_hi), drawn from the reference's stream(trial_seed, pid, 4).
     * fraction 0 and factors (1, 1) = the default policy (no draws). */
    double fraction_unannounced, factor_lo, factor_hi;
    uint16_t *week_days;            /* optional [52][n]: 2-bit day types
                                       (standard, active, movie, late) */
} gt_northern_args;
int gt_northern_protocol(const gt_northern_args *a, void *stream);

#ifdef __cplusplus
}
#endif
#endif
