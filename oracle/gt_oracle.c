/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into, imported by, or called
 * from the product path (paper_2202_13927_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm
 * may load it, and only as the checker / the timed CPU baseline.
 *
 * Plain-C restatement of the reference hot path of `glucotrial` 0.1.0
 * (/root/reference/pkg/src/glucotrial).  Every function cites the reference
 * file:line it restates.  Arithmetic is written in the reference's exact
 * left-to-right operation order and must be compiled WITHOUT floating-point
 * contraction (-ffp-contract=off, no -ffast-math): numba evaluates the
 * reference in strict IEEE order without FMA, so this file is
 * bitwise identical to the numba kernel on the same inputs.
 *
 * Parity pinned by tests/golden/ (vectors produced by importing the real
 * reference in the build container: tests/golden/make_golden.py).
 *
 * Third-party algorithm restated here: scipy.optimize.brentq (scipy 1.18.1,
 * scipy/optimize/Zeros/brentq.c — Brent's method as published in scipy),
 * called by hovorka.py:222-225.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>

/* State layout: hovorka.py:38 */
enum { IQ1, IQ2, IS1, IS2, II, IX1, IX2, IX3, ID1, ID2, IGSC, IZ1, IZ2, IE1, IE2, IE3, N_STATES };
/* Parameter layout: hovorka.py:53-55 */
enum { PW, PEGP0, PF01, PK12, PKA1, PKA2, PKA3, PSIT, PSID, PSIE, PKE, PVI, PVG,
       PTMAXI, PTMAXG, PAG, PTAUCGM, PTGLUC, PKEGLUC, PVGLUC, PSGLUC, PTAUHR,
       PTAUEX, PTAULATE, PALATE, PQEX, PSEX, PSIGEGP, PSIGGUT, PR, N_PARAMS };
/* Controller hyperparameters: controller.py:32-36 */
enum { HFILTER, HSETPOINT, HGLUCTHR, HHYST, HPREDHOR, HBKP, HBKD, HBFMAX, HSUPBG,
       HSUPFRAC, HSUSPMIN, HMICROUG, HLOCKMIN, HMICROTREND, HCFICR, HICRSTEP,
       HICRSTEPUP, HICRMIN, HICRMAX, HMEALWIN, HEXCHI, HUNDERBG, HMAXBOLUS,
       HMAXGLUC, HEXBOLUS, HEXBOLUSBG, HEXSETPOINT, HEXBFACTOR, HEXGLUCTHR,
       HEXMICROUG, N_HYPER };
/* Controller state: controller.py:40-41 */
enum { CFILT, CPREV, CMODE, CICR, CSUSPEND_UNTIL, CEXBOLUSDONE, CLASTGLUC, CWINEND,
       CWINPEAK, CWINMIN, CINIT, N_CSTATE };
/* scal carry: _kernel.py:26-30 */
enum { SCAL_MIN_BG, SCAL_MAX_BG, SCAL_SUM_BG, SCAL_LAST_Y };

#define N_THRESHOLDS 246
#define N_BG_BINS 247
#define MMOL_PER_G_CHO (1000.0 / 180.16) /* hovorka.py:64 */

/* ------------------------------------------------------------------------ */
/* hovorka.py:76-136  drift_vec                                              */
void oracle_drift(const double *x, const double *u, const double *d, const double *p,
                  double *out)
{
    double w = p[PW];
    double bg = x[IQ1] / (p[PVG] * w);
    double cho_mmol = d[0] * MMOL_PER_G_CHO;
    double tmaxg = p[PTMAXG];
    out[ID1] = p[PAG] * cho_mmol - x[ID1] / tmaxg;
    out[ID2] = (x[ID1] - x[ID2]) / tmaxg;
    double gut_appearance = x[ID2] / tmaxg;

    double tmaxi = p[PTMAXI];
    double u_ins = u[0] + u[1];
    out[IS1] = u_ins - x[IS1] / tmaxi;
    out[IS2] = (x[IS1] - x[IS2]) / tmaxi;
    double plasma_appearance = x[IS2] / tmaxi;

    out[II] = plasma_appearance / (p[PVI] * w) - p[PKE] * x[II];
    out[IX1] = p[PKA1] * (p[PSIT] * x[II] - x[IX1]);
    out[IX2] = p[PKA2] * (p[PSID] * x[II] - x[IX2]);
    out[IX3] = p[PKA3] * (p[PSIE] * x[II] - x[IX3]);

    double tg = p[PTGLUC];
    out[IZ1] = u[2] - x[IZ1] / tg;
    out[IZ2] = x[IZ1] / tg - p[PKEGLUC] * x[IZ2];
    double glucagon_conc = x[IZ2] / (p[PVGLUC] * w);

    out[IE1] = (d[1] - x[IE1]) / p[PTAUHR];
    out[IE2] = (x[IE1] - x[IE2]) / p[PTAUEX];
    out[IE3] = p[PALATE] * x[IE1] - x[IE3] / p[PTAULATE];

    double f01c, renal, egp;
    if (bg < 4.5)
        f01c = p[PF01] * w * bg / 4.5;
    else
        f01c = p[PF01] * w;
    if (bg > 9.0)
        renal = 0.003 * (bg - 9.0) * p[PVG] * w;
    else
        renal = 0.0;
    egp = p[PEGP0] * w * (1.0 - x[IX3]);
    if (egp < 0.0) egp = 0.0;
    egp += p[PSGLUC] * w * glucagon_conc;
    double uptake_boost = 1.0 + p[PQEX] * x[IE2];
    double action_boost = 1.0 + p[PSEX] * x[IE3];
    double x1 = x[IX1] * action_boost;
    double x2 = x[IX2] * action_boost;
    out[IQ1] = (gut_appearance - f01c * uptake_boost - x1 * x[IQ1]
                + p[PK12] * x[IQ2] - renal + egp);
    out[IQ2] = x1 * x[IQ1] - (p[PK12] + x2) * x[IQ2];
    out[IGSC] = (bg - x[IGSC]) / p[PTAUCGM];
}

/* hovorka.py:139-150  diffusion_diag */
static void oracle_diffusion(const double *x, const double *p, double *out)
{
    out[0] = p[PSIGEGP] * p[PW];
    out[1] = p[PSIGGUT] * x[ID1];
    out[2] = p[PSIGGUT] * x[ID2];
}

/* ------------------------------------------------------------------------ */
/* controller.py:343-458  controller_step_vec                                */
void oracle_controller_step(double *c, double y, double announced_cho_g,
                            double exercise_phase_s, double t_s, double period_s,
                            const double *hyper, double assumed_basal_uh, double *out)
{
    out[0] = 0.0; out[1] = 0.0; out[2] = 0.0;
    if (c[CINIT] == 0.0) {
        c[CFILT] = y; c[CPREV] = y; c[CINIT] = 1.0;
    } else {
        c[CPREV] = c[CFILT];
        c[CFILT] = (1.0 - hyper[HFILTER]) * c[CFILT] + hyper[HFILTER] * y;
    }
    double filt = c[CFILT];
    double trend = filt - c[CPREV];

    int exercising = exercise_phase_s >= 0.0;
    double setpoint, gluc_thr, micro;
    if (exercising) {
        setpoint = hyper[HEXSETPOINT]; gluc_thr = hyper[HEXGLUCTHR]; micro = hyper[HEXMICROUG];
    } else {
        setpoint = hyper[HSETPOINT]; gluc_thr = hyper[HGLUCTHR]; micro = hyper[HMICROUG];
    }

    if (exercising) {
        if (c[CEXBOLUSDONE] == 0.0) {
            c[CEXBOLUSDONE] = 1.0;
            if (filt < hyper[HEXBOLUSBG]) {
                double g = hyper[HEXBOLUS];
                if (g > hyper[HMAXGLUC]) g = hyper[HMAXGLUC];
                out[2] = g;
                c[CLASTGLUC] = t_s;
                return;
            }
        }
    } else {
        c[CEXBOLUSDONE] = 0.0;
    }

    double pred = filt + trend * (hyper[HPREDHOR] * 60.0 / period_s);
    if (c[CMODE] == 0.0) {
        if (filt < gluc_thr || pred < gluc_thr) c[CMODE] = 1.0;
    } else {
        if (filt >= gluc_thr + hyper[HHYST] && pred >= gluc_thr) c[CMODE] = 0.0;
    }

    if (c[CWINEND] > 0.0) {
        if (filt > c[CWINPEAK]) c[CWINPEAK] = filt;
        if (filt < c[CWINMIN]) c[CWINMIN] = filt;
        if (t_s >= c[CWINEND]) {
            double icr = c[CICR];
            if (c[CWINMIN] < hyper[HUNDERBG])
                icr *= 1.0 + hyper[HICRSTEPUP];
            else if (c[CWINPEAK] - hyper[HSETPOINT] > hyper[HEXCHI])
                icr *= 1.0 - hyper[HICRSTEP];
            if (icr < hyper[HICRMIN]) icr = hyper[HICRMIN];
            if (icr > hyper[HICRMAX]) icr = hyper[HICRMAX];
            c[CICR] = icr;
            c[CWINEND] = 0.0;
        }
    }

    if (c[CMODE] == 1.0) {
        if (filt < gluc_thr && trend < -hyper[HMICROTREND]
            && t_s - c[CLASTGLUC] >= hyper[HLOCKMIN] * 60.0) {
            if (micro > hyper[HMAXGLUC]) micro = hyper[HMAXGLUC];
            out[2] = micro;
            c[CLASTGLUC] = t_s;
        }
        return;
    }

    if (announced_cho_g > 0.0) {
        double bolus = announced_cho_g / c[CICR] + (filt - setpoint) / (hyper[HCFICR] * c[CICR]);
        if (filt > hyper[HSUPBG])
            bolus += hyper[HSUPFRAC] * assumed_basal_uh * hyper[HSUSPMIN] / 60.0;
        if (bolus < 0.0) bolus = 0.0;
        if (bolus > hyper[HMAXBOLUS]) bolus = hyper[HMAXBOLUS];
        out[1] = bolus;
        c[CSUSPEND_UNTIL] = t_s + hyper[HSUSPMIN] * 60.0;
        c[CWINEND] = t_s + hyper[HMEALWIN] * 60.0;
        c[CWINPEAK] = filt;
        c[CWINMIN] = filt;
    }

    if (t_s < c[CSUSPEND_UNTIL]) {
        out[0] = 0.0;
    } else {
        double factor = 1.0 + hyper[HBKP] * (filt - setpoint) + hyper[HBKD] * trend;
        if (factor < 0.0) factor = 0.0;
        if (factor > hyper[HBFMAX]) factor = hyper[HBFMAX];
        double basal = assumed_basal_uh * factor;
        if (exercising) basal *= hyper[HEXBFACTOR];
        out[0] = basal;
    }
}

/* CPython / numba float floor division (Objects/floatobject.c float_divmod;
 * numba/cpython/numbers.py real_divmod) as used by `t // 86400.0`
 * (_kernel.py:133, :148) and `day_totals // width` (analytics.py:256). */
/* ------------------------------------------------------------------------ */
/* PID + pump quantisation (paper_2202_13927_b200/pid.py pid_step_vec): the  */
/* BASELINE controller, a plug-in the reference runs through _python_block.  */
/* Restated operation by operation; same state-vector layout.                */
void oracle_pid_step(double *c, double y, double announced_cho_g, double exercise_phase_s,
                     double t_s, double period_s, const double *hyper, double assumed_basal_uh,
                     double *out)
{
    (void)exercise_phase_s; (void)t_s;
    const double a = hyper[0];
    if (c[CINIT] == 0.0) {
        c[CFILT] = y; c[CPREV] = y; c[CINIT] = 1.0;
    } else {
        c[CPREV] = c[CFILT];
        c[CFILT] = (1.0 - a) * c[CFILT] + a * y;
    }
    const double filt = c[CFILT];
    const double e = filt - hyper[1];
    const double trend = filt - c[CPREV];
    const double ph = period_s / 3600.0;
    double integ = c[CWINEND] + e * ph;
    const double imax = hyper[6];
    if (integ > imax) integ = imax;
    if (integ < -imax) integ = -imax;
    c[CWINEND] = integ;
    double factor = 1.0 + hyper[2] * e + hyper[3] * integ + hyper[4] * trend;
    if (factor < 0.0) factor = 0.0;
    if (factor > hyper[5]) factor = hyper[5];
    const double vol = assumed_basal_uh * factor * ph + c[CSUSPEND_UNTIL];
    const double q = hyper[7];
    double pulses = floor(vol / q);
    if (pulses < 0.0) pulses = 0.0;
    const double delivered = pulses * q;
    c[CSUSPEND_UNTIL] = vol - delivered;
    out[0] = delivered / ph;
    out[1] = 0.0;
    if (announced_cho_g > 0.0) {
        double b = announced_cho_g / c[CICR];
        if (b > hyper[9]) b = hyper[9];
        out[1] = floor(b / hyper[8]) * hyper[8];
    }
    out[2] = 0.0;
}

/* controller selected for oracle_simulate_block: 0 dual_hormone, 1 pid_pump */
static int g_controller = 0;
void oracle_set_controller(int code) { g_controller = code; }

double oracle_py_floordiv(double vx, double wx)
{
    double mod = fmod(vx, wx);
    double div = (vx - mod) / wx;
    if (mod != 0.0) {
        if ((wx < 0) != (mod < 0)) { mod += wx; div -= 1.0; }
    }
    double floordiv;
    if (div != 0.0) {
        floordiv = floor(div);
        if (div - floordiv > 0.5) floordiv += 1.0;
    } else {
        floordiv = copysign(0.0, vx / wx);
    }
    return floordiv;
}

/* numpy searchsorted(side="right") on a sorted array: number of a[i] <= v. */
static int64_t searchsorted_right(const double *a, int64_t n, double v)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (v < a[mid]) hi = mid; else lo = mid + 1;
    }
    return lo;
}

/* analytics.py:21-27 constants */
static double g_range_bounds[4] = {3.0, 3.9, 10.0, 13.9};
static double g_thresholds[N_THRESHOLDS];
static int g_tables_ready = 0;
static void init_tables(void)
{
    if (g_tables_ready) return;
    for (int i = 0; i < N_THRESHOLDS; ++i) g_thresholds[i] = (double)(5 + i) / 10.0;
    g_tables_ready = 1;
}

/* ------------------------------------------------------------------------ */
/* Hypoglycaemia events (BASELINE.json north_star output; the reference has no
 * such statistic — it counts only ticks below 3 mmol/L, analytics.py:129-135).
 * Definition used throughout the repo: an event is a
 * maximal run of consecutive ticks whose BG is below 3.9 (resp. 3.0) mmol/L
 * — the statistics' BG at each tick, _kernel.py:137 — lasting at least
 * min_ticks = ceil(900 s / dt) ticks.  The run state carries across blocks.
 * hypo = {run39, run30, events39, events30, min_ticks}. */
static void hypo_update(int64_t *hypo, double bg)
{
    hypo[0] = bg < 3.9 ? hypo[0] + 1 : 0;
    hypo[1] = bg < 3.0 ? hypo[1] + 1 : 0;
    hypo[2] += hypo[0] == hypo[4];
    hypo[3] += hypo[1] == hypo[4];
}

/* ------------------------------------------------------------------------ */
/* _kernel.py:38-182  simulate_block (one patient, one block).
 * Arrays exactly as the reference: day_dose [n_days][3], trace [n][8] or NULL,
 * wiener [n][3] or NULL (has_noise = wiener != NULL), meas [n/period_steps].
 * hypo: optional hypoglycaemia-event state (hypo_update), NULL to skip. */
static int simulate_block_hypo(
    double *x, double *c, const double *p, const double *hyper, double assumed_basal_uh,
    double t0_s, int64_t n_steps, double dt_s, int64_t period_steps, double period_s,
    const double *meals_start, const double *meals_end, const double *meals_rate,
    const double *meals_ann, int64_t n_meals,
    const double *ex_start, const double *ex_end, const double *ex_hrr,
    const double *ex_announced, int64_t n_ex,
    int64_t *ptrs, const double *wiener, const double *meas_norm,
    int64_t *tir_ticks, int64_t *bg_hist, double *scal, double *day_dose,
    double *timeline, int64_t grid_step_ticks, int64_t global_tick0, double *trace, int64_t *hypo)
{
    init_tables();
    int has_noise = wiener != NULL;
    double vg_w = p[PVG] * p[PW];
    double dt_min = dt_s / 60.0;
    double sqrt_dt_min = sqrt(dt_min);
    double sqrt_r = sqrt(p[PR]);
    double f[N_STATES], sig[3], dec[3], u[3] = {0, 0, 0}, d[2] = {0, 0};
    int64_t meal_ptr = ptrs[0], ann_ptr = ptrs[1], ex_ptr = ptrs[2];
    int64_t tick_idx = 0;
    double basal_uh = 0.0;

    for (int64_t i = 0; i < n_steps; ++i) {
        double t = t0_s + (double)i * dt_s;
        int64_t global_tick = global_tick0 + i;

        while (meal_ptr < n_meals && meals_end[meal_ptr] <= t) meal_ptr++;
        if (meal_ptr < n_meals && meals_start[meal_ptr] <= t) d[0] = meals_rate[meal_ptr];
        else d[0] = 0.0;
        while (ex_ptr < n_ex && ex_end[ex_ptr] <= t) ex_ptr++;
        int ex_active = ex_ptr < n_ex && ex_start[ex_ptr] <= t;
        d[1] = ex_active ? ex_hrr[ex_ptr] : 0.0;

        double bolus_u = 0.0, glucagon_ug = 0.0;
        if (i % period_steps == 0) {
            for (int k = 0; k < N_STATES; ++k)
                if (!isfinite(x[k])) return 1;
            while (ann_ptr < n_meals && meals_start[ann_ptr] < t) ann_ptr++;
            double announced = 0.0;
            int64_t j = ann_ptr;
            while (j < n_meals && meals_start[j] < t + period_s) {
                announced += meals_ann[j];
                j++;
            }
            double phase;
            if (ex_active && ex_announced[ex_ptr] != 0.0) phase = t - ex_start[ex_ptr];
            else phase = -1.0;
            double y = x[IGSC] + sqrt_r * meas_norm[tick_idx];
            tick_idx++;
            scal[SCAL_LAST_Y] = y;
            if (g_controller == 1)
                oracle_pid_step(c, y, announced, phase, t, period_s, hyper, assumed_basal_uh, dec);
            else
                oracle_controller_step(c, y, announced, phase, t, period_s, hyper,
                                       assumed_basal_uh, dec);
            basal_uh = dec[0]; bolus_u = dec[1]; glucagon_ug = dec[2];
            u[0] = basal_uh * 1000.0 / 60.0;
            u[1] = bolus_u * 1000.0 / (period_s / 60.0);
            u[2] = glucagon_ug / (period_s / 60.0);
            if (bolus_u > 0.0 || glucagon_ug > 0.0) {
                int64_t day = (int64_t)oracle_py_floordiv(t, 86400.0);
                day_dose[day * 3 + 1] += bolus_u;
                day_dose[day * 3 + 2] += glucagon_ug;
            }
        }

        double bg = x[IQ1] / vg_w;
        if (!isfinite(bg)) return 1;
        tir_ticks[searchsorted_right(g_range_bounds, 4, bg)] += 1;
        bg_hist[searchsorted_right(g_thresholds, N_THRESHOLDS, bg)] += 1;
        if (bg < scal[SCAL_MIN_BG]) scal[SCAL_MIN_BG] = bg;
        if (bg > scal[SCAL_MAX_BG]) scal[SCAL_MAX_BG] = bg;
        scal[SCAL_SUM_BG] += bg;
        int64_t day = (int64_t)oracle_py_floordiv(t, 86400.0);
        day_dose[day * 3 + 0] += basal_uh;
        if (global_tick % grid_step_ticks == 0) timeline[global_tick / grid_step_ticks] = bg;
        if (hypo) hypo_update(hypo, bg);
        if (trace) {
            double *tr = trace + i * 8;
            tr[0] = t; tr[1] = bg; tr[2] = scal[SCAL_LAST_Y]; tr[3] = d[0]; tr[4] = d[1];
            tr[5] = basal_uh; tr[6] = bolus_u; tr[7] = glucagon_ug;
        }

        oracle_drift(x, u, d, p, f);
        if (has_noise) {
            oracle_diffusion(x, p, sig);
            for (int k = 0; k < N_STATES; ++k) x[k] += f[k] * dt_min;
            x[IQ1] += sig[0] * sqrt_dt_min * wiener[i * 3 + 0];
            x[ID1] += sig[1] * sqrt_dt_min * wiener[i * 3 + 1];
            x[ID2] += sig[2] * sqrt_dt_min * wiener[i * 3 + 2];
        } else {
            for (int k = 0; k < N_STATES; ++k) x[k] += f[k] * dt_min;
        }
        for (int k = 0; k < N_STATES; ++k)
            if (x[k] < 0.0) x[k] = 0.0;
    }
    ptrs[0] = meal_ptr; ptrs[1] = ann_ptr; ptrs[2] = ex_ptr;
    return 0;
}

/* the reference's signature (_kernel.py:38-49) */
int oracle_simulate_block(
    double *x, double *c, const double *p, const double *hyper, double assumed_basal_uh,
    double t0_s, int64_t n_steps, double dt_s, int64_t period_steps, double period_s,
    const double *meals_start, const double *meals_end, const double *meals_rate,
    const double *meals_ann, int64_t n_meals,
    const double *ex_start, const double *ex_end, const double *ex_hrr,
    const double *ex_announced, int64_t n_ex,
    int64_t *ptrs, const double *wiener, const double *meas_norm,
    int64_t *tir_ticks, int64_t *bg_hist, double *scal, double *day_dose,
    double *timeline, int64_t grid_step_ticks, int64_t global_tick0, double *trace)
{
    return simulate_block_hypo(x, c, p, hyper, assumed_basal_uh, t0_s, n_steps, dt_s, period_steps,
                               period_s, meals_start, meals_end, meals_rate, meals_ann, n_meals,
                               ex_start, ex_end, ex_hrr, ex_announced, n_ex, ptrs, wiener, meas_norm,
                               tir_ticks, bg_hist, scal, day_dose, timeline, grid_step_ticks,
                               global_tick0, trace, NULL);
}

/* ------------------------------------------------------------------------ */
/* simulation.py:314-391  _simulate_arrays, fast-engine branch, with the
 * process/measurement noise injected as whole-horizon arrays (a one-shot
 * draw equals the concatenated block draws).
 * Block size: simulation.py:345.  scal starts [inf, -inf, 0, 0] (:329).
 * Returns status 0 ok / 1 nonfinite; *ticks_out = sum(tir_ticks) (:381). */
int oracle_simulate_patient(
    double *x, double *c, const double *p, const double *hyper, double assumed_basal_uh,
    int64_t horizon_ticks, double dt_s, int64_t period_steps, double period_s,
    const double *meals_start, const double *meals_end, const double *meals_rate,
    const double *meals_ann, int64_t n_meals,
    const double *ex_start, const double *ex_end, const double *ex_hrr,
    const double *ex_announced, int64_t n_ex,
    const double *wiener, const double *meas_norm,
    int64_t *tir_ticks, int64_t *bg_hist, double *scal, double *day_dose,
    double *timeline, int64_t grid_step_ticks, double *trace, int64_t *ticks_out, int64_t *hypo)
{
    int64_t ptrs[3] = {0, 0, 0};
    scal[0] = INFINITY; scal[1] = -INFINITY; scal[2] = 0.0; scal[3] = 0.0;
    int64_t block = period_steps * ((20160 / period_steps) > 1 ? (20160 / period_steps) : 1);
    int64_t done = 0;
    int status = 0;
    while (done < horizon_ticks) {
        int64_t n = horizon_ticks - done < block ? horizon_ticks - done : block;
        status = simulate_block_hypo(
            x, c, p, hyper, assumed_basal_uh, (double)done * dt_s, n, dt_s, period_steps, period_s,
            meals_start, meals_end, meals_rate, meals_ann, n_meals,
            ex_start, ex_end, ex_hrr, ex_announced, n_ex, ptrs,
            wiener ? wiener + done * 3 : NULL, meas_norm + done / period_steps,
            tir_ticks, bg_hist, scal, day_dose, timeline, grid_step_ticks, done,
            trace ? trace + done * 8 : NULL, hypo);
        if (status != 0) break;
        done += n;
    }
    int64_t s = 0;
    for (int r = 0; r < 5; ++r) s += tir_ticks[r];
    *ticks_out = s;
    return status;
}

/* ------------------------------------------------------------------------ */
/* hovorka.py:183-198  _net_glucose_flux_at */
double oracle_net_flux(double insulin_conc, double bg, const double *p)
{
    double w = p[PW];
    double q1 = bg * p[PVG] * w;
    double x1 = p[PSIT] * insulin_conc;
    double x2 = p[PSID] * insulin_conc;
    double x3 = p[PSIE] * insulin_conc;
    double q2 = x1 * q1 / (p[PK12] + x2);
    double f01c = bg < 4.5 ? p[PF01] * w * bg / 4.5 : p[PF01] * w;
    double renal = bg > 9.0 ? 0.003 * (bg - 9.0) * p[PVG] * w : 0.0;
    double v = p[PEGP0] * w * (1.0 - x3);
    double egp = v > 0.0 ? v : 0.0; /* python max(0.0, v) keeps 0.0 unless v > 0 */
    return -f01c - x1 * q1 + p[PK12] * q2 - renal + egp;
}

/* scipy/optimize/Zeros/brentq.c (scipy 1.18.1), restated. Returns root;
 * *err = 0 converged, 1 sign error, 2 no convergence. */
static double brentq_flux(double xa, double xb, double xtol, double rtol, int iter,
                          double bg, const double *p, int *err)
{
    double xpre = xa, xcur = xb;
    double xblk = 0., fpre, fcur, fblk = 0., spre = 0., scur = 0., sbis;
    double delta, stry, dpre, dblk;
    fpre = oracle_net_flux(xpre, bg, p);
    fcur = oracle_net_flux(xcur, bg, p);
    *err = 0;
    if (isnan(fpre) || isnan(fcur)) { *err = 3; return 0.0; }
    if (fpre == 0) return xpre;
    if (fcur == 0) return xcur;
    if (signbit(fpre) == signbit(fcur)) { *err = 1; return 0.0; }
    for (int i = 0; i < iter; i++) {
        if (fpre != 0 && fcur != 0 && (signbit(fpre) != signbit(fcur))) {
            xblk = xpre; fblk = fpre;
            spre = scur = xcur - xpre;
        }
        if (fabs(fblk) < fabs(fcur)) {
            xpre = xcur; xcur = xblk; xblk = xpre;
            fpre = fcur; fcur = fblk; fblk = fpre;
        }
        delta = (xtol + rtol * fabs(xcur)) / 2;
        sbis = (xblk - xcur) / 2;
        if (fcur == 0 || fabs(sbis) < delta) return xcur;
        if (fabs(spre) > delta && fabs(fcur) < fabs(fpre)) {
            if (xpre == xblk) {
                stry = -fcur * (xcur - xpre) / (fcur - fpre);
            } else {
                dpre = (fpre - fcur) / (xpre - xcur);
                dblk = (fblk - fcur) / (xblk - xcur);
                stry = -fcur * (fblk * dblk - fpre * dpre) / (dblk * dpre * (fblk - fpre));
            }
            double m1 = fabs(spre), m2 = 3 * fabs(sbis) - delta;
            if (2 * fabs(stry) < (m1 < m2 ? m1 : m2)) {
                spre = scur; scur = stry;
            } else {
                spre = sbis; scur = sbis;
            }
        } else {
            spre = sbis; scur = sbis;
        }
        xpre = xcur; fpre = fcur;
        if (fabs(scur) > delta) xcur += scur;
        else xcur += (sbis > 0 ? delta : -delta);
        fcur = oracle_net_flux(xcur, bg, p);
        if (isnan(fcur)) { *err = 3; return 0.0; }
    }
    *err = 2;
    return xcur;
}

/* hovorka.py:201-243  steady_state.  Returns 0 ok, 1 SteadyStateError. */
int oracle_steady_state(const double *p, double target_bg, double *x, double *u_basal_uh)
{
    if (target_bg <= 0) return 1;
    double w = p[PW];
    if (oracle_net_flux(0.0, target_bg, p) <= 0.0) return 1;
    double lo = 0.0, hi = 50.0;
    int found = 0;
    for (int k = 0; k < 30; ++k) {
        if (oracle_net_flux(hi, target_bg, p) < 0.0) { found = 1; break; }
        lo = hi; hi = hi * 2.0;
    }
    if (!found) return 1;
    int err = 0;
    double ic = brentq_flux(lo, hi, 1e-14, 8.9e-16, 200, target_bg, p, &err);
    if (err) return 1; /* scipy raises RuntimeError/ValueError: not a SteadyStateError in
                          the reference, but it cannot occur on a valid bracket */
    double u_basal_mU_min = ic * p[PKE] * p[PVI] * w;
    for (int k = 0; k < N_STATES; ++k) x[k] = 0.0;
    x[IQ1] = target_bg * p[PVG] * w;
    x[II] = ic;
    x[IX1] = p[PSIT] * ic;
    x[IX2] = p[PSID] * ic;
    x[IX3] = p[PSIE] * ic;
    x[IQ2] = x[IX1] * x[IQ1] / (p[PK12] + x[IX2]);
    x[IS1] = u_basal_mU_min * p[PTMAXI];
    x[IS2] = u_basal_mU_min * p[PTMAXI];
    x[IGSC] = target_bg;
    double u[3] = {u_basal_mU_min, 0.0, 0.0}, d[2] = {0.0, 0.0}, res[N_STATES];
    oracle_drift(x, u, d, p, res);
    double worst = 0.0;
    for (int k = 0; k < N_STATES; ++k) {
        double ax = fabs(x[k]);
        double scale = ax > 1.0 ? ax : 1.0;
        double r = fabs(res[k]) / scale;
        if (isnan(r)) { worst = NAN; break; } /* np.max propagates NaN */
        if (r > worst) worst = r;
    }
    if (worst > 1e-9) return 1; /* NaN compares False: no error, as in numpy */
    *u_basal_uh = u_basal_mU_min * 60.0 / 1000.0;
    return 0;
}
