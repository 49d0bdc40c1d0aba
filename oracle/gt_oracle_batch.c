/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see gt_oracle.c header).
 *
 * OpenMP batch drivers around oracle_simulate_patient:
 *   - oracle_run_batch_injected: per-patient protocol CSR + injected noise
 *     (the reference's own streams, drawn by numpy on the host), used by the
 *     parity tests at sizes the oracle finishes in seconds;
 *   - oracle_run_batch_philox: the bench workload (BASELINE configs[0..1]:
 *     3-meal generator + on-the-fly Philox4x32-7 noise) for the CPU
 *     baseline / `bench.py --impl reference` arm.  Noise and meals are
 *     generated per patient into thread-local buffers exactly as the
 *     reference generates its noise blocks per patient (simulation.py:350-357),
 *     so the timed CPU work includes noise generation.
 *
 * The Philox4x32-10 bijection (Salmon et al., SC'11 "Parallel random numbers:
 * as easy as 1, 2, 3"), the deterministic log and Acklam's inverse normal CDF
 * below restate the generator spec of the 3-meal disturbance generator
 * — an extension named by BASELINE.json configs[0] that has
 * no reference implementation ("parity unpinned" against the reference; pinned
 * against the product's Python twin and the device generator by tests).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_simulate_patient(
    double *x, double *c, const double *p, const double *hyper, double assumed_basal_uh,
    int64_t horizon_ticks, double dt_s, int64_t period_steps, double period_s,
    const double *meals_start, const double *meals_end, const double *meals_rate,
    const double *meals_ann, int64_t n_meals,
    const double *ex_start, const double *ex_end, const double *ex_hrr,
    const double *ex_announced, int64_t n_ex,
    const double *wiener, const double *meas_norm,
    int64_t *tir_ticks, int64_t *bg_hist, double *scal, double *day_dose,
    double *timeline, int64_t grid_step_ticks, double *trace, int64_t *ticks_out, int64_t *hypo);

/* ---------------------------------------------------------------- Philox */
static void philox4x32_r(const uint32_t ctr_in[4], uint32_t k0, uint32_t k1, uint32_t out[4], int rounds)
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    for (int r = 0; r < rounds; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c0 = hi1 ^ c1 ^ k0; c1 = lo1; c2 = hi0 ^ c3 ^ k1; c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void philox4x32_10(const uint32_t ctr_in[4], uint32_t k0, uint32_t k1, uint32_t out[4])
{
    philox4x32_r(ctr_in, k0, k1, out, 10);
}

void oracle_philox(const uint32_t *ctr, uint32_t k0, uint32_t k1, uint32_t *out)
{
    philox4x32_10(ctr, k0, k1, out);
}

/* Philox4x32 with R rounds (the fused kernel's noise stream uses R = 7). */
void oracle_philox_rounds(const uint32_t *ctr, uint32_t k0, uint32_t k1, uint32_t *out, int rounds)
{
    philox4x32_r(ctr, k0, k1, out, rounds);
}

/* Deterministic natural log from IEEE +,-,*,/ only (reproducible bit-for-bit
 * on any IEEE double implementation without contraction). */
double oracle_det_log(double x)
{
    int e;
    double m = frexp(x, &e); /* x = m * 2^e, m in [0.5, 1) */
    if (m < 0.70710678118654752440) { m = m * 2.0; e = e - 1; }
    double f = m - 1.0;
    double s = f / (2.0 + f);
    double z = s * s;
    double poly = 1.0 / 25.0;
    poly = 1.0 / 23.0 + z * poly;
    poly = 1.0 / 21.0 + z * poly;
    poly = 1.0 / 19.0 + z * poly;
    poly = 1.0 / 17.0 + z * poly;
    poly = 1.0 / 15.0 + z * poly;
    poly = 1.0 / 13.0 + z * poly;
    poly = 1.0 / 11.0 + z * poly;
    poly = 1.0 / 9.0 + z * poly;
    poly = 1.0 / 7.0 + z * poly;
    poly = 1.0 / 5.0 + z * poly;
    poly = 1.0 / 3.0 + z * poly;
    double logm = 2.0 * s + 2.0 * s * (z * poly);
    double de = (double)e;
    return de * 6.93147180369123816490e-01 + (de * 1.90821492927058770002e-10 + logm);
}

/* Acklam's inverse standard-normal CDF (relative error < 1.15e-9). */
double oracle_inv_norm(double p)
{
    static const double a[6] = {-3.969683028665376e+01, 2.209460984245205e+02,
                                -2.759285104469687e+02, 1.383577518672690e+02,
                                -3.066479806614716e+01, 2.506628277459239e+00};
    static const double b[5] = {-5.447609879822406e+01, 1.615858368580409e+02,
                                -1.556989798598866e+02, 6.680131188771972e+01,
                                -1.328068155288572e+01};
    static const double c[6] = {-7.784894002430293e-03, -3.223964580411365e-01,
                                -2.400758277161838e+00, -2.549732539343734e+00,
                                4.374664141464968e+00, 2.938163982698783e+00};
    static const double d[4] = {7.784695709041462e-03, 3.224671290700398e-01,
                                2.445134137142996e+00, 3.754408661907416e+00};
    const double plow = 0.02425, phigh = 1.0 - 0.02425;
    double q, r;
    if (p < plow) {
        q = sqrt(-2.0 * oracle_det_log(p));
        return (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
               ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
    }
    if (p > phigh) {
        q = sqrt(-2.0 * oracle_det_log(1.0 - p));
        return -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
               ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
    }
    q = p - 0.5;
    r = q * q;
    return (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
           (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
}

/* 3-meal generator: meal m = 3*day + slot for patient pid. */
typedef struct {
    double clock_s[3];
    double mean_g[3];
    double sd_g;
    int32_t jitter_s;
    double duration_s;
    uint32_t role;
} oracle_meal_spec;

void oracle_three_meal(const oracle_meal_spec *spec, uint64_t seed, uint32_t pid, int64_t m,
                       double *start, double *end, double *carbs)
{
    uint32_t ctr[4] = {(uint32_t)m, pid, spec->role, (uint32_t)((uint64_t)m >> 32)};
    uint32_t r[4];
    philox4x32_10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32), r);
    int64_t day = m / 3, slot = m % 3;
    uint32_t span = (uint32_t)(2 * spec->jitter_s + 1);
    int64_t jit = (int64_t)(((uint64_t)r[0] * span) >> 32) - spec->jitter_s;
    double st = (double)day * 86400.0 + spec->clock_s[slot] + (double)jit;
    uint64_t k = ((uint64_t)(r[1] >> 6) << 26) | (uint64_t)(r[2] >> 6);
    double u = ((double)(2 * k + 1)) * 1.1102230246251565404e-16; /* 2^-53 */
    double z = oracle_inv_norm(u);
    double g = spec->mean_g[slot] + spec->sd_g * z;
    if (g < 0.0) g = 0.0;
    *start = st;
    *end = st + spec->duration_s;
    *carbs = g;
}

/* ------------------------------------------------------------ batches */
int oracle_run_batch_injected(
    int64_t n, const double *params, const double *x0, const double *c0, const double *hyper,
    const double *assumed_basal, int64_t horizon_ticks, double dt_s, int64_t period_steps,
    double period_s, int64_t grid_step_ticks, int64_t n_days, int64_t n_grid,
    const int64_t *meal_off, const double *ms, const double *me, const double *mr,
    const double *ma, const int64_t *ex_off, const double *es, const double *ee,
    const double *eh, const double *ea, const double *wiener, const uint8_t *has_noise,
    const double *meas, int32_t *status, int64_t *ticks, int64_t *tir_ticks,
    int64_t *bg_hist, double *scal, double *day_dose, double *timeline, double *x_out,
    double *c_out, int32_t *hypo_events, int64_t hypo_min_ticks, double *trace, int nthreads)
{
    int64_t n_ctl = horizon_ticks / period_steps;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t i = 0; i < n; ++i) {
        double x[16], c[11];
        int64_t hypo[5] = {0, 0, 0, 0, hypo_min_ticks};
        memcpy(x, x0 + i * 16, sizeof x);
        memcpy(c, c0 + i * 11, sizeof c);
        int64_t mo = meal_off[i], eo = ex_off[i];
        status[i] = oracle_simulate_patient(
            x, c, params + i * 30, hyper, assumed_basal[i], horizon_ticks, dt_s, period_steps,
            period_s, ms + mo, me + mo, mr + mo, ma + mo, meal_off[i + 1] - mo, es + eo,
            ee + eo, eh + eo, ea + eo, ex_off[i + 1] - eo,
            has_noise[i] ? wiener + i * horizon_ticks * 3 : NULL, meas + i * n_ctl,
            tir_ticks + i * 5, bg_hist + i * 247, scal + i * 4, day_dose + i * n_days * 3,
            timeline + i * n_grid, grid_step_ticks, trace ? trace + i * horizon_ticks * 8 : NULL,
            ticks + i, hypo);
        if (hypo_events) { hypo_events[i * 2] = (int32_t)hypo[2]; hypo_events[i * 2 + 1] = (int32_t)hypo[3]; }
        if (x_out) memcpy(x_out + i * 16, x, sizeof x);
        if (c_out) memcpy(c_out + i * 11, c, sizeof c);
    }
    return 0;
}

/* Box–Muller in double (statistically equivalent to the device transform). */
static void bm_pair(uint32_t a, uint32_t b, double *z0, double *z1)
{
    double u1 = ((double)a + 0.5) * 2.3283064365386963e-10;
    double u2 = ((double)b + 0.5) * 2.3283064365386963e-10;
    double rad = sqrt(-2.0 * log(u1));
    double ang = 6.283185307179586 * u2;
    *z0 = rad * cos(ang);
    *z1 = rad * sin(ang);
}

int oracle_run_batch_philox(
    int64_t n, int64_t pid0, uint64_t seed, uint32_t noise_role, const oracle_meal_spec *spec,
    const double *params, const double *x0, const double *c0, const double *hyper,
    const double *assumed_basal, int64_t horizon_ticks, double dt_s, int64_t period_steps,
    double period_s, int64_t grid_step_ticks, int64_t n_days, int64_t n_grid,
    int32_t *status, int64_t *ticks, int64_t *tir_ticks, int64_t *bg_hist, double *scal,
    int32_t *hypo_events, int64_t hypo_min_ticks, int nthreads)
{
    int64_t n_ctl = horizon_ticks / period_steps;
    double horizon_s = (double)horizon_ticks * dt_s;
    int64_t n_meals_max = 3 * (n_days + 1);
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1)
    {
        double *wiener = (double *)malloc(sizeof(double) * horizon_ticks * 3);
        double *meas = (double *)malloc(sizeof(double) * (n_ctl + 1));
        double *mbuf = (double *)malloc(sizeof(double) * n_meals_max * 4);
        double *day_dose = (double *)malloc(sizeof(double) * n_days * 3);
        double *timeline = (double *)malloc(sizeof(double) * n_grid);
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < n; ++i) {
            uint32_t pid = (uint32_t)(pid0 + i);
            /* noise: one Philox4x32-7 call per tick -> 4 normals: 3 Wiener + 1 sensor
               (the sensor one is used on controller ticks only).  The device
               layout (csrc/gt_fast.cu philox_fast / philox_lane): fixed key,
               counter (pid, tick, seed_lo, seed_hi ^ role << 24). */
            int64_t ci = 0;
            for (int64_t k = 0; k < horizon_ticks; ++k) {
                uint32_t ctr[4] = {pid, (uint32_t)k, (uint32_t)seed,
                                   (uint32_t)(seed >> 32) ^ (noise_role << 24)};
                uint32_t r[4];
                philox4x32_r(ctr, 0xA4093822u, 0x299F31D0u, r, 7);  /* the device noise stream: 7 rounds */
                double z0, z1, z2, z3;
                bm_pair(r[0], r[1], &z0, &z1);
                bm_pair(r[2], r[3], &z2, &z3);
                wiener[k * 3 + 0] = z0; wiener[k * 3 + 1] = z1; wiener[k * 3 + 2] = z2;
                if (k % period_steps == 0) meas[ci++] = z3;
            }
            int64_t nm = 0;
            double *ms = mbuf, *me = mbuf + n_meals_max, *mr = mbuf + 2 * n_meals_max,
                   *ma = mbuf + 3 * n_meals_max;
            for (int64_t m = 0; m < n_meals_max; ++m) {
                double s, e, g;
                oracle_three_meal(spec, seed, pid, m, &s, &e, &g);
                if (s < horizon_s) {
                    ms[nm] = s; me[nm] = e; mr[nm] = g / ((e - s) / 60.0); ma[nm] = g; nm++;
                }
            }
            double x[16], c[11];
            memcpy(x, x0 + i * 16, sizeof x);
            memcpy(c, c0 + i * 11, sizeof c);
            memset(day_dose, 0, sizeof(double) * n_days * 3);
            for (int r = 0; r < 5; ++r) tir_ticks[i * 5 + r] = 0;
            for (int b = 0; b < 247; ++b) bg_hist[i * 247 + b] = 0;
            int64_t hypo[5] = {0, 0, 0, 0, hypo_min_ticks};
            status[i] = oracle_simulate_patient(
                x, c, params + i * 30, hyper, assumed_basal[i], horizon_ticks, dt_s,
                period_steps, period_s, ms, me, mr, ma, nm, NULL, NULL, NULL, NULL, 0, wiener,
                meas, tir_ticks + i * 5, bg_hist + i * 247, scal + i * 4, day_dose, timeline,
                grid_step_ticks, NULL, ticks + i, hypo);
            if (hypo_events) { hypo_events[i * 2] = (int32_t)hypo[2]; hypo_events[i * 2 + 1] = (int32_t)hypo[3]; }
        }
        free(wiener); free(meas); free(mbuf); free(day_dose); free(timeline);
    }
    return 0;
}

/* ------------------------------------------------------------ sampler twin */
/* Bitwise host twin of the device population sampler (csrc/gt_sampler.cu),
 * which restates population.py:148-173 (_positive_normal body weight) and
 * population.py:207-259 (sample_parameter_set: nonnegative values, normal
 * draws within 1 SD, a steady state at the target BG, u_basal >= 0.4 U/h)
 * with its own counter-based streams: Philox4x32-10 keyed by the trial seed,
 * counter (attempt, pid, role 0x12, pair) for the sampled values and
 * (draw, pid, role 0x13, 0) for the weight; normals by Acklam's inverse CDF of
 * a 52-bit uniform, lognormals by the deterministic exp below.  The draws are
 * counter-addressed, so the order in which an attempt's values are evaluated
 * cannot change them. */
double oracle_det_exp(double x)
{
    if (x > 709.0) return INFINITY;
    if (x < -745.0) return 0.0;
    double kf = floor(x * 1.44269504088896338700e+00 + 0.5);
    double r = (x - kf * 6.93147180369123816490e-01) - kf * 1.90821492927058770002e-10;
    static const double inv_fact[15] = {
        1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664, 0.008333333333333333,
        0.001388888888888889, 0.0001984126984126984, 2.48015873015873e-05, 2.7557319223985893e-06,
        2.755731922398589e-07, 2.505210838544172e-08, 2.08767569878681e-09, 1.6059043836821613e-10,
        1.1470745597729725e-11};
    double s = inv_fact[14];
    for (int j = 13; j >= 0; --j) s = inv_fact[j] + r * s;
    return ldexp(s, (int)kf);
}

int oracle_steady_state(const double *p, double target_bg, double *x, double *u_basal_uh);

static double u52(uint32_t a, uint32_t b)
{
    uint64_t k = ((uint64_t)(a >> 6) << 26) | (uint64_t)(b >> 6);
    return ((double)(2 * k + 1)) * 1.1102230246251565404e-16;
}

typedef struct {
    int32_t n_sampled;
    int32_t param_index[16];
    int32_t kind[16];        /* 0 normal(a = mean, b = sd), 1 lognormal(a = mu, b = sigma) */
    double a[16], b[16];
    double fixed_params[30];
    double weight_mean, weight_sd, target_bg, min_basal_uh;
    int32_t max_attempts, max_weight_redraws;
} oracle_sampler_spec;

int oracle_sample_patients(const oracle_sampler_spec *sp, uint64_t seed, int64_t pid0, int64_t n,
                           double *params, double *x0, double *ub_out, int32_t *attempts_out,
                           int32_t *status_out, int64_t *reject_counts, int nthreads)
{
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    int64_t rc0 = 0, rc1 = 0, rc2 = 0, rc3 = 0;
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads > 0 ? nthreads : 1) reduction(+:rc0, rc1, rc2, rc3)
    for (int64_t i = 0; i < n; ++i) {
        const uint32_t pid = (uint32_t)(pid0 + i);
        double p[30], x[16] = {0}, ub = 0.0;
        memcpy(p, sp->fixed_params, sizeof p);
        int status = 1;
        int32_t attempt = 0, total = 0;
        uint32_t wctr = 0;
        for (int wdraw = 0; wdraw <= sp->max_weight_redraws && status != 0; ++wdraw) {
            double w = 0.0;
            for (int t = 0; t < sp->max_attempts; ++t, ++wctr) {
                uint32_t ctr[4] = {wctr, pid, 0x13u, 0u}, r[4];
                philox4x32_10(ctr, k0, k1, r);
                double v = sp->weight_mean + sp->weight_sd * oracle_inv_norm(u52(r[0], r[1]));
                if (v > 0.0) { w = v; ++wctr; break; }
            }
            p[0] = w;
            for (attempt = 0; attempt < sp->max_attempts && w > 0.0; ++attempt) {
                const uint32_t actr = (uint32_t)(total + attempt);
                double vals[16];
                for (int q = 0; q < sp->n_sampled; q += 2) {
                    uint32_t ctr[4] = {actr, pid, 0x12u, (uint32_t)(q >> 1)}, r[4];
                    philox4x32_10(ctr, k0, k1, r);
                    double z[2] = {oracle_inv_norm(u52(r[0], r[1])), oracle_inv_norm(u52(r[2], r[3]))};
                    for (int h = 0; h < 2 && q + h < sp->n_sampled; ++h) {
                        int j = q + h;
                        vals[j] = sp->kind[j] == 0 ? sp->a[j] + sp->b[j] * z[h]
                                                   : oracle_det_exp(sp->a[j] + sp->b[j] * z[h]);
                    }
                }
                int neg = 0, outside = 0;
                for (int j = 0; j < sp->n_sampled; ++j) neg |= vals[j] < 0.0;
                if (neg) { ++rc0; continue; }
                for (int j = 0; j < sp->n_sampled; ++j)
                    if (sp->kind[j] == 0 && fabs(vals[j] - sp->a[j]) > sp->b[j]) { outside = 1; break; }
                if (outside) { ++rc1; continue; }
                for (int j = 0; j < sp->n_sampled; ++j) p[sp->param_index[j]] = vals[j];
                if (oracle_steady_state(p, sp->target_bg, x, &ub) != 0) { ++rc2; continue; }
                if (ub < sp->min_basal_uh) { ++rc3; continue; }
                status = 0;
                break;
            }
            total += status == 0 ? attempt + 1 : attempt;
        }
        memcpy(params + i * 30, p, sizeof p);
        for (int k = 0; k < 16; ++k) x0[i * 16 + k] = status == 0 ? x[k] : 0.0;
        ub_out[i] = status == 0 ? ub : 0.0;
        attempts_out[i] = total;
        status_out[i] = status;
    }
    reject_counts[0] = rc0; reject_counts[1] = rc1; reject_counts[2] = rc2; reject_counts[3] = rc3;
    return 0;
}
