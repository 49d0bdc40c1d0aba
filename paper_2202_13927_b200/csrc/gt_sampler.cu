// Population sampler (BASELINE north_star subsystem 1).
//
// Restates population.py:148-173 (_positive_normal body weight) and
// population.py:207-259 (sample_parameter_set rejection loop) per patient on
// device: one thread per patient, counter-based Philox4x32-10 keyed by
// (seed, global patient id), so the population is a pure function of
// (seed, n) and prefix-stable as n grows (population.py:10-13).  The
// acceptance rules are the reference's: every value nonnegative, every
// normal draw within one SD of its mean, a steady state at target BG exists
// (bitwise-exact brentq of gt_ref_model.cuh), u_basal >= 0.4 U/h.
// Normals come from Acklam's inverse CDF on 52-bit uniforms and lognormals
// from det_exp, both IEEE-op-only, so the oracle's C twin reproduces the
// device population bit for bit (tests/test_gpu_sampler.py).
// COMPILED WITH --fmad=false (exact translation unit).
#include <cmath>
#include "gt_ref_model.cuh"

namespace gt {

constexpr uint32_t kRoleSamplerParams = 0x12u;
constexpr uint32_t kRoleSamplerWeight = 0x13u;

__device__ __forceinline__ double u52(uint32_t a, uint32_t b) {
  const uint64_t k = ((uint64_t)(a >> 6) << 26) | (uint64_t)(b >> 6);
  return M_((double)(2 * k + 1), 1.1102230246251565404e-16);
}

__global__ void sampler_kernel(gt_sampler_args a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const uint32_t pid = (uint32_t)(a.pid0 + i);
  const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
  double p[GT_N_PARAMS];
  for (int k = 0; k < GT_N_PARAMS; ++k) p[k] = a.fixed_params[k];
  int status = 1;
  int32_t attempt = 0, total_attempts = 0;
  uint32_t wctr = 0;
  long long rej_neg = 0, rej_sd = 0, rej_ss = 0, rej_basal = 0;
  double x[GT_N_STATES], ub = 0.0;
  for (int wdraw = 0; wdraw <= a.max_weight_redraws && status != 0; ++wdraw) {
  // body weight: N(mean, sd) redrawn until > 0 (population.py:148-153)
  double w = 0.0;
  for (int t = 0; t < a.max_attempts; ++t, ++wctr) {
    const U4 r = philox4x32_10(wctr, pid, kRoleSamplerWeight, 0u, k0, k1);
    const double v = A_(a.weight_mean, M_(a.weight_sd, det_inv_norm(u52(r.x, r.y))));
    if (v > 0.0) { w = v; ++wctr; break; }
  }
  p[PW] = w;
  for (attempt = 0; attempt < a.max_attempts && w > 0.0; ++attempt) {
    const int32_t actr = total_attempts + attempt;
    // draw all sampled values in table order (population.py:207-214)
    double vals[16];
    for (int q = 0; q < a.n_sampled; q += 2) {
      const U4 r = philox4x32_10((uint32_t)actr, pid, kRoleSamplerParams, (uint32_t)(q >> 1), k0, k1);
      const double z0 = det_inv_norm(u52(r.x, r.y));
      const double z1 = det_inv_norm(u52(r.z, r.w));
      for (int h = 0; h < 2 && q + h < a.n_sampled; ++h) {
        const int j = q + h;
        const double z = h == 0 ? z0 : z1;
        vals[j] = a.kind[j] == 0 ? A_(a.a[j], M_(a.b[j], z))          // rng.normal(mean, sd)
                                 : det_exp(A_(a.a[j], M_(a.b[j], z)));  // rng.lognormal(mu, sigma)
      }
    }
    bool neg = false, outside = false;
    for (int j = 0; j < a.n_sampled; ++j) neg |= vals[j] < 0.0;
    if (neg) { ++rej_neg; continue; }
    for (int j = 0; j < a.n_sampled; ++j)
      if (a.kind[j] == 0 && fabs(S_(vals[j], a.a[j])) > a.b[j]) { outside = true; break; }
    if (outside) { ++rej_sd; continue; }
    for (int j = 0; j < a.n_sampled; ++j) p[a.param_index[j]] = vals[j];
    if (!steady_state_dev(p, a.target_bg, x, &ub)) { ++rej_ss; continue; }
    if (ub < a.min_basal_uh) { ++rej_basal; continue; }
    status = 0;
    break;
  }
  total_attempts += status == 0 ? attempt + 1 : attempt;
  }
  for (int k = 0; k < GT_N_PARAMS; ++k) a.params[i * GT_N_PARAMS + k] = p[k];
  for (int k = 0; k < GT_N_STATES; ++k) a.x0[i * GT_N_STATES + k] = status == 0 ? x[k] : 0.0;
  a.u_basal_uh[i] = status == 0 ? ub : 0.0;
  a.attempts[i] = total_attempts;
  a.status[i] = status;
  if (a.reject_counts) {
    if (rej_neg) atomicAdd((unsigned long long*)&a.reject_counts[0], (unsigned long long)rej_neg);
    if (rej_sd) atomicAdd((unsigned long long*)&a.reject_counts[1], (unsigned long long)rej_sd);
    if (rej_ss) atomicAdd((unsigned long long*)&a.reject_counts[2], (unsigned long long)rej_ss);
    if (rej_basal) atomicAdd((unsigned long long*)&a.reject_counts[3], (unsigned long long)rej_basal);
  }
}

// Materialise the 3-meal schedule (gt_common.cuh gen_meal).
__global__ void meals_kernel(int64_t n, int64_t pid0, uint64_t seed, gt_meal_gen g, int64_t n_meals,
                             double* start, double* end, double* carbs) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * n_meals) return;
  const int64_t i = t / n_meals, m = t - i * n_meals;
  const Meal ml = gen_meal(g, seed, (uint32_t)(pid0 + i), m);
  start[t] = ml.start; end[t] = ml.end; carbs[t] = ml.carbs;
}

}  // namespace gt

int gt_launch_sampler(const gt_sampler_args* a, cudaStream_t st) {
  if (a->n <= 0) return GT_OK;
  if (a->n_sampled < 0 || a->n_sampled > 16) {
    gt_set_error("gt_sample_population: n_sampled=%d out of range [0,16]", a->n_sampled);
    return GT_EINVAL;
  }
  const int bs = 128;
  gt::sampler_kernel<<<(unsigned)((a->n + bs - 1) / bs), bs, 0, st>>>(*a);
  return gt_check_launch("sampler_kernel");
}

int gt_launch_meals(int64_t n, int64_t pid0, uint64_t seed, const gt_meal_gen* g, int64_t n_meals,
                    double* start, double* end, double* carbs, cudaStream_t st) {
  const int64_t tot = n * n_meals;
  if (tot <= 0) return GT_OK;
  const int bs = 256;
  gt::meals_kernel<<<(unsigned)((tot + bs - 1) / bs), bs, 0, st>>>(n, pid0, seed, *g, n_meals, start, end, carbs);
  return gt_check_launch("meals_kernel");
}
