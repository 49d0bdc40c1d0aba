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
// device population bit for bit (oracle_sample_patients; tests/test_gpu_sampler.py).
// COMPILED WITH --fmad=false (exact translation unit).
#include <algorithm>
#include <cmath>
#include "gt_ref_model.cuh"

namespace gt {

constexpr uint32_t kRoleSamplerParams = 0x12u;
constexpr uint32_t kRoleSamplerWeight = 0x13u;

__device__ __forceinline__ double u52(uint32_t a, uint32_t b) {
  const uint64_t k = ((uint64_t)(a >> 6) << 26) | (uint64_t)(b >> 6);
  return M_((double)(2 * k + 1), 1.1102230246251565404e-16);
}

// One attempt's draw of sampled value j (counter-addressed: the order in which
// an attempt's values are evaluated cannot change them).
__device__ __forceinline__ double sampled_value(const gt_sampler_args& a, int j, double z) {
  return a.kind[j] == 0 ? A_(a.a[j], M_(a.b[j], z))         // rng.normal(mean, sd)
                        : det_exp(A_(a.a[j], M_(a.b[j], z)));  // rng.lognormal(mu, sigma)
}

// Persistent, warp-cooperative rejection sampler.  Each lane holds one
// patient at a time and takes the next from a global queue (one atomic per
// warp refill) when it finishes, so no lane idles while a neighbour works
// through a long rejection chain.  A round has two phases:
//   1. cheap rules: a lane draws only the normal values of its next attempts
//      (3 of the 7 Philox blocks) and applies the reference's first two
//      rules -- any value negative (lognormals never are), a normal draw
//      outside 1 SD (85 % of all rejections) -- until an attempt survives or
//      the attempt budget runs out;
//   2. the steady-state solve (brentq) of every lane's survivor, with the
//      lognormal values drawn only now; then the u_basal rule.
// Every lane of the warp reaches phase 2 with a survivor in hand, so the
// expensive solves run converged instead of one lane at a time.  The draws
// and the order of the rules are the reference's (population.py:217-259),
// so the population is bit-identical to the one-thread-per-patient loop
// (oracle_sample_patients, tests/test_gpu_sampler.py).
__global__ void __launch_bounds__(128) sampler_kernel(gt_sampler_args a, unsigned long long* queue) {
  const int lane = threadIdx.x & 31;
  const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
  double p[GT_N_PARAMS], x[GT_N_STATES], vals[16];
  double ub = 0.0, w = 0.0;
  int64_t i = -1;                       // this lane's patient (-1: none)
  int32_t attempt = 0, total = 0, wdraw = 0;
  uint32_t wctr = 0, pid = 0;
  long long rej_neg = 0, rej_sd = 0, rej_ss = 0, rej_basal = 0;
  bool drained = false;
  auto draw_weight = [&]() {             // population.py:148-153
    w = 0.0;
    for (int t = 0; t < a.max_attempts; ++t, ++wctr) {
      const U4 r = philox4x32_10(wctr, pid, kRoleSamplerWeight, 0u, k0, k1);
      const double v = A_(a.weight_mean, M_(a.weight_sd, det_inv_norm(u52(r.x, r.y))));
      if (v > 0.0) { w = v; ++wctr; break; }
    }
    p[PW] = w;
    attempt = 0;
  };
  auto finish = [&](int status) {
    for (int k = 0; k < GT_N_PARAMS; ++k) a.params[i * GT_N_PARAMS + k] = p[k];
    for (int k = 0; k < GT_N_STATES; ++k) a.x0[i * GT_N_STATES + k] = status == 0 ? x[k] : 0.0;
    a.u_basal_uh[i] = status == 0 ? ub : 0.0;
    a.attempts[i] = total;
    a.status[i] = status;
    i = -1;
  };
  for (;;) {
    // ---- refill: lanes without a patient take the next ids from the queue
    const unsigned need = __ballot_sync(0xffffffffu, i < 0 && !drained);
    if (need) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(queue, (unsigned long long)__popc(need));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (need >> lane & 1u) {
        const int64_t next = (int64_t)base + __popc(need & ((1u << lane) - 1u));
        if (next < a.n) {
          i = next;
          pid = (uint32_t)(a.pid0 + i);
          for (int k = 0; k < GT_N_PARAMS; ++k) p[k] = a.fixed_params[k];
          total = 0; wdraw = 0; wctr = 0;
          draw_weight();
        } else {
          drained = true;
        }
      }
    }
    if (__all_sync(0xffffffffu, i < 0)) break;
    // ---- phase 1: cheap rules until a survivor (or the budget is spent)
    bool survivor = false;
    if (i >= 0) {
      while (!survivor) {
        if (attempt >= a.max_attempts || !(w > 0.0)) {
          // budget spent for this body weight: redraw it or fail
          total += attempt;
          if (wdraw < a.max_weight_redraws) { ++wdraw; draw_weight(); continue; }
          finish(1);
          break;
        }
        const uint32_t actr = (uint32_t)(total + attempt);
        bool neg = false;
        for (int q = 0; q < a.n_sampled; q += 2) {
          const bool has_normal = a.kind[q] == 0 || (q + 1 < a.n_sampled && a.kind[q + 1] == 0);
          if (!has_normal) continue;
          const U4 r = philox4x32_10(actr, pid, kRoleSamplerParams, (uint32_t)(q >> 1), k0, k1);
          if (a.kind[q] == 0) vals[q] = sampled_value(a, q, det_inv_norm(u52(r.x, r.y)));
          if (q + 1 < a.n_sampled && a.kind[q + 1] == 0)
            vals[q + 1] = sampled_value(a, q + 1, det_inv_norm(u52(r.z, r.w)));
        }
        for (int j = 0; j < a.n_sampled; ++j) neg |= a.kind[j] == 0 && vals[j] < 0.0;
        if (neg) { ++rej_neg; ++attempt; continue; }
        bool outside = false;
        for (int j = 0; j < a.n_sampled; ++j)
          if (a.kind[j] == 0 && fabs(S_(vals[j], a.a[j])) > a.b[j]) { outside = true; break; }
        if (outside) { ++rej_sd; ++attempt; continue; }
        survivor = true;
      }
    }
    // ---- phase 2: the survivors' lognormal draws and steady-state solves
    if (survivor) {
      const uint32_t actr = (uint32_t)(total + attempt);
      for (int q = 0; q < a.n_sampled; q += 2) {
        const bool has_log = a.kind[q] == 1 || (q + 1 < a.n_sampled && a.kind[q + 1] == 1);
        if (!has_log) continue;
        const U4 r = philox4x32_10(actr, pid, kRoleSamplerParams, (uint32_t)(q >> 1), k0, k1);
        if (a.kind[q] == 1) vals[q] = sampled_value(a, q, det_inv_norm(u52(r.x, r.y)));
        if (q + 1 < a.n_sampled && a.kind[q + 1] == 1)
          vals[q + 1] = sampled_value(a, q + 1, det_inv_norm(u52(r.z, r.w)));
      }
      for (int j = 0; j < a.n_sampled; ++j) p[a.param_index[j]] = vals[j];
      if (!steady_state_dev(p, a.target_bg, x, &ub)) { ++rej_ss; ++attempt; }
      else if (ub < a.min_basal_uh) { ++rej_basal; ++attempt; }
      else { total += attempt + 1; finish(0); }
    }
  }
  if (a.reject_counts) {
    const unsigned long long c[4] = {(unsigned long long)rej_neg, (unsigned long long)rej_sd,
                                     (unsigned long long)rej_ss, (unsigned long long)rej_basal};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      unsigned long long v = c[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && v) atomicAdd((unsigned long long*)&a.reject_counts[k], v);
    }
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
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gt::sampler_kernel, bs, 0);
  if (per_sm < 1) per_sm = 1;
  // persistent grid: at most one resident wave, never more lanes than patients
  const int64_t blocks = std::min<int64_t>((int64_t)sms * per_sm, (a->n + bs - 1) / bs);
  unsigned long long* queue = nullptr;
  gt_keep_pool_mapped();
  if (cudaMallocAsync(&queue, sizeof(unsigned long long), st) != cudaSuccess) {
    gt_set_error("gt_sample_population: queue allocation failed");
    return GT_ECUDA;
  }
  cudaMemsetAsync(queue, 0, sizeof(unsigned long long), st);
  gt::sampler_kernel<<<(unsigned)blocks, bs, 0, st>>>(*a, queue);
  const int e = gt_check_launch("sampler_kernel");
  cudaFreeAsync(queue, st);
  return e;
}

int gt_launch_meals(int64_t n, int64_t pid0, uint64_t seed, const gt_meal_gen* g, int64_t n_meals,
                    double* start, double* end, double* carbs, cudaStream_t st) {
  const int64_t tot = n * n_meals;
  if (tot <= 0) return GT_OK;
  const int bs = 256;
  gt::meals_kernel<<<(unsigned)((tot + bs - 1) / bs), bs, 0, st>>>(n, pid0, seed, *g, n_meals, start, end, carbs);
  return gt_check_launch("meals_kernel");
}
