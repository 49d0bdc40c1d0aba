// extern "C" boundary of libglucosim.so (include/glucosim.h).  Argument
// validation and error reporting live here; kernels never throw.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cmath>
#include "gt_common.cuh"

static thread_local char g_err[1024] = "";

void gt_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

int gt_check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    gt_set_error("%s: CUDA launch failed: %s", what, cudaGetErrorString(e));
    return GT_ECUDA;
  }
  return GT_OK;
}

void gt_keep_pool_mapped() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
}

int gt_launch_parity(const gt_parity_args* a, cudaStream_t st);
int gt_launch_steady_state(int64_t n, const double* params, double target_bg, double* x0,
                           double* ub, int32_t* status, cudaStream_t st);
int gt_launch_controller_init(int64_t n, const double* hyper, double icr_initial_factor,
                              const double* basal, double* c0, cudaStream_t st);
int gt_launch_stage_fast(int64_t n, const double* params, const int32_t* ss_status, int32_t* active,
                         double* fixed, int32_t* mismatch, cudaStream_t st);
int gt_launch_fast(const gt_fast_args* a, cudaStream_t st);
int64_t gt_fast_scratch_need(int64_t n);
int gt_launch_noise_normals(int64_t n, int64_t pid0, uint64_t seed, uint32_t role, int64_t k0,
                            int64_t n_ticks, float* out, cudaStream_t st);
int gt_launch_northern(const gt_northern_args* a, cudaStream_t st);
int gt_launch_reduce(const gt_reduce_args* a, void* scratch_worst, int nblk, cudaStream_t st);
int gt_launch_sampler(const gt_sampler_args* a, cudaStream_t st);
int gt_launch_meals(int64_t n, int64_t pid0, uint64_t seed, const gt_meal_gen* g, int64_t n_meals,
                    double* start, double* end, double* carbs, cudaStream_t st);

#define REQUIRE(cond, ...)                 \
  do {                                     \
    if (!(cond)) {                         \
      gt_set_error(__VA_ARGS__);           \
      return GT_EINVAL;                    \
    }                                      \
  } while (0)

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int gt_abi_version(void) { return GT_ABI_VERSION; }

int gt_last_error(char* buf, int64_t len) {
  if (!buf || len <= 0) return GT_EINVAL;
  strncpy(buf, g_err, (size_t)len - 1);
  buf[len - 1] = '\0';
  return GT_OK;
}

int gt_device_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    gt_set_error("cudaDeviceGetAttribute failed for device %d", device);
    return GT_ECUDA;
  }
  return v;
}

int gt_steady_state(int64_t n, const double* params, double target_bg, double* x0,
                    double* u_basal_uh, int32_t* status, void* stream) {
  REQUIRE(n >= 0, "gt_steady_state: n=%lld < 0", (long long)n);
  REQUIRE(n == 0 || (params && x0 && u_basal_uh && status), "gt_steady_state: null pointer");
  return gt_launch_steady_state(n, params, target_bg, x0, u_basal_uh, status, S(stream));
}

int gt_controller_init(int64_t n, const double* hyper, double icr_initial_factor,
                       const double* assumed_basal_uh, double* c0, void* stream) {
  REQUIRE(n >= 0, "gt_controller_init: n < 0");
  REQUIRE(n == 0 || (hyper && assumed_basal_uh && c0), "gt_controller_init: null pointer");
  return gt_launch_controller_init(n, hyper, icr_initial_factor, assumed_basal_uh, c0, S(stream));
}

int gt_stage_fast(int64_t n, const double* params, const int32_t* ss_status, int32_t* active, double* fixed,
                  int32_t* mismatch, void* stream) {
  REQUIRE(n >= 1, "gt_stage_fast: n=%lld < 1 (row 0 is the reference row)", (long long)n);
  REQUIRE(params && fixed && mismatch, "gt_stage_fast: null pointer");
  return gt_launch_stage_fast(n, params, ss_status, active, fixed, mismatch, S(stream));
}

static int check_config(const char* who, double dt_s, double period_s, int64_t period_steps,
                        int64_t horizon_ticks, int64_t grid_step_ticks, int64_t n_days,
                        int64_t n_grid) {
  REQUIRE(dt_s > 0 && period_s > 0, "%s: dt_s and period_s must be positive", who);
  REQUIRE(period_steps > 0, "%s: period_steps must be positive", who);
  REQUIRE(horizon_ticks > 0 && horizon_ticks % period_steps == 0,
          "%s: horizon_ticks must be a positive multiple of period_steps", who);
  REQUIRE(grid_step_ticks > 0, "%s: grid_step_ticks must be positive", who);
  REQUIRE(n_grid == (horizon_ticks + grid_step_ticks - 1) / grid_step_ticks,
          "%s: n_grid inconsistent with horizon/grid step", who);
  // the kernels index day_dose by t // 86400 without a bound: the buffer
  // must hold every day of the horizon (advisor finding r01)
  const double days = std::ceil((double)horizon_ticks * dt_s / 86400.0);
  REQUIRE(n_days == (days < 1.0 ? 1 : (int64_t)days),
          "%s: n_days must be max(1, ceil(horizon_ticks * dt_s / 86400))", who);
  return GT_OK;
}

int gt_simulate_parity(const gt_parity_args* a, void* stream) {
  REQUIRE(a, "gt_simulate_parity: null args");
  REQUIRE(a->n >= 0, "gt_simulate_parity: n < 0");
  if (a->n == 0) return GT_OK;
  if (int e = check_config("gt_simulate_parity", a->dt_s, a->period_s, a->period_steps,
                           a->horizon_ticks, a->grid_step_ticks, a->n_days, a->n_grid))
    return e;
  REQUIRE(a->block_ticks > 0 && a->block_ticks % a->period_steps == 0,
          "gt_simulate_parity: block_ticks must be a positive multiple of period_steps");
  REQUIRE(a->params && a->x0 && a->c0 && a->hyper && a->assumed_basal && a->meal_off &&
              a->ex_off && a->wiener && a->has_noise && a->meas && a->status && a->ticks &&
              a->tir_ticks && a->bg_hist && a->scal && a->day_dose && a->timeline,
          "gt_simulate_parity: null required pointer");
  REQUIRE(a->controller == GT_CTRL_DUAL_HORMONE || a->controller == GT_CTRL_PID_PUMP,
          "gt_simulate_parity: unknown controller %d", a->controller);
  return gt_launch_parity(a, S(stream));
}

int64_t gt_fast_num_warps(int64_t n) { return (n + 31) / 32; }
int64_t gt_fast_scratch_bytes(int64_t n) { return n <= 0 ? 0 : gt_fast_scratch_need(n); }

int gt_simulate_fast(const gt_fast_args* a, void* stream) {
  REQUIRE(a, "gt_simulate_fast: null args");
  REQUIRE(a->n >= 0, "gt_simulate_fast: n < 0");
  if (a->n == 0) return GT_OK;
  if (int e = check_config("gt_simulate_fast", a->dt_s, a->period_s, a->period_steps,
                           a->horizon_ticks, a->grid_step_ticks, a->n_days, a->n_grid))
    return e;
  // tick-exact time arithmetic of the fused loop
  REQUIRE(a->dt_s == std::floor(a->dt_s) && a->period_s == std::floor(a->period_s),
          "gt_simulate_fast: dt_s and period_s must be whole seconds");
  REQUIRE(std::fmod(86400.0, a->period_s) == 0.0,
          "gt_simulate_fast: the controller period must divide one day");
  REQUIRE((double)a->horizon_ticks * a->dt_s < 2147483647.0,
          "gt_simulate_fast: horizon too long for int32 tick arithmetic");
  REQUIRE(a->n_slices >= 0, "gt_simulate_fast: n_slices must be >= 0 (0 = automatic)");
  REQUIRE(a->rerun_diverged >= 0 && a->rerun_diverged <= 2,
          "gt_simulate_fast: rerun_diverged must be 0, 1 (exclusion re-run) or 2 (abort-tick pass)");
  REQUIRE(!(a->rerun_diverged == 2 && a->trace), "gt_simulate_fast: the abort-tick pass takes no trace");
  REQUIRE(a->params && a->x0 && a->c0 && a->assumed_basal && a->status && a->ticks &&
              a->bg_hist && a->bg_stats && a->day_dose && a->hypo_events && a->timeline_warp,
          "gt_simulate_fast: null required pointer");
  REQUIRE(a->controller == GT_CTRL_DUAL_HORMONE || a->controller == GT_CTRL_PID_PUMP,
          "gt_simulate_fast: unknown controller %d", a->controller);
  if (a->proto_kind == GT_PROTO_CSR)
    REQUIRE(a->meal_off && a->meal_ks && a->meal_ke && a->meal_kp && a->meal_rate &&
                a->meal_ann && a->ex_off && a->ex_ks && a->ex_ke && a->ex_start_s && a->ex_hrr &&
                a->ex_announced,
            "gt_simulate_fast: CSR protocol arrays required");
  if (a->noise_kind == GT_NOISE_INJECTED)
    REQUIRE(a->wiener && a->has_noise && a->meas, "gt_simulate_fast: injected noise arrays required");
  REQUIRE(a->hypo_min_ticks > 0, "gt_simulate_fast: hypo_min_ticks must be positive");
  return gt_launch_fast(a, S(stream));
}

int gt_reduce_trial(const gt_reduce_args* a, void* stream) {
  REQUIRE(a, "gt_reduce_trial: null args");
  REQUIRE(a->n >= 0 && a->horizon_ticks > 0 && a->n_days >= 1, "gt_reduce_trial: bad sizes");
  REQUIRE(a->n_warps == (a->n + 31) / 32, "gt_reduce_trial: n_warps must be ceil(n/32)");
  REQUIRE(a->counts && a->tir_ticks_total && a->tir_hist && a->bg_hist_total && a->below_min &&
              a->below_max && a->minmax_bg_bits && a->timeline && a->dose_hist &&
              a->dose_sum_fp && a->worst,
          "gt_reduce_trial: null output pointer");
  REQUIRE(a->n == 0 || (a->status && a->ticks && a->bg_hist && a->bg_stats && a->day_dose &&
                        a->hypo_events && (a->n_grid == 0 || a->timeline_warp)),
          "gt_reduce_trial: null input pointer");
  REQUIRE((a->metric_tir == nullptr) == (a->metric_tbr70 == nullptr),
          "gt_reduce_trial: metric arrays must be all set or all NULL");
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) sms = v;
  }
  int nblk = sms * 4;
  const int64_t need = (a->n + 255) / 256;
  if (need < nblk) nblk = (int)(need > 0 ? need : 1);
  if (nblk * 24 > GT_REDUCE_SCRATCH_BYTES) nblk = GT_REDUCE_SCRATCH_BYTES / 24;
  void* scratch = a->scratch;
  const bool own = scratch == nullptr;
  if (own) {
    gt_keep_pool_mapped();
    if (cudaMallocAsync(&scratch, (size_t)nblk * 24, S(stream)) != cudaSuccess) {
      gt_set_error("gt_reduce_trial: cudaMallocAsync failed");
      return GT_ECUDA;
    }
  } else {
    REQUIRE(a->scratch_bytes >= (int64_t)nblk * 24, "gt_reduce_trial: scratch smaller than GT_REDUCE_SCRATCH_BYTES");
  }
  const int e = gt_launch_reduce(a, scratch, nblk, S(stream));
  if (own) cudaFreeAsync(scratch, S(stream));
  return e;
}

int gt_sample_population(const gt_sampler_args* a, void* stream) {
  REQUIRE(a, "gt_sample_population: null args");
  REQUIRE(a->n >= 0 && a->max_attempts > 0, "gt_sample_population: bad sizes");
  REQUIRE(a->n == 0 || (a->params && a->x0 && a->u_basal_uh && a->attempts && a->status),
          "gt_sample_population: null output pointer");
  for (int j = 0; j < a->n_sampled && j < 16; ++j)
    REQUIRE(a->param_index[j] >= 1 && a->param_index[j] < GT_N_PARAMS && a->kind[j] >= 0 &&
                a->kind[j] <= 1,
            "gt_sample_population: bad spec for sampled parameter %d", j);
  return gt_launch_sampler(a, S(stream));
}

int gt_generate_meals(int64_t n, int64_t pid0, uint64_t seed, const gt_meal_gen* gen,
                      int64_t n_meals, double* start_s, double* end_s, double* carbs_g,
                      void* stream) {
  REQUIRE(gen && n >= 0 && n_meals >= 0, "gt_generate_meals: bad arguments");
  REQUIRE(n * n_meals == 0 || (start_s && end_s && carbs_g), "gt_generate_meals: null output");
  REQUIRE(gen->jitter_s >= 0 && gen->duration_s > 0, "gt_generate_meals: bad generator spec");
  return gt_launch_meals(n, pid0, seed, gen, n_meals, start_s, end_s, carbs_g, S(stream));
}

int gt_noise_normals(int64_t n, int64_t pid0, uint64_t seed, uint32_t role, int64_t k0, int64_t n_ticks,
                     float* out, void* stream) {
  REQUIRE(n >= 0 && n_ticks >= 0 && k0 >= 0, "gt_noise_normals: bad sizes");
  REQUIRE(n * n_ticks == 0 || out, "gt_noise_normals: null output");
  REQUIRE(k0 + n_ticks <= (int64_t)UINT32_MAX + 1, "gt_noise_normals: tick index beyond 32 bits");
  return gt_launch_noise_normals(n, pid0, seed, role, k0, n_ticks, out, S(stream));
}

int gt_northern_protocol(const gt_northern_args* a, void* stream) {
  REQUIRE(a && a->n >= 0, "gt_northern_protocol: bad arguments");
  if (a->n == 0) return GT_OK;
  REQUIRE(a->params && a->meal_ks && a->meal_ke && a->meal_kp && a->meal_rate && a->meal_ann &&
          a->ex_ks && a->ex_ke && a->ex_start_s && a->ex_hrr && a->ex_announced,
          "gt_northern_protocol: null output pointer");
  REQUIRE(a->dt_s > 0 && a->period_s > 0, "gt_northern_protocol: bad time step");
  return gt_launch_northern(a, S(stream));
}

}  // extern "C"
