// Parity-mode kernels: bitwise restatements of the reference arithmetic.
// THIS TRANSLATION UNIT IS COMPILED WITH --fmad=false (see Makefile): every
// expression keeps the reference's left-to-right IEEE order with no FMA
// contraction, IEEE division and sqrt, so with injected reference noise the
// results equal the numba kernel bit for bit.
#include <cmath>
#include "gt_ref_model.cuh"

namespace gt {

// controller.py:343-458 controller_step_vec
// PID + pump quantisation (pid.py pid_step_vec), operation by operation; this
// translation unit is compiled without contraction.
__device__ void pid_ref(double* c, double y, double announced_cho_g, double period_s,
                        const double* hyper, double assumed_basal_uh, double* out) {
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

__device__ void controller_ref(double* c, double y, double announced_cho_g, double phase,
                               double t_s, double period_s, const double* hyper,
                               double assumed_basal_uh, double* out) {
  out[0] = 0.0; out[1] = 0.0; out[2] = 0.0;
  if (c[CINIT] == 0.0) {
    c[CFILT] = y; c[CPREV] = y; c[CINIT] = 1.0;
  } else {
    c[CPREV] = c[CFILT];
    c[CFILT] = (1.0 - hyper[HFILTER]) * c[CFILT] + hyper[HFILTER] * y;
  }
  const double filt = c[CFILT];
  const double trend = filt - c[CPREV];
  const bool exercising = phase >= 0.0;
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
  const double pred = filt + trend * (hyper[HPREDHOR] * 60.0 / period_s);
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
      if (c[CWINMIN] < hyper[HUNDERBG]) icr *= 1.0 + hyper[HICRSTEPUP];
      else if (c[CWINPEAK] - hyper[HSETPOINT] > hyper[HEXCHI]) icr *= 1.0 - hyper[HICRSTEP];
      if (icr < hyper[HICRMIN]) icr = hyper[HICRMIN];
      if (icr > hyper[HICRMAX]) icr = hyper[HICRMAX];
      c[CICR] = icr;
      c[CWINEND] = 0.0;
    }
  }
  if (c[CMODE] == 1.0) {
    if (filt < gluc_thr && trend < -hyper[HMICROTREND] &&
        t_s - c[CLASTGLUC] >= hyper[HLOCKMIN] * 60.0) {
      if (micro > hyper[HMAXGLUC]) micro = hyper[HMAXGLUC];
      out[2] = micro;
      c[CLASTGLUC] = t_s;
    }
    return;
  }
  if (announced_cho_g > 0.0) {
    double bolus = announced_cho_g / c[CICR] + (filt - setpoint) / (hyper[HCFICR] * c[CICR]);
    if (filt > hyper[HSUPBG]) bolus += hyper[HSUPFRAC] * assumed_basal_uh * hyper[HSUSPMIN] / 60.0;
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

__device__ __forceinline__ int64_t searchsorted_right(const double* a, int64_t n, double v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (v < a[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}

__device__ __forceinline__ bool finite(double v) { return isfinite(v); }

// simulation.py:314-391 (fast-engine branch) driving _kernel.py:38-182 per
// block.  One thread = one patient.
__global__ void parity_kernel(gt_parity_args a) {
  __shared__ double s_thr[GT_N_THRESHOLDS];
  __shared__ double s_rb[4];
  __shared__ double s_hyper[GT_N_HYPER];
  for (int i = threadIdx.x; i < GT_N_THRESHOLDS; i += blockDim.x) s_thr[i] = (double)(5 + i) / 10.0;
  if (threadIdx.x == 0) { s_rb[0] = 3.0; s_rb[1] = 3.9; s_rb[2] = 10.0; s_rb[3] = 13.9; }
  for (int i = threadIdx.x; i < GT_N_HYPER; i += blockDim.x) s_hyper[i] = a.hyper[i];
  __syncthreads();
  const int64_t pid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pid >= a.n) return;
  if (a.active && !a.active[pid]) { a.status[pid] = GT_STATUS_EXCLUDED; a.ticks[pid] = 0; return; }

  double p[GT_N_PARAMS], x[GT_N_STATES], c[GT_N_CSTATE];
  for (int k = 0; k < GT_N_PARAMS; ++k) p[k] = a.params[pid * GT_N_PARAMS + k];
  for (int k = 0; k < GT_N_STATES; ++k) x[k] = a.x0[pid * GT_N_STATES + k];
  for (int k = 0; k < GT_N_CSTATE; ++k) c[k] = a.c0[pid * GT_N_CSTATE + k];
  const double assumed = a.assumed_basal[pid];
  int64_t* tir = a.tir_ticks + pid * GT_N_RANGES;
  int64_t* hist = a.bg_hist + pid * GT_N_BG_BINS;
  double* dd = a.day_dose + pid * a.n_days * 3;
  double* tl = a.timeline + pid * a.n_grid;
  for (int r = 0; r < GT_N_RANGES; ++r) tir[r] = 0;
  for (int b = 0; b < GT_N_BG_BINS; ++b) hist[b] = 0;
  for (int64_t k = 0; k < a.n_days * 3; ++k) dd[k] = 0.0;
  for (int64_t k = 0; k < a.n_grid; ++k) tl[k] = 0.0;
  double scal[4] = {INFINITY, -INFINITY, 0.0, 0.0};

  const int64_t mo = a.meal_off[pid], n_meals = a.meal_off[pid + 1] - mo;
  const double *ms = a.meals_start + mo, *me = a.meals_end + mo, *mr = a.meals_rate + mo,
               *ma = a.meals_ann + mo;
  const int64_t eo = a.ex_off[pid], n_ex = a.ex_off[pid + 1] - eo;
  const double *es = a.ex_start + eo, *ee = a.ex_end + eo, *eh = a.ex_hrr + eo,
               *ea = a.ex_announced + eo;
  const bool has_noise = a.has_noise[pid] != 0;
  const double* wiener = a.wiener + pid * a.horizon_ticks * 3;
  const int64_t n_ctl = a.horizon_ticks / a.period_steps;
  const double* meas = a.meas + pid * n_ctl;
  double* trace = a.trace ? a.trace + pid * a.horizon_ticks * 8 : nullptr;

  const double vg_w = p[PVG] * p[PW];
  const double dt_s = a.dt_s, period_s = a.period_s;
  const double dt_min = dt_s / 60.0;
  const double sqrt_dt_min = sqrt(dt_min);
  const double sqrt_r = sqrt(p[PR]);
  int64_t meal_ptr = 0, ann_ptr = 0, ex_ptr = 0;
  int status = GT_STATUS_OK;
  int64_t done = 0;
  while (done < a.horizon_ticks && status == GT_STATUS_OK) {
    const int64_t n = a.horizon_ticks - done < a.block_ticks ? a.horizon_ticks - done : a.block_ticks;
    const double t0_s = (double)done * dt_s;
    double u[3] = {0.0, 0.0, 0.0}, d[2] = {0.0, 0.0}, f[GT_N_STATES], dec[3];
    double basal_uh = 0.0;
    int64_t tick_idx = done / a.period_steps;
    for (int64_t i = 0; i < n; ++i) {
      const double t = t0_s + (double)i * dt_s;
      const int64_t global_tick = done + i;
      while (meal_ptr < n_meals && me[meal_ptr] <= t) meal_ptr++;
      if (meal_ptr < n_meals && ms[meal_ptr] <= t) d[0] = mr[meal_ptr];
      else d[0] = 0.0;
      while (ex_ptr < n_ex && ee[ex_ptr] <= t) ex_ptr++;
      const bool ex_active = ex_ptr < n_ex && es[ex_ptr] <= t;
      d[1] = ex_active ? eh[ex_ptr] : 0.0;
      double bolus_u = 0.0, glucagon_ug = 0.0;
      if (i % a.period_steps == 0) {
        bool bad = false;
        for (int k = 0; k < GT_N_STATES; ++k) bad |= !finite(x[k]);
        if (bad) { status = GT_STATUS_NONFINITE; break; }
        while (ann_ptr < n_meals && ms[ann_ptr] < t) ann_ptr++;
        double announced = 0.0;
        int64_t j = ann_ptr;
        while (j < n_meals && ms[j] < t + period_s) { announced += ma[j]; j++; }
        double phase;
        if (ex_active && ea[ex_ptr] != 0.0) phase = t - es[ex_ptr];
        else phase = -1.0;
        const double y = x[IGSC] + sqrt_r * meas[tick_idx];
        tick_idx++;
        scal[3] = y;
        if (a.controller == GT_CTRL_PID_PUMP)
          pid_ref(c, y, announced, period_s, s_hyper, assumed, dec);
        else
          controller_ref(c, y, announced, phase, t, period_s, s_hyper, assumed, dec);
        basal_uh = dec[0]; bolus_u = dec[1]; glucagon_ug = dec[2];
        u[0] = basal_uh * 1000.0 / 60.0;
        u[1] = bolus_u * 1000.0 / (period_s / 60.0);
        u[2] = glucagon_ug / (period_s / 60.0);
        if (bolus_u > 0.0 || glucagon_ug > 0.0) {
          const int64_t day = (int64_t)py_floordiv(t, 86400.0);
          dd[day * 3 + 1] += bolus_u;
          dd[day * 3 + 2] += glucagon_ug;
        }
      }
      const double bg = x[IQ1] / vg_w;
      if (!finite(bg)) { status = GT_STATUS_NONFINITE; break; }
      tir[searchsorted_right(s_rb, 4, bg)] += 1;
      hist[searchsorted_right(s_thr, GT_N_THRESHOLDS, bg)] += 1;
      if (bg < scal[0]) scal[0] = bg;
      if (bg > scal[1]) scal[1] = bg;
      scal[2] += bg;
      const int64_t day = (int64_t)py_floordiv(t, 86400.0);
      dd[day * 3 + 0] += basal_uh;
      if (global_tick % a.grid_step_ticks == 0) tl[global_tick / a.grid_step_ticks] = bg;
      if (trace) {
        double* tr = trace + global_tick * 8;
        tr[0] = t; tr[1] = bg; tr[2] = scal[3]; tr[3] = d[0]; tr[4] = d[1];
        tr[5] = basal_uh; tr[6] = bolus_u; tr[7] = glucagon_ug;
      }
      drift_ref(x, u, d, p, f);
      if (has_noise) {
        const double sig0 = p[PSIGEGP] * p[PW];
        const double sig1 = p[PSIGGUT] * x[ID1];
        const double sig2 = p[PSIGGUT] * x[ID2];
        for (int k = 0; k < GT_N_STATES; ++k) x[k] += f[k] * dt_min;
        const double* wv = wiener + global_tick * 3;
        x[IQ1] += sig0 * sqrt_dt_min * wv[0];
        x[ID1] += sig1 * sqrt_dt_min * wv[1];
        x[ID2] += sig2 * sqrt_dt_min * wv[2];
      } else {
        for (int k = 0; k < GT_N_STATES; ++k) x[k] += f[k] * dt_min;
      }
      for (int k = 0; k < GT_N_STATES; ++k)
        if (x[k] < 0.0) x[k] = 0.0;
    }
    if (status == GT_STATUS_OK) done += n;
  }
  int64_t s = 0;
  for (int r = 0; r < GT_N_RANGES; ++r) s += tir[r];
  a.ticks[pid] = s;
  a.status[pid] = status;
  for (int k = 0; k < 4; ++k) a.scal[pid * 4 + k] = scal[k];
  if (a.x_out) for (int k = 0; k < GT_N_STATES; ++k) a.x_out[pid * GT_N_STATES + k] = x[k];
  if (a.c_out) for (int k = 0; k < GT_N_CSTATE; ++k) a.c_out[pid * GT_N_CSTATE + k] = c[k];
}

__global__ void steady_state_kernel(int64_t n, const double* params, double target_bg,
                                    double* x0, double* ub, int32_t* status) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[GT_N_PARAMS], x[GT_N_STATES], u = 0.0;
  for (int k = 0; k < GT_N_PARAMS; ++k) p[k] = params[i * GT_N_PARAMS + k];
  const bool ok = steady_state_dev(p, target_bg, x, &u);
  for (int k = 0; k < GT_N_STATES; ++k) x0[i * GT_N_STATES + k] = ok ? x[k] : 0.0;
  ub[i] = ok ? u : 0.0;
  status[i] = ok ? GT_STATUS_OK : GT_STATUS_NO_STEADY_STATE;
}

// gt_stage_fast (include/glucosim.h): active mask + fixed-block uniformity
__global__ void stage_fast_kernel(int64_t n, const double* params, const int32_t* ss_status, int32_t* active,
                                  double* fixed, int32_t* mismatch) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0)
    for (int k = 0; k < GT_N_PARAMS; ++k) fixed[k] = params[k];
  bool diff = false;
  for (int k = GT_FIXED_FIRST; k < GT_N_PARAMS; ++k) diff |= !(params[i * GT_N_PARAMS + k] == params[k]);
  if (diff) atomicOr(mismatch, 1);
  if (active) active[i] = ss_status == nullptr || ss_status[i] == GT_STATUS_OK;
}

// controller.py:241-250 initial_icr + ControllerState defaults (:183-195,
// to_vec :197-210).  np.clip propagates NaN.
__global__ void controller_init_kernel(int64_t n, const double* hyper, double icr_initial_factor,
                                       const double* basal, double* c0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double ub = basal[i];
  const double tdd = ub * 24.0 / 0.47;
  double icr = 500.0 / tdd * icr_initial_factor;
  if (!isnan(icr)) {
    if (icr < hyper[HICRMIN]) icr = hyper[HICRMIN];
    if (icr > hyper[HICRMAX]) icr = hyper[HICRMAX];
  }
  double* c = c0 + i * GT_N_CSTATE;
  c[CFILT] = 0.0; c[CPREV] = 0.0; c[CMODE] = 0.0; c[CICR] = icr; c[CSUSPEND_UNTIL] = 0.0;
  c[CEXBOLUSDONE] = 0.0; c[CLASTGLUC] = -1e18; c[CWINEND] = 0.0; c[CWINPEAK] = 0.0;
  c[CWINMIN] = 0.0; c[CINIT] = 0.0;
}

}  // namespace gt

// ------------------------------------------------------------- launchers
static inline unsigned grid_for(int64_t n, int bs) { return (unsigned)((n + bs - 1) / bs); }

int gt_launch_parity(const gt_parity_args* a, cudaStream_t st) {
  if (a->n <= 0) return GT_OK;
  const int bs = 64;
  gt::parity_kernel<<<grid_for(a->n, bs), bs, 0, st>>>(*a);
  return gt_check_launch("parity_kernel");
}

int gt_launch_steady_state(int64_t n, const double* params, double target_bg, double* x0,
                           double* ub, int32_t* status, cudaStream_t st) {
  if (n <= 0) return GT_OK;
  const int bs = 128;
  gt::steady_state_kernel<<<grid_for(n, bs), bs, 0, st>>>(n, params, target_bg, x0, ub, status);
  return gt_check_launch("steady_state_kernel");
}

int gt_launch_stage_fast(int64_t n, const double* params, const int32_t* ss_status, int32_t* active,
                         double* fixed, int32_t* mismatch, cudaStream_t st) {
  cudaMemsetAsync(mismatch, 0, sizeof(int32_t), st);
  if (n <= 0) return gt_check_launch("stage_fast (memset)");
  const int bs = 256;
  gt::stage_fast_kernel<<<grid_for(n, bs), bs, 0, st>>>(n, params, ss_status, active, fixed, mismatch);
  return gt_check_launch("stage_fast_kernel");
}

int gt_launch_controller_init(int64_t n, const double* hyper, double icr_initial_factor,
                              const double* basal, double* c0, cudaStream_t st) {
  if (n <= 0) return GT_OK;
  const int bs = 256;
  gt::controller_init_kernel<<<grid_for(n, bs), bs, 0, st>>>(n, hyper, icr_initial_factor, basal, c0);
  return gt_check_launch("controller_init_kernel");
}
