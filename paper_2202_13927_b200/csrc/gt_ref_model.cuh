// Reference-order model functions shared by the exact (--fmad=false)
// translation units gt_parity.cu and gt_sampler.cu.  Include ONLY from
// translation units compiled without FMA contraction.
#pragma once
#include <cmath>
#include "gt_common.cuh"

namespace gt {

// hovorka.py:76-136 drift_vec
__device__ __forceinline__ void drift_ref(const double* x, const double* u, const double* d,
                                          const double* p, double* out) {
  const double w = p[PW];
  const double bg = x[IQ1] / (p[PVG] * w);
  const double cho_mmol = d[0] * kMmolPerGCho;
  const double tmaxg = p[PTMAXG];
  out[ID1] = p[PAG] * cho_mmol - x[ID1] / tmaxg;
  out[ID2] = (x[ID1] - x[ID2]) / tmaxg;
  const double gut_appearance = x[ID2] / tmaxg;
  const double tmaxi = p[PTMAXI];
  const double u_ins = u[0] + u[1];
  out[IS1] = u_ins - x[IS1] / tmaxi;
  out[IS2] = (x[IS1] - x[IS2]) / tmaxi;
  const double plasma_appearance = x[IS2] / tmaxi;
  out[II] = plasma_appearance / (p[PVI] * w) - p[PKE] * x[II];
  out[IX1] = p[PKA1] * (p[PSIT] * x[II] - x[IX1]);
  out[IX2] = p[PKA2] * (p[PSID] * x[II] - x[IX2]);
  out[IX3] = p[PKA3] * (p[PSIE] * x[II] - x[IX3]);
  const double tg = p[PTGLUC];
  out[IZ1] = u[2] - x[IZ1] / tg;
  out[IZ2] = x[IZ1] / tg - p[PKEGLUC] * x[IZ2];
  const double glucagon_conc = x[IZ2] / (p[PVGLUC] * w);
  out[IE1] = (d[1] - x[IE1]) / p[PTAUHR];
  out[IE2] = (x[IE1] - x[IE2]) / p[PTAUEX];
  out[IE3] = p[PALATE] * x[IE1] - x[IE3] / p[PTAULATE];
  double f01c, renal, egp;
  if (bg < 4.5) f01c = p[PF01] * w * bg / 4.5;
  else f01c = p[PF01] * w;
  if (bg > 9.0) renal = 0.003 * (bg - 9.0) * p[PVG] * w;
  else renal = 0.0;
  egp = p[PEGP0] * w * (1.0 - x[IX3]);
  if (egp < 0.0) egp = 0.0;
  egp += p[PSGLUC] * w * glucagon_conc;
  const double uptake_boost = 1.0 + p[PQEX] * x[IE2];
  const double action_boost = 1.0 + p[PSEX] * x[IE3];
  const double x1 = x[IX1] * action_boost;
  const double x2 = x[IX2] * action_boost;
  out[IQ1] = (gut_appearance - f01c * uptake_boost - x1 * x[IQ1] + p[PK12] * x[IQ2] - renal + egp);
  out[IQ2] = x1 * x[IQ1] - (p[PK12] + x2) * x[IQ2];
  out[IGSC] = (bg - x[IGSC]) / p[PTAUCGM];
}

// ------------------------------------------------------------ steady state
// hovorka.py:183-198 _net_glucose_flux_at, with the terms that do not depend
// on the insulin concentration evaluated once per solve (same operations, same order, same values: the
// hoisted products are the left-most factors of the reference's expressions)
struct NetFlux {
  double q1, f01c, renal, egpw, k12, sit, sid, sie;
  __device__ explicit NetFlux(double bg, const double* p) {
    const double w = p[PW];
    q1 = bg * p[PVG] * w;
    f01c = bg < 4.5 ? p[PF01] * w * bg / 4.5 : p[PF01] * w;
    renal = bg > 9.0 ? 0.003 * (bg - 9.0) * p[PVG] * w : 0.0;
    egpw = p[PEGP0] * w;
    k12 = p[PK12]; sit = p[PSIT]; sid = p[PSID]; sie = p[PSIE];
  }
  __device__ double operator()(double ic) const {
    const double x1 = sit * ic, x2 = sid * ic, x3 = sie * ic;
    const double q2 = x1 * q1 / (k12 + x2);
    const double v = egpw * (1.0 - x3);
    const double egp = v > 0.0 ? v : 0.0;
    return -f01c - x1 * q1 + k12 * q2 - renal + egp;
  }
};

// scipy/optimize/Zeros/brentq.c (Brent's method), restated.  err: 0 ok.
static __device__ double brentq_flux(double xa, double xb, double xtol, double rtol, int iter,
                                     const NetFlux& f, int* err) {
  double xpre = xa, xcur = xb, xblk = 0., fpre, fcur, fblk = 0., spre = 0., scur = 0., sbis;
  double delta, stry, dpre, dblk;
  fpre = f(xpre);
  fcur = f(xcur);
  *err = 0;
  if (isnan(fpre) || isnan(fcur)) { *err = 3; return 0.0; }
  if (fpre == 0) return xpre;
  if (fcur == 0) return xcur;
  if (signbit(fpre) == signbit(fcur)) { *err = 1; return 0.0; }
  for (int i = 0; i < iter; i++) {
    if (fpre != 0 && fcur != 0 && (signbit(fpre) != signbit(fcur))) {
      xblk = xpre; fblk = fpre; spre = scur = xcur - xpre;
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
      const double m1 = fabs(spre), m2 = 3 * fabs(sbis) - delta;
      if (2 * fabs(stry) < (m1 < m2 ? m1 : m2)) { spre = scur; scur = stry; }
      else { spre = sbis; scur = sbis; }
    } else {
      spre = sbis; scur = sbis;
    }
    xpre = xcur; fpre = fcur;
    if (fabs(scur) > delta) xcur += scur;
    else xcur += (sbis > 0 ? delta : -delta);
    fcur = f(xcur);
    if (isnan(fcur)) { *err = 3; return 0.0; }
  }
  *err = 2;
  return xcur;
}

// hovorka.py:201-243 steady_state.  Returns true on success.
#ifndef GT_SS_NOINLINE
#define GT_SS_NOINLINE 0
#endif
#if GT_SS_NOINLINE
static __device__ __noinline__
#else
static __device__
#endif
bool steady_state_dev(const double* p, double target_bg, double* x, double* u_basal_uh) {
  if (!(target_bg > 0)) return false;
  const double w = p[PW];
  const NetFlux f(target_bg, p);
  if (f(0.0) <= 0.0) return false;
  double lo = 0.0, hi = 50.0;
  bool found = false;
  for (int k = 0; k < 30; ++k) {
    if (f(hi) < 0.0) { found = true; break; }
    lo = hi; hi = hi * 2.0;
  }
  if (!found) return false;
  int err = 0;
  const double ic = brentq_flux(lo, hi, 1e-14, 8.9e-16, 200, f, &err);
  if (err) return false;
  const double u_basal_mU_min = ic * p[PKE] * p[PVI] * w;
  for (int k = 0; k < GT_N_STATES; ++k) x[k] = 0.0;
  x[IQ1] = target_bg * p[PVG] * w;
  x[II] = ic;
  x[IX1] = p[PSIT] * ic;
  x[IX2] = p[PSID] * ic;
  x[IX3] = p[PSIE] * ic;
  x[IQ2] = x[IX1] * x[IQ1] / (p[PK12] + x[IX2]);
  x[IS1] = u_basal_mU_min * p[PTMAXI];
  x[IS2] = u_basal_mU_min * p[PTMAXI];
  x[IGSC] = target_bg;
  const double u[3] = {u_basal_mU_min, 0.0, 0.0}, d[2] = {0.0, 0.0};
  double res[GT_N_STATES];
  drift_ref(x, u, d, p, res);
  double worst = 0.0;
  for (int k = 0; k < GT_N_STATES; ++k) {
    const double ax = fabs(x[k]);
    const double scale = ax > 1.0 ? ax : 1.0;
    const double r = fabs(res[k]) / scale;
    if (isnan(r)) { worst = NAN; break; }
    if (r > worst) worst = r;
  }
  if (worst > 1e-9) return false;  // NaN compares false, as numpy's max does
  *u_basal_uh = u_basal_mU_min * 60.0 / 1000.0;
  return true;
}

}  // namespace gt
