// Shared device definitions for the glucosim kernels (sm_100a).
// Layouts restate the reference's packed-vector conventions:
//   states  hovorka.py:38, params hovorka.py:53-55,
//   hyper   controller.py:32-36, controller state controller.py:40-41.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/glucosim.h"

namespace gt {

enum { IQ1, IQ2, IS1, IS2, II, IX1, IX2, IX3, ID1, ID2, IGSC, IZ1, IZ2, IE1, IE2, IE3, NS };
enum { PW, PEGP0, PF01, PK12, PKA1, PKA2, PKA3, PSIT, PSID, PSIE, PKE, PVI, PVG,
       PTMAXI, PTMAXG, PAG, PTAUCGM, PTGLUC, PKEGLUC, PVGLUC, PSGLUC, PTAUHR,
       PTAUEX, PTAULATE, PALATE, PQEX, PSEX, PSIGEGP, PSIGGUT, PR, NP };
enum { HFILTER, HSETPOINT, HGLUCTHR, HHYST, HPREDHOR, HBKP, HBKD, HBFMAX, HSUPBG,
       HSUPFRAC, HSUSPMIN, HMICROUG, HLOCKMIN, HMICROTREND, HCFICR, HICRSTEP,
       HICRSTEPUP, HICRMIN, HICRMAX, HMEALWIN, HEXCHI, HUNDERBG, HMAXBOLUS,
       HMAXGLUC, HEXBOLUS, HEXBOLUSBG, HEXSETPOINT, HEXBFACTOR, HEXGLUCTHR,
       HEXMICROUG, NH };
enum { CFILT, CPREV, CMODE, CICR, CSUSPEND_UNTIL, CEXBOLUSDONE, CLASTGLUC, CWINEND,
       CWINPEAK, CWINMIN, CINIT, NC };

constexpr double kMmolPerGCho = 1000.0 / 180.16;  // hovorka.py:64
constexpr double kFpScale = 16777216.0;           // 2^24, analytics.py:40

// ---------------------------------------------------------------- Philox
// Philox4x32-10 (Salmon et al., SC'11). Counter = (index_lo, pid, role,
// index_hi); key = (seed_lo, seed_hi).
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                            uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return U4{c0, c1, c2, c3};
}

// ------------------------------------------- exactly reproducible arithmetic
// Explicit round-to-nearest intrinsics: never contracted into FMA even in a
// translation unit compiled with --fmad=true.  Used by the code that must be
// bit-identical to the host twin / reference (meal generator, steady state).
__device__ __forceinline__ double M_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double A_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double S_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double D_(double a, double b) { return __ddiv_rn(a, b); }

// Deterministic natural log from IEEE +,-,*,/ only (host twin:
// paper_2202_13927_b200/rng.py det_log).
__device__ __forceinline__ double det_log(double x) {
  int e;
  double m = frexp(x, &e);
  if (m < 0.70710678118654752440) { m = M_(m, 2.0); e = e - 1; }
  const double f = S_(m, 1.0);
  const double s = D_(f, A_(2.0, f));
  const double z = M_(s, s);
  double poly = 1.0 / 25.0;
  poly = A_(1.0 / 23.0, M_(z, poly));
  poly = A_(1.0 / 21.0, M_(z, poly));
  poly = A_(1.0 / 19.0, M_(z, poly));
  poly = A_(1.0 / 17.0, M_(z, poly));
  poly = A_(1.0 / 15.0, M_(z, poly));
  poly = A_(1.0 / 13.0, M_(z, poly));
  poly = A_(1.0 / 11.0, M_(z, poly));
  poly = A_(1.0 / 9.0, M_(z, poly));
  poly = A_(1.0 / 7.0, M_(z, poly));
  poly = A_(1.0 / 5.0, M_(z, poly));
  poly = A_(1.0 / 3.0, M_(z, poly));
  const double logm = A_(M_(2.0, s), M_(M_(2.0, s), M_(z, poly)));
  const double de = (double)e;
  return A_(M_(de, 6.93147180369123816490e-01), A_(M_(de, 1.90821492927058770002e-10), logm));
}

// Deterministic exp from IEEE +,-,* only: x = k*ln2 + r, Taylor(r) to
// degree 14 (|r| <= ln2/2) by Horner on the doubles nearest 1/j!, then an
// exact scaling by 2^k.  (No divisions: the sampler evaluates eight of these
// per steady-state candidate.)
__device__ __forceinline__ double det_exp(double x) {
  constexpr double kInvFact[15] = {
    1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664, 0.008333333333333333,
    0.001388888888888889, 0.0001984126984126984, 2.48015873015873e-05, 2.7557319223985893e-06,
    2.755731922398589e-07, 2.505210838544172e-08, 2.08767569878681e-09, 1.6059043836821613e-10,
    1.1470745597729725e-11};
  if (x > 709.0) return INFINITY;
  if (x < -745.0) return 0.0;
  const double kf = floor(A_(M_(x, 1.44269504088896338700e+00), 0.5));
  const double r = S_(S_(x, M_(kf, 6.93147180369123816490e-01)), M_(kf, 1.90821492927058770002e-10));
  double s = kInvFact[14];
#pragma unroll
  for (int j = 13; j >= 0; --j) s = A_(kInvFact[j], M_(r, s));
  return ldexp(s, (int)kf);
}

// Acklam's inverse normal CDF, evaluated with explicit IEEE operations.
__device__ __forceinline__ double det_inv_norm(double p) {
  const double a0 = -3.969683028665376e+01, a1 = 2.209460984245205e+02,
               a2 = -2.759285104469687e+02, a3 = 1.383577518672690e+02,
               a4 = -3.066479806614716e+01, a5 = 2.506628277459239e+00;
  const double b0 = -5.447609879822406e+01, b1 = 1.615858368580409e+02,
               b2 = -1.556989798598866e+02, b3 = 6.680131188771972e+01,
               b4 = -1.328068155288572e+01;
  const double c0 = -7.784894002430293e-03, c1 = -3.223964580411365e-01,
               c2 = -2.400758277161838e+00, c3 = -2.549732539343734e+00,
               c4 = 4.374664141464968e+00, c5 = 2.938163982698783e+00;
  const double d0 = 7.784695709041462e-03, d1 = 3.224671290700398e-01,
               d2 = 2.445134137142996e+00, d3 = 3.754408661907416e+00;
  const double plow = 0.02425, phigh = 1.0 - 0.02425;
  if (p < plow || p > phigh) {
    const bool upper = p > phigh;
    const double q = __dsqrt_rn(M_(-2.0, det_log(upper ? S_(1.0, p) : p)));
    const double num = A_(M_(A_(M_(A_(M_(A_(M_(A_(M_(c0, q), c1), q), c2), q), c3), q), c4), q), c5);
    const double den = A_(M_(A_(M_(A_(M_(A_(M_(d0, q), d1), q), d2), q), d3), q), 1.0);
    const double v = D_(num, den);
    return upper ? -v : v;
  }
  const double q = S_(p, 0.5);
  const double r = M_(q, q);
  const double num =
      M_(A_(M_(A_(M_(A_(M_(A_(M_(A_(M_(a0, r), a1), r), a2), r), a3), r), a4), r), a5), q);
  const double den =
      A_(M_(A_(M_(A_(M_(A_(M_(A_(M_(b0, r), b1), r), b2), r), b3), r), b4), r), 1.0);
  return D_(num, den);
}

// 3-meal disturbance generator: meal m = 3*day + slot.
struct Meal { double start, end, carbs; };
__device__ __forceinline__ Meal gen_meal(const gt_meal_gen& g, uint64_t seed, uint32_t pid,
                                         int64_t m) {
  const U4 r = philox4x32_10((uint32_t)m, pid, g.role, (uint32_t)((uint64_t)m >> 32),
                             (uint32_t)seed, (uint32_t)(seed >> 32));
  const int64_t day = m / 3;
  const int slot = (int)(m - day * 3);
  const uint32_t span = (uint32_t)(2 * g.jitter_s + 1);
  const int64_t jit = (int64_t)(((uint64_t)r.x * span) >> 32) - g.jitter_s;
  const double clock = slot == 0 ? g.clock_s[0] : (slot == 1 ? g.clock_s[1] : g.clock_s[2]);
  const double mean = slot == 0 ? g.mean_g[0] : (slot == 1 ? g.mean_g[1] : g.mean_g[2]);
  const double st = A_(A_(M_((double)day, 86400.0), clock), (double)jit);
  const uint64_t k = ((uint64_t)(r.y >> 6) << 26) | (uint64_t)(r.z >> 6);
  const double u = M_((double)(2 * k + 1), 1.1102230246251565404e-16);
  const double z = det_inv_norm(u);
  double carbs = A_(mean, M_(g.sd_g, z));
  if (carbs < 0.0) carbs = 0.0;
  return Meal{st, A_(st, (double)g.duration_s), carbs};
}

// CPython / numba float floor division (Objects/floatobject.c float_divmod),
// used by `t // 86400.0` (_kernel.py:133,148) and `x // width`
// (analytics.py:256).  fmod is exact.
__device__ __forceinline__ double py_floordiv(double vx, double wx) {
  double mod = fmod(vx, wx);
  double div = D_(S_(vx, mod), wx);
  if (mod != 0.0) {
    if ((wx < 0) != (mod < 0)) { mod = A_(mod, wx); div = S_(div, 1.0); }
  }
  double fl;
  if (div != 0.0) {
    fl = floor(div);
    if (S_(div, fl) > 0.5) fl = A_(fl, 1.0);
  } else {
    fl = copysign(0.0, D_(vx, wx));
  }
  return fl;
}

// Order-preserving int64 image of a double (for atomic min/max of floats).
__device__ __forceinline__ long long ordered_bits(double v) {
  long long b = __double_as_longlong(v);
  return b >= 0 ? b : (b ^ 0x7fffffffffffffffLL);
}

}  // namespace gt

// error plumbing (gt_capi.cu)
void gt_set_error(const char* fmt, ...);
int gt_check_launch(const char* what);
// Keep the current device's default stream-ordered pool mapped between
// calls (release threshold = max), so per-launch cudaMallocAsync fallbacks
// do not re-map memory after every synchronisation.
void gt_keep_pool_mapped();
