// Fast fused closed-loop integrator (BASELINE north_star subsystem 3).
//
// One thread = one virtual patient.  SDE state, Philox counters and per-step
// accumulators live in registers.  The 247-bin BG histogram of each patient
// lives in shared memory as uint8 counters: a counter that reaches 255
// drains into the patient's HBM column (a RED on that rare path only), and
// all drain at the end of a slice.  The state that changes only on controller ticks
// (controller memory, meal window, dose sums, BG extremes) lives in shared
// memory too, so HBM sees parameters in and metrics out only.
//
// Same model (hovorka.py:76-150), controller (controller.py:343-458) and
// statistics (_kernel.py:137-160) as the parity kernel, re-associated for
// the FP64 pipe: each linear update x += h*(b*y - x/tau) is evaluated as
// fma(x, 1-h/tau, h*b*y) with per-patient constants folded at start-up and
// launch-uniform constants (fixed parameters, controller hyperparameters) in
// the kernel-parameter bank; the noise Philox runs under a fixed key whose
// round keys are immediates.  For every state of that form the reference's
// projection max(x,0) is a no-op (monotone rounding of a - b with
// 0 <= b <= a), so it is applied only to Q1 and Q2 (and D1/D2 when arbitrary
// noise is injected: device Philox normals are bounded by 6.7 sigma, far
// inside the gut states' positivity margin of ~30 sigma).  Results agree with
// the parity path to rounding; DESIGN.md §4 documents the threshold ties.
//
// Scheduling: the kernel is persistent.  Each warp repeatedly claims a unit
// (chunk c, logical warp w) = 32 patients x one slice of the horizon, in
// chunk-major order, from a global counter; a unit with c > 0 waits until
// unit (c-1, w) has released its saved state.  Slicing the horizon removes
// the wave quantisation of one-thread-per-patient launches (100k patients =
// 3125 warps on 2368 resident warp slots = 1.32 waves) and, with several
// units per slot, lets the schedule balance the warps' unequal costs
// (choose_chunks).
//
// Loop structure is warp-uniform: outer loop over controller periods, inner
// loop over the period's integration steps; all lanes of a warp hit
// controller ticks, day boundaries and timeline grid points together.
#include <cmath>
#include <climits>
#include <cstdlib>
#include <cstdio>
#include "gt_common.cuh"

namespace gt {

// Debug builds (-DGT_DEBUG_BOUNDS) check every computed index of the fused
// kernel and trap with the failing site; release builds compile them out.
#ifdef GT_DEBUG_BOUNDS
#define GT_CHECK(c, tag) do { if (!(c)) { printf("GT_CHECK %s failed: block %d thread %d\n", tag, \
                                                  (int)blockIdx.x, (int)threadIdx.x); __trap(); } } while (0)
#else
#define GT_CHECK(c, tag) do { } while (0)
#endif

#ifndef GT_LASTCHECK
#define GT_LASTCHECK 1   // the state check at the horizon's last tick only (see the tick)
#endif
#ifndef GT_DAY_VOTE
#define GT_DAY_VOTE 1
#endif
// Per-instance code shape, a bit per (protocol, controller) as GT_PS5:
// 1 three_meal/pid_pump, 2 three_meal/dual_hormone, 4 csr/pid_pump,
// 8 csr/dual_hormone (measured with tools/ab_kernel.py, profiles/r02_ab_*.json).
#ifndef GT_PAIRS
#define GT_PAIRS 8      // plain steps in pairs (-4.7 % csr/dual_hormone; +3 to +24 % on three_meal)
#endif
#ifndef GT_NOPIPE
#define GT_NOPIPE 0     // instances drawing each tick's normals at use, not one step ahead (csr/pid_pump was -0.8 %
                        // in 128-thread blocks; pipelined is -0.5 % in 256-thread blocks)
#endif
#ifndef GT_LATE
#define GT_LATE 1       // controller after the tick's Euler update (only S1 / Z1 take its output)
#endif
#ifndef GT_NOISE_PIPE
#define GT_NOISE_PIPE 1  // draw tick k + 1's normals during step k
#endif
#ifndef GT_PS5
// instances whose 5-step controller period (dt 60 s, 300 s period) runs fully
// unrolled, a bit per (protocol, controller): 1 three_meal/pid_pump,
// 2 three_meal/dual_hormone, 4 csr/pid_pump, 8 csr/dual_hormone.  Measured
// (tools/ab_kernel.py, 100k x 4 w): the unrolled period is faster only for
// csr/pid_pump (-8 %); it spills more and is slower (+2.5 to +7 %) elsewhere.
#define GT_PS5 4
#endif
#ifndef GT_NOISE_ROUNDS
// Philox4x32 rounds of the integrator's noise stream.  7 is the smallest round
// count Salmon et al. (SC'11, Table 2) found Crush-resistant for Philox4x32
// (BigCrush passes); 10 is their default "safety margin".  The noise role only
// needs statistical parity (the parity path injects the reference's streams),
// and 7 rounds measured 6-13 % faster per launch (profiles/r02_ab_noise_rounds.json).
// The sampler and meal streams keep Philox4x32-10 (gt_common.cuh).
#define GT_NOISE_ROUNDS 7
#endif
#ifndef GT_DEAD_SINK
// instances (GT_PS5 bits) whose dead lanes count into the padding bin 247; the
// others count masked lanes into their own bins and never write them out
// (-0.6 % three_meal/pid_pump; +0.4 % on two other instances)
#define GT_DEAD_SINK 14
#endif
#ifndef GT_FKEY
#define GT_FKEY 1   // extremes / hypo-run branch keyed on FP32 bounds of the extremes (not bins)
#endif
#ifndef GT_KLOOP
#define GT_KLOOP 1  // plain-step loop over the tick index itself
#endif
#ifndef GT_EXFOLD
#define GT_EXFOLD 1  // exercise input h/tau_hr * HRR folded per session (one DMUL less per step on CSR)
#endif
#ifndef GT_RINT
#define GT_RINT 1   // instances (GT_PS5 bits) testing the near-edge bin as |t10 - rint(t10)| <= 1e-4:
                    // -0.7 % three_meal/pid_pump, +1.1 % three_meal/dual_hormone (profiles/r02_ab_code_shape.json)
#endif
#ifndef GT_DRAIN32
#define GT_DRAIN32 15  // instances (GT_PS5 bits) forming the drain address from a 32-bit element offset
                       // (-0.6 % three_meal/pid_pump, -0.9 % csr/dual_hormone, profiles/r02d_ab_fused.json)
#endif
#ifndef GT_SCALE
// States carried in a scaled form (a bit each), so that a per-step multiply
// folds into the update: 1 S1*hTI, 2 X1*h, 4 G/hS, 8 D1,D2*hTG.
#define GT_SCALE 15   // -1.7 % three_meal/pid_pump, -0.8 % three_meal/dual_hormone (profiles/r02d_ab_fused.json)
#endif
constexpr bool kScS1 = (GT_SCALE & 1) != 0, kScX1 = (GT_SCALE & 2) != 0, kScG = (GT_SCALE & 4) != 0,
               kScD = (GT_SCALE & 8) != 0;
// per instance (GT_PS5 bits): X2 carried as h*X2, S2 as dI*S2 (then S1 as hTI*dI*S1)
#ifndef GT_SCX2
#define GT_SCX2 15   // every instance (profiles/r02d_ab_fused.json)
#endif
#ifndef GT_SCS2
#define GT_SCS2 10   // the dual_hormone instances (a mask per controller keeps the 3-meal generator and
                     // the CSR form of the same schedule bit-identical)
#endif
static_assert(!GT_SCS2 || kScS1, "GT_SCS2: S2 carried as dI*S2 needs S1 carried as hTI*dI*S1");
#ifndef GT_LAZYZM
// instances (GT_PS5 bits) whose pipelined draws keep the 4th normal as
// (radius, angle), its sine taken only at ticks: -3.3 % three_meal/dual_hormone,
// +0.5 % three_meal/pid_pump (profiles/r02d_ab_fused.json)
#define GT_LAZYZM 14
#endif
#ifndef GT_F01Q
#define GT_F01Q 0
#endif
// timing ablations (results wrong): 1 drops the piece
#ifndef GT_ABL_TL
#define GT_ABL_TL 0      // timeline points
#endif
#ifndef GT_ABL_NOISE
#define GT_ABL_NOISE 0   // pipelined noise draws (the normals stay constant)
#endif
#ifndef GT_ABL_CTRL
#define GT_ABL_CTRL 0    // the late controller call (the last decision is held)
#endif
#ifndef GT_PIDFLAT
// instances (GT_PS5 bits) whose pid_pump controller runs its common path
// without branches (see control()): -0.65 % three_meal/pid_pump, +0.65 %
// csr/pid_pump (profiles/r02d_ab_fused.json)
#define GT_PIDFLAT 1
#endif
#ifndef GT_FAST_MINB
#define GT_FAST_MINB 2  // resident 256-thread blocks per SM (register budget 128: 16 warps per SM)
#endif
#ifndef GT_FAST_BS
#define GT_FAST_BS 256  // threads per block (lanes sharing the block's shared-memory slots); 256 against
                        // 128: -7 % NorthernYear/dual_hormone, -3 % NorthernYear/pid_pump, -0.4 %
                        // three_meal/pid_pump, +0.3 % three_meal/dual_hormone (profiles/r02d_ab_fused.json).
                        // The static shared memory (45 KB at 256) must stay under 48 KB.
#endif
constexpr int kFastBS = GT_FAST_BS;
constexpr int kHistWords = (GT_N_BG_BINS + 3) / 4;  // 62 packed uint8x4 words per lane
#ifndef GT_HISTLIN
// 1: each lane's 248 counter bytes contiguous (word tid * 62 + w), so a bin's
// byte address is one add; 0: word-interleaved (word w * kFastBS + tid), bank
// conflict free for any bins
#define GT_HISTLIN 1   // -0.7 to -1.5 % on every instance (profiles/r02d_ab_fused.json)
#endif
__device__ __forceinline__ int hword(int w, int tid) { return GT_HISTLIN ? tid * kHistWords + w : w * kFastBS + tid; }

// Launch-uniform constants derived from the fixed parameters (host-computed,
// passed by value -> constant bank operands, no registers).
struct Uni {
  double h, ginK, aS, hS, aZ1, hTg, aZ2, cG;
  double aE1, bE1, aE2, bE2, aE3, bE3, qex, sex;
  double sqG, sigEh, sqrtR, rK1, pred_k, u_basal_k, u_bolus_k, u_gluc_k;
  double dt, period, horizon_s, meal_dur_min, rs_agg, pid_ph;
  int32_t ps, n_ctl, ctl_per_day, grid_ctl, hypoL, agg;
  uint32_t nz_c2, nz_c3;  // noise counter words 2-3: seed_lo, seed_hi ^ role << 24
  uint32_t nz_a;          // hi(nz_c2 * M1) ^ K0(0): round 1's launch word (philox_lane)
  double hyper[GT_N_HYPER];  // controller hyperparameters (parameter bank: direct operands)
  double hc[6];              // hyper-derived controller constants (same IEEE values)
};

// Persistent work distribution (see the header comment).
struct Sched {
  int* counter;      // next unit to claim
  int* done;         // [n_warps] slices completed per logical warp
  double* sd;        // [SD_N][n] saved FP64 lane state between slices
  int* si;           // [SI_N][n] saved integer lane state between slices
  int n_units, n_warps, chunk_ctl, n_chunks;
};

// Per-patient constants (registers), in the integrator's precision R.
template <typename R>
struct PC {
  R invVGw, aG, hTG, aI, hTI, cI, dI, ax1, bx1, ax2, bx2, ax3, bx3;
  R hF01w45, hk12, aK12, hE, rK0, sqE;
  R hF01Q, Q45;   // GT_F01Q: h F01 / (4.5 VG) and 4.5 VG w (the flux on Q1 directly)
};

template <typename R, bool kScX2>
__device__ __forceinline__ void make_pc(const double* __restrict__ p, const Uni& u, PC<R>& c) {
  const double h = u.h, w = p[PW];
  // folded in FP64, then rounded once to R
  const double hTG = h / p[PTMAXG], hTI = h / p[PTMAXI], hk12 = h * p[PK12];
  c.invVGw = (R)(1.0 / (p[PVG] * w));
  c.hTG = (R)hTG; c.aG = (R)(1.0 - hTG);
  c.hTI = (R)hTI; c.aI = (R)(1.0 - hTI);
  c.cI = (R)(1.0 - h * p[PKE]); c.dI = (R)(hTI / (p[PVI] * w));
  c.ax1 = (R)(1.0 - h * p[PKA1]); c.bx1 = (R)((kScX1 ? h * h : h) * p[PKA1] * p[PSIT]);
  c.ax2 = (R)(1.0 - h * p[PKA2]); c.bx2 = (R)((kScX2 ? h * h : h) * p[PKA2] * p[PSID]);
  c.ax3 = (R)(1.0 - h * p[PKA3]); c.bx3 = (R)(h * p[PKA3] * p[PSIE]);
  c.hF01w45 = (R)(h * p[PF01] * w / 4.5);
  c.hF01Q = (R)(h * p[PF01] / (4.5 * p[PVG])); c.Q45 = (R)(4.5 * p[PVG] * w);
  c.hk12 = (R)hk12; c.aK12 = (R)(1.0 - hk12);
  c.hE = (R)(h * p[PEGP0] * w);
  c.rK0 = (R)(h * 0.003 * 9.0 * p[PVG] * w);
  c.sqE = (R)(u.sigEh * w);
}

// Explicit selects (setp + selp): the ternary forms below otherwise compile
// to the DSETP.MAX/MIN + NaN-quieting sequence of fmax/fmin (5 instructions).
__device__ __forceinline__ double zero_if_neg(double x) {   // x < 0 ? 0 : x (NaN kept)
  double r;
  asm("{\n\t.reg .pred p;\n\tsetp.lt.f64 p, %1, 0d0000000000000000;\n\t"
      "selp.f64 %0, 0d0000000000000000, %1, p;\n\t}" : "=d"(r) : "d"(x));
  return r;
}
__device__ __forceinline__ double pos_or_zero(double x) {   // x > 0 ? x : 0 (NaN -> 0)
  double r;
  asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %1, 0d0000000000000000;\n\t"
      "selp.f64 %0, %1, 0d0000000000000000, p;\n\t}" : "=d"(r) : "d"(x));
  return r;
}
__device__ __forceinline__ double lt_or(double x, double c) {  // x < c ? x : c (NaN -> c)
  double r;
  asm("{\n\t.reg .pred p;\n\tsetp.lt.f64 p, %1, %2;\n\tselp.f64 %0, %1, %2, p;\n\t}"
      : "=d"(r) : "d"(x), "d"(c));
  return r;
}
__device__ __forceinline__ float zero_if_neg(float x) { return x < 0.0f ? 0.0f : x; }
__device__ __forceinline__ float pos_or_zero(float x) { return x > 0.0f ? x : 0.0f; }
__device__ __forceinline__ float lt_or(float x, float c) { return x < c ? x : c; }

// Opaque copy: the compiler must keep the value (or spill it) rather than
// rematerialise it from its inputs (e.g. a reload of the parameters from HBM).
__device__ __forceinline__ double opaque(double x) { double r; asm("mov.b64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ __forceinline__ float opaque(float x) { float r; asm("mov.b32 %0, %1;" : "=f"(r) : "f"(x)); return r; }

// explicit-rounding multiply / fma in the integrator precision (no mixed
// overloads: a double constant reaching the FP32 integrator fails to compile)
__device__ __forceinline__ double MR_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float MR_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double FMR(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float FMR(float a, float b, float c) { return __fmaf_rn(a, b, c); }
// |x| bit pattern compared against the exponent-all-ones pattern (Inf/NaN)
__device__ __forceinline__ unsigned absbits(double x) { return (unsigned)__double2hiint(x) & 0x7fffffffu; }
__device__ __forceinline__ unsigned absbits(float x) { return __float_as_uint(x) & 0x7fffffffu; }
template <typename R> struct kNonfiniteBits;
template <> struct kNonfiniteBits<double> { static constexpr unsigned v = 0x7ff00000u; };
template <> struct kNonfiniteBits<float> { static constexpr unsigned v = 0x7f800000u; };

// ------------------------------------------------------------ noise
__device__ __forceinline__ void mulwide(uint32_t a, uint32_t b, uint32_t& lo, uint32_t& hi) {
  uint64_t p;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));  // one IMAD.WIDE.U32
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(p));
}

// Noise stream: Philox4x32-7 under a FIXED key, so the round keys are
// compile-time immediates of the LOP3s (no uniform registers, no constant
// loads); the trial seed enters the counter instead:
//   counter = (pid, index, seed_lo, seed_hi ^ role << 24)
// which is injective in (pid, index, seed) for the one role the kernel draws.
// Per round: 2 IMAD.WIDE.U32 + 2 LOP3.
constexpr uint32_t kNoiseKey0 = 0xA4093822u, kNoiseKey1 = 0x299F31D0u;  // digits of pi
__device__ __forceinline__ U4 philox_fast(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
#pragma unroll
  for (int r = 0; r < GT_NOISE_ROUNDS; ++r) {
    uint32_t lo0, hi0, lo1, hi1;
    mulwide(c0, 0xD2511F53u, lo0, hi0);
    mulwide(c2, 0xCD9E8D57u, lo1, hi1);
    const uint32_t n0 = hi1 ^ c1 ^ (kNoiseKey0 + (uint32_t)r * 0x9E3779B9u);
    const uint32_t n2 = hi0 ^ c3 ^ (kNoiseKey1 + (uint32_t)r * 0xBB67AE85u);
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return U4{c0, c1, c2, c3};
}

// The integrator's draws: Philox4x32-7 with the counter (pid, index, seed_lo,
// seed_hi ^ role << 24).  With the index in word 1 (xored, never multiplied in
// round 1), rounds 1-3 reduce to 2 multiplies and 4 xors per draw given four
// per-patient words (NoiseLane) and one launch word (Uni::nz_a):
//   round 1: (index ^ A, lo(s2*M1), B, lo(pid*M0))        B = hi(pid*M0) ^ s3 ^ K1(0)
//   round 2: (C, lo(B*M1), hi0 ^ D, lo0)  (lo0, hi0) = (index ^ A) * M0,
//            C = hi(B*M1) ^ lo(s2*M1) ^ K0(1), D = lo(pid*M0) ^ K1(1)
//   round 3: (hi1 ^ E, lo1, lo0 ^ F, lo(C*M0))  (lo1, hi1) = (hi0 ^ D) * M1,
//            E = lo(B*M1) ^ K0(2), F = hi(C*M0) ^ K1(2)
// then rounds 4-7 as usual: the same outputs as philox_fast(pid, index, s2, s3).
struct NoiseLane { uint32_t d, e, f, loc; };
__device__ __forceinline__ uint32_t noise_k0(int r) { return kNoiseKey0 + (uint32_t)r * 0x9E3779B9u; }
__device__ __forceinline__ uint32_t noise_k1(int r) { return kNoiseKey1 + (uint32_t)r * 0xBB67AE85u; }
__device__ __forceinline__ NoiseLane noise_lane(uint32_t pid, uint32_t s2, uint32_t s3) {
  uint32_t lo0p, hi0p, lo1u, hi1u, loB, hiB, loC, hiC;
  mulwide(pid, 0xD2511F53u, lo0p, hi0p);
  mulwide(s2, 0xCD9E8D57u, lo1u, hi1u);
  const uint32_t B = hi0p ^ s3 ^ noise_k1(0);
  mulwide(B, 0xCD9E8D57u, loB, hiB);
  const uint32_t C = hiB ^ lo1u ^ noise_k0(1);
  mulwide(C, 0xD2511F53u, loC, hiC);
  NoiseLane L;
  L.d = lo0p ^ noise_k1(1); L.e = loB ^ noise_k0(2); L.f = hiC ^ noise_k1(2); L.loc = loC;
  return L;
}
__device__ __forceinline__ U4 philox_lane(uint32_t index, const NoiseLane& L, uint32_t nz_a) {
  uint32_t lo0, hi0, lo1, hi1;
  mulwide(index ^ nz_a, 0xD2511F53u, lo0, hi0);       // round 2, word 0 product
  mulwide(hi0 ^ L.d, 0xCD9E8D57u, lo1, hi1);         // round 3, word 2 product
  uint32_t c0 = hi1 ^ L.e, c1 = lo1, c2 = lo0 ^ L.f, c3 = L.loc;
#pragma unroll
  for (int r = 3; r < GT_NOISE_ROUNDS; ++r) {
    uint32_t a0, b0, a1, b1;
    mulwide(c0, 0xD2511F53u, a0, b0);
    mulwide(c2, 0xCD9E8D57u, a1, b1);
    const uint32_t n0 = b1 ^ c1 ^ noise_k0(r);
    const uint32_t n2 = b0 ^ c3 ^ noise_k1(r);
    c0 = n0; c1 = a1; c2 = n2; c3 = a0;
  }
  return U4{c0, c1, c2, c3};
}

// Raw SFU approximations (MUFU.LG2 / SQRT / SIN / COS), no denormal or
// special-value paths: every argument below is a normal, finite float.
__device__ __forceinline__ float lg2_approx(float x) {
  float r; asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float r; asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r;
}
__device__ __forceinline__ float sin_approx(float x) {
  float r; asm("sin.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r;
}
__device__ __forceinline__ float cos_approx(float x) {
  float r; asm("cos.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r;
}

// Box-Muller in FP32 on the SFU: u1 in [2^-33, 1] (never 0), radius
// sqrt(-2 ln u1) by MUFU.SQRT (u1 = 1 gives radius 0, as it should), angle
// 2*pi*u2 in [0, 2*pi).
__device__ __forceinline__ void bm_polar(uint32_t a, uint32_t b, float& rad, float& ang) {
  const float u1 = fmaf((float)a, 2.3283064365386963e-10f, 1.1641532182693481e-10f);
  ang = (float)b * 1.4629180792671596e-09f;  // 2*pi * 2^-32
  const float t = lg2_approx(u1) * -1.3862943611198906f;  // -2 ln 2 * log2(u1) > 0
  rad = sqrt_approx(t);
}
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float& z0, float& z1) {
  float rad, ang;
  bm_polar(a, b, rad, ang);
  z0 = rad * cos_approx(ang);
  z1 = rad * sin_approx(ang);
}

// ------------------------------------------------------------ meals
// Meals in tick units: active while ks <= k < ke; announced on controller
// period kp (start in [kp*P, (kp+1)*P)).  Exhausted sources return INT_MAX.
struct MealT { int32_t ks, ke, kp; double rate, carbs; };

__device__ __noinline__ MealT three_meal_at(const gt_meal_gen* g, uint64_t seed, uint32_t pid,
                                            int32_t m, double dt, double period, double horizon_s) {
  const Meal ml = gen_meal(*g, seed, pid, m);
  MealT r;
  if (ml.start >= horizon_s) {  // compile_protocol filter (simulation.py:157)
    r.ks = r.ke = r.kp = INT_MAX; r.rate = 0.0; r.carbs = 0.0; return r;
  }
  r.ks = (int32_t)ceil(ml.start / dt);
  r.ke = (int32_t)ceil(ml.end / dt);
  r.kp = (int32_t)floor(ml.start / period);
  r.carbs = ml.carbs;
  r.rate = ml.carbs / ((ml.end - ml.start) / 60.0);  // simulation.py:162
  return r;
}

__device__ __forceinline__ long long warp_sum64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long warp_min64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { long long w = __shfl_xor_sync(0xffffffffu, v, o); v = w < v ? w : v; }
  return v;
}
__device__ __forceinline__ long long warp_max64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { long long w = __shfl_xor_sync(0xffffffffu, v, o); v = w > v ? w : v; }
  return v;
}

// Exact per-warp timeline partials on 64-bit values (rare: a live BG >= 128
// mmol/L or non-finite); out of line to keep the step loop small.
__device__ __noinline__ void timeline_partials64(bool alive, long long v, long long& ssum, long long& smin,
                                                 long long& smax) {
  ssum = warp_sum64(alive ? v : 0LL);
  smin = warp_min64(alive ? v : LLONG_MAX);
  smax = warp_max64(alive ? v : LLONG_MIN);
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// Saved slice state is written with an L2 evict_last policy so it stays in
// L2 until the next slice of the same warp reads it, and the read lines are
// then discarded (no write-back): the state round trip does not reach HBM.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_keep(double* a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" :: "l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_keep(int* a, int v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" :: "l"(a), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void l2_discard_line(const void* a) {  // a: 128-byte aligned
  asm volatile("discard.global.L2 [%0], 128;" :: "l"(a) : "memory");
}

// Shared-memory per-lane slots (SoA, [slot][tid]).
enum { SC_FILT, SC_ICR, SC_SUSP, SC_LASTG, SC_WEND, SC_WPEAK, SC_WMIN,
       SC_BGMIN, SC_BGMAX, SC_DBOLUS, SC_DGLUC, SC_ANNCARBS, SC_ASSUMED, N_SC };
enum { SI_FLAGS, SI_ANNKP, SI_ANNM, SI_MEALM, SI_EXPTR, N_SI };  // flags: mode | exdone<<1 | init<<2

// Saved lane state between horizon slices ([field][n] in Sched::sd / si).
enum { SD_Q1, SD_Q2, SD_S1, SD_S2, SD_I, SD_X1, SD_X2, SD_X3, SD_D1, SD_D2, SD_G, SD_Z1, SD_Z2,
       SD_E1, SD_E2, SD_E3, SD_BGSUM, SD_DAYBASAL, SD_HUINS, SD_HU2, SD_GIN, SD_MC0, SD_MC1,
       SD_MC2, SD_SC0, SD_N = SD_SC0 + N_SC };
enum { SV_MKS, SV_MKE, SV_KBMIN, SV_KBMAX, SV_RUN39, SV_RUN30, SV_EV39,
       SV_EV30, SV_ALIVE, SV_STATUS, SV_DEATH, SV_MK0, SV_SI0 = SV_MK0 + 9, SV_H0 = SV_SI0 + N_SI,
       SV_N = SV_H0 + kHistWords };  // SV_H0: the packed uint8 histogram counters

template <int PROTO, int NOISE, typename R, bool AGG, bool TRACE, int CTRL, int PSC>
__global__ void __launch_bounds__(kFastBS, GT_FAST_MINB)
fast_kernel(const gt_fast_args a, const Uni u, const Sched sch) {
  constexpr bool HAS_EX = (PROTO == GT_PROTO_CSR);
  constexpr int kShape = (PROTO == GT_PROTO_CSR ? 4 : 1) << (CTRL == GT_CTRL_PID_PUMP ? 0 : 1);
  constexpr bool kScX2 = (GT_SCX2 & kShape) != 0, kScS2 = (GT_SCS2 & kShape) != 0;
  constexpr bool CLAMP_GUT = (NOISE == GT_NOISE_INJECTED);
  // s_thr[k+1] = bits of THRESHOLDS[k]; s_thr[0] = -inf, s_thr[247] = +inf
  __shared__ long long s_thr[GT_N_THRESHOLDS + 2];
  constexpr int kPulseTab = 64;
  __shared__ double s_prate[kPulseTab];  // PID: basal rate of p whole pulses, (p * q) / P_h
  extern __shared__ uint32_t s_hist[];  // [kHistWords * kFastBS], dynamic (> 48 KB total)
  __shared__ double s_d[N_SC * kFastBS];   // [field][lane], flat
  __shared__ int32_t s_i[N_SI * kFastBS];
  __shared__ gt_meal_gen s_gen;
  __shared__ uint16_t s_mk[3][3][kFastBS];  // THREE_MEAL day window: ks, ke, kp offsets
  __shared__ double s_mc[3][kFastBS];       // THREE_MEAL day window: carbs (g)
  const int tid = threadIdx.x;
  for (int q = tid; q < GT_N_THRESHOLDS + 2; q += kFastBS)
    s_thr[q] = q == 0 ? LLONG_MIN : (q == GT_N_THRESHOLDS + 1 ? LLONG_MAX
                                                               : __double_as_longlong((double)(4 + q) / 10.0));
  for (int q = tid; q < kHistWords * kFastBS; q += kFastBS) s_hist[q] = 0u;
  if (tid == 0) s_gen = a.meal_gen;
  __syncthreads();
  if (CTRL == GT_CTRL_PID_PUMP)
    for (int q = tid; q < kPulseTab; q += kFastBS) s_prate[q] = D_(M_((double)q, u.hyper[7]), u.pid_ph);
  __syncthreads();  // no block-wide barrier after this point: warps run independently

  const int lane = tid & 31;
  // this lane's controller / extremes slots, field stride kFastBS; the lane
  // index is opaque so the base is kept instead of rebuilt from SR_TID
  int tid_o;
  asm("mov.b32 %0, %1;" : "=r"(tid_o) : "r"(tid));
  double* const sdl = s_d + tid_o;
  int32_t* const sil = s_i + tid_o;
  const int64_t n = a.n;
  const int64_t n_warps = sch.n_warps;
  // shared address of this lane's bin-0 byte, opaque to the compiler so it
  // stays in one register instead of being rebuilt every step
  uint32_t hist_lane;
  asm("mov.b32 %0, %1;" : "=r"(hist_lane)
      : "r"((uint32_t)__cvta_generic_to_shared(s_hist) + 4u * (GT_HISTLIN ? kHistWords * tid : tid)));
  // PSC > 0: the controller period's step count is a compile-time constant and
  // the period's plain steps are unrolled (no loop control, no register
  // rotation of the loop-carried noise / states)
  const int ps = PSC > 0 ? PSC : u.ps;
  const int cpd = u.ctl_per_day;

  for (;;) {
    // ------------------------------------------------------ claim a unit
    int unit = 0;
    if (lane == 0) unit = atomicAdd(sch.counter, 1);
    unit = __shfl_sync(0xffffffffu, unit, 0);
    if (unit >= sch.n_units) break;
    const int chunk = unit / sch.n_warps;
    const int64_t warp_global = unit - (int64_t)chunk * sch.n_warps;
    GT_CHECK(warp_global >= 0 && warp_global < sch.n_warps && chunk < sch.n_chunks, "unit");
    const int ctl_lo = chunk * sch.chunk_ctl;
    const int ctl_hi = min(u.n_ctl, ctl_lo + sch.chunk_ctl);
    const bool first = chunk == 0, last = chunk == sch.n_chunks - 1;
    const int64_t i = warp_global * 32 + lane;
    const bool inrange = i < n;
    const int64_t ii = inrange ? i : 0;
    const uint32_t pid = (uint32_t)(a.pid0 + i);
    const NoiseLane nlane = noise_lane(pid, u.nz_c2, u.nz_c3);
    auto philox_draw = [&](uint32_t index) -> U4 {
      return philox_lane(index, nlane, u.nz_a);
    };

    // rerun mode: only warps holding a diverged lane re-simulate (lanes masked).
    // Abort-tick pass (TRACE instance, rerun_diverged == 2): only the diverged
    // lanes run, with the reference's per-tick state check and per-step BG
    // check, and write nothing but their status and abort tick.
    const bool was_bad = a.rerun_diverged && inrange && a.status[i] == GT_STATUS_NONFINITE;
    const bool abort_pass = TRACE && a.rerun_diverged == 2;
    if (a.rerun_diverged && !__any_sync(0xffffffffu, was_bad)) {
      __syncwarp();
      if (lane == 0) st_release(sch.done + warp_global, chunk + 1);
      continue;
    }
    if (!first) {  // wait for the previous slice of these 32 patients
      if (lane == 0)
        while (ld_acquire(sch.done + warp_global) < chunk) __nanosleep(256);
      __syncwarp();
      __threadfence();
    }

    // ---- per-patient constants (recomputed per slice: cheap, register-free)
    PC<R> pc;
    {
      double p[NP];
#pragma unroll
      for (int k = 0; k < NP; ++k) p[k] = a.params[ii * NP + k];
      make_pc<R, kScX2>(p, u, pc);
    }
    R sqE = opaque(pc.sqE), sqG = (R)u.sqG;   // kept, not re-derived from the parameters in HBM
    if (NOISE == GT_NOISE_INJECTED && a.has_noise[ii] == 0) { sqE = 0; sqG = 0; }
    int64_t moff = 0, n_meals_csr = 0, ex_lo = 0, n_ex = 0;
    if (PROTO == GT_PROTO_CSR) {
      moff = a.meal_off[ii]; n_meals_csr = a.meal_off[ii + 1] - moff;
      ex_lo = a.ex_off[ii]; n_ex = a.ex_off[ii + 1] - ex_lo;
    }
    auto meal_at = [&](int32_t m) -> MealT {
      if (PROTO == GT_PROTO_CSR) {
        MealT r;
        if (m >= n_meals_csr) { r.ks = r.ke = r.kp = INT_MAX; r.rate = 0.0; r.carbs = 0.0; return r; }
        const int64_t q = moff + m;
        r.ks = a.meal_ks[q]; r.ke = a.meal_ke[q]; r.kp = a.meal_kp[q]; r.rate = a.meal_rate[q];
        r.carbs = a.meal_ann[q];
        return r;
      }
      return three_meal_at(&s_gen, a.seed, pid, m, u.dt, u.period, u.horizon_s);
    };

    // ---- lane state: initialise (first slice) or restore
    R Q1, Q2, S1, S2, I, X1, X2, X3, D1, D2, G, Z1, Z2, E1 = 0, E2 = 0, E3 = 0;
    R hu_ins, hu2, gin;  // per-step inputs, in the integrator precision
    double bg_sum, day_basal;
    int32_t m_ks, m_ke, act_lo = 0;
    int ann_rel = 0xFFFF;  // THREE_MEAL: period (from the day start) of the day's next announcement
    uint32_t act_len = 0;  // THREE_MEAL: meal input on for steps act_lo <= s < act_lo + act_len of this period
    int kb_min, kb_max, run39, run30, ev39, ev30, trig_lo;
    // GT_FKEY: FP32 round-toward-zero keys of the extremes so far and of the
    // low trigger.  rz is monotone, so bg < min_bg implies rz(bg) <= f_mn, bg >
    // max_bg implies rz(bg) >= f_mx and bg < 3.9 implies rz(bg) <= rz(3.9):
    // the branch is entered on a superset of the ticks that can change an
    // extreme or a hypo run, and decides exactly inside.
    float f_mn, f_mx, f_lo;
    constexpr uint32_t kF39Bits = 0x40799999u;   // rz(3.9) as FP32
    double tr_rate = 0.0, tr_y = 0.0, tr_basal = 0.0;  // TRACE only (held trace columns)
    bool alive;
    int status, death_tick;
    if (first) {
      alive = abort_pass ? was_bad : inrange && !was_bad && (a.active == nullptr || a.active[i] != 0);
      status = (inrange && !alive) ? GT_STATUS_EXCLUDED : GT_STATUS_OK;
      death_tick = -1;
      const double* x0 = a.x0 + ii * NS;
      Q1 = (R)x0[IQ1]; Q2 = (R)x0[IQ2]; S1 = (R)x0[IS1]; S2 = (R)x0[IS2]; I = (R)x0[II];
      X1 = (R)x0[IX1]; X2 = (R)x0[IX2]; X3 = (R)x0[IX3]; D1 = (R)x0[ID1]; D2 = (R)x0[ID2];
      G = (R)x0[IGSC]; Z1 = (R)x0[IZ1]; Z2 = (R)x0[IZ2];
      // scaled carried forms (GT_SCALE); the saved slice state keeps them scaled
      if (kScS1) S1 = (R)(x0[IS1] * (double)pc.hTI * (kScS2 ? (double)pc.dI : 1.0));
      if (kScS2) S2 = (R)(x0[IS2] * (double)pc.dI);
      if (kScX1) X1 = (R)(x0[IX1] * u.h);
      if (kScX2) X2 = (R)(x0[IX2] * u.h);
      if (kScG) G = (R)(x0[IGSC] / u.hS);
      if (kScD) { D1 = (R)(x0[ID1] * (double)pc.hTG); D2 = (R)(x0[ID2] * (double)pc.hTG); }
      if (CTRL == GT_CTRL_PID_PUMP) {  // no glucagon: Z1 = Z2 = 0 throughout (GT_STATUS_BAD_INITIAL_STATE)
        if (alive && (x0[IZ1] != 0.0 || x0[IZ2] != 0.0)) { alive = false; status = GT_STATUS_BAD_INITIAL_STATE; }
        Z1 = 0; Z2 = 0;
      }
      if (HAS_EX) { E1 = (R)x0[IE1]; E2 = (R)x0[IE2]; E3 = (R)x0[IE3]; }
      const double* c0 = a.c0 + ii * NC;
      sdl[(SC_FILT) * kFastBS] = c0[CFILT]; sdl[(SC_ICR) * kFastBS] = c0[CICR];
      sdl[(SC_SUSP) * kFastBS] = c0[CSUSPEND_UNTIL]; sdl[(SC_LASTG) * kFastBS] = c0[CLASTGLUC];
      sdl[(SC_WEND) * kFastBS] = c0[CWINEND]; sdl[(SC_WPEAK) * kFastBS] = c0[CWINPEAK]; sdl[(SC_WMIN) * kFastBS] = c0[CWINMIN];
      sil[(SI_FLAGS) * kFastBS] = (c0[CMODE] != 0.0) | ((c0[CEXBOLUSDONE] != 0.0) << 1) | ((c0[CINIT] != 0.0) << 2);
      sdl[(SC_ASSUMED) * kFastBS] = a.assumed_basal[ii];
      sdl[(SC_BGMIN) * kFastBS] = INFINITY;
      sdl[(SC_BGMAX) * kFastBS] = -INFINITY;
      sdl[(SC_DBOLUS) * kFastBS] = 0.0;
      sdl[(SC_DGLUC) * kFastBS] = 0.0;
      bg_sum = 0.0; day_basal = 0.0; hu_ins = 0; hu2 = 0;
      kb_min = INT_MAX; kb_max = -1; run39 = run30 = ev39 = ev30 = 0;
      f_mn = INFINITY; f_mx = -INFINITY;
      m_ks = m_ke = INT_MAX; gin = 0;
      if (PROTO == GT_PROTO_CSR) {
        const MealT m0 = meal_at(0);
        m_ks = m0.ks; m_ke = m0.ke; gin = (R)(u.ginK * m0.rate * (kScD ? (double)pc.hTG : 1.0));
        if (TRACE) tr_rate = m0.rate;
        sil[(SI_MEALM) * kFastBS] = 0;
        sil[(SI_ANNM) * kFastBS] = 0;
        sil[(SI_ANNKP) * kFastBS] = m0.kp;
        sdl[(SC_ANNCARBS) * kFastBS] = m0.carbs;
        sil[(SI_EXPTR) * kFastBS] = 0;
      }
      if (inrange && !abort_pass)
        for (int b = 0; b < GT_N_BG_BINS; ++b) a.bg_hist[(int64_t)b * n + i] = 0;
    } else {
      // every lane (padding included) restores its own slot: a padding lane
      // must not read a patient slot another warp may still be writing
      const int64_t npad = (int64_t)sch.n_warps * 32;
      const double* sd = sch.sd + i;
      const int* si = sch.si + i;
#define LDD(f) sd[(int64_t)(f) * npad]
#define LDI(f) si[(int64_t)(f) * npad]
      Q1 = (R)LDD(SD_Q1); Q2 = (R)LDD(SD_Q2); S1 = (R)LDD(SD_S1); S2 = (R)LDD(SD_S2); I = (R)LDD(SD_I);
      X1 = (R)LDD(SD_X1); X2 = (R)LDD(SD_X2); X3 = (R)LDD(SD_X3); D1 = (R)LDD(SD_D1); D2 = (R)LDD(SD_D2);
      G = (R)LDD(SD_G); Z1 = (R)LDD(SD_Z1); Z2 = (R)LDD(SD_Z2);
      if (CTRL == GT_CTRL_PID_PUMP) { Z1 = 0; Z2 = 0; }
      if (HAS_EX) { E1 = (R)LDD(SD_E1); E2 = (R)LDD(SD_E2); E3 = (R)LDD(SD_E3); }
      bg_sum = LDD(SD_BGSUM); day_basal = LDD(SD_DAYBASAL);
      hu_ins = (R)LDD(SD_HUINS); hu2 = (R)LDD(SD_HU2); gin = (R)LDD(SD_GIN);
      for (int q = 0; q < N_SC; ++q) sdl[(q) * kFastBS] = LDD(SD_SC0 + q);
      for (int q = 0; q < N_SI; ++q) sil[(q) * kFastBS] = LDI(SV_SI0 + q);
      // the histogram counters carried over from the previous slice
      for (int w = 0; w < kHistWords; ++w) s_hist[hword(w, tid)] = (uint32_t)LDI(SV_H0 + w);
      asm volatile("" ::: "memory");  // before the asm increments
      if (PROTO == GT_PROTO_THREE_MEAL) {
        for (int j = 0; j < 3; ++j) {
          s_mc[j][tid] = LDD(SD_MC0 + j);
          for (int f = 0; f < 3; ++f) s_mk[f][j][tid] = (uint16_t)LDI(SV_MK0 + 3 * f + j);
        }
      }
      m_ks = LDI(SV_MKS); m_ke = LDI(SV_MKE);  // act_lo / act_len are set at the slice's first tick
      if (PROTO == GT_PROTO_THREE_MEAL) {
        const int j = sil[(SI_ANNM) * kFastBS];
        GT_CHECK(j >= 0 && j <= 3, "restore ann cursor");
        ann_rel = j < 3 ? (int)s_mk[2][j][tid] : 0xFFFF;
      }
      kb_min = LDI(SV_KBMIN); kb_max = LDI(SV_KBMAX); run39 = LDI(SV_RUN39); run30 = LDI(SV_RUN30);
      f_mn = __int_as_float(kb_min); f_mx = __int_as_float(kb_max);   // (GT_FKEY: the slots hold the keys)
      ev39 = LDI(SV_EV39); ev30 = LDI(SV_EV30); alive = LDI(SV_ALIVE) != 0;
      status = LDI(SV_STATUS); death_tick = LDI(SV_DEATH);
#undef LDD
#undef LDI
      // every lane of the warp has read its slots: drop this warp's slot
      // lines (2 x 128 B per FP64 field, 128 B per int field) from L2
      __syncwarp();
      for (int r = lane; r < 2 * SD_N + SV_N; r += 32) {
        const char* line = r < 2 * SD_N
            ? reinterpret_cast<const char*>(sch.sd + (int64_t)(r >> 1) * npad + warp_global * 32) + (r & 1) * 128
            : reinterpret_cast<const char*>(sch.si + (int64_t)(r - 2 * SD_N) * npad + warp_global * 32);
        l2_discard_line(line);
      }
      alive = alive && inrange && !was_bad;  // padding lanes read patient 0's slot
    }

    // without the dead-lane sink (GT_DEAD_SINK bit off) a lane masked from the start (excluded, re-run mask, bad
    // initial state) counts into its shared bins like any other, and its
    // counts are never written out; a lane that dies during the run is
    // aborted and its statistics are discarded by the host either way
    const bool ran = status == GT_STATUS_OK || status == GT_STATUS_NONFINITE;
    // extremes / hypo-run bookkeeping is needed only for a bin <= trig_lo or >= kb_max
    trig_lo = run39 > 0 ? INT_MAX : max(kb_min, 34);  // 34: bg < 3.9 (THRESHOLDS[34])
    f_lo = run39 > 0 ? INFINITY : fmaxf(f_mn, __int_as_float(kF39Bits));

    // THREE_MEAL day window: the day's 3 meals, generated warp-uniformly at
    // the day's first tick (no divergence), tick offsets relative to the day
    // start (uint16, 0xFFFF = no meal) and carbs.
    int32_t day_ctl0 = (ctl_lo / cpd) * cpd;
    int32_t day_k0 = day_ctl0 * ps;
    auto load_slot = [&](int j) {
      GT_CHECK(j >= 0 && j < 3, "load_slot");
      const int ks = s_mk[0][j][tid];
      if (ks == 0xFFFF) { m_ks = m_ke = INT_MAX; gin = 0; return; }
      m_ks = day_k0 + ks; m_ke = day_k0 + s_mk[1][j][tid];
      gin = (R)(u.ginK * (s_mc[j][tid] / u.meal_dur_min)   // rate = g / duration (simulation.py:162)
                * (kScD ? (double)pc.hTG : 1.0));
      if (TRACE) tr_rate = s_mc[j][tid] / u.meal_dur_min;
    };
    auto gen_day = [&](int32_t d) {
      for (int j = 0; j < 3; ++j) {
        const MealT mt = three_meal_at(&s_gen, a.seed, pid, 3 * d + j, u.dt, u.period, u.horizon_s);
        const bool ok = mt.ks != INT_MAX;
        s_mk[0][j][tid] = ok ? (uint16_t)(mt.ks - day_k0) : (uint16_t)0xFFFF;
        s_mk[1][j][tid] = ok ? (uint16_t)(mt.ke - day_k0) : (uint16_t)0xFFFF;
        s_mk[2][j][tid] = ok ? (uint16_t)(mt.kp - day_ctl0) : (uint16_t)0xFFFF;
        s_mc[j][tid] = mt.carbs;
      }
      sil[(SI_MEALM) * kFastBS] = 0;
      load_slot(0);
      sil[(SI_ANNM) * kFastBS] = 0;
      ann_rel = s_mk[2][0][tid];
    };
    // flush the lane's uint8 histogram into its HBM column (bins 0..246;
    // bin 247 is the dead-lane sink) and clear it
    auto flush_hist = [&]() {
      asm volatile("" ::: "memory");  // order after the asm increments
      for (int w = 0; w < kHistWords; ++w) {
        const uint32_t word = s_hist[hword(w, tid)];
        if (word == 0u) continue;
        s_hist[hword(w, tid)] = 0u;
        if (!inrange || abort_pass) continue;
        if (!(GT_DEAD_SINK & kShape) && !ran) continue;   // a masked lane's counts are dropped
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint32_t c = (word >> (8 * b)) & 0xFFu;
          const int bin = 4 * w + b;
          // fire-and-forget RED (no load-use wait); the column is this lane's own
          if (c && bin < GT_N_BG_BINS) atomicAdd(&a.bg_hist[(int64_t)bin * n + i], (int32_t)c);
        }
      }
    };
    double hrr = 0.0;
    // CSR exercise: the current session (first with end > k) held in registers;
    // the cursor in shared memory moves only when a session ends
    int32_t ex_ks_c = INT_MAX, ex_ke_c = INT_MAX;
    double ex_hrr_c = 0.0;
    R ex_e1_c = 0;   // GT_EXFOLD: h/tau_hr * HRR of the current session, folded at session change
    auto load_session = [&](int p) {
      if (p < n_ex) { ex_ks_c = a.ex_ks[ex_lo + p]; ex_ke_c = a.ex_ke[ex_lo + p]; ex_hrr_c = a.ex_hrr[ex_lo + p]; }
      else { ex_ks_c = ex_ke_c = INT_MAX; ex_hrr_c = 0.0; }
      ex_e1_c = (R)(u.bE1 * ex_hrr_c);
    };
    if (HAS_EX) load_session(sil[(SI_EXPTR) * kFastBS]);
    // warp-uniform cursors derived from the slice start
    int next_grid_ctl = ((ctl_lo + u.grid_ctl - 1) / u.grid_ctl) * u.grid_ctl;
    int g_idx = next_grid_ctl / u.grid_ctl;
    int next_day_ctl = ((ctl_lo + cpd - 1) / cpd) * cpd;  // day start: flush (ctl > 0), day window

    // software-pipelined noise: the normals of tick k + 1 are drawn during
    // step k, next to its Euler update, so no step waits on its own Philox
    constexpr int kShapeBit = (PROTO == GT_PROTO_CSR ? 4 : 1) << (CTRL == GT_CTRL_PID_PUMP ? 0 : 1);
    constexpr bool PIPE = GT_NOISE_PIPE && !(GT_NOPIPE & kShapeBit) && NOISE == GT_NOISE_PHILOX && !AGG;
    constexpr bool PAIRS = (GT_PAIRS & kShapeBit) != 0;
    float pz0 = 0.f, pz1 = 0.f, pz2 = 0.f, pz3 = 0.f;   // GT_LAZYZM: pz3 holds the angle
    float prad = 0.f;
    constexpr bool LAZYZM = (GT_LAZYZM & kShapeBit) != 0;
    auto draw_pipe = [&](int32_t kk) {
      const U4 r = philox_draw((uint32_t)kk);
      box_muller(r.x, r.y, pz0, pz1);
      if (LAZYZM) { bm_polar(r.z, r.w, prad, pz3); pz2 = prad * cos_approx(pz3); }
      else box_muller(r.z, r.w, pz2, pz3);
    };
    if (PIPE) draw_pipe(ctl_lo * ps);

    // ---------------------------------------------------------- one step
    auto step = [&](const int32_t k, const bool tick, const int32_t ctl, const int32_t sk) {
      // noise for tick k (counter = (k, pid, role, 0)).  On a controller tick
      // the reading's normal is needed first; otherwise the draw is placed
      // next to the Euler update, in one basic block with the FP64 model
      // arithmetic, so the Philox chain overlaps it.
      R z0, z1, z2;
      double zm = 0.0;
      double tr_bolus = 0.0, tr_gluc = 0.0;  // TRACE only
      auto draw_noise = [&]() {
        if (PIPE) {
          z0 = pz0; z1 = pz1; z2 = pz2;
          if (tick) zm = LAZYZM ? prad * sin_approx(pz3) : pz3;
        } else if (NOISE == GT_NOISE_PHILOX) {
          if (!AGG) {
            const U4 r = philox_draw((uint32_t)k);
            float f0, f1, f2, f3;
            box_muller(r.x, r.y, f0, f1);
            box_muller(r.z, r.w, f2, f3);
            z0 = f0; z1 = f1; z2 = f2;
            if (tick) zm = f3;
          } else {
            // Brownian aggregation: this step's increment is the sum of the agg
            // fine increments at counters k*agg + j (the path a run at dt/agg
            // draws), rescaled to unit variance; the reading uses fine tick k*agg
            R s0 = 0, s1 = 0, s2 = 0;
            const uint32_t kf = (uint32_t)k * (uint32_t)u.agg;
            for (int j = 0; j < u.agg; ++j) {
              const U4 r = philox_draw(kf + (uint32_t)j);
              float f0, f1, f2, f3;
              box_muller(r.x, r.y, f0, f1);
              box_muller(r.z, r.w, f2, f3);
              s0 += (R)f0; s1 += (R)f1; s2 += (R)f2;
              if (j == 0 && tick) zm = f3;
            }
            const R sc = (R)u.rs_agg;
            z0 = s0 * sc; z1 = s1 * sc; z2 = s2 * sc;
          }
        } else {
          const double* wv = a.wiener + (ii * (int64_t)a.horizon_ticks + k) * 3;
          z0 = (R)wv[0]; z1 = (R)wv[1]; z2 = (R)wv[2];
          if (tick) zm = a.meas[ii * (int64_t)u.n_ctl + ctl];
        }
      };
      if (tick || PIPE) draw_noise();
      // disturbances at tick k (_kernel.py:85-94)
      if (PROTO == GT_PROTO_CSR) {
        while (k >= m_ke) {
          const int32_t m = sil[(SI_MEALM) * kFastBS] + 1;
          sil[(SI_MEALM) * kFastBS] = m;
          const MealT mt = meal_at(m);
          m_ks = mt.ks; m_ke = mt.ke; gin = (R)(u.ginK * mt.rate * (kScD ? (double)pc.hTG : 1.0));
          if (TRACE) tr_rate = mt.rate;
        }
      } else if (tick) {
        // generated meals are >= one period apart, so the active window of
        // the current meal within this period [act_lo, act_hi) is fixed here
        while (m_ke <= k) {
          const int j = ++sil[(SI_MEALM) * kFastBS];
          if (j < 3) load_slot(j);
          else { m_ks = m_ke = INT_MAX; gin = 0; }
        }
        // opaque moves: kept in two registers rather than rebuilt from m_ks/m_ke every step
        asm("mov.b32 %0, %1;" : "=r"(act_lo) : "r"(m_ks - k));
        asm("mov.b32 %0, %1;" : "=r"(act_len) : "r"(m_ke - m_ks));
      }
      const R gin_k = PROTO == GT_PROTO_CSR ? ((k >= m_ks) ? gin : (R)0)
                      : GT_KLOOP ? ((uint32_t)(k - m_ks) < act_len ? gin : (R)0)
                                 : ((uint32_t)(sk - act_lo) < act_len ? gin : (R)0);
      bool ex_active = false;
      if (HAS_EX) {
        if (__builtin_expect(k >= ex_ke_c, 0)) {  // the session ended: advance the cursor
          int p = sil[(SI_EXPTR) * kFastBS];
          while (p < n_ex && k >= a.ex_ke[ex_lo + p]) ++p;
          sil[(SI_EXPTR) * kFastBS] = p;
          load_session(p);
        }
        ex_active = k >= ex_ks_c;   // (k < ex_ke_c here)
        if (!GT_EXFOLD || TRACE) hrr = ex_active ? ex_hrr_c : 0.0;
      }
      // controller tick (_kernel.py:98-135): the check, the announcement and
      // the reading here.  Under kLateControl the controller itself runs
      // after the Euler update of the other states (only S1 / Z1 take its
      // output), so its serial FP64 chain overlaps the model's
      double t_s = 0.0, announced = 0.0, phase = -1.0, y = 0.0;
      if (tick) {
        t_s = (double)k * u.dt;
        // The reference checks every state at every tick (_kernel.py:98-103).
        // Non-finiteness is absorbing here: a linear update a*x + b (a > 0)
        // keeps Inf/NaN, a projected Q1/Q2 at +Inf turns NaN the next step
        // (Inf - Inf) and NaN survives the projection; so a state that is
        // non-finite at any tick is non-finite at the horizon's last tick,
        // and that one check is equivalent to the reference's per-tick checks.
        // (The injected-noise gut clamp is the one exception, beyond ~30 sigma.)
        // (a traced launch checks every tick, as the reference does, so its
        // abort tick is the reference's: the abort-tick pass relies on it)
        if ((!GT_LASTCHECK || TRACE || ctl == u.n_ctl - 1) && alive) {
          // x * 0 is +-0 for finite x and NaN for Inf/NaN: one FMA per state,
          // in four short chains
          const R z = 0;
          R a0 = FMR(Q1, z, FMR(Q2, z, FMR(S1, z, z)));
          R a1 = FMR(S2, z, FMR(I, z, FMR(X1, z, z)));
          R a2 = FMR(X2, z, FMR(X3, z, FMR(D1, z, z)));
          R a3 = FMR(D2, z, FMR(G, z, FMR(Z1, z, FMR(Z2, z, z))));
          if (HAS_EX) { a0 = FMR(E1, z, a0); a1 = FMR(E2, z, a1); a2 = FMR(E3, z, a2); }
          const R acc = (a0 + a1) + (a2 + a3);
          if (acc != acc) { alive = false; status = GT_STATUS_NONFINITE; death_tick = k; }
        }
        // announced carbs starting within [t, t+P)
        if (PROTO == GT_PROTO_THREE_MEAL) {
          // meals are >= 1 h apart, so at most one starts in a period: the
          // day's next announcement is a cursor (0 + carbs = the reference's sum)
          if (ctl - day_ctl0 == ann_rel) {
            const int j = sil[(SI_ANNM) * kFastBS];
            GT_CHECK(j >= 0 && j < 3, "announce cursor");
            announced = A_(0.0, s_mc[j][tid]);
            sil[(SI_ANNM) * kFastBS] = j + 1;
            ann_rel = j + 1 < 3 ? (int)s_mk[2][j + 1][tid] : 0xFFFF;
          }
        }
        int32_t akp = PROTO == GT_PROTO_CSR ? sil[(SI_ANNKP) * kFastBS] : INT_MAX;
        if (akp <= ctl) {
          int32_t am = sil[(SI_ANNM) * kFastBS];
          double carbs = sdl[(SC_ANNCARBS) * kFastBS];
          while (akp <= ctl) {
            if (akp == ctl) announced += carbs;
            ++am;
            const MealT mt = meal_at(am);
            akp = mt.kp; carbs = mt.carbs;
          }
          sil[(SI_ANNM) * kFastBS] = am; sil[(SI_ANNKP) * kFastBS] = akp; sdl[(SC_ANNCARBS) * kFastBS] = carbs;
        }
        if (HAS_EX && ex_active) {
          const int p = sil[(SI_EXPTR) * kFastBS];
          if (a.ex_announced[ex_lo + p] != 0.0) phase = t_s - a.ex_start_s[ex_lo + p];
        }
        y = A_(kScG ? (double)G * u.hS : (double)G, M_(u.sqrtR, zm));
        if (TRACE) tr_y = y;
      }
      constexpr bool kPidFlat = CTRL == GT_CTRL_PID_PUMP && (GT_PIDFLAT & kShapeBit) != 0;
      auto control = [&]() {
        // ---- controller_step_vec (controller.py:343-458); state in shared
        // memory.  Explicit IEEE operations in the reference's order: the
        // controller is bit-identical to the reference's for identical readings.
        int flags = sil[(SI_FLAGS) * kFastBS];
        double filt = sdl[(SC_FILT) * kFastBS], prev;
        if (kPidFlat) {   // the same values by selects (no branch: one basic block with the model)
          const bool init = (flags & 4) != 0;
          const double fn = A_(M_(u.hc[1], filt), M_(u.hyper[HFILTER], y));
          prev = init ? filt : y;
          filt = init ? fn : y;
          flags |= 4;
        } else if (!(flags & 4)) { filt = y; prev = y; flags |= 4; }
        else { prev = filt; filt = A_(M_(u.hc[1], filt), M_(u.hyper[HFILTER], y)); }
        sdl[(SC_FILT) * kFastBS] = filt;
        const double trend = S_(filt, prev);
        double b_basal = 0.0, b_bolus = 0.0, b_gluc = 0.0;
        if (CTRL == GT_CTRL_PID_PUMP) {   // the controller is a template parameter: one per kernel
          // ---- PID + pump quantisation (pid.py pid_step_vec), same filter;
          // slots: SC_WEND = integral, SC_SUSP = pump carry
          const double e = S_(filt, u.hyper[1]);
          const double ph = u.pid_ph;   // period / 3600, folded on the host (same IEEE quotient)
          double integ = A_(sdl[(SC_WEND) * kFastBS], M_(e, ph));
          if (integ > u.hyper[6]) integ = u.hyper[6];
          if (integ < -u.hyper[6]) integ = -u.hyper[6];
          sdl[(SC_WEND) * kFastBS] = integ;
          double factor = A_(A_(A_(1.0, M_(u.hyper[2], e)), M_(u.hyper[3], integ)), M_(u.hyper[4], trend));
          if (factor < 0.0) factor = 0.0;
          if (factor > u.hyper[5]) factor = u.hyper[5];
          const double vol = A_(M_(M_(sdl[(SC_ASSUMED) * kFastBS], factor), ph), sdl[(SC_SUSP) * kFastBS]);
          // floor(vol / q) of the IEEE quotient: vol * RN(1/q) is within 1e-13
          // of it, so its floor is exact unless it lies within 1e-9 of an
          // integer (then the division is done)
          const double qf = M_(vol, u.hc[5]);
          double pulses = floor(qf);
          const double fr = S_(qf, pulses);
          const bool exact = fr > 1e-9 && fr < 1.0 - 1e-9 && qf < 1e6;
          if (kPidFlat) {
            // the common path without branches (selects, the table lookup on a
            // clamped index); the division cases and the meal bolus -- a few
            // ticks per day -- in one rare branch that recomputes exactly what
            // the branchy form below computes
            pulses = pulses < 0.0 ? 0.0 : pulses;
            double delivered = M_(pulses, u.hyper[7]);
            double susp = S_(vol, delivered);
            const bool tab = pulses < (double)kPulseTab;
            b_basal = s_prate[tab ? (int)pulses : 0];
            if (__builtin_expect(!exact || !tab || announced > 0.0, 0)) {
              if (!exact) {
                pulses = floor(D_(vol, u.hyper[7]));
                if (pulses < 0.0) pulses = 0.0;
                delivered = M_(pulses, u.hyper[7]);
                susp = S_(vol, delivered);
              }
              b_basal = pulses < (double)kPulseTab ? s_prate[(int)pulses] : D_(delivered, ph);
              if (announced > 0.0) {
                double bb = D_(announced, sdl[(SC_ICR) * kFastBS]);
                if (bb > u.hyper[9]) bb = u.hyper[9];
                b_bolus = M_(floor(D_(bb, u.hyper[8])), u.hyper[8]);
              }
            }
            sdl[(SC_SUSP) * kFastBS] = susp;
          } else {
          if (!exact) pulses = floor(D_(vol, u.hyper[7]));
          if (pulses < 0.0) pulses = 0.0;
          const double delivered = M_(pulses, u.hyper[7]);
          sdl[(SC_SUSP) * kFastBS] = S_(vol, delivered);
          // (p * q) / P_h from the table (same operations), else computed
          b_basal = pulses < (double)kPulseTab ? s_prate[(int)pulses] : D_(delivered, ph);
          if (announced > 0.0) {
            double bb = D_(announced, sdl[(SC_ICR) * kFastBS]);
            if (bb > u.hyper[9]) bb = u.hyper[9];
            b_bolus = M_(floor(D_(bb, u.hyper[8])), u.hyper[8]);
          }
          }
        } else {
        const bool exercising = HAS_EX && phase >= 0.0;
        const double setpoint = exercising ? u.hyper[HEXSETPOINT] : u.hyper[HSETPOINT];
        const double gluc_thr = exercising ? u.hyper[HEXGLUCTHR] : u.hyper[HGLUCTHR];
        double micro = exercising ? u.hyper[HEXMICROUG] : u.hyper[HMICROUG];
        bool done = false;
        if (exercising) {
          if (!(flags & 2)) {
            flags |= 2;
            if (filt < u.hyper[HEXBOLUSBG]) {
              b_gluc = fmin(u.hyper[HEXBOLUS], u.hyper[HMAXGLUC]);
              sdl[(SC_LASTG) * kFastBS] = t_s;
              done = true;
            }
          }
        } else {
          flags &= ~2;
        }
        if (!done) {
          const double pred = A_(filt, M_(trend, u.hc[0]));
          if (!(flags & 1)) {
            if (filt < gluc_thr || pred < gluc_thr) flags |= 1;
          } else {
            if (filt >= (exercising ? u.hc[4] : u.hc[3]) && pred >= gluc_thr) flags &= ~1;
          }
          const double wend = sdl[(SC_WEND) * kFastBS];
          if (wend > 0.0) {
            const double wpeak = fmax(sdl[(SC_WPEAK) * kFastBS], filt);
            const double wmin = fmin(sdl[(SC_WMIN) * kFastBS], filt);
            sdl[(SC_WPEAK) * kFastBS] = wpeak; sdl[(SC_WMIN) * kFastBS] = wmin;
            if (t_s >= wend) {
              double icr = sdl[(SC_ICR) * kFastBS];
              if (wmin < u.hyper[HUNDERBG]) icr = M_(icr, A_(1.0, u.hyper[HICRSTEPUP]));
              else if (S_(wpeak, u.hyper[HSETPOINT]) > u.hyper[HEXCHI]) icr = M_(icr, S_(1.0, u.hyper[HICRSTEP]));
              if (icr < u.hyper[HICRMIN]) icr = u.hyper[HICRMIN];
              if (icr > u.hyper[HICRMAX]) icr = u.hyper[HICRMAX];
              sdl[(SC_ICR) * kFastBS] = icr;
              sdl[(SC_WEND) * kFastBS] = 0.0;
            }
          }
          if (flags & 1) {
            if (filt < gluc_thr && trend < -u.hyper[HMICROTREND] && S_(t_s, sdl[(SC_LASTG) * kFastBS]) >= u.hc[2]) {
              if (micro > u.hyper[HMAXGLUC]) micro = u.hyper[HMAXGLUC];
              b_gluc = micro;
              sdl[(SC_LASTG) * kFastBS] = t_s;
            }
          } else {
            const double assumed = sdl[(SC_ASSUMED) * kFastBS];
            if (announced > 0.0) {
              const double icr = sdl[(SC_ICR) * kFastBS];
              double b = A_(D_(announced, icr), D_(S_(filt, setpoint), M_(u.hyper[HCFICR], icr)));
              if (filt > u.hyper[HSUPBG]) b = A_(b, D_(M_(M_(u.hyper[HSUPFRAC], assumed), u.hyper[HSUSPMIN]), 60.0));
              if (b < 0.0) b = 0.0;
              if (b > u.hyper[HMAXBOLUS]) b = u.hyper[HMAXBOLUS];
              b_bolus = b;
              sdl[(SC_SUSP) * kFastBS] = A_(t_s, M_(u.hyper[HSUSPMIN], 60.0));
              sdl[(SC_WEND) * kFastBS] = A_(t_s, M_(u.hyper[HMEALWIN], 60.0));
              sdl[(SC_WPEAK) * kFastBS] = filt;
              sdl[(SC_WMIN) * kFastBS] = filt;
            }
            if (!(t_s < sdl[(SC_SUSP) * kFastBS])) {
              double factor = A_(A_(1.0, M_(u.hyper[HBKP], S_(filt, setpoint))), M_(u.hyper[HBKD], trend));
              if (factor < 0.0) factor = 0.0;
              if (factor > u.hyper[HBFMAX]) factor = u.hyper[HBFMAX];
              double b = M_(assumed, factor);
              if (exercising) b = M_(b, u.hyper[HEXBFACTOR]);
              b_basal = b;
            }
          }
        }
        }  // dual_hormone
        sil[(SI_FLAGS) * kFastBS] = flags;
        day_basal = fma(b_basal, (double)ps, day_basal);  // basal held for the whole period
        if (TRACE) { tr_basal = b_basal; tr_bolus = b_bolus; tr_gluc = b_gluc; }
        hu_ins = (R)fma(b_bolus, u.u_bolus_k, b_basal * u.u_basal_k);   // h * (u[0] + u[1])
        if (kScS1) hu_ins = hu_ins * pc.hTI;                            // carried S1 is hTI * S1
        if (kScS2) hu_ins = hu_ins * pc.dI;                             //   (times dI)
        hu2 = (R)(b_gluc * u.u_gluc_k);                                 // h * u[2]
        if (b_bolus > 0.0 || b_gluc > 0.0) {
          sdl[(SC_DBOLUS) * kFastBS] += b_bolus;
          sdl[(SC_DGLUC) * kFastBS] += b_gluc;
        }
      };
      // late control measured -1.2 % under pid_pump and +3.8 % under
      // dual_hormone (whose larger controller then spills), and +2 % on the
      // CSR (NorthernYear) path: pid_pump with the generated meals only
      constexpr bool kLateControl = !TRACE && (GT_LATE & kShapeBit) != 0;
      if (tick && !kLateControl) control();
      // statistics at tick k (_kernel.py:137-160)
      double bg = (double)MR_(Q1, pc.invVGw);  // explicit: never fused into the sums below
      if (tick && ctl == 0) {
        // the steady state puts BG(0) on a histogram edge (6.0 = THRESHOLDS[55],
        // SURVEY.md §7): use the reference's exact division for that tick
        bg = Q1 / (a.params[ii * NP + PVG] * a.params[ii * NP + PW]);
      }
      // traced launches: the reference's per-step BG check (_kernel.py:139-141),
      // so the abort tick is exact; other launches check bg_sum after the horizon
      if (TRACE && alive && !(fabs(bg) < INFINITY)) { alive = false; status = GT_STATUS_NONFINITE; death_tick = k; }
      if (!GT_ABL_TL && tick && ctl == next_grid_ctl) {  // timeline point (warp-uniform)
        next_grid_ctl += u.grid_ctl;
        const long long v = __double2ll_rn(bg * kFpScale);
        // 0 <= v < 2^31 (bg < 128 mmol/L) for every live lane: four 32-bit
        // REDUX; otherwise (or a NaN) the exact 64-bit shuffle path, out of line
        long long ssum, smin, smax;
        if (__builtin_expect(__any_sync(0xffffffffu, alive && (v < 0 || v > 0x7FFFFFFELL)), 0)) {
          timeline_partials64(alive, v, ssum, smin, smax);
        } else {
          const unsigned vv = alive ? (unsigned)v : 0u;
          const unsigned lo = __reduce_add_sync(0xffffffffu, vv & 0xFFFFu);
          const unsigned hi = __reduce_add_sync(0xffffffffu, vv >> 16);
          const unsigned mn = __reduce_min_sync(0xffffffffu, alive ? vv : 0xFFFFFFFFu);
          const int mx = __reduce_max_sync(0xffffffffu, alive ? (int)vv : -1);
          ssum = ((long long)hi << 16) + (long long)lo;
          smin = mn == 0xFFFFFFFFu ? LLONG_MAX : (long long)mn;
          smax = mx < 0 ? LLONG_MIN : (long long)mx;
        }
        if (lane == 0 && !abort_pass) {
          GT_CHECK(g_idx >= 0 && g_idx < a.n_grid, "timeline");
          long long* dst = (long long*)a.timeline_warp + ((int64_t)g_idx * n_warps + warp_global) * 3;
          dst[0] = ssum; dst[1] = smin; dst[2] = smax;
        }
        if (a.timeline_pp && inrange && !abort_pass) a.timeline_pp[(int64_t)g_idx * n + i] = alive ? bg : 0.0;
        ++g_idx;
      }
      if (TRACE && inrange && a.trace) {  // the parity kernel's 8 trace columns (simulation.py:61-64)
        double* tr = a.trace + ((int64_t)i * a.horizon_ticks + k) * 8;
        tr[0] = (double)k * u.dt; tr[1] = bg; tr[2] = tr_y; tr[3] = gin_k != (R)0 ? tr_rate : 0.0;
        tr[4] = hrr; tr[5] = tr_basal; tr[6] = tr_bolus; tr[7] = tr_gluc;
      }
      if (PIPE && !GT_ABL_NOISE) draw_pipe(k + 1);
      else if (!tick) draw_noise();
      // Euler–Maruyama step, re-associated (hovorka.py:76-150)
      // (in R: launch-uniform constants are rounded to R at their use)
      const R bgR = (R)bg, zero = 0, one = 1;
      const R ab = HAS_EX ? FMR((R)u.sex, E3, one) : one;
      const R ub = HAS_EX ? FMR((R)u.qex, E2, one) : one;
      const R x1e = X1 * ab, x2e = X2 * ab;   // (kScX1: x1e is h * X1 * ab)
      // Q1's loop-carried chain is kept short: the Q1-independent terms
      // (gut, Q2 exchange, EGP, noise) are summed first, off the chain, and
      // the Q1 terms enter as one FMA plus the two clamped fluxes
      const R egp = FMR(-pc.hE, X3, pc.hE);
      // pid_pump doses no glucagon: Z2 = 0 exactly and cG * 0 + e == e
      const R hegp = CTRL == GT_CTRL_PID_PUMP ? pos_or_zero(egp) : FMR((R)u.cG, Z2, pos_or_zero(egp));
      R pq = FMR(pc.hk12, Q2, kScD ? D2 : D2 * pc.hTG) + hegp;
      pq = FMR(sqE, z0, pq);
      const R a1 = kScX1 ? one - x1e : FMR(-(R)u.h, x1e, one);  // 1 - h x1e
      // h F01 w min(bg/4.5, 1); GT_F01Q: as h F01/(4.5 VG) min(Q1, 4.5 VG w), off the bg multiply
      const R hf01 = GT_F01Q ? MR_(pc.hF01Q, lt_or(Q1, pc.Q45)) : MR_(pc.hF01w45, lt_or(bgR, (R)4.5));
      const R hren = pos_or_zero(FMR(Q1, (R)u.rK1, -pc.rK0));
      R q1n = FMR(Q1, a1, pq);
      q1n = FMR(-hf01, ub, q1n);
      q1n = q1n - hren;
      // projection max(x, 0) (_kernel.py:175-177): keeps NaN like `if x < 0: x = 0`
      const R q2n = FMR(Q2, kScX2 ? pc.aK12 - x2e : FMR(-(R)u.h, x2e, pc.aK12), (kScX1 ? x1e : (R)u.h * x1e) * Q1);
      const R nQ1 = zero_if_neg(q1n);
      const R nQ2 = zero_if_neg(q2n);
      R nD1 = FMR(D1, FMR(sqG, z1, pc.aG), gin_k);
      R nD2 = FMR(D2, FMR(sqG, z2, pc.aG), D1 * pc.hTG);
      if (CLAMP_GUT) { nD1 = zero_if_neg(nD1); nD2 = zero_if_neg(nD2); }
      const R nS2 = FMR(S2, pc.aI, kScS1 ? S1 : S1 * pc.hTI);
      if (!tick || !kLateControl) S1 = FMR(S1, pc.aI, hu_ins);
      const R nI = FMR(I, pc.cI, kScS2 ? S2 : S2 * pc.dI);
      S2 = nS2;
      X1 = FMR(X1, pc.ax1, I * pc.bx1);
      X2 = FMR(X2, pc.ax2, I * pc.bx2);
      X3 = FMR(X3, pc.ax3, I * pc.bx3);
      I = nI;
      if (CTRL != GT_CTRL_PID_PUMP) {  // (pid_pump: the chain stays at 0)
        const R nZ2 = FMR(Z2, (R)u.aZ2, Z1 * (R)u.hTg);
        if (!tick || !kLateControl) Z1 = FMR(Z1, (R)u.aZ1, hu2);
        Z2 = nZ2;
      }
      if (HAS_EX) {
        const R nE2 = FMR(E2, (R)u.aE2, E1 * (R)u.bE2);
        const R nE3 = FMR(E3, (R)u.aE3, E1 * (R)u.bE3);
        E1 = FMR(E1, (R)u.aE1, GT_EXFOLD ? (ex_active ? ex_e1_c : (R)0) : (R)(u.bE1 * hrr));
        E2 = nE2; E3 = nE3;
      }
      G = kScG ? FMR(G, (R)u.aS, bgR) : FMR(G, (R)u.aS, bgR * (R)u.hS);
      Q1 = nQ1; Q2 = nQ2; D1 = nD1; D2 = nD2;
      if (tick && kLateControl) {  // the controller, then the two states that take its output
        if (!GT_ABL_CTRL) control();
        S1 = FMR(S1, pc.aI, hu_ins);
        if (CTRL != GT_CTRL_PID_PUMP) Z1 = FMR(Z1, (R)u.aZ1, hu2);
      }
      // Statistics of tick k's BG, binned after the update so the bin chain
      // overlaps the model's FP64 chain.  A non-finite bg (_kernel.py:139-141)
      // is caught lazily: bg_sum absorbs Inf/NaN and is checked after the last
      // step.  Until then the lane's statistics are garbage but in range; an
      // aborted patient's are discarded and its warp re-run with it masked.
      {
        // searchsorted(THRESHOLDS, bg, 'right') for bg >= 0.  THRESHOLDS[i] =
        // RN((5+i)/10), so away from a threshold the bin is floor(10 bg) - 4
        // (clamped to [0, 246]); the FP32 estimate decides whenever 10 bg is
        // more than 1e-4 from an integer (its error is < 4e-5 up to bg = 25.6)
        // and the exact int64 compare against the table settles the rest.
        const float fbg = __double2float_rz(bg);
        const float t10 = fbg * 10.0f;
        const float fl = floorf(t10);
        int kb = min(max((int)fl - 4, 0), GT_N_THRESHOLDS);
        // near an integer: |t10 - rint(t10)| <= 1e-4 (one FSETP on |x|)
        const bool near_edge = (GT_RINT & kShapeBit) ? !(fabsf(t10 - rintf(t10)) > 1e-4f)
                                       : !((t10 - fl) > 1e-4f && (t10 - fl) < 0.9999f);
        if (__builtin_expect(near_edge, 0)) {
          const long long bb = __double_as_longlong(bg);
          kb = min(max(kb, 0), GT_N_THRESHOLDS);
          kb += (s_thr[kb + 1] <= bb) - (s_thr[kb] > bb);
        }
        if (GT_DEAD_SINK & kShape) kb = alive ? kb : GT_N_BG_BINS;  // dead lanes count into the padding bin 247
        {  // byte ((kb >> 2) * kFastBS + tid) * 4 + (kb & 3)
          GT_CHECK(kb >= 0 && kb <= GT_N_BG_BINS, "histogram bin");
          const uint32_t ha = GT_HISTLIN ? hist_lane + (uint32_t)kb
                                         : hist_lane + (uint32_t)(kb & ~3) * (uint32_t)kFastBS + (uint32_t)(kb & 3);
          uint32_t c;
          asm volatile("{\n\t.reg .u32 t;\n\tld.shared.u8 t, [%1];\n\tadd.u32 %0, t, 1;\n\t"
                       "st.shared.u8 [%1], %0;\n\t}" : "=r"(c) : "r"(ha));
          // a full counter drains into the HBM column (1 tick in 255): the
          // column address is formed only on that path
          if (__builtin_expect(c == 255u, 0)) {
            asm volatile("st.shared.u8 [%0], 0;" :: "r"(ha) : "memory");
            if (kb < GT_N_BG_BINS && inrange && !abort_pass && ((GT_DEAD_SINK & kShape) || ran)) {
              // 32-bit element offset (the launcher bounds 247 n < 2^31): the drain
              // path then needs fewer scratch registers than a 64-bit index
              if (GT_DRAIN32 & kShapeBit) atomicAdd(a.bg_hist + (uint32_t)(kb * (uint32_t)n + (uint32_t)i), 255);
              else atomicAdd(a.bg_hist + ((int64_t)kb * n + i), 255);
            }
          }
        }
        bg_sum += bg;
        // extremes: only a tick in the lowest/highest bin so far can move them;
        // hypo runs: only ticks below 3.9 mmol/L (or ending such a run) matter
        if (GT_FKEY) {
          if (__builtin_expect(fbg <= f_lo || fbg >= f_mx, 0) && alive) {
            const double omn = sdl[(SC_BGMIN) * kFastBS], omx = sdl[(SC_BGMAX) * kFastBS];
            if (bg < omn) { sdl[(SC_BGMIN) * kFastBS] = bg; f_mn = fbg; }   // _kernel.py:144-147
            if (bg > omx) { sdl[(SC_BGMAX) * kFastBS] = bg; f_mx = fbg; }
            run39 = kb <= 34 ? run39 + 1 : 0;  // bg < 3.9 (THRESHOLDS[34])
            run30 = kb <= 25 ? run30 + 1 : 0;  // bg < 3.0 (THRESHOLDS[25])
            ev39 += run39 == u.hypoL;
            ev30 += run30 == u.hypoL;
            f_lo = run39 > 0 ? INFINITY : fmaxf(f_mn, __int_as_float(kF39Bits));
          }
        } else if (__builtin_expect(kb <= trig_lo || kb >= kb_max, 0) && alive) {
          if (kb <= kb_min) { const double o = sdl[(SC_BGMIN) * kFastBS]; sdl[(SC_BGMIN) * kFastBS] = bg < o ? bg : o; kb_min = kb; }
          if (kb >= kb_max) { const double o = sdl[(SC_BGMAX) * kFastBS]; sdl[(SC_BGMAX) * kFastBS] = bg > o ? bg : o; kb_max = kb; }
          run39 = kb <= 34 ? run39 + 1 : 0;  // bg < 3.9 (THRESHOLDS[34])
          run30 = kb <= 25 ? run30 + 1 : 0;  // bg < 3.0 (THRESHOLDS[25])
          ev39 += run39 == u.hypoL;
          ev30 += run30 == u.hypoL;
          trig_lo = run39 > 0 ? INT_MAX : max(kb_min, 34);
        }
      }
    };

    // ------------------------------------------------- the slice's periods
    int ctl = ctl_lo;
    for (; ctl < ctl_hi; ++ctl) {
      // day boundary: flush the finished day's dose sums (_kernel.py:133-149)
      if (ctl == next_day_ctl) {
        next_day_ctl += cpd;
        // flush the finished day's dose sums (_kernel.py:133-149)
        if (ctl > 0) {
          const int64_t day = ctl / cpd - 1;
          GT_CHECK(day >= 0 && day < a.n_days, "day flush");
          if (inrange && !abort_pass) {
            double* dd = a.day_dose + (day * 3) * n + i;
            dd[0] = day_basal; dd[n] = sdl[(SC_DBOLUS) * kFastBS]; dd[2 * n] = sdl[(SC_DGLUC) * kFastBS];
          }
          day_basal = 0.0; sdl[(SC_DBOLUS) * kFastBS] = 0.0; sdl[(SC_DGLUC) * kFastBS] = 0.0;
        }
        if (PROTO == GT_PROTO_THREE_MEAL) {
          day_ctl0 = ctl; day_k0 = ctl * ps;
          gen_day(ctl / cpd);
        }
        // lanes die only at the horizon's last tick: an all-dead warp is one
        // masked from the start (excluded / re-run lanes); checked per day
        if (GT_DAY_VOTE && __all_sync(0xffffffffu, !alive)) break;
      }
      if (!GT_DAY_VOTE && __all_sync(0xffffffffu, !alive)) break;
      const int32_t kb0 = ctl * ps;
      step(kb0, true, ctl, 0);
      if (PSC > 0) {
#pragma unroll
        for (int s = 1; s < PSC; ++s) step(kb0 + s, false, ctl, s);
      } else if (GT_KLOOP == 2 || PAIRS) {   // pairs of plain steps (loop-carried registers alternate)
        const int32_t kend = kb0 + ps;
        int32_t k = kb0 + 1;
        for (; k + 1 < kend; k += 2) { step(k, false, ctl, 0); step(k + 1, false, ctl, 0); }
        if (k < kend) step(k, false, ctl, 0);
      } else if (GT_KLOOP) {
        const int32_t kend = kb0 + ps;
        for (int32_t k = kb0 + 1; k < kend; ++k) step(k, false, ctl, 0);
      } else {
        for (int s = 1; s < ps; ++s) step(kb0 + s, false, ctl, s);
      }
    }
    // an all-dead warp stops early: its remaining timeline partials are identities
    for (; next_grid_ctl < ctl_hi; next_grid_ctl += u.grid_ctl, ++g_idx)
      if (lane == 0 && !abort_pass) {
        GT_CHECK(g_idx >= 0 && g_idx < a.n_grid, "timeline tail");
        long long* dst = (long long*)a.timeline_warp + ((int64_t)g_idx * n_warps + warp_global) * 3;
        dst[0] = 0; dst[1] = LLONG_MAX; dst[2] = LLONG_MIN;
      }
    // the last slice drains the counters into the HBM columns; earlier ones
    // carry them in the saved lane state (no read-modify-write of the
    // [247][n] columns per slice).  Either way the shared counters end empty.
    if (last) flush_hist();

    if (last && alive && !(fabs(bg_sum) < INFINITY)) {  // the lazy bg check (see the step)
      alive = false; status = GT_STATUS_NONFINITE; death_tick = (int)a.horizon_ticks;
    }
    if (!last) {
      // ---- save the lane state for the next slice (padding lanes too); the
      // warp barrier orders these stores after the other lanes' discards of
      // the same lines at this unit's restore
      __syncwarp();
      {
        const int64_t npad = (int64_t)sch.n_warps * 32;
        double* sd = sch.sd + i;
        int* si = sch.si + i;
        const uint64_t keep = l2_evict_last_policy();
#define STD(f, v) st_keep(sd + (int64_t)(f) * npad, (double)(v), keep)
#define STI(f, v) st_keep(si + (int64_t)(f) * npad, (int)(v), keep)
        STD(SD_Q1, Q1); STD(SD_Q2, Q2); STD(SD_S1, S1); STD(SD_S2, S2); STD(SD_I, I);
        STD(SD_X1, X1); STD(SD_X2, X2); STD(SD_X3, X3); STD(SD_D1, D1); STD(SD_D2, D2);
        STD(SD_G, G); STD(SD_Z1, Z1); STD(SD_Z2, Z2);
        if (HAS_EX) { STD(SD_E1, E1); STD(SD_E2, E2); STD(SD_E3, E3); }
        STD(SD_BGSUM, bg_sum); STD(SD_DAYBASAL, day_basal); STD(SD_HUINS, hu_ins);
        STD(SD_HU2, hu2); STD(SD_GIN, gin);
        for (int q = 0; q < N_SC; ++q) STD(SD_SC0 + q, sdl[(q) * kFastBS]);
        for (int q = 0; q < N_SI; ++q) STI(SV_SI0 + q, sil[(q) * kFastBS]);
        asm volatile("" ::: "memory");  // after the asm increments
        for (int w = 0; w < kHistWords; ++w) {
          STI(SV_H0 + w, (int)s_hist[hword(w, tid)]);
          s_hist[hword(w, tid)] = 0u;
        }
        if (PROTO == GT_PROTO_THREE_MEAL) {
          for (int j = 0; j < 3; ++j) {
            STD(SD_MC0 + j, s_mc[j][tid]);
            for (int f = 0; f < 3; ++f) STI(SV_MK0 + 3 * f + j, s_mk[f][j][tid]);
          }
        }
        STI(SV_MKS, m_ks); STI(SV_MKE, m_ke);
        if (GT_FKEY) { STI(SV_KBMIN, __float_as_int(f_mn)); STI(SV_KBMAX, __float_as_int(f_mx)); }
        else { STI(SV_KBMIN, kb_min); STI(SV_KBMAX, kb_max); }
        STI(SV_RUN39, run39); STI(SV_RUN30, run30);
        STI(SV_EV39, ev39); STI(SV_EV30, ev30); STI(SV_ALIVE, alive ? 1 : 0);
        STI(SV_STATUS, status); STI(SV_DEATH, death_tick);
#undef STD
#undef STI
      }
    } else if (abort_pass) {   // the diverged lanes' exact abort tick (simulation.py:381)
      if (was_bad) {
        a.status[i] = status == GT_STATUS_OK ? GT_STATUS_NONFINITE : status;
        a.ticks[i] = status == GT_STATUS_OK ? a.horizon_ticks : (death_tick < 0 ? 0 : death_tick);
      }
    } else if (inrange && !was_bad) {  // a rerun keeps the diverged lanes' outputs
      // ---- final outputs
      const int64_t last_day = a.n_days - 1;
      double* dd = a.day_dose + (last_day * 3) * n + i;
      dd[0] = day_basal; dd[n] = sdl[(SC_DBOLUS) * kFastBS]; dd[2 * n] = sdl[(SC_DGLUC) * kFastBS];
      a.status[i] = status;
      a.ticks[i] = status == GT_STATUS_OK ? a.horizon_ticks : (death_tick < 0 ? 0 : death_tick);
      a.bg_stats[i] = sdl[(SC_BGMIN) * kFastBS];
      a.bg_stats[n + i] = sdl[(SC_BGMAX) * kFastBS];
      a.bg_stats[2 * n + i] = bg_sum;
      a.hypo_events[i] = ev39;
      a.hypo_events[n + i] = ev30;
      if (a.x_out) {
        const double hTG = (double)pc.hTG;
        const double fS1 = (kScS1 ? (double)pc.hTI : 1.0) * (kScS2 ? (double)pc.dI : 1.0);
        const double xs[NS] = {(double)Q1, (double)Q2, (double)S1 / fS1,
                               kScS2 ? (double)S2 / (double)pc.dI : (double)S2, (double)I,
                               kScX1 ? (double)X1 / u.h : (double)X1,
                               kScX2 ? (double)X2 / u.h : (double)X2, (double)X3, kScD ? (double)D1 / hTG : (double)D1,
                               kScD ? (double)D2 / hTG : (double)D2, kScG ? (double)G * u.hS : (double)G,
                               (double)Z1, (double)Z2, (double)E1, (double)E2, (double)E3};
        for (int k = 0; k < NS; ++k) a.x_out[(int64_t)k * n + i] = xs[k];
      }
    }
    // ---- release this slice
    __syncwarp();
    __threadfence();
    if (lane == 0) st_release(sch.done + warp_global, chunk + 1);
  }
}

// host-side folding of the fixed parameters (same expressions as make_pc)
static Uni make_uni(const gt_fast_args& a) {
  const double* f = a.fixed;
  Uni u{};
  const double h = a.dt_s / 60.0;
  u.h = h;
  u.ginK = h * f[PAG] * kMmolPerGCho;
  u.hS = h / f[PTAUCGM]; u.aS = 1.0 - u.hS;
  u.hTg = h / f[PTGLUC]; u.aZ1 = 1.0 - u.hTg; u.aZ2 = 1.0 - h * f[PKEGLUC];
  u.cG = h * f[PSGLUC] / f[PVGLUC];
  u.bE1 = h / f[PTAUHR]; u.aE1 = 1.0 - u.bE1;
  u.bE2 = h / f[PTAUEX]; u.aE2 = 1.0 - u.bE2;
  u.aE3 = 1.0 - h / f[PTAULATE]; u.bE3 = h * f[PALATE];
  u.qex = f[PQEX]; u.sex = f[PSEX];
  u.sqG = f[PSIGGUT] * std::sqrt(h);
  u.sigEh = f[PSIGEGP] * std::sqrt(h);
  u.sqrtR = std::sqrt(f[PR]);
  u.rK1 = h * 0.003;
  u.dt = a.dt_s; u.period = a.period_s;
  u.horizon_s = (double)a.horizon_ticks * a.dt_s;
  u.meal_dur_min = (double)a.meal_gen.duration_s / 60.0;
  u.u_basal_k = h * (1000.0 / 60.0);
  u.u_bolus_k = h * (1000.0 / (a.period_s / 60.0));
  u.u_gluc_k = h * (1.0 / (a.period_s / 60.0));
  u.ps = (int32_t)a.period_steps;
  u.n_ctl = (int32_t)(a.horizon_ticks / a.period_steps);
  u.ctl_per_day = (int32_t)std::llround(86400.0 / a.period_s);
  u.grid_ctl = (int32_t)(a.grid_step_ticks / a.period_steps);
  u.hypoL = (int32_t)a.hypo_min_ticks;
  u.agg = a.noise_agg < 1 ? 1 : a.noise_agg;
  u.rs_agg = 1.0 / std::sqrt((double)u.agg);
  u.pid_ph = a.period_s / 3600.0;
  // controller constants: single IEEE operations, identical on host and device
  // (controller.py:393 prediction factor, filter complement, lock-out, hysteresis)
  for (int k = 0; k < GT_N_HYPER; ++k) u.hyper[k] = a.hyper[k];
  const double* hy = a.hyper;
  u.hc[0] = (hy[HPREDHOR] * 60.0) / a.period_s;
  u.hc[1] = 1.0 - hy[HFILTER];
  u.hc[2] = hy[HLOCKMIN] * 60.0;
  u.hc[3] = hy[HGLUCTHR] + hy[HHYST];
  u.hc[4] = hy[HEXGLUCTHR] + hy[HHYST];
  u.hc[5] = a.controller == GT_CTRL_PID_PUMP ? 1.0 / hy[7] : 0.0;   // PID: RN(1 / pulse size)
  u.nz_c2 = (uint32_t)a.seed;
  u.nz_c3 = (uint32_t)(a.seed >> 32) ^ (a.noise_role << 24);
  u.nz_a = (uint32_t)(((uint64_t)u.nz_c2 * 0xCD9E8D57u) >> 32) ^ kNoiseKey0;
  return u;
}

}  // namespace gt

// Number of horizon slices.  Per-warp cost varies with the patients'
// trajectories (hypo runs, meals), so the persistent schedule balances better
// with several units per resident warp slot: aim for >= 6 rounds of units,
// then take the fewest slices whose wave quantisation ceil(c * warps / slots)
// / c is within 1 % of the least in that range.  A slice keeps >= 48
// controller periods; each boundary moves ~0.65 KB per lane through L2.
// Measured on 100k x 4 weeks (PID): 5 slices 38.0 ms, 9-25 slices 35.9-36.6 ms.
static int choose_chunks(int64_t warps, int64_t slots, int n_ctl) {
  const int c_max = std::max(1, std::min(32, n_ctl / 48));
  // (fewer warps than slots: one slice; a warp's slices run in sequence anyway)
  const int c_min = warps < slots ? 1
                                  : (int)std::max<int64_t>(1, std::min<int64_t>(c_max, (6 * slots + warps - 1) / warps));
  // the fewest slices whose quantised rounds come within 1 % of the best:
  // every slice boundary saves and restores ~0.65 KB per lane
  auto t_of = [&](int c) { return (double)((c * warps + slots - 1) / slots) / c; };
  double best_t = 1e300;
  for (int c = c_min; c <= c_max; ++c) best_t = std::min(best_t, t_of(c));
  for (int c = c_min; c <= c_max; ++c)
    if (t_of(c) <= best_t * 1.01) return c;
  return c_min;
}

template <int PROTO, int NOISE, typename R, bool AGG, bool TRACE, int CTRL, int PSC = 0>
static int launch_sched(const gt_fast_args* a, const gt::Uni& u, cudaStream_t st) {
  constexpr int kBit = (PROTO == GT_PROTO_CSR ? 4 : 1) << (CTRL == GT_CTRL_PID_PUMP ? 0 : 1);
  constexpr bool kPs5 = (GT_PS5 & kBit) != 0 && !TRACE && !AGG;
  if (PSC == 0 && kPs5 && a->period_steps == 5)
    return launch_sched<PROTO, NOISE, R, AGG, TRACE, CTRL, kPs5 ? 5 : 0>(a, u, st);
  constexpr int kDyn = gt::kHistWords * gt::kFastBS * 4;
  auto kern = gt::fast_kernel<PROTO, NOISE, R, AGG, TRACE, CTRL, PSC>;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  // the > 48 KB dynamic shared-memory opt-in is a per-device attribute: set
  // it on every launch (cheap) rather than once per process
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kDyn) != cudaSuccess) {
    gt_set_error("gt_simulate_fast: cudaFuncSetAttribute(MaxDynamicSharedMemorySize) failed");
    return GT_ECUDA;
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, gt::kFastBS, kDyn);
  if (per_sm < 1) per_sm = 1;
  const int64_t warps = (a->n + 31) / 32;
  const int64_t slots = (int64_t)sms * per_sm * (gt::kFastBS / 32);
  const int n_ctl = u.n_ctl;
  // a traced launch runs unsliced (the held trace columns are not saved between slices)
  // an explicit slice count is clamped to the horizon's periods and to the
  // 32-bit unit counter (warps * slices < 2^31; advisor finding r01)
  const int max_chunks = (int)std::max<int64_t>(1, std::min<int64_t>(n_ctl, INT32_MAX / std::max<int64_t>(warps, 1)));
  const int chunks = TRACE ? 1 : a->n_slices > 0 ? std::min(a->n_slices, max_chunks) : std::min(choose_chunks(warps, slots, n_ctl), max_chunks);
  gt::Sched s{};
  s.n_warps = (int)warps;
  s.n_chunks = chunks;
  s.chunk_ctl = (n_ctl + chunks - 1) / chunks;
  s.n_chunks = (n_ctl + s.chunk_ctl - 1) / s.chunk_ctl;
  s.n_units = (int)(warps * s.n_chunks);
  // scratch: counter + done flags (+ saved lane state when slicing)
  const size_t bytes_i = sizeof(int) * (1 + (size_t)warps);
  const size_t n_pad = (size_t)warps * 32;   // every lane of a warp owns a saved-state slot
  const size_t bytes_state = s.n_chunks > 1 ? n_pad * (gt::SD_N * sizeof(double) + gt::SV_N * sizeof(int)) : 0;
  const size_t need = bytes_i + 256 + bytes_state;  // state rows 256-byte aligned (L2 line discards)
  char* scratch = static_cast<char*>(a->scratch);
  const bool own = scratch == nullptr;
  if (own) {
    gt_keep_pool_mapped();
    if (cudaMallocAsync(&scratch, need, st) != cudaSuccess) {
      gt_set_error("gt_simulate_fast: scratch allocation failed");
      return GT_ECUDA;
    }
  } else if (a->scratch_bytes < (int64_t)need || (reinterpret_cast<uintptr_t>(scratch) & 15u)) {
    gt_set_error("gt_simulate_fast: scratch must be 16-byte aligned and >= gt_fast_scratch_bytes(n)");
    return GT_EINVAL;
  }
  cudaMemsetAsync(scratch, 0, bytes_i, st);
  s.counter = reinterpret_cast<int*>(scratch);
  s.done = s.counter + 1;
  if (bytes_state) {
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(scratch) + bytes_i + 255) & ~uintptr_t(255));
    s.sd = reinterpret_cast<double*>(base);
    s.si = reinterpret_cast<int*>(base + n_pad * gt::SD_N * sizeof(double));
  }
  const int64_t blocks_needed = (warps + gt::kFastBS / 32 - 1) / (gt::kFastBS / 32);
  const unsigned grid = (unsigned)std::min<int64_t>((int64_t)sms * per_sm, blocks_needed);
  kern<<<grid, gt::kFastBS, kDyn, st>>>(*a, u, s);
  const int e = gt_check_launch("fast_kernel");
  if (own) cudaFreeAsync(scratch, st);
  return e;
}

template <int PROTO, int NOISE, typename R = double, bool AGG = false>
static int launch_one(const gt_fast_args* a, const gt::Uni& u, cudaStream_t st) {
  const bool pid = a->controller == GT_CTRL_PID_PUMP;
  if (a->trace || a->rerun_diverged == 2)   // traced, or the abort-tick pass (exact checks)
    return pid ? launch_sched<PROTO, NOISE, R, AGG, true, GT_CTRL_PID_PUMP>(a, u, st)
               : launch_sched<PROTO, NOISE, R, AGG, true, GT_CTRL_DUAL_HORMONE>(a, u, st);
  return pid ? launch_sched<PROTO, NOISE, R, AGG, false, GT_CTRL_PID_PUMP>(a, u, st)
             : launch_sched<PROTO, NOISE, R, AGG, false, GT_CTRL_DUAL_HORMONE>(a, u, st);
}

// The fused kernel's noise stream, materialised: out[(i * n_ticks + j) * 4 + l]
// = normal l of tick k0 + j of patient pid0 + i, drawn exactly as the kernel
// draws it (philox_lane: Philox4x32-7, + FP32 SFU Box-Muller; lanes 0-2 = Wiener, 3 = CGM).
namespace gt {
__global__ void noise_normals_kernel(int64_t n, int64_t pid0, int64_t k0, int64_t n_ticks, const Uni u,
                                     float* out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * n_ticks) return;
  const int64_t i = idx / n_ticks, j = idx - i * n_ticks;
  const U4 r = philox_lane((uint32_t)(k0 + j), noise_lane((uint32_t)(pid0 + i), u.nz_c2, u.nz_c3), u.nz_a);
  float f0, f1, f2, f3;
  box_muller(r.x, r.y, f0, f1);
  box_muller(r.z, r.w, f2, f3);
  float* o = out + idx * 4;
  o[0] = f0; o[1] = f1; o[2] = f2; o[3] = f3;
}
}  // namespace gt

int gt_launch_noise_normals(int64_t n, int64_t pid0, uint64_t seed, uint32_t role, int64_t k0,
                            int64_t n_ticks, float* out, cudaStream_t st) {
  if (n <= 0 || n_ticks <= 0) return GT_OK;
  gt::Uni u{};
  u.nz_c2 = (uint32_t)seed;
  u.nz_c3 = (uint32_t)(seed >> 32) ^ (role << 24);
  u.nz_a = (uint32_t)(((uint64_t)u.nz_c2 * 0xCD9E8D57u) >> 32) ^ gt::kNoiseKey0;
  const int64_t total = n * n_ticks;
  gt::noise_normals_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(n, pid0, k0, n_ticks, u, out);
  return gt_check_launch("noise_normals_kernel");
}

// Upper bound of launch_one's scratch (sliced schedule) for n patients.
int64_t gt_fast_scratch_need(int64_t n) {
  const int64_t warps = (n + 31) / 32;
  const int64_t bytes_i = (int64_t)sizeof(int) * (1 + warps);
  return bytes_i + 256 + warps * 32 * (int64_t)(gt::SD_N * sizeof(double) + gt::SV_N * sizeof(int));
}

int gt_launch_fast(const gt_fast_args* a, cudaStream_t st) {
  if (a->n <= 0) return GT_OK;
  if (a->grid_step_ticks % a->period_steps != 0) {
    gt_set_error("gt_simulate_fast: grid step must be a multiple of the controller period");
    return GT_EUNSUPPORTED;
  }
  if (a->proto_kind == GT_PROTO_THREE_MEAL) {
    const gt_meal_gen& g = a->meal_gen;
    const bool in_day = g.clock_s[0] - g.jitter_s >= 0.0 &&
                        g.clock_s[2] + g.jitter_s + g.duration_s <= 86400.0;
    const double span = 2.0 * g.jitter_s + g.duration_s;
    const bool apart = g.clock_s[1] - g.clock_s[0] >= span + a->period_s &&
                       g.clock_s[2] - g.clock_s[1] >= span + a->period_s;
    if ((double)g.duration_s < a->dt_s || a->dt_s < 2.0 || !in_day || !apart) {
      gt_set_error("gt_simulate_fast: 3-meal generator needs meals within the day, >= one "
                   "controller period apart, lasting >= one step, and dt >= 2 s");
      return GT_EUNSUPPORTED;
    }
  }
  if (a->n * (int64_t)GT_N_BG_BINS > (int64_t)INT32_MAX) {  // the histogram drain's 32-bit element offsets
    gt_set_error("gt_simulate_fast: too many patients for one launch (247 n must fit 31 bits); shard the population");
    return GT_EINVAL;
  }
  if ((a->n + 31) / 32 > INT32_MAX / 8) {
    gt_set_error("gt_simulate_fast: too many patients for one launch; shard the population");
    return GT_EINVAL;
  }
  if (a->noise_agg < 1 || (a->noise_agg > 1 && a->noise_kind != GT_NOISE_PHILOX) ||
      (int64_t)a->noise_agg * a->horizon_ticks > (int64_t)UINT32_MAX) {
    gt_set_error("gt_simulate_fast: noise_agg must be >= 1, > 1 only with Philox noise, and "
                 "noise_agg * horizon_ticks must fit the 32-bit tick counter");
    return GT_EINVAL;
  }
  const gt::Uni u = gt::make_uni(*a);
  const int pk = a->proto_kind, nk = a->noise_kind;
  if (a->precision == 1) {  // FP32 integrator: the generated-meal / Philox path only
    if (pk == GT_PROTO_THREE_MEAL && nk == GT_NOISE_PHILOX)
      return u.agg > 1 ? launch_one<GT_PROTO_THREE_MEAL, GT_NOISE_PHILOX, float, true>(a, u, st)
                       : launch_one<GT_PROTO_THREE_MEAL, GT_NOISE_PHILOX, float, false>(a, u, st);
    gt_set_error("gt_simulate_fast: the FP32 integrator supports the 3-meal generator with "
                 "Philox noise only");
    return GT_EUNSUPPORTED;
  }
  if (a->precision != 0) {
    gt_set_error("gt_simulate_fast: precision must be 0 (FP64) or 1 (FP32)");
    return GT_EINVAL;
  }
  if (pk == GT_PROTO_THREE_MEAL && nk == GT_NOISE_PHILOX)
    return u.agg > 1 ? launch_one<GT_PROTO_THREE_MEAL, GT_NOISE_PHILOX, double, true>(a, u, st)
                     : launch_one<GT_PROTO_THREE_MEAL, GT_NOISE_PHILOX>(a, u, st);
  if (pk == GT_PROTO_THREE_MEAL && nk == GT_NOISE_INJECTED)
    return launch_one<GT_PROTO_THREE_MEAL, GT_NOISE_INJECTED>(a, u, st);
  if (pk == GT_PROTO_CSR && nk == GT_NOISE_PHILOX)
    return u.agg > 1 ? launch_one<GT_PROTO_CSR, GT_NOISE_PHILOX, double, true>(a, u, st)
                     : launch_one<GT_PROTO_CSR, GT_NOISE_PHILOX>(a, u, st);
  if (pk == GT_PROTO_CSR && nk == GT_NOISE_INJECTED)
    return launch_one<GT_PROTO_CSR, GT_NOISE_INJECTED>(a, u, st);
  gt_set_error("gt_simulate_fast: unsupported proto_kind=%d noise_kind=%d", pk, nk);
  return GT_EUNSUPPORTED;
}
