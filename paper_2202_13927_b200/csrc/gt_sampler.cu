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
#include <climits>
#include <cmath>
// the steady-state solve is one out-of-line function (code size: the kernel is
// instruction-fetch bound when every call site inlines it)
#define GT_SS_NOINLINE 1
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
// through a long rejection chain.  Each round:
//   1. cheap rules: a lane without a pending survivor draws only the normal
//      values of its next attempt (3 of the 7 Philox blocks) and applies the
//      reference's first two rules -- any value negative (lognormals never
//      are), a normal draw outside 1 SD (85 % of all rejections);
//   2. once kBatch lanes hold a survivor (or every lane still working does),
//      those lanes draw the survivor's lognormal values and run the
//      steady-state solve (brentq) together, then the u_basal rule.
// A lane keeps its survivor across rounds until the batch fills, so the
// expensive solves run with most of the warp converged.  The draws are
// counter-addressed and the rules are applied in the reference's order
// (population.py:217-259), so the population is bit-identical to the
// one-thread-per-patient loop (oracle_sample_patients, tests/test_gpu_sampler.py).
// A patient still without an accepted set after kPark attempts of one body
// weight (~0.5 % of patients: light weights have low acceptance; a weight
// below ~30 kg never succeeds and spends the whole 10 000-attempt budget) is
// handed to straggler_kernel, which searches its remaining attempts 128 at a
// time with a whole block instead of one lane.
// One attempt's values written into the packed parameter vector.
__device__ __noinline__ void fill_attempt_p(const gt_sampler_args& a, uint32_t actr, uint32_t pid, uint32_t k0,
                                            uint32_t k1, double* p) {
#pragma unroll 1
  for (int q = 0; q < a.n_sampled; q += 2) {
    const U4 r = philox4x32_10(actr, pid, kRoleSamplerParams, (uint32_t)(q >> 1), k0, k1);
    p[a.param_index[q]] = sampled_value(a, q, det_inv_norm(u52(r.x, r.y)));
    if (q + 1 < a.n_sampled) p[a.param_index[q + 1]] = sampled_value(a, q + 1, det_inv_norm(u52(r.z, r.w)));
  }
}

// ---- cheap rules on the uniform key
// A normal value v = a + b * inv_norm(u52(k)) is a monotone function of the
// 52-bit key k (the uniform's integer image), so each of the reference's
// cheap rules -- v < 0, v - a < -b, v - a > b -- flips once along k.  A setup
// kernel locates each flip with the exact device arithmetic (bisection on k);
// phase 1 then decides a value from k alone, and evaluates it exactly only
// when k falls within a band around a flip (about 1e-5 of the draws).  The
// band (|k - K| <= min(K, 2^52 - K) / 2^16 + 2^16, i.e. ~1e-5 relative in u)
// is many orders wider than the ulp-level non-monotonicity of the
// floating-point inverse CDF, so every decision equals the exact one.
struct KeyRule {
  unsigned long long e[3], w[3];  // band of flip f: k - e[f] < w[f] (unsigned); f: 0 neg, 1 low, 2 high
  unsigned long long k_neg, k_lo, k_hi;  // neg: k < k_neg; low: k < k_lo; high: k >= k_hi
};
constexpr unsigned long long kKeyEnd = 1ull << 52;

__device__ __forceinline__ unsigned long long key52(uint32_t a, uint32_t b) {
  return ((unsigned long long)(a >> 6) << 26) | (unsigned long long)(b >> 6);
}
__device__ __forceinline__ double normal_at(const gt_sampler_args& a, int j, unsigned long long k) {
  return A_(a.a[j], M_(a.b[j], det_inv_norm(M_((double)(2 * k + 1), 1.1102230246251565404e-16))));
}
// rule f at key k, exactly (f 0: v < 0; 1: v - a < -b; 2: v - a > b)
__device__ bool rule_exact(const gt_sampler_args& a, int j, int f, unsigned long long k) {
  const double v = normal_at(a, j, k);
  if (f == 0) return v < 0.0;
  const double d = S_(v, a.a[j]);
  return f == 1 ? d < -a.b[j] : d > a.b[j];
}

// thread (j, f): the flip of rule f of sampled normal j
__global__ void key_rules_kernel(gt_sampler_args a, KeyRule* rules) {
  const int j = threadIdx.x / 3, f = threadIdx.x % 3;
  if (j >= a.n_sampled) return;
  unsigned long long K;
  if (a.kind[j] != 0) {
    K = f == 2 ? kKeyEnd : 0;                     // lognormals: no cheap rule
  } else if (f < 2) {                             // true below the flip
    unsigned long long lo = 0, hi = kKeyEnd;      // rule(lo) true, rule(hi) false
    if (!rule_exact(a, j, f, 0)) K = 0;
    else {
      while (hi - lo > 1) {
        const unsigned long long mid = lo + (hi - lo) / 2;
        if (rule_exact(a, j, f, mid)) lo = mid; else hi = mid;
      }
      K = hi;
    }
  } else {                                        // true from the flip on
    unsigned long long lo = 0, hi = kKeyEnd - 1;  // rule(lo) false, rule(hi) true
    if (!rule_exact(a, j, f, hi)) K = kKeyEnd;
    else if (rule_exact(a, j, f, 0)) K = 0;
    else {
      while (hi - lo > 1) {
        const unsigned long long mid = lo + (hi - lo) / 2;
        if (rule_exact(a, j, f, mid)) hi = mid; else lo = mid;
      }
      K = hi;
    }
  }
  const bool flips = a.kind[j] == 0 && K > 0 && K < kKeyEnd;
  const unsigned long long m = flips ? ((K < kKeyEnd - K ? K : kKeyEnd - K) >> 16) + (1ull << 16) : 0;
  const unsigned long long e = K > m ? K - m : 0;
  rules[j].e[f] = e;
  rules[j].w[f] = flips ? K + m + 1 - e : 0;
  // a normal entry whose value is not increasing in k (sd <= 0 or not finite):
  // no flip structure to rely on, every draw is evaluated exactly
  if (a.kind[j] == 0 && f == 0 && !(a.b[j] > 0.0 && a.b[j] < INFINITY && fabs(a.a[j]) < INFINITY)) {
    rules[j].e[0] = 0;
    rules[j].w[0] = kKeyEnd + 1;
  }
  (f == 0 ? rules[j].k_neg : f == 1 ? rules[j].k_lo : rules[j].k_hi) = K;
}

// The reference's first two rules on one normal draw (population.py:234-244),
// from its key: exact inside a flip band, by the flips elsewhere.
// bit 0: v < 0, bit 1: outside one SD (out of line: rare)
__device__ __noinline__ int key_exact(const gt_sampler_args& a, int j, unsigned long long k) {
  const double v = normal_at(a, j, k);
  return (v < 0.0 ? 1 : 0) | (fabs(S_(v, a.a[j])) > a.b[j] ? 2 : 0);
}
__device__ __forceinline__ void key_verdict(const gt_sampler_args& a, const KeyRule& r, int j,
                                            unsigned long long k, bool& neg, bool& outside) {
  if (k - r.e[0] < r.w[0] || k - r.e[1] < r.w[1] || k - r.e[2] < r.w[2]) {
    const int v = key_exact(a, j, k);
    neg |= (v & 1) != 0;
    outside |= (v & 2) != 0;
  } else {
    neg |= k < r.k_neg;
    outside |= k < r.k_lo || k >= r.k_hi;
  }
}

#ifndef GT_SAMPLER_PARK
#define GT_SAMPLER_PARK 384
#endif
constexpr int kPark = GT_SAMPLER_PARK;   // attempts of one body weight before a patient is parked
#ifndef GT_STRAG_BS
#define GT_STRAG_BS 512
#endif
constexpr int kStragBS = GT_STRAG_BS;    // straggler_kernel: attempts evaluated per round
#ifndef GT_SAMPLER_CAP
#define GT_SAMPLER_CAP 1   // with solve batching: 1 ~ 2 ~ 8 (tools/ab_sampler.sh); 4 was best without
#endif
constexpr int kCap = GT_SAMPLER_CAP;   // cheap attempts per lane per round
#ifndef GT_SAMPLER_BATCH
#define GT_SAMPLER_BATCH 24
#endif
constexpr int kBatch = GT_SAMPLER_BATCH;  // lanes holding a survivor before the warp solves
constexpr int kMaxSampled = 16;
struct Straggler {
  int64_t i;
  int32_t total, attempt, wdraw, last_surv;  // last_surv: counter of the latest cheap-rule survivor, -1 none
  uint32_t wctr, pad;
  double w;
};

// population.py:148-153 _positive_normal: the next positive weight draw of
// the patient's weight stream (0 when the budget is spent); advances *wctr.
__device__ __noinline__ double draw_weight_dev(const gt_sampler_args& a, uint32_t pid, uint32_t* wctr,
                                               uint32_t k0, uint32_t k1) {
  uint32_t c = *wctr;
  double w = 0.0;
  for (int t = 0; t < a.max_attempts; ++t, ++c) {
    const U4 r = philox4x32_10(c, pid, kRoleSamplerWeight, 0u, k0, k1);
    const double v = A_(a.weight_mean, M_(a.weight_sd, det_inv_norm(u52(r.x, r.y))));
    if (v > 0.0) { w = v; ++c; break; }
  }
  *wctr = c;
  return w;
}

#ifndef GT_SAMPLER_MINB
#define GT_SAMPLER_MINB 2
#endif
__global__ void __launch_bounds__(128, GT_SAMPLER_MINB) sampler_kernel(gt_sampler_args a, const KeyRule* rules,
                                                      unsigned long long* queue,
                                                      Straggler* park, unsigned int* n_park, int park_cap) {
  __shared__ KeyRule s_rules[kMaxSampled];
  for (int t = threadIdx.x; t < a.n_sampled; t += blockDim.x) s_rules[t] = rules[t];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
  // the attempt's values go straight into p (no separate value registers)
  double p[GT_N_PARAMS], x[GT_N_STATES];
  double ub = 0.0, w = 0.0;
  int64_t i = -1;                       // this lane's patient (-1: none)
  int32_t attempt = 0, total = 0, wdraw = 0, last_surv = -1;
  uint32_t wctr = 0, pid = 0;
  bool park_full = false;
  bool survivor = false;   // holds a cheap-rule survivor awaiting its solve (phase 2)
  long long rej_neg = 0, rej_sd = 0, rej_ss = 0, rej_basal = 0;
  bool drained = false;
  auto draw_weight = [&]() {             // population.py:148-153
    w = draw_weight_dev(a, pid, &wctr, k0, k1);
    p[PW] = w;
    attempt = 0;
  };
  auto finish = [&](int status) {
    if (status != 0) {
      // the sequential loop's last p holds the latest survivor's values (or the
      // fixed ones if none survived); phase 1 wrote later attempts' normals
      for (int j = 0; j < a.n_sampled; ++j) p[a.param_index[j]] = a.fixed_params[a.param_index[j]];
      if (last_surv >= 0) fill_attempt_p(a, (uint32_t)last_surv, pid, k0, k1, p);
    }
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
          total = 0; wdraw = 0; wctr = 0; last_surv = -1;
          draw_weight();
        } else {
          drained = true;
        }
      }
    }
    if (__all_sync(0xffffffffu, i < 0)) break;
    // ---- phase 1: cheap rules until a survivor, at most kCap attempts this
    // round (a lane without a survivor skips phase 2 and continues next round:
    // the warp never waits for one lane's long rejection chain)
    if (i >= 0 && !survivor) {
      for (int c = 0; c < kCap && !survivor && i >= 0; ++c) {
        if (attempt >= a.max_attempts || !(w > 0.0)) {
          // budget spent for this body weight: redraw it or fail
          total += attempt;
          if (wdraw < a.max_weight_redraws) { ++wdraw; draw_weight(); continue; }
          finish(1);
          break;
        }
        if (attempt >= kPark && !park_full) {   // hand the rest of this patient to straggler_kernel
          const unsigned slot = atomicAdd(n_park, 1u);
          if ((int)slot < park_cap) {
            park[slot] = Straggler{i, total, attempt, wdraw, last_surv, wctr, 0u, w};
            i = -1;
            break;
          }
          park_full = true;   // list full: carry on in this lane
        }
        const uint32_t actr = (uint32_t)(total + attempt);
        // the normal draws' keys only (lognormals are never negative and have no SD rule)
        bool neg = false, outside = false;
#pragma unroll 1
        for (int q = 0; q < kMaxSampled; q += 2) {
          if (q >= a.n_sampled) break;
          const bool n0 = a.kind[q] == 0, n1 = q + 1 < a.n_sampled && a.kind[q + 1] == 0;
          if (!(n0 || n1)) continue;
          const U4 r = philox4x32_10(actr, pid, kRoleSamplerParams, (uint32_t)(q >> 1), k0, k1);
          if (n0) key_verdict(a, s_rules[q], q, key52(r.x, r.y), neg, outside);
          if (n1) key_verdict(a, s_rules[q + 1], q + 1, key52(r.z, r.w), neg, outside);
        }
        if (neg) { ++rej_neg; ++attempt; continue; }          // population.py:234-236
        if (outside) { ++rej_sd; ++attempt; continue; }       // population.py:237-244
        survivor = true;
      }
    }
    // ---- phase 2: the survivors' lognormal draws and steady-state solves, once
    // enough lanes hold one (kBatch) or every lane still working does, so the
    // solves run with most of the warp converged on them
    const unsigned hold = __ballot_sync(0xffffffffu, survivor);
    const unsigned busy = __ballot_sync(0xffffffffu, i >= 0);
    const bool go = __popc(hold) >= kBatch || hold == busy;
    if (survivor && go) {
      survivor = false;
      const uint32_t actr = (uint32_t)(total + attempt);
      fill_attempt_p(a, actr, pid, k0, k1, p);   // the survivor's values, normals included
      last_surv = (int32_t)actr;
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

// One attempt's values (all sampled parameters), counter-addressed.
__device__ __noinline__ void draw_attempt(const gt_sampler_args& a, uint32_t actr, uint32_t pid, uint32_t k0,
                                          uint32_t k1, double* vals) {
#pragma unroll 1
  for (int q = 0; q < a.n_sampled; q += 2) {
    const U4 r = philox4x32_10(actr, pid, kRoleSamplerParams, (uint32_t)(q >> 1), k0, k1);
    vals[q] = sampled_value(a, q, det_inv_norm(u52(r.x, r.y)));
    if (q + 1 < a.n_sampled) vals[q + 1] = sampled_value(a, q + 1, det_inv_norm(u52(r.z, r.w)));
  }
}

// The parked patients, one block each.  A round takes the next kStragBS x
// kStragC attempts of the current body weight: every thread applies the cheap
// rules to kStragC consecutive attempts, the survivors are compacted in
// attempt order (block scan) and solved in parallel, the lowest accepted
// attempt wins, and only the attempts before it are counted -- exactly the
// sequential loop's result and rejection counts.  A body weight that never
// succeeds (its 10 000-attempt budget spent) takes 3 rounds, each about one
// solve long, instead of 20.
#ifndef GT_STRAG_C
#define GT_STRAG_C 8
#endif
constexpr int kStragC = GT_STRAG_C;

// cheap-rule code of one attempt: 1 a negative value, 2 outside one SD, 3 survivor
__device__ __forceinline__ int cheap_code(const gt_sampler_args& a, const KeyRule* rules, uint32_t actr,
                                          uint32_t pid, uint32_t k0, uint32_t k1) {
  bool neg = false, outside = false;   // the normal draws' keys (as sampler_kernel's phase 1)
  for (int q = 0; q < a.n_sampled; q += 2) {
    const bool n0 = a.kind[q] == 0, n1 = q + 1 < a.n_sampled && a.kind[q + 1] == 0;
    if (!(n0 || n1)) continue;
    const U4 r = philox4x32_10(actr, pid, kRoleSamplerParams, (uint32_t)(q >> 1), k0, k1);
    if (n0) key_verdict(a, rules[q], q, key52(r.x, r.y), neg, outside);
    if (n1) key_verdict(a, rules[q + 1], q + 1, key52(r.z, r.w), neg, outside);
  }
  return neg ? 1 : (outside ? 2 : 3);
}

__global__ void __launch_bounds__(kStragBS) straggler_kernel(gt_sampler_args a, const KeyRule* rules,
                                                        const Straggler* park,
                                                        const unsigned int* n_park, int park_cap,
                                                        unsigned int* next) {
  __shared__ int s_amin, s_last, s_j, s_nsurv;
  __shared__ int s_wsum[kStragBS / 32];
  __shared__ int s_list[kStragBS * kStragC];            // survivors' attempt numbers, in order
  __shared__ unsigned char s_code[kStragBS * kStragC];  // their outcome: 3 no steady state, 4 basal, 5 accepted
  __shared__ KeyRule s_rules[kMaxSampled];
  for (int q = threadIdx.x; q < a.n_sampled; q += blockDim.x) s_rules[q] = rules[q];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
  const int n_list = min((int)*n_park, park_cap);
  long long rej[4] = {0, 0, 0, 0};
  double p[GT_N_PARAMS], x[GT_N_STATES], vals[16];
  for (;;) {
    if (t == 0) s_j = (int)atomicAdd(next, 1u);
    __syncthreads();
    const int j = s_j;
    __syncthreads();
    if (j >= n_list) break;
    const Straggler st = park[j];
    const int64_t i = st.i;
    const uint32_t pid = (uint32_t)(a.pid0 + i);
    int32_t total = st.total, a0 = st.attempt, wdraw = st.wdraw, last_surv = st.last_surv;
    uint32_t wctr = st.wctr;
    double w = st.w;
    for (int k = 0; k < GT_N_PARAMS; ++k) p[k] = a.fixed_params[k];
    p[PW] = w;
    int status = 1;
    for (;;) {
      if (a0 >= a.max_attempts || !(w > 0.0)) {   // this body weight's budget is spent
        total += a0 < a.max_attempts ? a0 : a.max_attempts;
        if (wdraw >= a.max_weight_redraws) break;
        ++wdraw;
        w = draw_weight_dev(a, pid, &wctr, k0, k1);   // population.py:148-153 (every thread, same draws)
        p[PW] = w;
        a0 = 0;
        continue;
      }
      // ---- 1. cheap rules on kStragC consecutive attempts per thread
      const int32_t base = a0 + t * kStragC;
      unsigned codes = 0;   // 2 bits per attempt: 0 past the budget, else cheap_code
      int n_s = 0;
      for (int c = 0; c < kStragC; ++c) {
        const int32_t att = base + c;
        if (att >= a.max_attempts) break;
        const int code = cheap_code(a, s_rules, (uint32_t)(total + att), pid, k0, k1);
        codes |= (unsigned)code << (2 * c);
        n_s += code == 3;
      }
      // ---- 2. survivors compacted in attempt order (block exclusive scan)
      int incl = n_s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane == 31) s_wsum[wid] = incl;
      if (t == 0) { s_amin = INT_MAX; s_last = -1; }
      __syncthreads();
      if (t == 0) {
        int run = 0;
        for (int w2 = 0; w2 < kStragBS / 32; ++w2) { const int v = s_wsum[w2]; s_wsum[w2] = run; run += v; }
        s_nsurv = run;
      }
      __syncthreads();
      int pos = s_wsum[wid] + incl - n_s;
      for (int c = 0; c < kStragC; ++c)
        if (((codes >> (2 * c)) & 3u) == 3u) s_list[pos++] = base + c;
      __syncthreads();
      const int n_surv = s_nsurv;
      // ---- 3. the survivors' values and steady-state solves, in parallel
      for (int q = t; q < n_surv; q += kStragBS) {
        const int32_t att = s_list[q];
        double ub = 0.0;
        draw_attempt(a, (uint32_t)(total + att), pid, k0, k1, vals);
        for (int m = 0; m < a.n_sampled; ++m) p[a.param_index[m]] = vals[m];
        const int code = !steady_state_dev(p, a.target_bg, x, &ub) ? 3 : (ub < a.min_basal_uh ? 4 : 5);
        s_code[q] = (unsigned char)code;
        if (code == 5) atomicMin(&s_amin, att);
      }
      __syncthreads();
      const int amin = s_amin;
      // ---- 4. count what the sequential loop reaches (attempts <= amin)
      for (int c = 0; c < kStragC; ++c) {
        const unsigned code = (codes >> (2 * c)) & 3u;
        if ((code == 1u || code == 2u) && base + c < amin) ++rej[code - 1];
      }
      int mine = -1;   // the list entry of the accepted attempt, if this thread holds it
      for (int q = t; q < n_surv; q += kStragBS) {
        const int32_t att = s_list[q];
        if (att > amin) continue;
        const int code = s_code[q];
        if (code == 3 || code == 4) ++rej[code - 1];
        atomicMax(&s_last, (int)(total + att));   // the latest survivor reached (accepted included)
        if (att == amin) mine = q;
      }
      __syncthreads();
      if (s_last >= 0) last_surv = s_last;
      if (amin != INT_MAX) {
        total += amin + 1;
        status = 0;
        if (mine >= 0) {   // the accepted attempt writes the patient (its solve repeated: same values)
          double ub = 0.0;
          draw_attempt(a, (uint32_t)(total - 1), pid, k0, k1, vals);
          for (int m = 0; m < a.n_sampled; ++m) p[a.param_index[m]] = vals[m];
          steady_state_dev(p, a.target_bg, x, &ub);
          for (int k = 0; k < GT_N_PARAMS; ++k) a.params[i * GT_N_PARAMS + k] = p[k];
          for (int k = 0; k < GT_N_STATES; ++k) a.x0[i * GT_N_STATES + k] = x[k];
          a.u_basal_uh[i] = ub;
          a.attempts[i] = total;
          a.status[i] = 0;
        }
        break;
      }
      a0 += kStragBS * kStragC;
      __syncthreads();
    }
    if (status != 0 && t == 0) {   // exhausted: the sequential loop's last p (latest survivor's values)
      for (int k = 0; k < GT_N_PARAMS; ++k) p[k] = a.fixed_params[k];
      p[PW] = w;
      if (last_surv >= 0) {
        draw_attempt(a, (uint32_t)last_surv, pid, k0, k1, vals);
        for (int q = 0; q < a.n_sampled; ++q) p[a.param_index[q]] = vals[q];
      }
      for (int k = 0; k < GT_N_PARAMS; ++k) a.params[i * GT_N_PARAMS + k] = p[k];
      for (int k = 0; k < GT_N_STATES; ++k) a.x0[i * GT_N_STATES + k] = 0.0;
      a.u_basal_uh[i] = 0.0;
      a.attempts[i] = total;
      a.status[i] = 1;
    }
    __syncthreads();
  }
  if (a.reject_counts)
    for (int k = 0; k < 4; ++k)
      if (rej[k]) atomicAdd((unsigned long long*)&a.reject_counts[k], (unsigned long long)rej[k]);
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
  int strag_per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&strag_per_sm, gt::straggler_kernel, gt::kStragBS, 0);
  if (strag_per_sm < 1) strag_per_sm = 1;
  // persistent grid: at most one resident wave, never more lanes than patients
  const int64_t blocks = std::min<int64_t>((int64_t)sms * per_sm, (a->n + bs - 1) / bs);
  // workspace: patient queue, straggler count and cursor, straggler list
  // ~0.5 % of patients (light body weights: low acceptance) pass 384 attempts
  const int cap = (int)std::min<int64_t>(std::max<int64_t>(1024, a->n / 16), 1 << 22);
  const size_t head = 64 + sizeof(gt::KeyRule) * gt::kMaxSampled;
  char* ws = nullptr;
  gt_keep_pool_mapped();
  if (cudaMallocAsync(&ws, head + sizeof(gt::Straggler) * (size_t)cap, st) != cudaSuccess) {
    gt_set_error("gt_sample_population: workspace allocation failed");
    return GT_ECUDA;
  }
  cudaMemsetAsync(ws, 0, 64, st);
  auto* queue = reinterpret_cast<unsigned long long*>(ws);
  auto* n_park = reinterpret_cast<unsigned int*>(ws + 8);
  auto* cursor = reinterpret_cast<unsigned int*>(ws + 16);
  auto* rules = reinterpret_cast<gt::KeyRule*>(ws + 64);
  auto* park = reinterpret_cast<gt::Straggler*>(ws + head);
  gt::key_rules_kernel<<<1, 3 * gt::kMaxSampled, 0, st>>>(*a, rules);
  int e = gt_check_launch("key_rules_kernel");
  if (e == GT_OK) {
    gt::sampler_kernel<<<(unsigned)blocks, bs, 0, st>>>(*a, rules, queue, park, n_park, cap);
    e = gt_check_launch("sampler_kernel");
  }
  if (e == GT_OK) {
    gt::straggler_kernel<<<(unsigned)(sms * strag_per_sm), gt::kStragBS, 0, st>>>(*a, rules, park, n_park, cap, cursor);
    e = gt_check_launch("straggler_kernel");
  }
  cudaFreeAsync(ws, st);
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
