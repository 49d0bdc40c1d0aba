// Population reduction (BASELINE north_star subsystem 4): restates
// TrialAccumulator.add_patient / merge (analytics.py:234-302) over a whole
// shard on device.  Every field is an exact integer (counts, fixed-point 2^24
// sums with numpy rint, min/max), so warp-shuffle + shared-memory +
// global-atomic reduction order cannot change the result — the same
// order-independence the reference's merge relies on (analytics.py:1-13).
#include <cmath>
#include <climits>
#include "gt_common.cuh"

namespace gt {

constexpr int kRedBS = 256;
#ifndef GT_RED_UNROLL
#define GT_RED_UNROLL 8
#endif
constexpr int kRedUnroll = GT_RED_UNROLL;
constexpr int kTirBins = GT_TIR_BINS + 1;
constexpr int kDoseBins = GT_DOSE_BINS + 1;

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// DOUBLE_pairwise_sum) as used by np.sum on a strided float64 column, plus
// the reduction's 0.0 initial value (analytics.py:258; verified against
// numpy 2.3 in tests/test_host.py).  Leaves of <= 128 elements use 8
// interleaved partial sums; larger ranges split at n/2 rounded down to a
// multiple of 8.  Iterative with an explicit stack; `val(d)` yields element d.
template <class F>
__device__ double pw_leaf(const F& val, int64_t lo, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t q = 0; q < n; ++q) res = A_(res, val(lo + q));
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = val(lo + j);
  int64_t q = 8;
  for (; q < n - (n % 8); q += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = A_(r[j], val(lo + q + j));
  }
  double res = A_(A_(A_(r[0], r[1]), A_(r[2], r[3])), A_(A_(r[4], r[5]), A_(r[6], r[7])));
  for (; q < n; ++q) res = A_(res, val(lo + q));
  return res;
}

template <class F>
__device__ double pairwise_sum(const F& val, int64_t n) {
  int64_t off[40], len[40];
  double acc[40];
  unsigned char st[40];
  int sp = 0;
  off[0] = 0; len[0] = n; st[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    if (len[sp] <= 128) {
      ret = pw_leaf(val, off[sp], len[sp]);
      --sp;
      while (sp >= 0) {
        if (st[sp] == 1) {  // left child finished: descend into the right one
          acc[sp] = ret; st[sp] = 2;
          int64_t n2 = len[sp] / 2; n2 -= n2 % 8;
          off[sp + 1] = off[sp] + n2; len[sp + 1] = len[sp] - n2; st[sp + 1] = 0;
          ++sp;
          break;
        }
        ret = A_(acc[sp], ret);  // right child finished
        --sp;
      }
    } else {
      st[sp] = 1;
      int64_t n2 = len[sp] / 2; n2 -= n2 % 8;
      off[sp + 1] = off[sp]; len[sp + 1] = n2; st[sp + 1] = 0;
      ++sp;
    }
  }
  return A_(0.0, ret);
}

__device__ __forceinline__ long long wsum64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long wmin64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { long long w = __shfl_xor_sync(0xffffffffu, v, o); v = w < v ? w : v; }
  return v;
}
__device__ __forceinline__ long long wmax64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { long long w = __shfl_xor_sync(0xffffffffu, v, o); v = w > v ? w : v; }
  return v;
}

// Unsigned 128-bit accumulation as a low word + carry word (the reference's
// fixed-point sums are Python ints): every partial is >= 0, so a wrapped low
// word (old + v < old) carries exactly one into the high word.
__device__ __forceinline__ void add_u128(unsigned long long* lo, unsigned long long* hi, unsigned long long v) {
  const unsigned long long old = atomicAdd(lo, v);
  if (old + v < old) atomicAdd(hi, 1ull);
}

struct Worst { long long kb; long long neg_t3; long long pid; };
__device__ __forceinline__ bool worst_less(const Worst& a, const Worst& b) {
  // analytics.py:150-153: (min_bg, -ticks_below_3, patient_id)
  if (a.kb != b.kb) return a.kb < b.kb;
  if (a.neg_t3 != b.neg_t3) return a.neg_t3 < b.neg_t3;
  return a.pid < b.pid;
}

__global__ void reduce_init_kernel(gt_reduce_args a, Worst* wblk, int nblk) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < 6) a.counts[t] = 0;
  if (t < GT_N_RANGES) a.tir_ticks_total[t] = 0;
  if (t < GT_N_RANGES * kTirBins) a.tir_hist[t] = 0;
  if (t < GT_N_BG_BINS) a.bg_hist_total[t] = 0;
  if (t < GT_N_THRESHOLDS) { a.below_min[t] = LLONG_MAX; a.below_max[t] = 0; }
  if (t == 0) { a.minmax_bg_bits[0] = LLONG_MAX; a.minmax_bg_bits[1] = LLONG_MIN; }
  if (t < 3 * kDoseBins) a.dose_hist[t] = 0;
  if (t < 6) a.dose_sum_fp[t] = 0;  // low words [0..2], carry words [3..5]
  if (a.metric_hist && t < 7 * kTirBins) a.metric_hist[t] = 0;
  if (t < nblk) wblk[t] = Worst{LLONG_MAX, LLONG_MAX, LLONG_MAX};
}

// One count per valid lane into h[bin]: lanes with the same bin are merged
// (match.any) and their leader adds the group size, so the 32 lanes of a warp
// -- whose patients mostly share a bin (similar daily doses) -- cost one
// shared-memory atomic per distinct bin instead of 32 serialised ones.
// Called by all 32 lanes.
__device__ __forceinline__ void warp_hist_add(unsigned* h, int bin, bool valid) {
  const unsigned vm = __ballot_sync(0xffffffffu, valid);
  const unsigned grp = __match_any_sync(0xffffffffu, valid ? bin : -1) & vm;
  const int lane = threadIdx.x & 31;
  if (valid && (grp & ((1u << lane) - 1u)) == 0u) atomicAdd(&h[bin], (unsigned)__popc(grp));
}

__global__ void __launch_bounds__(kRedBS) reduce_patients_kernel(gt_reduce_args a, Worst* wblk) {
  __shared__ unsigned long long s_bg[GT_N_BG_BINS];
  __shared__ int s_bmin[GT_N_THRESHOLDS], s_bmax[GT_N_THRESHOLDS];
  // per-block patient histograms: 32-bit counts (a block folds at most
  // kRedBS patients per pass), filled by warp-aggregated adds (warp_hist_add)
  __shared__ unsigned s_tirh[GT_N_RANGES * kTirBins];
  __shared__ unsigned s_doseh[3 * kDoseBins];
  __shared__ unsigned s_mh[2 * kTirBins];  // hypo-event histograms
  __shared__ unsigned s_mr[3 * kTirBins];  // tbr70, tar180 combined-range hists
  __shared__ unsigned long long s_tir[GT_N_RANGES];
  __shared__ long long s_misc[8];  // n_ok, n_abort, sum_fp, d0, d1, d2, minb, maxb
  __shared__ unsigned long long s_carry[4];  // carry words of sum_fp, d0, d1, d2
  __shared__ Worst s_w[kRedBS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int k = tid; k < GT_N_BG_BINS; k += kRedBS) s_bg[k] = 0;
  for (int k = tid; k < GT_N_THRESHOLDS; k += kRedBS) { s_bmin[k] = INT_MAX; s_bmax[k] = 0; }
  for (int k = tid; k < GT_N_RANGES * kTirBins; k += kRedBS) s_tirh[k] = 0;
  for (int k = tid; k < 3 * kDoseBins; k += kRedBS) s_doseh[k] = 0;
  for (int k = tid; k < 2 * kTirBins; k += kRedBS) s_mh[k] = 0;
  for (int k = tid; k < 3 * kTirBins; k += kRedBS) s_mr[k] = 0;
  if (tid < GT_N_RANGES) s_tir[tid] = 0;
  if (tid < 8) s_misc[tid] = (tid == 6) ? LLONG_MAX : (tid == 7 ? LLONG_MIN : 0);
  if (tid < 4) s_carry[tid] = 0;
  __syncthreads();

  const int64_t n = a.n;
  const int64_t H = a.horizon_ticks;
  Worst wbest{LLONG_MAX, LLONG_MAX, LLONG_MAX};
  long long n_ok = 0, n_ab = 0;
  for (int64_t base = (int64_t)blockIdx.x * kRedBS; base < n; base += (int64_t)gridDim.x * kRedBS) {
    const int64_t i = base + tid;
    const bool inr = i < n;
    const int stv = inr ? a.status[i] : GT_STATUS_EXCLUDED;
    const bool ok = inr && stv == GT_STATUS_OK;
    n_ok += ok;
    n_ab += inr && (stv == GT_STATUS_NONFINITE || stv == GT_STATUS_NO_STEADY_STATE ||
                    stv == GT_STATUS_BAD_INITIAL_STATE);
    // ---- histogram, below-threshold envelope, TIR ticks
    int cum = 0, c25 = 0, c34 = 0, c95 = 0, c134 = 0;
    const int* hcol = a.bg_hist + (ok ? i : 0);
#pragma unroll (kRedUnroll)
    for (int b = 0; b < GT_N_BG_BINS; ++b) {
      const int v = ok ? __ldg(hcol + (int64_t)b * n) : 0;
      cum += v;  // below[b] = cumsum(hist)[b] (analytics.py:129-131)
      if (b == 25) c25 = cum;
      if (b == 34) c34 = cum;
      if (b == 95) c95 = cum;
      if (b == 134) c134 = cum;
      const unsigned sv = __reduce_add_sync(0xffffffffu, (unsigned)v);
      if (b < GT_N_THRESHOLDS) {
        const int mn = __reduce_min_sync(0xffffffffu, ok ? cum : INT_MAX);
        const int mx = __reduce_max_sync(0xffffffffu, ok ? cum : 0);
        if (lane == 0) {
          atomicMin(&s_bmin[b], mn);
          atomicMax(&s_bmax[b], mx);
        }
      }
      if (lane == 0 && sv) atomicAdd(&s_bg[b], (unsigned long long)sv);
    }
    const int tir[5] = {c25, c34 - c25, c95 - c34, c134 - c95, cum - c134};
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      // analytics.py:240: min(TIR_BINS, ticks*200 // horizon)
      long long fb = ((long long)tir[r] * GT_TIR_BINS) / H;
      if (fb > GT_TIR_BINS) fb = GT_TIR_BINS;
      warp_hist_add(s_tirh, r * kTirBins + (int)fb, ok);
    }
    // BASELINE metrics: TBR<70 = r0+r1, TAR>180 = r3+r4 (TIR, TBR<54, TAR>250 are r2, r0, r4)
    const int comb[2] = {tir[0] + tir[1], tir[3] + tir[4]};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      long long fb = ((long long)comb[q] * GT_TIR_BINS) / H;
      if (fb > GT_TIR_BINS) fb = GT_TIR_BINS;
      warp_hist_add(s_mr, q * kTirBins + (int)fb, ok);
    }
    {
      const int e39 = ok ? a.hypo_events[i] : 0, e30 = ok ? a.hypo_events[n + i] : 0;
      warp_hist_add(s_mh, min(e39, GT_TIR_BINS), ok);
      warp_hist_add(s_mh, kTirBins + min(e30, GT_TIR_BINS), ok);
    }
    if (ok) {
      if (a.metric_tir) {
        const float fH = (float)H;
        a.metric_tir[i] = tir[2] / fH;
        a.metric_tbr70[i] = comb[0] / fH;
        a.metric_tbr54[i] = tir[0] / fH;
        a.metric_tar180[i] = comb[1] / fH;
        a.metric_tar250[i] = tir[4] / fH;
      }
    }
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const unsigned sv = __reduce_add_sync(0xffffffffu, ok ? (unsigned)tir[r] : 0u);
      if (lane == 0) atomicAdd(&s_tir[r], (unsigned long long)sv);
    }
    // ---- BG sum (fixed point), extremes
    const double mnb = ok ? a.bg_stats[i] : 0.0;
    const double mxb = ok ? a.bg_stats[n + i] : 0.0;
    const double smb = ok ? a.bg_stats[2 * n + i] : 0.0;
    const long long sfp = ok ? __double2ll_rn(smb * kFpScale) : 0;  // analytics.py:56-57
    const long long ws = wsum64(sfp);
    const long long wmn = wmin64(ok ? ordered_bits(mnb) : LLONG_MAX);
    const long long wmx = wmax64(ok ? ordered_bits(mxb) : LLONG_MIN);
    if (lane == 0) {
      add_u128((unsigned long long*)&s_misc[2], &s_carry[0], (unsigned long long)ws);
      atomicMin(&s_misc[6], wmn);
      atomicMax(&s_misc[7], wmx);
    }
    // ---- daily doses (analytics.py:123-127, 253-258)
    for (int k = 0; k < 3; ++k) {
      const double* col = a.day_dose + (int64_t)k * n + (ok ? i : 0);
      const int64_t stride = 3 * n;
      const double width = k == 2 ? 10.0 : 0.5;  // DOSE_BIN_WIDTH, analytics.py:36
      const double dt = a.dt_s;
      // day_totals[:, 0] = day_dose[:, 0] * dt_s / 3600.0 (analytics.py:126)
      // One pass over the days: numpy's pairwise sum visits every element once,
      // in index order, so each day's value is binned as the sum reads it.
      // Every lane walks the days (the bins are warp-aggregated, and the sum's
      // control flow depends on n_days only); a lane without a patient reads
      // patient 0's column and counts nothing.
      auto val = [&](int64_t d) {
        const double v0 = col[d * stride];
        const double v = k == 0 ? D_(M_(v0, dt), 3600.0) : v0;
        // Python's floordiv; for the 0.5 U widths (a power of two) and v >= 0
        // it is exactly floor(2 v): fmod(v, 0.5) is exact and so is v - fmod
        long long bin = !ok ? 0
                        : (k < 2 && v >= 0.0) ? (long long)floor(M_(v, 2.0))
                        : (v == 0.0 ? 0 : (long long)py_floordiv(v, width));
        if (bin > GT_DOSE_BINS) bin = GT_DOSE_BINS;
        warp_hist_add(s_doseh, k * kDoseBins + (int)bin, ok);
        return v;
      };
      const double psum = pairwise_sum(val, a.n_days);
      const long long fp = ok ? __double2ll_rn(psum * kFpScale) : 0;   // (0 for a lane without a patient)
      const long long wsf = wsum64(fp);
      if (lane == 0) add_u128((unsigned long long*)&s_misc[3 + k], &s_carry[1 + k], (unsigned long long)wsf);
    }
    // ---- worst case candidate (analytics.py:150-153, 260-265)
    if (ok) {
      const Worst c{ordered_bits(mnb), -(long long)c25, (long long)(a.pid0 + i)};
      if (worst_less(c, wbest)) wbest = c;
    }
  }
  // warp-level worst
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Worst w{__shfl_xor_sync(0xffffffffu, wbest.kb, o), __shfl_xor_sync(0xffffffffu, wbest.neg_t3, o),
            __shfl_xor_sync(0xffffffffu, wbest.pid, o)};
    if (worst_less(w, wbest)) wbest = w;
  }
  if (lane == 0) s_w[warp] = wbest;
  const long long tok = wsum64(n_ok), tab = wsum64(n_ab);
  if (lane == 0) {
    atomicAdd((unsigned long long*)&s_misc[0], (unsigned long long)tok);
    atomicAdd((unsigned long long*)&s_misc[1], (unsigned long long)tab);
  }
  __syncthreads();
  if (tid == 0) {
    Worst b = s_w[0];
    for (int w = 1; w < kRedBS / 32; ++w) if (worst_less(s_w[w], b)) b = s_w[w];
    wblk[blockIdx.x] = b;
  }
  // ---- flush block accumulators
  for (int k = tid; k < GT_N_BG_BINS; k += kRedBS)
    if (s_bg[k]) atomicAdd((unsigned long long*)&a.bg_hist_total[k], s_bg[k]);
  for (int k = tid; k < GT_N_THRESHOLDS; k += kRedBS) {
    if (s_bmin[k] != INT_MAX) atomicMin((long long*)&a.below_min[k], (long long)s_bmin[k]);
    atomicMax((long long*)&a.below_max[k], (long long)s_bmax[k]);
  }
  for (int k = tid; k < GT_N_RANGES * kTirBins; k += kRedBS)
    if (s_tirh[k]) atomicAdd((unsigned long long*)&a.tir_hist[k], (unsigned long long)s_tirh[k]);
  for (int k = tid; k < 3 * kDoseBins; k += kRedBS)
    if (s_doseh[k]) atomicAdd((unsigned long long*)&a.dose_hist[k], (unsigned long long)s_doseh[k]);
  if (a.metric_hist) {
    // rows: 0 tir(normo) 1 tbr70 2 tbr54 3 tar180 4 tar250 5 events<3.9 6 events<3.0
    for (int k = tid; k < kTirBins; k += kRedBS) {
      if (s_tirh[2 * kTirBins + k]) atomicAdd((unsigned long long*)&a.metric_hist[0 * kTirBins + k], (unsigned long long)s_tirh[2 * kTirBins + k]);
      if (s_mr[k]) atomicAdd((unsigned long long*)&a.metric_hist[1 * kTirBins + k], (unsigned long long)s_mr[k]);
      if (s_tirh[k]) atomicAdd((unsigned long long*)&a.metric_hist[2 * kTirBins + k], (unsigned long long)s_tirh[k]);
      if (s_mr[kTirBins + k]) atomicAdd((unsigned long long*)&a.metric_hist[3 * kTirBins + k], (unsigned long long)s_mr[kTirBins + k]);
      if (s_tirh[4 * kTirBins + k]) atomicAdd((unsigned long long*)&a.metric_hist[4 * kTirBins + k], (unsigned long long)s_tirh[4 * kTirBins + k]);
      if (s_mh[k]) atomicAdd((unsigned long long*)&a.metric_hist[5 * kTirBins + k], (unsigned long long)s_mh[k]);
      if (s_mh[kTirBins + k]) atomicAdd((unsigned long long*)&a.metric_hist[6 * kTirBins + k], (unsigned long long)s_mh[kTirBins + k]);
    }
  }
  if (tid < GT_N_RANGES) atomicAdd((unsigned long long*)&a.tir_ticks_total[tid], s_tir[tid]);
  if (tid == 0) {
    atomicAdd((unsigned long long*)&a.counts[0], (unsigned long long)s_misc[0]);
    atomicAdd((unsigned long long*)&a.counts[1], (unsigned long long)s_misc[1]);
    // sum_bg_fp and the dose sums can exceed int64 (1M x 52-week trials; the
    // reference uses Python ints): 128-bit accumulation, low word + carry
    // word, per warp into the block partial and per block into the output
    add_u128((unsigned long long*)&a.counts[2], (unsigned long long*)&a.counts[4], (unsigned long long)s_misc[2]);
    if (s_carry[0]) atomicAdd((unsigned long long*)&a.counts[4], s_carry[0]);
    atomicAdd((unsigned long long*)&a.counts[3], (unsigned long long)(s_misc[0] * a.n_days));
    for (int k = 0; k < 3; ++k) {
      add_u128((unsigned long long*)&a.dose_sum_fp[k], (unsigned long long*)&a.dose_sum_fp[3 + k],
               (unsigned long long)s_misc[3 + k]);
      if (s_carry[1 + k]) atomicAdd((unsigned long long*)&a.dose_sum_fp[3 + k], s_carry[1 + k]);
    }
    atomicMin((long long*)&a.minmax_bg_bits[0], s_misc[6]);
    atomicMax((long long*)&a.minmax_bg_bits[1], s_misc[7]);
  }
}

__global__ void reduce_worst_kernel(const Worst* wblk, int nblk, long long* out) {
  __shared__ Worst s[kRedBS];
  Worst b{LLONG_MAX, LLONG_MAX, LLONG_MAX};
  for (int k = threadIdx.x; k < nblk; k += kRedBS) if (worst_less(wblk[k], b)) b = wblk[k];
  s[threadIdx.x] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < kRedBS; ++k) if (worst_less(s[k], b)) b = s[k];
    out[0] = b.kb; out[1] = -b.neg_t3; out[2] = b.pid; out[3] = b.pid != LLONG_MAX;
  }
}

// timeline: [n_grid][n_warps][3] per-warp partials -> [3][n_grid]
__global__ void reduce_timeline_kernel(const long long* tw, int64_t n_grid, int64_t n_warps, long long* out) {
  __shared__ long long s_s[kRedBS / 32], s_mn[kRedBS / 32], s_mx[kRedBS / 32];
  for (int64_t g = blockIdx.x; g < n_grid; g += gridDim.x) {
    long long su = 0, mn = LLONG_MAX, mx = LLONG_MIN;
    for (int64_t w = threadIdx.x; w < n_warps; w += kRedBS) {
      const long long* p = tw + (g * n_warps + w) * 3;
      su += p[0]; mn = p[1] < mn ? p[1] : mn; mx = p[2] > mx ? p[2] : mx;
    }
    su = wsum64(su); mn = wmin64(mn); mx = wmax64(mx);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { s_s[warp] = su; s_mn[warp] = mn; s_mx[warp] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
      su = s_s[0]; mn = s_mn[0]; mx = s_mx[0];
      for (int w = 1; w < kRedBS / 32; ++w) {
        su += s_s[w]; mn = s_mn[w] < mn ? s_mn[w] : mn; mx = s_mx[w] > mx ? s_mx[w] : mx;
      }
      out[g] = su; out[n_grid + g] = mn; out[2 * n_grid + g] = mx;
    }
    __syncthreads();
  }
}

}  // namespace gt

int gt_launch_reduce(const gt_reduce_args* a, void* scratch_worst, int nblk, cudaStream_t st) {
  gt::Worst* wblk = reinterpret_cast<gt::Worst*>(scratch_worst);
  gt::reduce_init_kernel<<<8, 256, 0, st>>>(*a, wblk, nblk);
  if (int e = gt_check_launch("reduce_init_kernel")) return e;
  if (a->n > 0) {
    gt::reduce_patients_kernel<<<nblk, gt::kRedBS, 0, st>>>(*a, wblk);
    if (int e = gt_check_launch("reduce_patients_kernel")) return e;
  }
  gt::reduce_worst_kernel<<<1, gt::kRedBS, 0, st>>>(wblk, nblk, (long long*)a->worst);
  if (int e = gt_check_launch("reduce_worst_kernel")) return e;
  if (a->n_grid > 0) {
    const int g = (int)(a->n_grid < 4096 ? a->n_grid : 4096);
    gt::reduce_timeline_kernel<<<g, gt::kRedBS, 0, st>>>((const long long*)a->timeline_warp, a->n_grid, a->n_warps, (long long*)a->timeline);
    if (int e = gt_check_launch("reduce_timeline_kernel")) return e;
  }
  return GT_OK;
}
