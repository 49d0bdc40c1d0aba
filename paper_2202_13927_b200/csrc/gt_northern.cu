// On-device NorthernYearProtocol: the reference's
// 52-week lifestyle schedule (simulation.py:420-453 -> protocol.py:191-394),
// built per patient on the GPU and emitted in the fused kernel's tick-compiled
// CSR form (protocol.compile_protocol + compile_ticks) at a fixed per-patient
// stride: every seed yields exactly GT_NY_MEALS meals and GT_NY_EX exercise
// sessions per year (the Table-1 compositions fix the day-type counts).
//
// The plan draws from the reference's own keyed stream, so it restates
// numpy exactly:
//   derive_seed(trial_seed, pid, ROLE_PROTOCOL)      rng.py:42-48
//     = SeedSequence(entropy, spawn_key).generate_state(2)   (pool size 4)
//   stream(derived, 0) = Generator(Philox(SeedSequence(derived, (0,))))
//     Philox4x64-10, key = generate_state(2, uint64), counter pre-incremented
//   Generator.shuffle(list) = for i = n-1..1: swap(i, random_interval(i))
//     random_interval: mask rejection on next_uint32 (low half of a uint64
//     first, then the high half)
// Host twins: rng.seed_sequence_state / NumpyPhiloxTwin, northern.plan_year.
// Events past the horizon are written as inert records (ticks = INT_MAX), the
// fused kernel's "no further event" value, so the CSR needs no compaction.
#include <climits>
#include <cmath>
#include "gt_common.cuh"

namespace gt {
namespace ny {

// ---- numpy SeedSequence (numpy/random/bit_generator.pyx), pool size 4
struct Entropy { uint32_t w[8]; int n; };

__device__ void push_words(Entropy& e, uint64_t v) {
  if (v == 0) { e.w[e.n++] = 0u; return; }
  while (v) { e.w[e.n++] = (uint32_t)v; v >>= 32; }
}

__device__ void seed_sequence(const Entropy& run_in, const Entropy& spawn, uint32_t* out, int n_out) {
  Entropy ent = run_in;
  if (spawn.n > 0) while (ent.n < 4) ent.w[ent.n++] = 0u;
  for (int k = 0; k < spawn.n; ++k) ent.w[ent.n++] = spawn.w[k];
  uint32_t hc = 0x43B0D7E5u;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= 0x931E8875u;
    v *= hc;
    return v ^ (v >> 16);
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = 0xCA01F9DDu * x - 0x4973F715u * y;
    return r ^ (r >> 16);
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < ent.n ? ent.w[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int s = 4; s < ent.n; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent.w[s]));
  uint32_t hb = 0x8B51F9DDu;
  for (int i = 0; i < n_out; ++i) {
    uint32_t v = pool[i & 3] ^ hb;
    hb *= 0x58F38DEDu;
    v *= hb;
    out[i] = v ^ (v >> 16);
  }
}

// ---- numpy Philox (Philox4x64-10) bit generator
struct Stream {
  uint64_t key0, key1, ctr0, ctr1, ctr2, ctr3;
  uint64_t buf[4];
  int pos;
  bool has32;
  uint32_t u32;

  __device__ void refill() {
    if (++ctr0 == 0 && ++ctr1 == 0 && ++ctr2 == 0) ++ctr3;  // 256-bit increment
    uint64_t c0 = ctr0, c1 = ctr1, c2 = ctr2, c3 = ctr3, k0 = key0, k1 = key1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0);
      const uint64_t lo1 = 0xCA5A826395121157ull * c2, hi1 = __umul64hi(0xCA5A826395121157ull, c2);
      const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
      c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
      k0 += 0x9E3779B97F4A7C15ull; k1 += 0xBB67AE8584CAA73Bull;
    }
    buf[0] = c0; buf[1] = c1; buf[2] = c2; buf[3] = c3;
    pos = 0;
  }
  __device__ uint64_t next64() {
    if (pos >= 4) refill();
    return buf[pos++];
  }
  __device__ double next_double() {  // numpy next_double: (next_uint64 >> 11) * 2^-53
    return (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
  }
  __device__ uint32_t next32() {
    if (has32) { has32 = false; return u32; }
    const uint64_t v = next64();
    has32 = true; u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  __device__ uint32_t interval(uint32_t mx) {  // random_interval for mx < 2^32
    if (mx == 0) return 0;
    uint32_t mask = mx;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
    uint32_t v;
    while ((v = next32() & mask) > mx) {}
    return v;
  }
  template <int N>
  __device__ void shuffle(uint8_t (&x)[N], int n) {
    for (int i = n - 1; i > 0; --i) {
      const int j = (int)interval((uint32_t)i);
      const uint8_t t = x[i]; x[i] = x[j]; x[j] = t;
    }
  }
};

// Table 1 (protocol.py:33-45): week types standard, active, vacation; day
// types standard, active, movie_night, late_night; seasons winter, spring,
// summer, autumn.
__constant__ int8_t kSeasonWeeks[4][3] = {{6, 4, 3}, {6, 6, 1}, {7, 3, 3}, {9, 3, 1}};
__constant__ int8_t kWeekDays[3][4] = {{4, 1, 1, 1}, {3, 3, 1, 0}, {5, 0, 0, 2}};

// Basis days (data/basis_days.yaml): per (day type, season class) the day's
// events in clock order; class >= 0 = meal class (large, medium, small,
// snack), -1 = exercise.  Season class 0 = winter/autumn, 1 = summer/spring.
struct Ev { int32_t clock_s; int8_t cls; };
__constant__ Ev kBasis[4][2][7] = {
    // standard
    {{{27000, 1}, {43200, 1}, {55800, 3}, {66600, 0}, {0, -2}, {0, -2}, {0, -2}},
     {{27000, 1}, {36000, 3}, {43200, 1}, {66600, 1}, {0, -2}, {0, -2}, {0, -2}}},
    // active: + exercise 17:00
    {{{27000, 1}, {43200, 1}, {55800, 3}, {61200, -1}, {66600, 0}, {0, -2}, {0, -2}},
     {{27000, 1}, {36000, 3}, {43200, 1}, {61200, -1}, {66600, 1}, {0, -2}, {0, -2}}},
    // movie night: + snack 21:30
    {{{27000, 1}, {43200, 1}, {55800, 3}, {66600, 0}, {77400, 3}, {0, -2}, {0, -2}},
     {{27000, 1}, {36000, 3}, {43200, 1}, {66600, 1}, {77400, 3}, {0, -2}, {0, -2}}},
    // late night: + snacks 22:00 and 23:30
    {{{27000, 1}, {43200, 1}, {55800, 3}, {66600, 0}, {79200, 3}, {84600, 3}, {0, -2}},
     {{27000, 1}, {36000, 3}, {43200, 1}, {66600, 1}, {79200, 3}, {84600, 3}, {0, -2}}},
};
__constant__ double kChoPerKg[4] = {1.29, 0.86, 0.57, 0.29};
constexpr double kMealDurS = 900.0;
constexpr double kExDurS = 45.0 * 60.0;
constexpr double kExHrr = 0.5;

__global__ void northern_kernel(const gt_northern_args a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const uint64_t pid = (uint64_t)(a.pid0 + i);
  // derived = derive_seed(trial_seed, pid, ROLE_PROTOCOL)
  Entropy run{}, spawn{};
  push_words(run, a.trial_seed);
  push_words(spawn, pid);
  push_words(spawn, 3u);
  uint32_t w2[2];
  seed_sequence(run, spawn, w2, 2);
  const uint64_t derived = (uint64_t)w2[0] | ((uint64_t)w2[1] << 32);
  // stream(derived, 0)
  Entropy run2{}, spawn2{};
  push_words(run2, derived);
  push_words(spawn2, 0u);
  uint32_t w4[4];
  seed_sequence(run2, spawn2, w4, 4);
  Stream g{};
  g.key0 = (uint64_t)w4[0] | ((uint64_t)w4[1] << 32);
  g.key1 = (uint64_t)w4[2] | ((uint64_t)w4[3] << 32);
  g.pos = 4;

  // announcement policy stream: stream(trial_seed, pid, ROLE_ANNOUNCEMENT = 4)
  // (rng.py:26-39), used only when the policy is not the default
  // (simulation.py:441-444)
  const bool policy = a.fraction_unannounced > 0.0 || a.factor_lo != 1.0 || a.factor_hi != 1.0;
  Stream ga{};
  if (policy) {
    Entropy run3{}, spawn3{};
    push_words(run3, a.trial_seed);
    push_words(spawn3, pid);
    push_words(spawn3, 4u);
    uint32_t k4[4];
    seed_sequence(run3, spawn3, k4, 4);
    ga.key0 = (uint64_t)k4[0] | ((uint64_t)k4[1] << 32);
    ga.key1 = (uint64_t)k4[2] | ((uint64_t)k4[3] << 32);
    ga.pos = 4;
  }
  const double w = a.params[i * NP + PW];
  const double dt = a.dt_s, period = a.period_s, horizon = a.horizon_s;
  int32_t* mks = a.meal_ks + i * GT_NY_MEALS;
  int32_t* mke = a.meal_ke + i * GT_NY_MEALS;
  int32_t* mkp = a.meal_kp + i * GT_NY_MEALS;
  double* mrate = a.meal_rate + i * GT_NY_MEALS;
  double* mann = a.meal_ann + i * GT_NY_MEALS;
  int32_t* eks = a.ex_ks + i * GT_NY_EX;
  int32_t* eke = a.ex_ke + i * GT_NY_EX;
  double* est = a.ex_start_s + i * GT_NY_EX;
  double* ehrr = a.ex_hrr + i * GT_NY_EX;
  double* eann = a.ex_announced + i * GT_NY_EX;
  int nm = 0, ne = 0, nm_h = 0, ne_h = 0;

  int wi = 0;
  for (int season = 0; season < 4; ++season) {
    uint8_t wk[13];
    int nw = 0;
    for (int t = 0; t < 3; ++t)
      for (int c = 0; c < kSeasonWeeks[season][t]; ++c) wk[nw++] = (uint8_t)t;
    g.shuffle(wk, 13);
    const int sc = (season == 0 || season == 3) ? 0 : 1;
    for (int k = 0; k < 13; ++k, ++wi) {
      const int wt = wk[k];
      uint8_t days[7];
      int nd = 0;
      for (int d = 0; d < 4; ++d)
        for (int c = 0; c < kWeekDays[wt][d]; ++c) days[nd++] = (uint8_t)d;
      const bool constrained = kWeekDays[wt][1] > 0 && kWeekDays[wt][3] > 0;
      bool ok = false;
      for (int attempt = 0; attempt < 1000 && !ok; ++attempt) {
        g.shuffle(days, 7);
        ok = true;
        if (constrained)
          for (int d = 0; d + 1 < 7; ++d)
            if ((days[d] == 1 && days[d + 1] == 3) || (days[d] == 3 && days[d + 1] == 1)) ok = false;
      }
      if (!ok) { if (a.n_meals) a.n_meals[i] = -1; return; }  // reference raises ValueError
      if (a.week_days) {
        uint32_t code = 0;
        for (int d = 0; d < 7; ++d) code |= (uint32_t)days[d] << (2 * d);
        a.week_days[(int64_t)wi * a.n + i] = (uint16_t)code;
      }
      for (int d = 0; d < 7; ++d) {
        const double offset = (double)wi * 604800.0 + (double)d * 86400.0;
        for (int e = 0; e < 7; ++e) {
          const Ev ev = kBasis[days[d]][sc][e];
          if (ev.cls == -2) break;
          const double start = offset + (double)ev.clock_s;
          const bool in_h = start < horizon;  // compile_protocol filter (simulation.py:157)
          if (ev.cls >= 0) {
            const double end = start + kMealDurS;
            const double mag = kChoPerKg[ev.cls] * w;
            // apply_announcement_policy (protocol.py:373-394), every meal of the
            // year in compose order: Generator.random() < fraction -> unannounced,
            // else magnitude * (lo if lo == hi else Generator.uniform(lo, hi))
            double ann = mag;
            if (policy) {
              if (ga.next_double() < a.fraction_unannounced) ann = 0.0;
              else ann = mag * (a.factor_lo == a.factor_hi ? a.factor_lo
                                                           : a.factor_lo + (a.factor_hi - a.factor_lo) * ga.next_double());
            }
            mks[nm] = in_h ? (int32_t)ceil(start / dt) : INT_MAX;
            mke[nm] = in_h ? (int32_t)ceil(end / dt) : INT_MAX;
            mkp[nm] = in_h ? (int32_t)floor(start / period) : INT_MAX;
            mrate[nm] = in_h ? mag / ((end - start) / 60.0) : 0.0;
            mann[nm] = in_h ? ann : 0.0;
            ++nm; nm_h += in_h;
          } else {
            const double end = start + kExDurS;
            eks[ne] = in_h ? (int32_t)ceil(start / dt) : INT_MAX;
            eke[ne] = in_h ? (int32_t)ceil(end / dt) : INT_MAX;
            est[ne] = start;
            ehrr[ne] = in_h ? kExHrr : 0.0;
            eann[ne] = 1.0;
            ++ne; ne_h += in_h;
          }
        }
      }
    }
  }
  if (a.n_meals) a.n_meals[i] = nm == GT_NY_MEALS && ne == GT_NY_EX ? nm_h : -2;
  if (a.n_ex) a.n_ex[i] = ne_h;
}

}  // namespace ny
}  // namespace gt

int gt_launch_northern(const gt_northern_args* a, cudaStream_t st) {
  if (a->n <= 0) return GT_OK;
  const int bs = 128;
  const unsigned grid = (unsigned)((a->n + bs - 1) / bs);
  gt::ny::northern_kernel<<<grid, bs, 0, st>>>(*a);
  return gt_check_launch("northern_kernel");
}
