"""Random streams.

Two families:

* the reference's keyed streams (rng.py:18-48 of the reference): numpy
  ``Generator(Philox(SeedSequence(entropy=seed, spawn_key=key)))`` — used to
  draw the reference's own process / measurement noise on the host when a
  trial must reproduce the reference bit for bit ("injected" noise);
* the device family: Philox4x32-10 keyed by the trial seed with counter
  ``(index_lo, patient_id, role, index_hi)`` (include/glucosim.h).  The numpy
  twins below evaluate the same bijection and the same IEEE-only transforms
  (deterministic log / exp, Acklam's inverse normal CDF) so host and device
  agree bit for bit where the device uses them (meal generator, sampler).
"""

from __future__ import annotations

import numpy as np

# reference roles (rng.py:18-23) — part of the reproducibility contract
ROLE_DEMOGRAPHICS = 1
ROLE_PARAMETERS = 2
ROLE_PROTOCOL = 3
ROLE_ANNOUNCEMENT = 4
ROLE_PROCESS_NOISE = 5
ROLE_MEASUREMENT_NOISE = 6
# device roles (new streams; never collide with the reference's)
ROLE_DEVICE_NOISE = 0x10
ROLE_MEALS = 0x11
ROLE_SAMPLER_PARAMS = 0x12
ROLE_SAMPLER_WEIGHT = 0x13


def stream(seed: int, *key: int) -> np.random.Generator:
    """The reference's keyed generator (rng.py:26-39)."""
    if seed < 0:
        raise ValueError("seed must be nonnegative")
    for k in key:
        if not 0 <= k < 2**32:
            raise ValueError(f"stream key component out of range: {k}")
    ss = np.random.SeedSequence(entropy=seed, spawn_key=tuple(key))
    return np.random.Generator(np.random.Philox(ss))


def derive_seed(seed: int, *key: int) -> int:
    """64-bit child seed (rng.py:42-48)."""
    ss = np.random.SeedSequence(entropy=seed, spawn_key=tuple(key))
    lo, hi = ss.generate_state(2)
    return int(lo) | (int(hi) << 32)


def reference_noise(seed: int, pid: int, horizon_ticks: int, period_steps: int,
                    process_on: bool, sensor_on: bool):
    """The reference's noise for one patient-run, drawn once for the whole
    horizon (equal to its per-block draws, simulation.py:333-357):
    ``(wiener [H,3] or None, meas [H/period_steps])``."""
    wiener = (stream(seed, pid, ROLE_PROCESS_NOISE).standard_normal((horizon_ticks, 3))
              if process_on else None)
    n_ctl = horizon_ticks // period_steps
    meas = (stream(seed, pid, ROLE_MEASUREMENT_NOISE).standard_normal(n_ctl)
            if sensor_on else np.zeros(n_ctl))
    return wiener, meas


# --------------------------------------------------------------- Philox twin
_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = 0x9E3779B9, 0xBB67AE85
_MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr: np.ndarray, seed: int) -> np.ndarray:
    """Philox4x32-10 over rows of ``ctr`` (uint32 [N,4]) with key = seed."""
    c = np.asarray(ctr, dtype=np.uint64).reshape(-1, 4)
    c0, c1, c2, c3 = (c[:, j].copy() for j in range(4))
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    for r in range(10):
        if r > 0:
            k0 = (k0 + _W0) & 0xFFFFFFFF
            k1 = (k1 + _W1) & 0xFFFFFFFF
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0
    return np.stack([c0, c1, c2, c3], axis=1).astype(np.uint32)


def philox_counters(index, pid, role) -> np.ndarray:
    index = np.asarray(index, dtype=np.uint64)
    out = np.empty(index.shape + (4,), dtype=np.uint32)
    out[..., 0] = (index & _MASK).astype(np.uint32)
    out[..., 1] = np.uint32(pid) if np.isscalar(pid) else np.asarray(pid, dtype=np.uint32)
    out[..., 2] = np.uint32(role)
    out[..., 3] = (index >> np.uint64(32)).astype(np.uint32)
    return out


# ------------------------------------------------ IEEE-only transforms (twins)
_LN2_HI = 6.93147180369123816490e-01
_LN2_LO = 1.90821492927058770002e-10


def det_log(x: np.ndarray) -> np.ndarray:
    """Natural log from +,-,*,/ only (device: gt_common.cuh det_log)."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)
    small = m < 0.70710678118654752440
    m = np.where(small, m * 2.0, m)
    e = np.where(small, e - 1, e)
    f = m - 1.0
    s = f / (2.0 + f)
    z = s * s
    poly = np.full_like(s, 1.0 / 25.0)
    for d in (23.0, 21.0, 19.0, 17.0, 15.0, 13.0, 11.0, 9.0, 7.0, 5.0, 3.0):
        poly = 1.0 / d + z * poly
    logm = 2.0 * s + (2.0 * s) * (z * poly)
    de = e.astype(np.float64)
    return de * _LN2_HI + (de * _LN2_LO + logm)


# doubles nearest 1/j!, j = 0..14 (Horner coefficients of det_exp)
_INV_FACT = (1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664, 0.008333333333333333,
             0.001388888888888889, 0.0001984126984126984, 2.48015873015873e-05, 2.7557319223985893e-06,
             2.755731922398589e-07, 2.505210838544172e-08, 2.08767569878681e-09, 1.6059043836821613e-10,
             1.1470745597729725e-11)


def det_exp(x: np.ndarray) -> np.ndarray:
    """exp from +,-,*,/ only (device: gt_common.cuh det_exp)."""
    x = np.asarray(x, dtype=np.float64)
    kf = np.floor(x * 1.44269504088896338700e+00 + 0.5)
    r = (x - kf * _LN2_HI) - kf * _LN2_LO
    s = np.full_like(r, _INV_FACT[14])
    for j in range(13, -1, -1):
        s = _INV_FACT[j] + r * s
    out = np.ldexp(s, kf.astype(np.int64))
    out = np.where(x > 709.0, np.inf, out)
    return np.where(x < -745.0, 0.0, out)


_A = (-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
      1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00)
_B = (-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
      6.680131188771972e+01, -1.328068155288572e+01)
_C = (-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
      -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00)
_D = (7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
      3.754408661907416e+00)


def det_inv_norm(p: np.ndarray) -> np.ndarray:
    """Acklam's inverse standard-normal CDF (relative error < 1.15e-9),
    IEEE operations in a fixed order (device: det_inv_norm)."""
    p = np.asarray(p, dtype=np.float64)
    out = np.empty_like(p)
    plow, phigh = 0.02425, 1.0 - 0.02425
    tail = (p < plow) | (p > phigh)
    mid = ~tail
    q = p[mid] - 0.5
    r = q * q
    num = (((((_A[0] * r + _A[1]) * r + _A[2]) * r + _A[3]) * r + _A[4]) * r + _A[5]) * q
    den = (((((_B[0] * r + _B[1]) * r + _B[2]) * r + _B[3]) * r + _B[4]) * r + 1.0)
    out[mid] = num / den
    if tail.any():
        pt = p[tail]
        upper = pt > phigh
        arg = np.where(upper, 1.0 - pt, pt)
        qt = np.sqrt(-2.0 * det_log(arg))
        num = (((((_C[0] * qt + _C[1]) * qt + _C[2]) * qt + _C[3]) * qt + _C[4]) * qt + _C[5])
        den = ((((_D[0] * qt + _D[1]) * qt + _D[2]) * qt + _D[3]) * qt + 1.0)
        v = num / den
        out[tail] = np.where(upper, -v, v)
    return out


def u52(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Open-interval uniform from two uint32 words (device: u52 / gen_meal)."""
    k = ((a.astype(np.uint64) >> np.uint64(6)) << np.uint64(26)) | (b.astype(np.uint64) >> np.uint64(6))
    return (2 * k + 1).astype(np.float64) * 1.1102230246251565404e-16


# ------------------------------------------------- numpy stream restatement
# The device NorthernYear planner (csrc/gt_northern.cu) draws from the
# reference's own keyed streams, so it restates numpy's SeedSequence,
# Philox4x64-10 bit generator and Generator.shuffle bit for bit.  These
# pure-integer twins are that restatement on the host (checked against numpy
# in tests/test_northern.py).
_M32 = 0xFFFFFFFF
_M64 = 0xFFFFFFFFFFFFFFFF


def _u32_words(v: int) -> list:
    """numpy _int_to_uint32_array: little-endian 32-bit words, [0] for 0."""
    if v < 0:
        raise ValueError("negative entropy")
    if v == 0:
        return [0]
    out = []
    while v > 0:
        out.append(v & _M32)
        v >>= 32
    return out


def seed_sequence_state(entropy: int, spawn_key: tuple, n_words32: int) -> list:
    """SeedSequence(entropy, spawn_key).generate_state(n_words32, uint32),
    pool size 4 (numpy/random/bit_generator.pyx)."""
    run = _u32_words(entropy)
    spawn = [w for k in spawn_key for w in _u32_words(int(k))]
    if spawn and len(run) < 4:
        run = run + [0] * (4 - len(run))
    ent = run + spawn
    hc = 0x43B0D7E5

    def hashmix(v):
        nonlocal hc
        v = (v ^ hc) & _M32
        hc = (hc * 0x931E8875) & _M32
        v = (v * hc) & _M32
        return v ^ (v >> 16)

    def mix(x, y):
        r = (0xCA01F9DD * x - 0x4973F715 * y) & _M32
        return r ^ (r >> 16)

    pool = [hashmix(ent[i]) if i < len(ent) else hashmix(0) for i in range(4)]
    for s in range(4):
        for d in range(4):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(4, len(ent)):
        for d in range(4):
            pool[d] = mix(pool[d], hashmix(ent[s]))
    hb = 0x8B51F9DD
    out = []
    for i in range(n_words32):
        v = pool[i % 4] ^ hb
        hb = (hb * 0x58F38DED) & _M32
        v = (v * hb) & _M32
        out.append(v ^ (v >> 16))
    return out


def derive_seed_twin(seed: int, *key: int) -> int:
    w = seed_sequence_state(seed, key, 2)
    return w[0] | (w[1] << 32)


def philox4x64_10(ctr: list, key: list) -> list:
    c, k0, k1 = list(ctr), key[0], key[1]
    for _ in range(10):
        p0 = 0xD2E7470EE14C6C93 * c[0]
        p1 = 0xCA5A826395121157 * c[2]
        c = [((p1 >> 64) ^ c[1] ^ k0) & _M64, p1 & _M64, ((p0 >> 64) ^ c[3] ^ k1) & _M64, p0 & _M64]
        k0 = (k0 + 0x9E3779B97F4A7C15) & _M64
        k1 = (k1 + 0xBB67AE8584CAA73B) & _M64
    return c


class NumpyPhiloxTwin:
    """numpy.random.Philox(SeedSequence(entropy, spawn_key)) as used by
    ``stream``: next_uint64 / next_uint32 (low half first) / random_interval."""

    def __init__(self, entropy: int, spawn_key: tuple):
        w = seed_sequence_state(entropy, spawn_key, 4)
        self.key = [w[0] | (w[1] << 32), w[2] | (w[3] << 32)]
        self.ctr = [0, 0, 0, 0]
        self.buf, self.pos = [0] * 4, 4
        self.has32, self.u32 = False, 0

    def next_uint64(self) -> int:
        if self.pos < 4:
            self.pos += 1
            return self.buf[self.pos - 1]
        for i in range(4):   # 256-bit counter increment with carry
            self.ctr[i] = (self.ctr[i] + 1) & _M64
            if self.ctr[i]:
                break
        self.buf, self.pos = philox4x64_10(self.ctr, self.key), 1
        return self.buf[0]

    def next_uint32(self) -> int:
        if self.has32:
            self.has32 = False
            return self.u32
        v = self.next_uint64()
        self.has32, self.u32 = True, v >> 32
        return v & _M32

    def random_interval(self, mx: int) -> int:
        if mx == 0:
            return 0
        mask = mx
        for s in (1, 2, 4, 8, 16, 32):
            mask |= mask >> s
        if mx <= _M32:
            while True:
                v = self.next_uint32() & mask
                if v <= mx:
                    return v
        while True:
            v = self.next_uint64() & mask
            if v <= mx:
                return v

    def shuffle(self, x: list) -> None:
        for i in range(len(x) - 1, 0, -1):
            j = self.random_interval(i)
            x[i], x[j] = x[j], x[i]
