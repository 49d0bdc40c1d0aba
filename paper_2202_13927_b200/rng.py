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


def det_exp(x: np.ndarray) -> np.ndarray:
    """exp from +,-,*,/ only (device: gt_common.cuh det_exp)."""
    x = np.asarray(x, dtype=np.float64)
    kf = np.floor(x * 1.44269504088896338700e+00 + 0.5)
    r = (x - kf * _LN2_HI) - kf * _LN2_LO
    s = np.ones_like(r)
    for j in range(14, 0, -1):
        s = 1.0 + (r * s) / float(j)
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
