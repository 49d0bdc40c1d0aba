"""Population statistics and the trial report.

The device reduction (csrc/gt_reduce.cu) produces the exact integer fields
of the reference's ``TrialAccumulator`` (analytics.py:179-269); this module
holds them (``TrialAccumulator``), merges shards exactly (``merge``,
analytics.py:272-302), folds per-patient host statistics for the parity
path (``TrialAccumulator.add_patient``, analytics.py:234-265) and renders
the byte-stable report (analytics.py:305-431, storage.py:229-231).
BASELINE's extra outputs — 5/95 % quantiles and per-metric histograms — are
built from the same nearest-rank primitive.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from .layout import (DOSE_BIN_COUNT, DOSE_BIN_WIDTH, DOSE_SIGNALS, FP_SCALE, IDX_3_MMOL,
                     METRIC_NAMES, N_BG_BINS, N_THRESHOLDS, RANGE_BOUNDS, RANGE_NAMES,
                     SCHEMA_REPORT, THRESHOLDS, TIR_BINS)

I64_MAX = np.iinfo(np.int64).max
I64_MIN = np.iinfo(np.int64).min


class GridMismatchError(ValueError):
    pass


def rint_fp(x) -> np.ndarray:
    """Fixed-point image rint(x * 2^24) (analytics.py:56-61)."""
    return np.rint(np.asarray(x, dtype=np.float64) * FP_SCALE).astype(np.int64)


@dataclass
class PatientStats:
    """Per-patient streaming statistics (analytics.py:64-135)."""
    dt_s: float
    horizon_ticks: int
    n_days: int
    n_grid: int
    ticks: int = 0
    tir_ticks: np.ndarray = None
    bg_hist: np.ndarray = None
    min_bg: float = np.inf
    max_bg: float = -np.inf
    sum_bg: float = 0.0
    timeline_bg: np.ndarray = None
    day_dose: np.ndarray = None

    def __post_init__(self):
        if self.tir_ticks is None:
            self.tir_ticks = np.zeros(5, dtype=np.int64)
        if self.bg_hist is None:
            self.bg_hist = np.zeros(N_BG_BINS, dtype=np.int64)
        if self.timeline_bg is None:
            self.timeline_bg = np.zeros(self.n_grid)
        if self.day_dose is None:
            self.day_dose = np.zeros((self.n_days, 3))

    def day_totals(self) -> np.ndarray:
        out = self.day_dose.copy()
        out[:, 0] = out[:, 0] * self.dt_s / 3600.0
        return out

    def below_threshold_ticks(self) -> np.ndarray:
        return np.cumsum(self.bg_hist)[:N_THRESHOLDS]

    @property
    def ticks_below_3(self) -> int:
        return int(self.below_threshold_ticks()[IDX_3_MMOL])


@dataclass
class WorstCase:
    patient_id: int
    min_bg: float
    max_bg: float
    ticks_below_3: int
    ticks: int
    tir_ticks: np.ndarray
    bg_hist: np.ndarray


def _worst_key(w) -> tuple:
    # lower min BG is worse; ties: more time below 3 mmol/L, then lower id
    return (w.min_bg, -w.ticks_below_3, w.patient_id)


@dataclass
class TrialAccumulator:
    """Exact population statistics (field-for-field the reference's)."""
    dt_s: float
    horizon_ticks: int
    n_days: int
    n_grid: int
    grid_step_s: float
    n_patients: int = 0
    n_aborted: int = 0
    aborted_ids: tuple = ()
    tir_ticks_total: np.ndarray = None
    tir_hist: np.ndarray = None
    bg_hist_total: np.ndarray = None
    below_min: np.ndarray = None
    below_max: np.ndarray = None
    sum_bg_fp: int = 0
    min_bg: float = np.inf
    max_bg: float = -np.inf
    timeline_sum_fp: np.ndarray = None
    timeline_min_fp: np.ndarray = None
    timeline_max_fp: np.ndarray = None
    dose_hist: dict = None
    dose_sum_fp: list = None
    n_patient_days: int = 0
    worst: WorstCase | None = None
    # BASELINE extras (not part of the reference report)
    metric_hist: np.ndarray = None   # [7][201]

    def __post_init__(self):
        z = lambda n: np.zeros(n, dtype=np.int64)
        if self.tir_ticks_total is None:
            self.tir_ticks_total = z(5)
        if self.tir_hist is None:
            self.tir_hist = np.zeros((5, TIR_BINS + 1), dtype=np.int64)
        if self.bg_hist_total is None:
            self.bg_hist_total = z(N_BG_BINS)
        if self.below_min is None:
            self.below_min = np.full(N_THRESHOLDS, I64_MAX, dtype=np.int64)
        if self.below_max is None:
            self.below_max = z(N_THRESHOLDS)
        if self.timeline_sum_fp is None:
            self.timeline_sum_fp = z(self.n_grid)
        if self.timeline_min_fp is None:
            self.timeline_min_fp = np.full(self.n_grid, I64_MAX, dtype=np.int64)
        if self.timeline_max_fp is None:
            self.timeline_max_fp = np.full(self.n_grid, I64_MIN, dtype=np.int64)
        if self.dose_hist is None:
            self.dose_hist = {s: z(DOSE_BIN_COUNT[s] + 1) for s in DOSE_SIGNALS}
        if self.dose_sum_fp is None:
            self.dose_sum_fp = [0, 0, 0]
        if self.metric_hist is None:
            self.metric_hist = np.zeros((len(METRIC_NAMES), TIR_BINS + 1), dtype=np.int64)

    def grid_meta(self) -> tuple:
        return (self.dt_s, self.horizon_ticks, self.n_days, self.n_grid, self.grid_step_s)

    # -------------------------------------------------- host fold (parity path)
    def add_patient(self, patient_id: int, stats: PatientStats, hypo_events=(0, 0)) -> None:
        if stats.ticks != self.horizon_ticks:
            raise ValueError("patient tick count does not match the trial horizon")
        H = self.horizon_ticks
        self.n_patients += 1
        self.tir_ticks_total += stats.tir_ticks
        fb = np.minimum(stats.tir_ticks * TIR_BINS // H, TIR_BINS)
        self.tir_hist[np.arange(5), fb] += 1
        self.bg_hist_total += stats.bg_hist
        below = stats.below_threshold_ticks()
        np.minimum(self.below_min, below, out=self.below_min)
        np.maximum(self.below_max, below, out=self.below_max)
        self.sum_bg_fp += int(rint_fp(stats.sum_bg))
        self.min_bg = min(self.min_bg, float(stats.min_bg))
        self.max_bg = max(self.max_bg, float(stats.max_bg))
        tl = rint_fp(stats.timeline_bg)
        self.timeline_sum_fp += tl
        np.minimum(self.timeline_min_fp, tl, out=self.timeline_min_fp)
        np.maximum(self.timeline_max_fp, tl, out=self.timeline_max_fp)
        totals = stats.day_totals()
        for k, s in enumerate(DOSE_SIGNALS):
            bins = np.minimum((totals[:, k] // DOSE_BIN_WIDTH[s]).astype(np.int64), DOSE_BIN_COUNT[s])
            np.add.at(self.dose_hist[s], bins, 1)
            self.dose_sum_fp[k] += int(rint_fp(float(np.sum(totals[:, k]))))
        self.n_patient_days += self.n_days
        t = stats.tir_ticks
        for row, ticks in enumerate((t[2], t[0] + t[1], t[0], t[3] + t[4], t[4])):
            self.metric_hist[row, min(TIR_BINS, int(ticks) * TIR_BINS // H)] += 1
        self.metric_hist[5, min(TIR_BINS, int(hypo_events[0]))] += 1
        self.metric_hist[6, min(TIR_BINS, int(hypo_events[1]))] += 1
        cand = WorstCase(patient_id, float(stats.min_bg), float(stats.max_bg),
                         stats.ticks_below_3, stats.ticks, stats.tir_ticks.copy(),
                         stats.bg_hist.copy())
        if self.worst is None or _worst_key(cand) < _worst_key(self.worst):
            self.worst = cand

    def add_aborted(self, patient_id: int) -> None:
        self.n_aborted += 1
        self.aborted_ids = tuple(sorted(self.aborted_ids + (int(patient_id),)))


def merge(a: TrialAccumulator, b: TrialAccumulator) -> TrialAccumulator:
    """Exact, associative, commutative combination (analytics.py:272-302)."""
    if a.grid_meta() != b.grid_meta():
        raise GridMismatchError("accumulators were built with different grids")
    out = TrialAccumulator(a.dt_s, a.horizon_ticks, a.n_days, a.n_grid, a.grid_step_s)
    out.n_patients = a.n_patients + b.n_patients
    out.n_aborted = a.n_aborted + b.n_aborted
    out.aborted_ids = tuple(sorted(a.aborted_ids + b.aborted_ids))
    for name in ("tir_ticks_total", "tir_hist", "bg_hist_total", "timeline_sum_fp", "metric_hist"):
        setattr(out, name, getattr(a, name) + getattr(b, name))
    out.below_min = np.minimum(a.below_min, b.below_min)
    out.below_max = np.maximum(a.below_max, b.below_max)
    out.timeline_min_fp = np.minimum(a.timeline_min_fp, b.timeline_min_fp)
    out.timeline_max_fp = np.maximum(a.timeline_max_fp, b.timeline_max_fp)
    out.sum_bg_fp = a.sum_bg_fp + b.sum_bg_fp
    out.min_bg = min(a.min_bg, b.min_bg)
    out.max_bg = max(a.max_bg, b.max_bg)
    out.dose_hist = {s: a.dose_hist[s] + b.dose_hist[s] for s in DOSE_SIGNALS}
    out.dose_sum_fp = [x + y for x, y in zip(a.dose_sum_fp, b.dose_sum_fp)]
    out.n_patient_days = a.n_patient_days + b.n_patient_days
    cands = [w for w in (a.worst, b.worst) if w is not None]
    out.worst = min(cands, key=_worst_key) if cands else None
    return out


# ------------------------------------------------------------- report
def quantile_bin_center(hist, n: int, num: int, den: int, width: float) -> float:
    """Nearest-rank quantile q = num/den from binned counts (analytics.py:305-317)."""
    target = -(-num * n // den)
    cum = np.cumsum(np.asarray(hist, dtype=np.int64))
    idx = int(np.searchsorted(cum, target, side="left"))
    if idx >= len(cum):
        return (len(cum) - 0.5) * width
    return (idx + 0.5) * width


def box_stats(hist, n: int, width: float) -> dict:
    """Box-plot summary with 1.5 IQR whiskers (analytics.py:320-337)."""
    hist = np.asarray(hist)
    q1 = quantile_bin_center(hist, n, 1, 4, width)
    med = quantile_bin_center(hist, n, 1, 2, width)
    q3 = quantile_bin_center(hist, n, 3, 4, width)
    iqr = q3 - q1
    lo, hi = q1 - 1.5 * iqr, q3 + 1.5 * iqr
    nz = np.nonzero(hist)[0]
    centers = (nz + 0.5) * width
    inside = centers[(centers >= lo) & (centers <= hi)]
    return {
        "q1": q1, "median": med, "q3": q3,
        "whisker_lo": float(inside[0]) if inside.size else q1,
        "whisker_hi": float(inside[-1]) if inside.size else q3,
        "n_outliers_lo": int(np.sum(hist[nz[centers < lo]])) if nz.size else 0,
        "n_outliers_hi": int(np.sum(hist[nz[centers > hi]])) if nz.size else 0,
    }


def _nonempty(acc):
    if acc.n_patients == 0:
        raise ValueError("empty accumulator")


def tir_report(acc) -> dict:
    _nonempty(acc)
    denom = acc.n_patients * acc.horizon_ticks
    return {
        "ranges": list(RANGE_NAMES), "n_patients": acc.n_patients,
        "mean": [int(t) / denom for t in acc.tir_ticks_total],
        "worst_case": [int(t) / acc.worst.ticks for t in acc.worst.tir_ticks],
        "box": {name: box_stats(acc.tir_hist[r], acc.n_patients, 1.0 / TIR_BINS)
                for r, name in enumerate(RANGE_NAMES)},
    }


def bg_cdf_report(acc) -> dict:
    _nonempty(acc)
    denom = acc.n_patients * acc.horizon_ticks
    return {
        "thresholds_mmol_per_l": [float(t) for t in THRESHOLDS],
        "mean": [int(t) / denom for t in np.cumsum(acc.bg_hist_total)[:N_THRESHOLDS]],
        "min": [int(t) / acc.horizon_ticks for t in acc.below_min],
        "max": [int(t) / acc.horizon_ticks for t in acc.below_max],
        "worst_case": [int(t) / acc.worst.ticks for t in np.cumsum(acc.worst.bg_hist)[:N_THRESHOLDS]],
    }


def dose_report(acc) -> dict:
    _nonempty(acc)
    sig = {}
    for k, s in enumerate(DOSE_SIGNALS):
        nb = DOSE_BIN_COUNT[s]
        sig[s] = {
            "bin_width": DOSE_BIN_WIDTH[s], "bin_edges_start": 0.0,
            "counts": [int(c) for c in acc.dose_hist[s][:nb]],
            "overflow": int(acc.dose_hist[s][nb]),
            "mean_daily": acc.dose_sum_fp[k] / FP_SCALE / acc.n_patient_days,
        }
    return {"n_patient_days": acc.n_patient_days, "signals": sig}


def timeline_report(acc) -> dict:
    _nonempty(acc)
    return {
        "grid_step_s": acc.grid_step_s,
        "times_s": [i * acc.grid_step_s for i in range(acc.n_grid)],
        "mean": [int(v) / FP_SCALE / acc.n_patients for v in acc.timeline_sum_fp],
        "min": [int(v) / FP_SCALE for v in acc.timeline_min_fp],
        "max": [int(v) / FP_SCALE for v in acc.timeline_max_fp],
    }


def build_trial_report(acc, run_meta: dict) -> dict:
    """JSON-ready report, schema ``glucotrial/trial-report/1``."""
    _nonempty(acc)
    denom = acc.n_patients * acc.horizon_ticks
    w = acc.worst
    return {
        "schema": SCHEMA_REPORT,
        "run": dict(run_meta),
        "n_patients": acc.n_patients,
        "n_aborted": acc.n_aborted,
        "aborted_ids": list(acc.aborted_ids),
        "horizon_ticks": acc.horizon_ticks,
        "dt_s": acc.dt_s,
        "bg": {"mean": acc.sum_bg_fp / FP_SCALE / denom, "min": acc.min_bg, "max": acc.max_bg},
        "worst_case": {"patient_id": w.patient_id, "min_bg": w.min_bg, "max_bg": w.max_bg,
                       "ticks_below_3_mmol": w.ticks_below_3},
        "tir": tir_report(acc),
        "cdf": bg_cdf_report(acc),
        "doses": dose_report(acc),
        "timeline": timeline_report(acc),
    }


def report_bytes(report: dict) -> bytes:
    """Canonical serialisation (storage.py:229-231)."""
    return (json.dumps(report, sort_keys=True, indent=2) + "\n").encode()


QUANTILES = ((1, 20), (1, 4), (1, 2), (3, 4), (19, 20))  # 5/25/50/75/95 %


def metric_quantiles(acc) -> dict:
    """BASELINE population quantiles (5/25/50/75/95 %) of every metric, by the
    reference's nearest-rank bin-centre rule; range fractions in [0, 1] at
    0.5 % bins, hypo-event counts at unit bins."""
    out = {}
    for row, name in enumerate(METRIC_NAMES):
        width = 1.0 / TIR_BINS if row < 5 else 1.0
        shift = 0.0 if row < 5 else -0.5   # unit bins: report the integer count
        out[name] = {f"p{int(100 * a / b)}": quantile_bin_center(acc.metric_hist[row], acc.n_patients, a, b, width) + shift
                     for a, b in QUANTILES}
    return out
