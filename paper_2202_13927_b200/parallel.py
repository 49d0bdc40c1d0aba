"""Multi-GPU sharding: one process per GPU, patients partitioned into
contiguous global-id ranges, exact accumulators combined after compute.

Patients never interact, so the data path has no collective;
the only exchange is the final combination of the exact integer
accumulator fields — int64 SUM / MIN / MAX all-reduces (NCCL over NVLink on
GPUs, gloo on CPU) plus an all-gather of the per-rank worst-case candidates
and aborted ids.  Because every field is an integer (or a min/max) the
result is identical for any world size, mirroring the reference's
worker-count invariance (simulation.py:54-56, test_simulation.py:242-250).
"""

from __future__ import annotations

import numpy as np

from .analytics import TrialAccumulator, WorstCase
from .layout import DOSE_SIGNALS


def shard_range(n_total: int, rank: int, world: int) -> tuple:
    """Contiguous [lo, hi) global patient ids of `rank` (balanced)."""
    base, rem = divmod(n_total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def _ordered(v: float) -> int:
    b = int(np.array([v], dtype=np.float64).view(np.int64)[0])
    return b if b >= 0 else b ^ 0x7FFFFFFFFFFFFFFF


def _unordered(b: int) -> float:
    if b < 0:
        b ^= 0x7FFFFFFFFFFFFFFF
    return float(np.array([b], dtype=np.int64).view(np.float64)[0])


def allreduce_accumulator(acc: TrialAccumulator, device=None, group=None) -> TrialAccumulator:
    """Combine per-rank accumulators into the global one on every rank."""
    import torch
    import torch.distributed as dist
    dev = device if device is not None else torch.device("cpu")
    i64 = torch.int64
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int64), device=dev)

    sums = [np.array([acc.n_patients, acc.n_aborted, acc.n_patient_days], dtype=np.int64),
            acc.tir_ticks_total, acc.tir_hist.reshape(-1), acc.bg_hist_total, acc.timeline_sum_fp,
            np.concatenate([acc.dose_hist[s] for s in DOSE_SIGNALS]),
            np.array(acc.dose_sum_fp, dtype=np.int64), acc.metric_hist.reshape(-1)]
    sizes = [len(s) for s in sums]
    st = T(np.concatenate(sums))
    dist.all_reduce(st, op=dist.ReduceOp.SUM, group=group)
    mins = T(np.concatenate([acc.below_min, acc.timeline_min_fp, [_ordered(acc.min_bg)]]))
    dist.all_reduce(mins, op=dist.ReduceOp.MIN, group=group)
    maxs = T(np.concatenate([acc.below_max, acc.timeline_max_fp, [_ordered(acc.max_bg)]]))
    dist.all_reduce(maxs, op=dist.ReduceOp.MAX, group=group)
    # python-int pieces (128-bit BG sum), worst candidates, aborted ids
    objs = [None] * dist.get_world_size(group)
    w = acc.worst
    mine = (int(acc.sum_bg_fp), tuple(acc.aborted_ids),
            None if w is None else (w.min_bg, w.ticks_below_3, w.patient_id, w.max_bg, w.ticks,
                                    w.tir_ticks.tolist(), w.bg_hist.tolist()))
    dist.all_gather_object(objs, mine, group=group)

    out = TrialAccumulator(acc.dt_s, acc.horizon_ticks, acc.n_days, acc.n_grid, acc.grid_step_s)
    s = st.cpu().numpy()
    parts = np.split(s, np.cumsum(sizes)[:-1])
    out.n_patients, out.n_aborted, out.n_patient_days = (int(v) for v in parts[0])
    out.tir_ticks_total = parts[1]
    out.tir_hist = parts[2].reshape(acc.tir_hist.shape)
    out.bg_hist_total = parts[3]
    out.timeline_sum_fp = parts[4]
    dh = np.split(parts[5], len(DOSE_SIGNALS))
    out.dose_hist = {sname: dh[k] for k, sname in enumerate(DOSE_SIGNALS)}
    out.dose_sum_fp = [int(v) for v in parts[6]]
    out.metric_hist = parts[7].reshape(acc.metric_hist.shape)
    m = mins.cpu().numpy()
    M = maxs.cpu().numpy()
    nb = len(acc.below_min)
    out.below_min, out.timeline_min_fp = m[:nb], m[nb:-1]
    out.below_max, out.timeline_max_fp = M[:nb], M[nb:-1]
    out.min_bg = _unordered(int(m[-1])) if out.n_patients else np.inf
    out.max_bg = _unordered(int(M[-1])) if out.n_patients else -np.inf
    out.sum_bg_fp = sum(o[0] for o in objs)
    out.aborted_ids = tuple(sorted(i for o in objs for i in o[1]))
    cands = [o[2] for o in objs if o[2] is not None]
    if cands:
        best = min(cands, key=lambda c: (c[0], -c[1], c[2]))
        out.worst = WorstCase(patient_id=best[2], min_bg=best[0], max_bg=best[3], ticks_below_3=best[1],
                              ticks=best[4], tir_ticks=np.array(best[5], np.int64),
                              bg_hist=np.array(best[6], np.int64))
    return out


def gather_per_patient(arrays: dict, lo: int, n_total: int, device=None, group=None) -> dict:
    """All-gather per-patient arrays (same keys on every rank, this rank's
    contiguous slice starting at global id ``lo``) into global-id order.
    Shards differ in size by at most one patient, so every rank pads to the
    largest shard (one collective per array, NCCL all-gather over NVLink on
    GPUs, gloo on CPU).  Device tensors stay on the device (no host round
    trip before the collective); the result is numpy."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = device if device is not None else torch.device("cpu")
    sizes = [shard_range(n_total, r, world) for r in range(world)]
    width = max(hi - l for l, hi in sizes)
    out = {}
    for k in sorted(arrays):
        a = arrays[k]
        if not isinstance(a, torch.Tensor):
            a = torch.as_tensor(np.ascontiguousarray(a))
        a = a.to(dev)
        t = torch.zeros((width,) + tuple(a.shape[1:]), dtype=a.dtype, device=dev)
        t[: a.shape[0]] = a
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        out[k] = torch.cat([p[: hi - l] for p, (l, hi) in zip(parts, sizes)]).cpu().numpy()
    return out


def run_trial_sharded(n_total: int, population_seed: int, generator, controller_id: str, profile, config, *,
                      device=None, group=None, gather_metrics: bool = False, hypo_min_s: float = 900.0):
    """One rank's part of a multi-GPU trial (launch one process per GPU, e.g.
    torchrun): this rank samples and simulates global ids
    ``shard_range(n_total, rank, world)`` with pid-keyed streams, then the
    exact accumulators are combined.  Every rank returns the same
    ``(report, accumulator, metrics)``; ``metrics`` (per-patient arrays in
    global-id order) only with ``gather_metrics``."""
    import torch.distributed as dist
    from . import analytics
    from .population import generate_population
    from .trial import FastTrial
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = shard_range(n_total, rank, world)
    pop = generate_population(population_seed, hi - lo, pid0=lo, device=device, on_exhausted="redraw_weight")
    ft = FastTrial(lo, pop.params_device, pop.basal_device, generator, profile, config, controller_id,
                   device, hypo_min_s=hypo_min_s, per_patient_metrics=gather_metrics,
                   x0=pop.x0_device if pop.target_bg == config.initial_bg_mmol_per_l else None)
    ft.step()
    acc = allreduce_accumulator(ft.accumulator(), device, group)
    metrics = gather_per_patient(ft.metrics(), lo, n_total, device, group) if gather_metrics else None
    return analytics.build_trial_report(acc, {}), acc, metrics
