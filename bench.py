"""Benchmark: simulated patient-weeks per second of the closed-loop Monte
Carlo hot path (BASELINE.json metric) on B200s, with the FP64 roofline of
the fused integrator and the reference-path CPU baseline.

Workload (BASELINE configs[1]): 100,000 virtual patients x 4 weeks per GPU,
FP64, Euler-Maruyama at 1-min step with process noise, 5-min CGM with sensor
noise, the BASELINE's PID controller with pump quantisation (pid.py; its
golden run is the reference's own generic engine) -- or, with
--controller dual_hormone, the reference's own AP controller -- 3 meals/day ~N(50/70/80 g, 10 g) with U(+-30 min)
jitter, seed 1, population drawn by the device sampler from the reference
distribution table.  One "step" = one pass of the hot path over the batch:
fused integrator + population reduction (histograms, quantile bins, exact
accumulator).  Multi-GPU (torchrun): weak scaling, each rank simulates its
own 100k-patient shard (global patient ids rank*n ...), exact accumulators
are combined with NCCL all-reduce (sum/min/max) — the only collective.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself
under ``python -m torch.distributed.run --nproc-per-node N`` (127.0.0.1
rendezvous), one rank per GPU; rank 0 prints the one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

N_PATIENTS = 100_000
WEEKS = 4
DT_S = 60.0
SEED = 1
METRIC = "simulated patient-weeks/sec"
FP64_PEAK_FILES = [os.path.join(REPO, "profiles", f) for f in ("fp64_peak_r02.jsonl", "fp64_peak_r01.jsonl")]


def fp64_peak():
    """Measured DFMA peak (tools/fp64_peak.py on this pool's B200, SM clock
    sampled during the run); MEASURED_PEAKS.json carries no FP64 figure.
    Returns (peak for the bench's back-to-back kernel = the SUSTAINED figure
    when recorded, burst figure, source)."""
    for path in FP64_PEAK_FILES:
        best, sus, clk = 0.0, None, None
        try:
            for line in open(path):
                d = json.loads(line)
                if d.get("kernel") == "dfma":
                    best = max(best, d["tflops"])
                if d.get("kernel") == "dfma_sustained":
                    sus = d["tflops"]
                if d.get("summary"):
                    clk = d.get("clocks", {}).get("sm_mhz")
        except OSError:
            continue
        if best:
            rel = os.path.relpath(path, REPO)
            if sus:
                return sus, best, f"measured DFMA, sustained 4 s back to back ({rel}, median SM clock {clk} MHz)"
            return best, best, f"measured DFMA, best burst ({rel})"
    return 37.2, 37.2, "nominal 148 SM x 64 DFMA x 2 x 1.965 GHz (fallback)"


PIPE_FILES = {"pid_pump": "fast_kernel_pid_pipes.json", "dual_hormone": "fast_kernel_dual_pipes.json"}


def measured_pipes(controller):
    """Pipe utilisation of the fused kernel from the newest committed ncu
    --set full capture of this workload (profiles/*_fast_kernel_*_pipes.json)."""
    import glob
    paths = sorted(glob.glob(os.path.join(REPO, "profiles", "r*_" + PIPE_FILES[controller])))
    if not paths:
        return None
    d = json.load(open(paths[-1]))
    d["file"] = os.path.relpath(paths[-1], REPO)
    return d


TRAFFIC_FILES = {"pid_pump": "fast_kernel_pid_traffic.json", "dual_hormone": "fast_kernel_dual_traffic.json"}


def measured_traffic(n_patients, controller="pid_pump"):
    """DRAM bytes (read + write) per launch of the fused kernel from the
    newest committed ncu --set full capture of this exact workload, else None."""
    import glob
    paths = sorted(glob.glob(os.path.join(REPO, "profiles", "r*_" + TRAFFIC_FILES[controller])))
    if not paths or n_patients != N_PATIENTS:
        return None
    d = json.load(open(paths[-1]))
    return d["dram_bytes_read"] + d["dram_bytes_write"]


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args, argv) -> int | None:
    """--gpus N > 1 outside torchrun: re-launch this script as N ranks (one
    process per GPU) and return their exit status; None when no spawn is
    needed (already a rank, or N = 1).  NCCL's INFO log (communicator set-up,
    transports) goes to per-rank files so stdout keeps the one JSON line."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if not args.dry_run and args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT,COLL")
    env.setdefault("NCCL_DEBUG_FILE", os.path.join(REPO, "gpurun_out" if os.path.isdir(os.path.join(REPO, "gpurun_out"))
                                                   else "/tmp", "nccl_bench.%h.%p.log"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + list(argv)
    return subprocess.run(cmd, env=env).returncode


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self):
        """NVML polling (microseconds per query): a sample every 10 ms."""
        import pynvml as nv
        import torch
        nv.nvmlInit()
        try:  # the CUDA device's own GPU (CUDA_VISIBLE_DEVICES may renumber it)
            h = nv.nvmlDeviceGetHandleByUUID("GPU-" + str(torch.cuda.get_device_properties(self.index).uuid))
        except Exception:
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
        while not self._stop.is_set():
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            r = get_reasons(h)
            self.rows.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits])
            self._stop.wait(0.01)

    def _run(self):
        try:
            self._run_nvml()
            return
        except Exception:
            pass
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 2 + k and r[2 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def controller_setup(controller_id: str):
    """(profile, device code, config label) of the benchmarked controller."""
    if controller_id == "pid_pump":
        from paper_2202_13927_b200.pid import PIDProfile
        return PIDProfile(), 1, "pid_pump (PID basal + pump quantisation 0.05 U, meal bolus; BASELINE)"
    from paper_2202_13927_b200.controller import ControllerHyperparameters
    return ControllerHyperparameters(), 0, "dual_hormone (reference AP: PD basal + heuristic meal bolus)"


CPU_SAMPLE_SECONDS = 10.0   # target CPU work per baseline sample


def cpu_sample_size(weeks: int, threads: int, controller_id: str) -> int:
    """Patients per CPU-baseline sample: a short pilot run sizes the sample
    to about CPU_SAMPLE_SECONDS of work on this host."""
    pilot = max(threads * 16, 128)
    rate, _wall = cpu_baseline(pilot, weeks, threads, controller_id)
    return int(min(max(pilot, rate * CPU_SAMPLE_SECONDS / weeks), 400_000))


def cpu_baseline(n_sample: int, weeks: int, threads: int, controller_id: str = "pid_pump"):
    """Reference path on the host cores: the oracle's C restatement of the
    numba kernel (bitwise equal to it on injected inputs), OpenMP over
    patients, per-patient noise + schedule generation included."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle
    from paper_2202_13927_b200.config import SimulationConfig, sizes
    from paper_2202_13927_b200.controller import initial_icr
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.rng import ROLE_DEVICE_NOISE
    cfg = SimulationConfig(horizon_s=weeks * 7 * 86400.0, seed=SEED, dt_s=DT_S)
    sz = sizes(cfg)
    pop = golden_population(n_sample)
    params, ub, x0 = pop
    prof, code, _ = controller_setup(controller_id)
    oracle.set_controller(code)
    c0 = np.zeros((n_sample, 11))
    c0[:, 3] = [initial_icr(u, prof) for u in ub]
    c0[:, 6] = -1e18
    t0 = time.perf_counter()
    out = oracle.run_batch_philox(ThreeMealProtocol(), SEED, 0, params, x0, c0, prof.to_vec(), ub, sz,
                                  cfg.dt_s, cfg.controller_period_s, ROLE_DEVICE_NOISE, nthreads=threads)
    wall = time.perf_counter() - t0
    assert np.all(out["status"] == 0)
    return n_sample * weeks / wall, wall


def golden_population(n):
    """Host population for the CPU arm: the 64 parameter sets the reference's
    own sampler drew for seed 0 (tests/golden/population.npz), tiled to n
    patients (each patient id gets its own noise and meal streams)."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle
    g = np.load(os.path.join(REPO, "tests", "golden", "population.npz"))
    params = np.ascontiguousarray(np.resize(g["s0_params"], (n, 30)))
    ub = np.resize(g["s0_ubasal"], n).astype(np.float64)
    x0 = np.zeros((n, 16))
    for i in range(min(n, 64)):
        x0[i], _ = oracle.steady_state(params[i])
    x0 = np.ascontiguousarray(np.resize(x0[:min(n, 64)], (n, 16)))
    return params, ub, x0


REF_DIR = os.path.join(REPO, "baseline", "_ref")


def reference_available() -> bool:
    """The unmodified reference (glucotrial, pip-installed into baseline/_ref)
    and its numba JIT importable on this host."""
    if not os.path.isdir(os.path.join(REF_DIR, "glucotrial")):
        return False
    try:
        import numba  # noqa: F401
    except ImportError:
        return False
    return True


_REF_CACHE = {}


class _RefPatient:
    """The two Patient fields the reference's simulation reads (id, weight)."""

    def __init__(self, pid, w):
        self.id, self.body_weight_kg = pid, w


def reference_numba(n_sample: int, weeks: int, threads: int):
    """The reference's OWN CPU path on the host cores: glucotrial.simulation.
    run_trial(..., workers=threads) from baseline/_ref on its numba fast engine
    (hovorka_ext + dual_hormone, simulation.py:301-311; the BASELINE's PID runs
    only on the reference's ~300x slower generic engine, so the reference's
    own controller is the conservative baseline), after _warmup_fast_path()
    (simulation.py:534-548).  Same shape as the GPU workload: 3-meal generator
    (the product's plug-in through the reference's generator contract), dt
    60 s, seed 1, the reference sampler's own seed-7 parameter sets tiled to
    n_sample patients.  Returns (patient-weeks/s over run_trial's own wall_s,
    wall_s)."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    from glucotrial.controller import load_profile
    from glucotrial.population import ParameterSet, load_parameter_table
    from glucotrial.simulation import SimulationConfig as RefConfig
    from glucotrial.simulation import _warmup_fast_path, run_trial
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    if n_sample not in _REF_CACHE:
        g = np.load(os.path.join(REPO, "tests", "golden", "population_s7_n4000.npz"))
        fixed = load_parameter_table().fixed
        names = [str(x) for x in g["names"]]

        entries = []
        for i in range(n_sample):
            j = i % g["weights"].size
            v = {"weight_kg": float(g["weights"][j])}
            v.update({k: float(x) for k, x in zip(names, g["sampled"][j])})
            v.update(fixed)
            entries.append((_RefPatient(i, float(g["weights"][j])), ParameterSet(values=v, u_basal_u_per_h=float(g["ubasal"][j]))))
        _REF_CACHE[n_sample] = entries
    _warmup_fast_path()
    cfg = RefConfig(horizon_s=weeks * 7 * 86400.0, seed=SEED, dt_s=DT_S)
    res = run_trial(_REF_CACHE[n_sample], ThreeMealProtocol(), "dual_hormone", load_profile(), "hovorka_ext", cfg,
                    workers=threads)
    assert res.accumulator.n_patients == n_sample
    return n_sample * weeks / res.wall_s, res.wall_s


def reference_sample_size(weeks: int, threads: int) -> int:
    """Patients per reference sample: a pilot sizes it to about
    CPU_SAMPLE_SECONDS of reference work on this host."""
    pilot = max(threads * 32, 256)
    rate, _ = reference_numba(pilot, weeks, threads)
    return int(min(max(pilot, rate * CPU_SAMPLE_SECONDS / weeks), 400_000))


def cpu_reference_or_port(weeks: int, threads: int, controller_id: str):
    """The CPU baseline of record: the reference itself (numba) when it is
    installed, else the oracle's C port.  Returns (value, wall_s, kind, sample)."""
    if reference_available():
        n = reference_sample_size(weeks, threads)
        v, wall = reference_numba(n, weeks, threads)
        return v, wall, "reference", (f"{n} patients x {weeks} weeks, dt 60 s: glucotrial.simulation.run_trial("
                                      f"workers={threads}) from baseline/_ref, numba fast engine, dual_hormone, "
                                      f"3-meal plug-in ({wall:.1f} s wall)")
    n = cpu_sample_size(weeks, threads, controller_id)
    v, wall = cpu_baseline(n, weeks, threads, controller_id)
    return v, wall, "port", (f"{n} patients x {weeks} weeks (oracle C restatement, OpenMP, {wall:.1f} s wall; "
                             "reference not installed)")


def run_reference_arm(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    use_ref = reference_available()
    n_sample = reference_sample_size(WEEKS, threads) if use_ref else cpu_sample_size(WEEKS, threads, args.controller)
    vals = []
    for i in range(args.warmup + args.steps):
        if use_ref:
            v, wall = reference_numba(n_sample, WEEKS, threads)
        else:
            v, wall = cpu_baseline(n_sample, WEEKS, threads, args.controller)
        if i >= args.warmup:
            vals.append(v)
    v = float(np.mean(vals))
    # the oracle's C port on the same host, for the record (kind "port")
    port_n = cpu_sample_size(WEEKS, threads, "dual_hormone")
    port_v, port_wall = cpu_baseline(port_n, WEEKS, threads, "dual_hormone")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "patient-weeks/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * n_sample * WEEKS / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"BASELINE configs[1] shape ({N_PATIENTS} patients x {WEEKS} weeks), "
                               f"timed on a {n_sample}-patient sample at full horizon",
                   "dt_s": DT_S, "seed": SEED,
                   "controller": ("dual_hormone (the reference's own controller on its numba fast engine; "
                                  "the BASELINE's PID runs only on its ~300x slower generic engine)")
                   if use_ref else controller_setup(args.controller)[2],
                   "protocol": "three_meal"},
        "cpu_baseline": {"value": v, "unit": "patient-weeks/s", "cores": threads,
                         "kind": "reference" if use_ref else "port",
                         "sample": (f"{n_sample} patients x {WEEKS} weeks, dt 60 s: glucotrial.simulation.run_trial("
                                    f"workers={threads}) from baseline/_ref (numba), after _warmup_fast_path()")
                         if use_ref else f"{n_sample} patients x {WEEKS} weeks, dt 60 s, all {threads} host threads"},
        "port": {"value": port_v, "unit": "patient-weeks/s", "kind": "port", "threads": threads,
                 "sample": f"{port_n} patients x {WEEKS} weeks, dual_hormone, oracle C restatement (OpenMP)"},
        "e2e": {"value": v, "unit": "patient-weeks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)
    from paper_2202_13927_b200 import analytics, engine, flops
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.parallel import allreduce_accumulator
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial, run_population_arrays

    n = args.patients
    cfg = SimulationConfig(horizon_s=WEEKS * 7 * 86400.0, seed=SEED, dt_s=DT_S)
    pid0 = rank * n
    prof, _code, ctl_label = controller_setup(args.controller)
    gen = ThreeMealProtocol()
    t_s0 = time.perf_counter()
    pop = generate_population(SEED, n, pid0=pid0, device=device, on_exhausted="redraw_weight")
    torch.cuda.synchronize()
    sampler_s = time.perf_counter() - t_s0
    ft = FastTrial(pid0, pop.params_device, pop.basal_device, gen, prof, cfg, controller_id=args.controller,
                   device=device,
                   per_patient_metrics=True)
    stream = torch.cuda.current_stream(device)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)  # > 126 MB L2

    def one_step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        ft.simulate()
        if ev is not None:
            ev[1].record(stream)
        ft._rerun_if_diverged()
        ft.reduce()
        if ev is not None:
            ev[2].record(stream)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()                 # L2 flush between timed iterations
            one_step(evs[k])
        torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    sim_ms = np.array([e[0].elapsed_time(e[1]) for e in evs])
    step_ms = np.array([e[0].elapsed_time(e[2]) for e in evs])
    tot_ms = float(step_ms.sum())
    if ws > 1:
        t = torch.tensor([tot_ms], device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot_ms = float(t.item())
    acc = ft.accumulator()
    acc_all = allreduce_accumulator(acc, device) if ws > 1 else acc

    # end-to-end through the public array API with host (pinned) buffers
    params_h = pop.params_device.cpu().pin_memory()
    basal_h = pop.basal_device.cpu().pin_memory()
    e2e_ms = []
    for k in range(max(1, min(args.steps, 3)) + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        acc_e, met = run_population_arrays(params_h, basal_h, gen, prof, cfg, pid0=pid0, device=device,
                                           controller_id=args.controller)
        torch.cuda.synchronize()
        if k > 0:
            e2e_ms.append(1000 * (time.perf_counter() - t0))
    e2e = float(np.median(e2e_ms))
    if ws > 1:
        t = torch.tensor([e2e], device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e = float(t.item())
    assert analytics.report_bytes(analytics.build_trial_report(acc_e, {})) == \
        analytics.report_bytes(analytics.build_trial_report(acc, {})), "e2e result differs"

    # the reference-signature drop-in (simulation.run_trial, simulation.py:551
    # semantics) with host Patient / ParameterSet objects: packing the
    # population on the host is part of that call (one measurement, rank 0)
    api = None
    if rank == 0 and ws == 1:
        from paper_2202_13927_b200.simulation import run_trial
        entries = pop.entries()
        walls = []
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = run_trial(entries, gen, args.controller, prof, "hovorka_ext", cfg, noise="philox", device=device)
            walls.append(time.perf_counter() - t0)
        assert analytics.report_bytes(analytics.build_trial_report(res.accumulator, {})) == \
            analytics.report_bytes(analytics.build_trial_report(acc, {})), "run_trial result differs"
        api = {"value": n * WEEKS / walls[-1], "unit": "patient-weeks/s", "wall_s": walls[-1],
               "path": "simulation.run_trial(population=[(Patient, ParameterSet)] * n, noise='philox'): host "
                       "packing of the reference's objects + staging + fused kernel + reduction + report"}
    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return 0
    pw_per_step = n * WEEKS * ws
    value = pw_per_step / (tot_ms / args.steps / 1000.0)
    F = flops.flops_per_step(ft.sz["period_steps"], args.controller)
    F_nt = flops.flops_per_step_nontrivial(ft.sz["period_steps"], args.controller, exercise=False)
    flop_per_launch = F * n * ft.sz["horizon_ticks"]
    sim_s = float(np.mean(sim_ms)) / 1000.0
    peak, peak_burst, peak_src = fp64_peak()
    achieved = flop_per_launch / sim_s / 1e12
    cpu_v, cpu_wall, cpu_kind, cpu_sample = None, None, None, None
    if not args.no_cpu_baseline and ws == 1:   # the CPU baseline: rank 0 at N = 1 only
        threads = os.cpu_count() or 1
        cpu_v, cpu_wall, cpu_kind, cpu_sample = cpu_reference_or_port(WEEKS, threads, args.controller)
    q = analytics.metric_quantiles(acc_all)
    h2d = params_h.numel() * 8 + basal_h.numel() * 8
    d2h = n * (5 * 4 + 2 * 4 + 4) + 8 * (4 + 5 + 5 * 201 + 247 + 2 * 246 + 2 + 3 * ft.sz["n_grid"] + 603 + 3 + 4 + 7 * 201)
    line = {
        "metric": METRIC, "value": value, "unit": "patient-weeks/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (device-sampled population from the reference distribution table; "
                "3-meal generator; on-device Philox noise)",
        "config": {"workload": f"BASELINE configs[1]: {n} patients x {WEEKS} weeks per GPU, dt 60 s, "
                               "controller period 300 s, seed 1",
                   "patients_per_gpu": n, "weeks": WEEKS, "dt_s": DT_S, "seed": SEED,
                   "controller": ctl_label,
                   "protocol": "three_meal N(50/70/80,10) g, U(+-30 min)", "noise": "philox4x32-7 (fixed key, counter (pid, tick, seed))",
                   "parallelism": f"patients sharded over {ws} GPU(s), NCCL all-reduce of exact accumulators",
                   "l2": "flushed (256 MB write) between timed iterations"},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": measured_traffic(n, args.controller),
                     # the same kernel time over the work that is not structurally zero in this
                     # workload (no exercise sessions; pid_pump doses no glucagon): flops.py
                     "frac_nontrivial": achieved * F_nt / F / peak, "flops_per_step_nontrivial": F_nt,
                     "frac_vs_burst_peak": achieved / peak_burst, "peak_burst": peak_burst,
                     "pipes_ncu": measured_pipes(args.controller),
                     "kernel": "gt::fast_kernel<THREE_MEAL, PHILOX>",
                     "algorithmic_flops_per_launch": flop_per_launch,
                     "flops_per_step": F, "peak_source": peak_src,
                     "kernel_ms": sim_s * 1000.0, "share_of_step": float(np.mean(sim_ms) / np.mean(step_ms))},
        "cpu_baseline": ({"value": cpu_v, "unit": "patient-weeks/s", "cores": os.cpu_count(), "kind": cpu_kind,
                          "sample": cpu_sample} if cpu_v else None),
        "e2e": {"value": pw_per_step / (e2e / 1000.0), "unit": "patient-weeks/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "path": "trial.run_population_arrays (pinned host params -> report fields + per-patient metrics)"},
        "e2e_run_trial_api": api,
        "gpu_launches": args.steps * 7,   # per step: fused kernel + exclusion re-run + abort-tick pass + 4 reduction kernels
        "clocks": clk.summary(),
        "sampler_s": sampler_s,
        "trial": {"n_patients": acc_all.n_patients, "n_aborted": acc_all.n_aborted,
                  "mean_bg": acc_all.sum_bg_fp / 2**24 / (acc_all.n_patients * acc_all.horizon_ticks),
                  "quantiles": q},
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def run_trial1m(args):
    """BASELINE configs[2] / the north_star's headline trial: 1M patients x 52
    weeks, seed 2, strong-scaled over the launched ranks (each rank samples and
    simulates shard_range(1M, rank, world) with global-id streams; the exact
    accumulators are combined with NCCL).  Wall-clock = device sampler +
    staging + fused kernel + reduction + combine, max over ranks."""
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)
    from paper_2202_13927_b200 import analytics
    from paper_2202_13927_b200.config import SimulationConfig
    from paper_2202_13927_b200.parallel import allreduce_accumulator, gather_per_patient, shard_range
    from paper_2202_13927_b200.population import generate_population
    from paper_2202_13927_b200.protocol import ThreeMealProtocol
    from paper_2202_13927_b200.trial import FastTrial
    n_total, weeks = args.patients if args.patients != N_PATIENTS else 1_000_000, 52
    cfg = SimulationConfig(horizon_s=weeks * 7 * 86400.0, seed=2, dt_s=DT_S)
    prof, _code, ctl_label = controller_setup(args.controller)
    lo, hi = shard_range(n_total, rank, ws)
    walls = []
    for it in range(args.warmup + args.steps):
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pop = generate_population(2, hi - lo, pid0=lo, device=device, on_exhausted="redraw_weight")
        ft = FastTrial(lo, pop.params_device, pop.basal_device, ThreeMealProtocol(), prof, cfg,
                       controller_id=args.controller, device=device, per_patient_metrics=True,
                       x0=pop.x0_device if pop.target_bg == cfg.initial_bg_mmol_per_l else None)
        ft.step()
        acc = ft.accumulator()
        if ws > 1:
            acc = allreduce_accumulator(acc, device)
            # the per-patient metric arrays, gathered over NCCL in global-id order
            metrics = gather_per_patient(ft.metrics_device(), lo, n_total, device)
        else:
            metrics = ft.metrics()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if ws > 1:
            t = torch.tensor([wall], device=device)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            wall = float(t.item())
        if it >= args.warmup:
            walls.append(wall)
        del ft, pop
    if rank == 0:
        w = float(np.median(walls))
        ok = metrics["status"] == 0
        assert metrics["tir"].shape[0] == n_total and int(ok.sum()) == acc.n_patients
        # exact per-patient quantiles of the gathered arrays next to the
        # histogram (0.5 % bin) quantiles of the accumulator
        exact = {k: {str(q): float(np.quantile(metrics[k][ok].astype(np.float64), q, method="inverted_cdf"))
                     for q in (0.05, 0.25, 0.5, 0.75, 0.95)}
                 for k in ("tir", "tbr70", "tbr54", "tar180", "tar250", "hypo_events_lt70", "hypo_events_lt54")}
        print(json.dumps({
            "metric": "1M-patient x 52-week trial wall-clock", "value": w, "unit": "s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": False, "scaling": "strong",
            "patient_weeks_per_s": n_total * weeks / w, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"BASELINE configs[2]: {n_total} patients x {weeks} weeks, seed 2, dt 60 s",
                       "controller": ctl_label, "protocol": "three_meal",
                       "timed": "sampler + staging + fused kernel + reduction + NCCL all-reduce of the exact "
                                "accumulators + NCCL all-gather of the per-patient metric arrays (host wall, "
                                "max over ranks)"},
            "gathered_patients": int(metrics["tir"].shape[0]),
            "quantiles": analytics.metric_quantiles(acc), "quantiles_exact_per_patient": exact}), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def run_dry(args):
    """--dry-run: the multi-rank plumbing without a GPU (gloo): the spawn, the
    per-rank shard ids, barrier-bracketed timing with the max over ranks and
    the whole-job aggregation of the JSON line.  The per-rank 'step' is a
    fixed host wait, so the value is NOT a measurement (tests only)."""
    import torch
    import torch.distributed as dist
    from paper_2202_13927_b200.parallel import shard_range
    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    n = args.patients
    lo, hi = rank * n, (rank + 1) * n
    for _ in range(args.warmup):
        time.sleep(0.002)
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        time.sleep(0.005)
    ms = 1000.0 * (time.perf_counter() - t0)
    ids = torch.tensor([lo, hi], dtype=torch.int64)
    parts = [torch.zeros(2, dtype=torch.int64) for _ in range(ws)]
    if ws > 1:
        dist.barrier()
        t = torch.tensor([ms])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.all_gather(parts, ids)
    else:
        parts = [ids]
    if rank == 0:
        shards = [tuple(int(v) for v in p) for p in parts]
        print(json.dumps({"metric": METRIC + " (dry run: no GPU work)", "value": n * WEEKS * ws / (ms / args.steps / 1000.0),
                          "unit": "patient-weeks/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": ms / args.steps, "dry_run": True, "scaling": "weak",
                          "shards": shards, "trial1m_shards": [shard_range(1_000_000, r, ws) for r in range(ws)]}),
              flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--patients", type=int, default=N_PATIENTS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--controller", default="pid_pump", choices=["pid_pump", "dual_hormone"])
    ap.add_argument("--workload", default="c1", choices=["c1", "trial1m"],
                    help="c1: BASELINE configs[1] throughput (default); trial1m: the 1M x 52 w trial wall-clock")
    ap.add_argument("--dry-run", action="store_true",
                    help="multi-rank plumbing check on CPU (gloo, no GPU work; tests only)")
    argv = sys.argv[1:]
    args = ap.parse_args(argv)
    rc = spawn_ranks(args, argv)
    if rc is not None:
        return rc
    if args.dry_run:
        return run_dry(args)
    if args.workload == "trial1m" and args.impl == "ours":
        return run_trial1m(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
