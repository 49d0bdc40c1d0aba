"""Host-side inputs of the bitwise parity path (``run_trial(noise="reference")``),
prepared in worker processes.

The reference draws each patient's process and measurement noise from its own
keyed numpy stream (rng.py:26-39; simulation.py:333-357) and builds each
patient's protocol in Python (simulation.py:500-505).  Both are per-patient,
independent and held under the GIL, so the parity path spreads them over the
host cores the way the reference spreads whole patients over its process pool
(simulation.py:572-599): a persistent spawn-context process pool, the noise
written straight into a shared-memory block the caller then hands to the
device, the protocols returned by value.  The values are the reference's
(same streams, same draws, same order); only where they are computed moves.
"""

from __future__ import annotations

import atexit
import os
import threading
from concurrent.futures import ProcessPoolExecutor
from multiprocessing import get_context
from multiprocessing.shared_memory import SharedMemory

import numpy as np

_POOL = None
_POOL_PID = None


def workers() -> int:
    """Worker processes for the host inputs (GLUCOSIM_HOST_WORKERS, default:
    the usable host cores)."""
    env = os.environ.get("GLUCOSIM_HOST_WORKERS")
    if env:
        return max(1, int(env))
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:   # pragma: no cover (non-Linux)
        return max(1, os.cpu_count() or 1)


def pool():
    """The persistent worker pool (None with one worker)."""
    global _POOL, _POOL_PID
    if workers() <= 1:
        return None
    if _POOL is None or _POOL_PID != os.getpid():
        _POOL = ProcessPoolExecutor(max_workers=workers(), mp_context=get_context("spawn"))
        _POOL_PID = os.getpid()
        atexit.register(_POOL.shutdown, wait=False, cancel_futures=True)
    return _POOL


class NoiseBlock:
    """wiener [n, H, 3] and meas [n, H/period_steps] float64 in one
    shared-memory block (workers attach by name and fill their rows)."""

    def __init__(self, n: int, horizon_ticks: int, n_ctl: int, shared: bool = True):
        self.shape_w, self.shape_m = (n, horizon_ticks, 3), (n, n_ctl)
        nbytes = 8 * (n * horizon_ticks * 3 + n * n_ctl)
        # a tmpfs too small for the block would fault on write, not on creation:
        # check the free space first and fall back to process-local memory
        self.shm = SharedMemory(create=True, size=max(8, nbytes)) if shared and _shm_room(nbytes) else None
        buf = self.shm.buf if self.shm is not None else np.empty(max(1, nbytes // 8)).data
        self.wiener = np.ndarray(self.shape_w, dtype=np.float64, buffer=buf)
        self.meas = np.ndarray(self.shape_m, dtype=np.float64, buffer=buf, offset=self.wiener.nbytes)

    @property
    def shared(self) -> bool:
        return self.shm is not None

    def pin(self) -> "NoiseBlock":
        """Page-lock the block for the device copy (cudaHostRegister): the
        injected noise then moves at DMA speed instead of through a pageable
        staging copy.  A no-op when the runtime refuses."""
        self._pinned = False
        try:
            import torch
            nbytes = self.wiener.nbytes + self.meas.nbytes
            if nbytes and torch.cuda.is_available():
                self._pinned = int(torch.cuda.cudart().cudaHostRegister(self.wiener.ctypes.data, nbytes, 0)) == 0
        except Exception:
            self._pinned = False
        return self

    def close(self) -> None:
        if getattr(self, "_pinned", False):
            import torch
            torch.cuda.cudart().cudaHostUnregister(self.wiener.ctypes.data)
            self._pinned = False
        self.wiener = self.meas = None
        if self.shm is None:
            return
        try:
            self.shm.close()
        except BufferError:   # a view still alive (e.g. held by a traceback): freed with it
            pass
        self.shm.unlink()


_BLOCKS: dict = {}
# one bitwise trial at a time uses the cached blocks (threads of one process
# running trials concurrently take turns)
LOCK = threading.Lock()


def blocks(n: int, horizon_ticks: int, n_ctl: int, shared: bool, count: int = 2) -> list:
    """``count`` page-locked NoiseBlocks of at least n rows, kept between
    calls: pinning a gigabyte of shared memory costs ~0.3 s, so a process
    that runs several trials pays it once (freed at exit)."""
    key = (horizon_ticks, n_ctl, shared)
    cur = _BLOCKS.get(key)
    if cur is None or cur[0].shape_w[0] < n or len(cur) < count:
        if cur is not None:
            for b in cur:
                b.close()
        cur = [NoiseBlock(n, horizon_ticks, n_ctl, shared=shared).pin() for _ in range(count)]
        _BLOCKS[key] = cur
    return cur[:count]


@atexit.register
def _free_blocks() -> None:
    for bl in _BLOCKS.values():
        for b in bl:
            try:
                b.close()
            except Exception:
                pass
    _BLOCKS.clear()


def _shm_room(nbytes: int) -> bool:
    try:
        st = os.statvfs("/dev/shm")
    except OSError:
        return False
    return st.f_bavail * st.f_frsize >= 2 * nbytes + (64 << 20)


def fill_noise(w: np.ndarray, m: np.ndarray, seed: int, pids, proc, sens) -> None:
    """Rows of the reference's noise (rng.reference_noise), drawn in place."""
    from .rng import ROLE_MEASUREMENT_NOISE, ROLE_PROCESS_NOISE, stream
    for j, pid in enumerate(pids):
        if proc[j]:
            stream(seed, int(pid), ROLE_PROCESS_NOISE).standard_normal(w.shape[1:], out=w[j])
        else:
            w[j] = 0.0
        if sens[j]:
            stream(seed, int(pid), ROLE_MEASUREMENT_NOISE).standard_normal(m.shape[1], out=m[j])
        else:
            m[j] = 0.0


def _noise_task(args):
    name, shape_w, shape_m, lo, hi, seed, pids, proc, sens = args
    # (spawned workers share the parent's resource tracker: attaching registers
    # the name again, idempotently, and the parent's unlink releases it)
    shm = SharedMemory(name=name)
    try:
        w = np.ndarray(shape_w, dtype=np.float64, buffer=shm.buf)
        m = np.ndarray(shape_m, dtype=np.float64, buffer=shm.buf, offset=w.nbytes)
        fill_noise(w[lo:hi], m[lo:hi], seed, pids, proc, sens)
        del w, m
    finally:
        shm.close()
    return hi - lo


def build_protocols(generator, seed: int, patients, horizon_s: float) -> list:
    from .protocol import compile_protocol
    return [compile_protocol(generator.build(seed, p), horizon_s) for p in patients]


def _protocol_task(args):
    generator, seed, patients, horizon_s = args
    return build_protocols(generator, seed, patients, horizon_s)


class Prepared:
    """One chunk's host inputs in flight; ``result()`` -> (protocol arrays,
    NoiseBlock).  A protocol span whose objects fail to pickle is built in
    this process instead (same values)."""

    def __init__(self, spans, proto_futs, noise_futs, block, local):
        self.spans, self.proto_futs, self.noise_futs, self.block, self.local = (spans, proto_futs, noise_futs,
                                                                              block, local)

    def result(self):
        pas = []
        for (lo, hi), f in zip(self.spans, self.proto_futs):
            try:
                pas.extend(f.result())
            except Exception:
                pas.extend(self.local(lo, hi))
        for f in self.noise_futs:
            f.result()
        return pas, self.block


def prepare(generator, seed: int, patients, pids, proc, sens, horizon_s: float, horizon_ticks: int,
            n_ctl: int, min_parallel: int = 64, block: NoiseBlock | None = None) -> Prepared:
    """Start the host inputs of one chunk of patients (rows [0, n) of
    ``block``, a new block when None): in the worker pool when the chunk is
    large enough and the block is shared, else in this process."""
    n = len(pids)
    p = pool() if n >= min_parallel else None
    if block is None:
        block = NoiseBlock(n, horizon_ticks, n_ctl, shared=p is not None)
    if not block.shared:
        p = None
    local = lambda lo, hi: build_protocols(generator, seed, patients[lo:hi], horizon_s)
    if p is None:
        pas = local(0, n)
        fill_noise(block.wiener[:n], block.meas[:n], seed, pids, proc, sens)
        done = _Done(pas)
        return Prepared([(0, n)], [done], [], block, local)
    k = workers()
    bounds = [(n * j) // k for j in range(k + 1)]
    spans = [(lo, hi) for lo, hi in zip(bounds[:-1], bounds[1:]) if hi > lo]
    noise = [p.submit(_noise_task, (block.shm.name, block.shape_w, block.shape_m, lo, hi, seed,
                                    [int(x) for x in pids[lo:hi]], [bool(x) for x in proc[lo:hi]],
                                    [bool(x) for x in sens[lo:hi]]))
             for lo, hi in spans]
    proto = [p.submit(_protocol_task, (generator, seed, list(patients[lo:hi]), horizon_s)) for lo, hi in spans]
    return Prepared(spans, proto, noise, block, local)


class _Done:
    def __init__(self, value):
        self.value = value

    def result(self):
        return self.value
