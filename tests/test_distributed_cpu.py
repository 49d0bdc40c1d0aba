"""World-size-2 gloo test of the multi-GPU combination logic (CPU): the
all-reduced accumulator of two shards equals the single-process merge, and
the shard ranges tile the population."""

import os
import socket

import numpy as np
import pytest

from paper_2202_13927_b200 import analytics
from paper_2202_13927_b200.parallel import shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _acc(seed):
    from test_host import _random_acc
    return _random_acc(seed)


def _worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist
    from paper_2202_13927_b200.parallel import allreduce_accumulator
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    acc = _acc(100 + rank)
    acc.add_aborted(1000 + rank)
    acc.sum_bg_fp += (1 << 70) * (rank + 1)   # beyond int64: python-int path
    out = allreduce_accumulator(acc)
    q.put((rank, analytics.report_bytes(analytics.build_trial_report(out, {})), out.sum_bg_fp,
           out.aborted_ids))
    dist.destroy_process_group()


def test_allreduce_equals_merge_world2():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = _acc(100), _acc(101)
    a.add_aborted(1000)
    b.add_aborted(1001)
    a.sum_bg_fp += 1 << 70
    b.sum_bg_fp += 2 << 70
    ref = analytics.merge(a, b)
    want = analytics.report_bytes(analytics.build_trial_report(ref, {}))
    for rank, rep, s, ab in res:
        assert rep == want
        assert s == ref.sum_bg_fp
        assert ab == (1000, 1001)


@pytest.mark.parametrize("n,world", [(100_000, 1), (1_000_000, 8), (7, 3), (5, 8)])
def test_shard_ranges_tile(n, world):
    got = [shard_range(n, r, world) for r in range(world)]
    assert got[0][0] == 0 and got[-1][1] == n
    for (a, b), (c, d) in zip(got, got[1:]):
        assert b == c
    sizes = [b - a for a, b in got]
    assert max(sizes) - min(sizes) <= 1


def _gather_worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    import torch.distributed as dist
    from paper_2202_13927_b200.parallel import gather_per_patient, shard_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 11
    lo, hi = shard_range(n, rank, world)
    ids = np.arange(lo, hi)
    out = gather_per_patient({"tir": (ids * 0.5).astype(np.float32), "status": ids.astype(np.int32) % 3},
                             lo, n)
    q.put((rank, out["tir"].tolist(), out["status"].tolist()))
    dist.destroy_process_group()


def test_gather_per_patient_world3():
    """Per-patient arrays of unequal shards come back in global-id order."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gather_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, tir, st in res:
        assert tir == [i * 0.5 for i in range(11)] and st == [i % 3 for i in range(11)]


def _bench_line(*extra):
    import json
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--dry-run", "--steps", "4", "--warmup", "1",
                          *extra], capture_output=True, text=True, timeout=300, env=env, cwd=repo)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout       # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_spawns_ranks_for_gpus_n():
    """bench.py --gpus 2 outside torchrun re-launches itself as 2 ranks
    (torch.distributed.run, 127.0.0.1 rendezvous); the plumbing runs on CPU
    with gloo under --dry-run: one JSON line, n_gpus 2, global-id shards
    tiling the population, whole-job value (2 shards over the max rank time)."""
    one = _bench_line()
    two = _bench_line("--gpus", "2")
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["shards"] == [[0, 100000], [100000, 200000]]
    assert two["trial1m_shards"] == [[0, 500000], [500000, 1000000]]
    assert two["value"] > 1.5 * one["value"]
