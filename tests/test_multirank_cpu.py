"""Multi-rank host logic on CPU (gloo, world size 2): each rank generates its
own trace shard from the counter-based generator, computes its outcome
histogram (here with the oracle; on GPUs with K3), and the one SUM allreduce
yields exactly the single-process histogram of all traces."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_24259_b200.shard import allreduce_histogram, shard_range, weak_range

TOTAL, T, N = 96, 64, 256


def _hist(cfgs, ops):
    from parity_util import oracle_hist, run_ref
    ref = run_ref(cfgs, ops, N=N, nthreads=2)
    return oracle_hist(ref, ops.shape[0])


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_24259_b200 import gen
    b, e = shard_range(rank, world, TOTAL)
    cfgs, ops = gen.random_traces(3, 5, b, e - b, T, N)
    h = torch.from_numpy(_hist(cfgs, ops))
    allreduce_histogram(h)
    if rank == 0:
        out.put(h.numpy().tolist())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges_partition():
    for world in (1, 2, 3, 4, 8):
        for total in (0, 1, 7, 100, 1_000_000):
            rs = [shard_range(r, world, total) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in rs]
            assert max(sizes) - min(sizes) <= 1
    assert weak_range(3, 100_000) == (300_000, 400_000)


def test_gloo_world2_histogram_allreduce_equals_single_process():
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = np.array(q.get(timeout=300), dtype=np.int64)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from paper_2605_24259_b200 import gen
    cfgs, ops = gen.random_traces(3, 5, 0, TOTAL, T, N)
    whole = _hist(cfgs, ops)
    assert (got == whole).all()
