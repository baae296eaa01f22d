"""bench.py's own multi-rank code path on CPU (gloo, world size 2).

1. `python bench.py --gpus 2` without a launcher re-runs itself under torchrun
   with two ranks (rendezvous on 127.0.0.1); rank 0 alone prints one JSON
   line, the other rank exits 0 (here with the reference arm, which needs no
   GPU).
2. bench.shard() + the histogram SUM allreduce bench.py performs
   (shard.allreduce_histogram): every rank replays its own trace range of a
   strong-scaling workload (c5 layout, shrunk), and the allreduced outcome
   histogram equals the single-process histogram of all traces.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOTAL, T, N = 90, 48, 256


def test_bench_without_launcher_spawns_two_ranks():
    env = {**os.environ, "PYTHONPATH": ROOT}
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "0", "--config", "c3"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["impl"] == "reference" and out["n_gpus"] == 2 and out["value"] > 0
    assert out["config"]["parallelism"] == "trace-sharded x2"


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    import bench
    from paper_2605_24259_b200 import gen
    from paper_2605_24259_b200.shard import allreduce_histogram
    from parity_util import oracle_hist, run_ref
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bench.select_workload("c5")
    bench.WL = dict(bench.WL, traces=TOTAL)                 # c5's strong-scaling split, shrunk
    first, n = bench.shard(rank, world)
    cfgs, ops = gen.random_traces(3, bench.SEED, first, n, T, N)
    h = torch.from_numpy(oracle_hist(run_ref(cfgs, ops, N=N, nthreads=2), T))
    allreduce_histogram(h)
    if rank == 0:
        q.put((h.numpy().tolist(), [bench.shard(r, world) for r in range(world)]))
    dist.barrier()
    dist.destroy_process_group()


def test_bench_shard_and_histogram_allreduce_gloo():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, shards = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert shards == [(0, 45), (45, 45)]
    from paper_2605_24259_b200 import gen
    from parity_util import oracle_hist, run_ref
    cfgs, ops = gen.random_traces(3, 0, 0, TOTAL, T, N)
    whole = oracle_hist(run_ref(cfgs, ops, N=N, nthreads=2), T)
    assert (np.array(got, dtype=np.int64) == whole).all()
