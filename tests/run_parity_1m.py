"""Bit-exact parity of the CUDA path with the oracle on 10^6 random c3 traces
(BASELINE.json north_star: "bit-exact agreement with the CPU oracle across the
full litmus suite and 10^6 random traces").  Test infrastructure, run by hand
on a GPU box (about 10 minutes with 16 host threads), not collected by pytest:

    python tests/run_parity_1m.py [--traces 1000000] [--chunk 20000] [--steps 256] [--single-pool]

Trace ids [0, traces) of the c3 recipe are replayed chunk by chunk (traces are
independent): the GPU pool through the C ABI, the oracle on the host
cores; per chunk every counter, every event record (in (trace, step, seq)
order) and the full final state (header, blocks, claims, requests, objects)
must be equal byte for byte.  Prints one line per chunk and a JSON summary.

--single-pool: the bench's own launch configuration instead -- ONE pool of all
the traces (c5: 10^6 traces, 512 events per trace, ops resident in HBM), one
256-step replay, telemetry read once; the oracle then checks it chunk by chunk.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--traces", type=int, default=1_000_000)
    ap.add_argument("--chunk", type=int, default=20_000)
    ap.add_argument("--steps", type=int, default=256)
    ap.add_argument("--blocks", type=int, default=1024)
    ap.add_argument("--config", type=int, default=3, help="generator recipe (3 = c3/c5, 6 = c6 hits)")
    ap.add_argument("--single-pool", action="store_true")
    ap.add_argument("--slots", type=int, nargs=3, default=(16, 16, 64), metavar=("C", "Q", "O"))
    ap.add_argument("--u-range", type=int, nargs=2, default=None, metavar=("LO", "HI"),
                    help="draw each trace's usable blocks from [LO, HI] (seeded) instead of N")
    a = ap.parse_args()
    import torch
    from paper_2605_24259_b200 import gen
    from parity_util import assert_parity, run_gpu, run_ref
    threads = os.cpu_count() or 1
    t0 = time.time()
    n_ev = n_ops = 0
    if a.single_pool:
        return single_pool(a, threads, t0)
    for begin in range(0, a.traces, a.chunk):
        n = min(a.chunk, a.traces - begin)
        cfgs, ops = gen.random_traces(a.config, seed=0, trace_begin=begin, n_traces=n, T=a.steps, N=a.blocks)
        g = run_gpu(cfgs, ops, N=a.blocks, ept=512)
        o = run_ref(cfgs, ops, N=a.blocks, nthreads=threads)
        assert_parity(g, o, views=True, what=f"traces [{begin}, {begin + n})")
        n_ev += len(g["events"])
        n_ops += int((ops["kind"] != 0).sum())
        del g, o
        torch.cuda.empty_cache()
        print(f"traces [{begin:7d}, {begin + n:7d}) bit-exact: counters, {n_ev} events so far, "
              f"final state ({time.time() - t0:.0f} s)", flush=True)
    print(json.dumps({"config": a.config, "traces": a.traces, "steps": a.steps, "pool_blocks": a.blocks,
                      "non_nop_ops": n_ops, "events": n_ev, "result": "bit-exact",
                      "host_threads": threads, "seconds": round(time.time() - t0, 1)}))


def single_pool(a, threads, t0):
    import torch
    from paper_2605_24259_b200 import gen, rkc
    from parity_util import VIEW_KEYS, first_event_mismatch, run_ref
    C, Q, O = a.slots
    cfgs, ops = gen.random_traces(a.config, seed=0, trace_begin=0, n_traces=a.traces, T=a.steps,
                                  N=a.blocks, C=C, Q=Q, O=O)
    if a.u_range:
        cfgs["U"] = np.random.default_rng(0).integers(a.u_range[0], a.u_range[1] + 1, size=a.traces)
    ept = max(512, 4 * a.steps + 64)
    pool = rkc.Pool(cfgs, a.blocks, C, Q, O, events_per_trace=ept)
    pool.rkc_step_batch(torch.from_numpy(ops.view(np.uint8).reshape(-1)).cuda(), a.steps)
    torch.cuda.synchronize()
    counters, events, _ = pool.read_all()
    idx = np.searchsorted(events["trace"], np.arange(a.traces + 1))
    print(f"one pool of {a.traces} traces replayed: {len(events)} events ({time.time() - t0:.0f} s)",
          flush=True)
    n_ops = 0
    for begin in range(0, a.traces, a.chunk):
        n = min(a.chunk, a.traces - begin)
        sub = np.ascontiguousarray(ops[:, begin:begin + n])
        o = run_ref(cfgs[begin:begin + n], sub, N=a.blocks, C=C, Q=Q, O=O, nthreads=threads)
        oe = o["events"]
        oe["trace"] += begin
        ge = events[idx[begin]:idx[begin + n]]
        mm = first_event_mismatch(ge, oe)
        assert mm is None, f"traces [{begin}, {begin + n}) first event mismatch at {mm}"
        assert (counters[begin:begin + n] == o["counters"]).all(), f"counters [{begin}, {begin + n})"
        g = pool.rkc_state_export(begin, n)
        for k in VIEW_KEYS:
            assert g[k].tobytes() == o[k].tobytes(), f"{k} [{begin}, {begin + n})"
        for f in ("seq_ctr", "free_blocks", "alive", "protected_total"):
            assert (g["header"][f] == o["header"][f]).all(), f"header {f}"
        n_ops += int((sub["kind"] != 0).sum())
        print(f"traces [{begin:7d}, {begin + n:7d}) bit-exact in the single pool "
              f"({time.time() - t0:.0f} s)", flush=True)
    print(json.dumps({"config": a.config, "traces": a.traces, "steps": a.steps, "pool_blocks": a.blocks,
                      "slots": [C, Q, O], "u_range": a.u_range,
                      "layout": "one pool of all traces (the bench launch configuration)",
                      "non_nop_ops": n_ops, "events": len(events), "result": "bit-exact",
                      "host_threads": threads, "seconds": round(time.time() - t0, 1)}))


if __name__ == "__main__":
    main()
