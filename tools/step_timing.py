"""A/B timing of one c3 replay (256 lockstep steps) through the C ABI, for
kernel experiments (never a bench number: no clocks check, no L2 flush).

usage: python tools/step_timing.py [--nop] [--reps 5] [--tag name]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--traces", type=int, default=100_000)
    ap.add_argument("--steps", type=int, default=256)
    ap.add_argument("--blocks", type=int, default=1024)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--objects", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--nop", action="store_true", help="all-NOP op stream (launch floor)")
    ap.add_argument("--tag", default="")
    ap.add_argument("--per-step", action="store_true", help="time every lockstep step separately")
    a = ap.parse_args()
    import torch
    from paper_2605_24259_b200 import gen, rkc
    cfgs, ops = gen.random_traces(a.config, 0, 0, a.traces, a.steps, a.blocks, 16, 16, a.objects)
    if a.nop:
        ops[:] = np.zeros((), dtype=ops.dtype)
    non_nop = int((ops["kind"] != 0).sum())
    d = torch.from_numpy(ops.view(np.uint8).reshape(-1)).cuda()
    ept = max(64, 2 * a.steps + 64)
    pool = rkc.Pool(cfgs, a.blocks, 16, 16, a.objects, events_per_trace=ept)
    ts = []
    for r in range(a.reps + 1):
        pool.rkc_pool_reset()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pool.rkc_step_batch(d, a.steps)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    if a.per_step:  # one more replay, one rkc_step_batch call and one event pair per step
        pool.rkc_pool_reset()
        torch.cuda.synchronize()
        row = a.traces * 16
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
        evs[0].record()
        for st in range(a.steps):
            pool.rkc_step_batch(d[st * row:(st + 1) * row], 1)
            evs[st + 1].record()
        torch.cuda.synchronize()
        us = [1000 * evs[i].elapsed_time(evs[i + 1]) for i in range(a.steps)]
        print(f"{a.tag:16s} per-step us: " + " ".join(f"{i}:{us[i]:.0f}" for i in range(0, a.steps, 16)) +
              f"  sum {sum(us) / 1000:.2f} ms")
    ctr = torch.zeros(a.traces * 32, dtype=torch.int32, device="cuda")
    pool.rkc_telemetry_read(counters_out=ctr)
    w = torch.arange(1, a.traces * 32 + 1, device="cuda", dtype=torch.int64) % 1000003
    chk = int((ctr.to(torch.int64) * w).sum().item())
    print(f"{a.tag:16s} replay_ms {ms:8.3f} step_us {1000 * ms / a.steps:7.1f} "
          f"events/s {non_nop / ms * 1e3:.4e} ctrsum {chk}")


if __name__ == "__main__":
    main()
