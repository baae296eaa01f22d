"""Profiling driver: one c3 replay through the C ABI (for ncu launch lists and
--set full captures; never used for bench numbers)."""
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
    ap.add_argument("--replays", type=int, default=1)
    a = ap.parse_args()
    import torch
    from paper_2605_24259_b200 import build, gen
    build.build()
    from paper_2605_24259_b200 import rkc
    cfgs, ops = gen.random_traces(a.config, 0, 0, a.traces, a.steps, a.blocks, 16, 16, a.objects)
    d = torch.from_numpy(ops.view(np.uint8).reshape(-1)).cuda()
    pool = rkc.Pool(cfgs, a.blocks, 16, 16, a.objects, events_per_trace=max(64, 2 * a.steps + 64))
    ev = torch.empty(a.traces * max(64, 2 * a.steps + 64) * 32, dtype=torch.uint8, device="cuda")
    hist = torch.zeros(128, dtype=torch.int64, device="cuda")
    for _ in range(a.replays):
        pool.rkc_pool_reset()
        pool.rkc_step_batch(d, a.steps)
        pool.rkc_telemetry_read(events_out=ev, hist_out=hist)
    torch.cuda.synchronize()
    print("hist[48:56]", hist[48:56].tolist())


if __name__ == "__main__":
    main()
