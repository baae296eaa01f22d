"""Replay one bench shard (c5 recipe, traces [first, first + n)) in its own pool on one GPU and
report the C-ABI status of the replay and the telemetry read (debugging multi-rank runs)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--first", type=int, default=500000)
    ap.add_argument("--n", type=int, default=500000)
    ap.add_argument("--steps", type=int, default=256)
    a = ap.parse_args()
    import torch
    from paper_2605_24259_b200 import gen, rkc
    cfgs, ops = gen.random_traces(3, 0, a.first, a.n, a.steps, 1024, 16, 16, 64)
    d = torch.from_numpy(ops.view(np.uint8).reshape(-1)).cuda()
    ept = 512
    pool = rkc.Pool(cfgs, 1024, 16, 16, 64, events_per_trace=ept)
    ev = torch.empty(a.n * ept * 32, dtype=torch.uint8, device="cuda")
    hist = torch.zeros(rkc.RKC_NHIST, dtype=torch.int64, device="cuda")
    for rep in range(2):
        pool.rkc_pool_reset()
        pool.rkc_step_batch(d, a.steps)
        try:
            torch.cuda.synchronize()
            print("replay", rep, "sync ok")
        except Exception as e:  # noqa: BLE001
            print("replay", rep, "sync failed:", e)
            return 1
        try:
            st = pool.rkc_telemetry_read(events_out=ev, hist_out=hist)
            print("telemetry", st, hist[:8].tolist())
        except Exception as e:  # noqa: BLE001
            print("telemetry failed:", e)
            return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
