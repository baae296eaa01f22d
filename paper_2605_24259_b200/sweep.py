"""the paper's capacity sweep as one
GPU batch.  Every (resident R, active A, usable U, policy) cell is one trace
of the litmus capacity-sweep recipe, all replayed together through the C ABI;
the outcome of each cell (active served / refused, resident preserved) is
read back from its claim-level telemetry.  "Hard resident exclusion preserves
the accepted resident claim and converts infeasible active/resident
coexistence into scheduler-visible refusal. At and above R + A usable blocks,
active and resident KV can coexist".

  python -m paper_2605_24259_b200.sweep [--resident 60 --active 70 --umin 75 --umax 135]
"""
from __future__ import annotations

import argparse

import numpy as np

from .gen import litmus

EV_REFUSED, EV_SERVED, EV_REUSE_PROBE = 8, 11, 13


def run_sweep(pairs, usable_for=None, device: int = 0):
    """pairs: iterable of (R, A); usable_for(R, A) -> iterable of U (default
    max(R, A) .. R + A + 10).  Returns a list of cell dicts."""
    import torch
    from . import rkc
    cfg_list, op_lists, params = [], [], []
    for R, A in pairs:
        us = list(usable_for(R, A) if usable_for else range(max(R, A), R + A + 11))
        c, o, p = litmus.capacity_sweep(R, A, us)
        cfg_list.append(c)
        for i in range(o.shape[1]):
            op_lists.append(o[:, i])
        params.extend(p)
    cfgs = np.concatenate(cfg_list)
    T = max(len(x) for x in op_lists)
    ops = np.zeros((T, len(op_lists)), dtype=op_lists[0].dtype)
    for i, x in enumerate(op_lists):
        ops[: len(x), i] = x
    N = int(cfgs["U"].max())
    pool = rkc.Pool(cfgs, N, events_per_trace=4 * T + 16, device=device)
    pool.rkc_step_batch(torch.from_numpy(np.ascontiguousarray(ops).view(np.uint8).reshape(-1))
                        .to(f"cuda:{device}"), T)
    torch.cuda.synchronize(device)
    _, ev, _ = pool.read_all()
    idx = np.searchsorted(ev["trace"], np.arange(len(params) + 1))
    cells = []
    for i, p in enumerate(params):
        e = ev[idx[i]:idx[i + 1]]
        probe = e[e["type"] == EV_REUSE_PROBE][-1]
        cells.append(dict(p, served=bool((e["type"] == EV_SERVED).any()),
                          refused=bool((e["type"] == EV_REFUSED).any()),
                          resident_kept=int(probe["f"][1]) == p["R"],
                          resident_leading=int(probe["f"][1])))
    return cells


def flip_points(cells):
    """Smallest usable size at which each (R, A, policy) serves the active
    request with the resident preserved."""
    out = {}
    for c in cells:
        key = (c["R"], c["A"], c["policy"])
        if c["served"] and c["resident_kept"]:
            out[key] = min(out.get(key, 1 << 30), c["U"])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--resident", type=int, default=60)
    ap.add_argument("--active", type=int, default=70)
    ap.add_argument("--umin", type=int, default=75)
    ap.add_argument("--umax", type=int, default=135)
    a = ap.parse_args()
    cells = run_sweep([(a.resident, a.active)], lambda R, A: range(a.umin, a.umax + 1))
    print(f"{'U':>5s} " + " ".join(f"{p:>22s}" for p in ("hard", "native", "noadmit")))
    by = {(c["U"], c["policy"]): c for c in cells}
    for U in range(a.umin, a.umax + 1):
        row = []
        for pol in ("hard", "native", "noadmit"):
            c = by.get((U, pol))
            row.append("-" if c is None else
                       f"{'served' if c['served'] else 'REFUSED'}/{'kept' if c['resident_kept'] else 'lost'}")
        print(f"{U:5d} " + " ".join(f"{r:>22s}" for r in row))
    print("flip (served with resident kept):", flip_points(cells))


if __name__ == "__main__":
    main()
