"""Helpers for GPU-vs-oracle parity tests (test infrastructure).

GPU results come only through the C ABI (paper_2605_24259_b200.rkc); oracle
results only through oracle/.  Records are compared byte for byte.
"""
import numpy as np

from oracle import oracle as orc

VIEW_KEYS = ("blocks", "claims", "requests", "objects")


def run_gpu(cfgs, ops, N, C=16, Q=16, O=64, ept=None, device_ops=True, views=True):
    import torch
    from paper_2605_24259_b200 import rkc
    T = ops.shape[0]
    if ept is None:
        ept = max(64, 4 * T + 16)
    pool = rkc.Pool(cfgs, N, C, Q, O, events_per_trace=ept)
    if T:
        if device_ops:
            d = torch.from_numpy(np.ascontiguousarray(ops).view(np.uint8).reshape(-1)).cuda()
            pool.rkc_step_batch(d, T)
        else:
            pool.rkc_step_batch(np.ascontiguousarray(ops), T)
    torch.cuda.synchronize()
    counters, events, hist = pool.read_all()
    out = dict(counters=counters, events=events, hist=hist, pool=pool)
    if views:
        out.update(pool.rkc_state_export())
    return out


def run_ref(cfgs, ops, N, C=16, Q=16, O=64, views=True, nthreads=8, trace_offset=0):
    b = orc.OracleBatch(cfgs, N, C, Q, O)
    b.run(ops, nthreads=nthreads, trace_offset=trace_offset)
    out = dict(counters=b.counters(), events=b.events(), batch=b)
    if views:
        ex = [b.export(i) for i in range(len(cfgs))]
        out["header"] = np.stack([e["header"] for e in ex])
        for k in VIEW_KEYS:
            out[k] = np.stack([e[k] for e in ex])
    return out


def oracle_hist(ref, n_steps):
    """The outcome histogram of DESIGN.md / rkc.h computed from oracle views."""
    h = np.zeros(128, dtype=np.int64)
    cl = ref["claims"]
    for st, md in zip(cl["state"].ravel(), cl["mode"].ravel()):
        if st != 0:
            h[0 + int(st) * 6 + int(md)] += 1
    for st in ref["requests"]["status"].ravel():
        if st != 0:
            h[42 + int(st)] += 1
    h[48:80] = ref["counters"].astype(np.int64).sum(0)
    return h


def first_event_mismatch(ge, oe):
    n = min(len(ge), len(oe))
    gb = ge.view(np.uint8).reshape(-1, 32)[:n]
    ob = oe.view(np.uint8).reshape(-1, 32)[:n]
    bad = np.nonzero((gb != ob).any(1))[0]
    if len(bad):
        i = int(bad[0])
        return i, ge[i], oe[i]
    if len(ge) != len(oe):
        return n, ge[n] if n < len(ge) else None, oe[n] if n < len(oe) else None
    return None


def assert_parity(g, o, views=True, what=""):
    mm = first_event_mismatch(g["events"], o["events"])
    assert mm is None, f"{what} first event mismatch at {mm[0]}: gpu={mm[1]} oracle={mm[2]}"
    assert g["events"].tobytes() == o["events"].tobytes()
    diff = np.nonzero((g["counters"] != o["counters"]).any(1))[0]
    assert len(diff) == 0, f"{what} counters differ for traces {diff[:10]}: " \
        f"gpu={g['counters'][diff[0]]} oracle={o['counters'][diff[0]]}"
    if views:
        for k in VIEW_KEYS:
            gb, ob = g[k], o[k]
            bad = np.nonzero((gb.view(np.uint8).reshape(len(gb), -1) !=
                              ob.view(np.uint8).reshape(len(ob), -1)).any(1))[0]
            assert len(bad) == 0, f"{what} {k} differ for traces {bad[:10]}"
        for f in ("seq_ctr", "free_blocks", "alive", "protected_total"):
            assert (g["header"][f] == o["header"][f]).all(), f"{what} header {f}"
