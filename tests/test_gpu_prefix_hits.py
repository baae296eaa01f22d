"""GPU parity of the prefix-hit extension (G28-G30).

The CUDA path (through the C ABI) equals the oracle bit for bit -- every
event record, counter and state view (incl. the request's `hit` word and the
header's A, which counts pinned blocks once) -- on hit litmus traces, on
random c6 traces (c3 + prefix hits) at several pool sizes, on a 128-object
build, and on the big-pool build.  Integer path: exact equality."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2605_24259_b200 import gen
from paper_2605_24259_b200.gen import (ADVANCE, COMPLETE, CONTRACT, HARD, HIT_ADMIT, INSERT, NATIVE,
                                       NONE, PEAK, SUBMIT, TOUCH, ADMIT, make_cfg, op, pack_ops)
from parity_util import assert_parity, oracle_hist, run_gpu, run_ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_24259_b200 import build
    build.build()


def _litmus():
    """The hit closed-form templates of tests/test_oracle_prefix_hits.py, one trace each."""
    traces, cfgs = [], []
    rng = np.random.default_rng(0)
    for _ in range(200):
        R = int(rng.integers(1, 100)); A = int(rng.integers(1, 120))
        U = int(rng.integers(R, R + A + 10))
        cfgs.append(make_cfg(U, CONTRACT, PEAK, defer_budget=int(rng.integers(0, 2))))
        traces.append([op(INSERT, 0, x=R), op(SUBMIT, 0, 0, HARD, R, R, 0),
                       op(HIT_ADMIT, 0, 0, 0, 16 * A, 16 * A, 0), op(ADVANCE, 0), op(ADVANCE, 0),
                       op(COMPLETE, 0), op(TOUCH, 0)])
    for _ in range(200):
        U = int(rng.integers(4, 200)); R = int(rng.integers(1, U + 1)); A = int(rng.integers(1, U + 1))
        cfgs.append(make_cfg(U, NATIVE, NONE))
        traces.append([op(INSERT, 0, x=R), op(HIT_ADMIT, 0, 0, 0, 16 * A, 16 * A, 0),
                       op(ADVANCE, 0), op(TOUCH, 0), op(HIT_ADMIT, 1, 0, 0, 16 * A + 3, 48, 5),
                       op(ADMIT, 2, 1, 1, 16 * (U // 2), 64, 0), op(ADVANCE, 2), op(COMPLETE, 0),
                       op(ADVANCE, 1), op(COMPLETE, 1), op(TOUCH, 0)])
    from paper_2605_24259_b200.gen import DEMOTABLE
    for _ in range(100):  # auto-demotion inside the hit's PEAK check, then the backstop (G29)
        R = int(rng.integers(2, 80)); A = int(rng.integers(R + 1, 140))
        U = int(rng.integers(A - R + 1, R + A + 5))
        cfgs.append(make_cfg(U, CONTRACT, PEAK, defer_budget=int(rng.integers(0, 2)), auto_demote=1))
        traces.append([op(INSERT, 0, x=R), op(SUBMIT, 0, 0, DEMOTABLE, R, R, 0),
                       op(HIT_ADMIT, 0, 0, 0, 16 * A, 16 * A, 0), op(ADVANCE, 0), op(ADVANCE, 0),
                       op(COMPLETE, 0), op(TOUCH, 0)])
    return np.stack(cfgs), pack_ops(traces)


def test_hit_litmus_parity():
    cfgs, ops = _litmus()
    g = run_gpu(cfgs, ops, N=256)
    o = run_ref(cfgs, ops, N=256)
    assert_parity(g, o, what="hit litmus")
    assert (g["hist"] == oracle_hist(o, ops.shape[0])).all()
    assert g["counters"][:, orc.K["prefix_hits"]].sum() > 300


@pytest.mark.parametrize("N", [128, 333, 1024, 2000])
def test_random_c6_parity(N):
    cfgs, ops = gen.random_traces(6, seed=600 + N, trace_begin=0, n_traces=1000, T=256, N=N)
    rng = np.random.default_rng(N)
    cfgs["U"] = rng.integers(max(1, N // 2), N + 1, size=len(cfgs))
    g = run_gpu(cfgs, ops, N=N)
    o = run_ref(cfgs, ops, N=N)
    assert_parity(g, o, what=f"c6 N={N}")
    assert (g["hist"] == oracle_hist(o, 256)).all()
    assert g["counters"][:, orc.K["hit_tokens"]].sum() > 0
    assert (g["header"]["alive"] == o["header"]["alive"]).all()


def test_c6_slot_limits_o128():
    cfgs, ops = gen.random_traces(6, seed=61, trace_begin=0, n_traces=400, T=200, N=256,
                                  C=32, Q=32, O=128)
    g = run_gpu(cfgs, ops, N=256, C=32, Q=32, O=128)
    o = run_ref(cfgs, ops, N=256, C=32, Q=32, O=128)
    assert_parity(g, o, what="c6 O128")


def test_c6_big_pool_parity():
    """The crew build (N > 1024): pins streamed by the leader warp."""
    cfgs, ops = gen.random_traces(6, seed=62, trace_begin=0, n_traces=64, T=160, N=4096)
    g = run_gpu(cfgs, ops, N=4096)
    o = run_ref(cfgs, ops, N=4096)
    assert_parity(g, o, what="c6 big")


def test_state_injection_with_pins():
    """Import a mid-run c6 state (running hit requests, pinned blocks) into a
    fresh pool; continuing on the GPU equals continuing in the oracle."""
    from paper_2605_24259_b200 import rkc
    import torch
    cfgs, ops = gen.random_traces(6, seed=63, trace_begin=0, n_traces=200, T=200, N=512)
    g = run_gpu(cfgs, np.ascontiguousarray(ops[:100]), N=512)
    assert (g["requests"]["hit"] > 0).any()
    pool = rkc.Pool(cfgs, 512, events_per_trace=1024)
    hdr = g["header"].copy()
    pool.rkc_state_import(0, hdr, g["blocks"], g["claims"], g["requests"], g["objects"])
    pool.rkc_state_set_step(100)
    rest = np.ascontiguousarray(ops[100:])
    pool.rkc_step_batch(torch.from_numpy(rest.view(np.uint8).reshape(-1)).cuda(), rest.shape[0])
    torch.cuda.synchronize()
    counters, events, _ = pool.read_all()
    o = run_ref(cfgs, ops, N=512, views=False)
    oe = o["events"][o["events"]["step"] >= 100]
    assert events.tobytes() == oe.tobytes()
