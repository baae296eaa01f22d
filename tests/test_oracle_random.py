"""Oracle on random c3/c4-recipe traces: invariants I1-I9 hold at full pool
size, runs are deterministic, and results do not depend on the thread count
or on which trace range a worker generated (the counter-based generator)."""
import numpy as np

from oracle import oracle as orc
from paper_2605_24259_b200 import gen


def test_random_c3_invariants():
    cfgs, ops = gen.random_traces(3, seed=7, trace_begin=0, n_traces=24, T=256, N=1024)
    b = orc.OracleBatch(cfgs, N=1024)
    assert b.run(ops, nthreads=8, check=True) == 0
    ctr = b.counters().astype(np.int64).sum(0)
    # the workload exercises every lifecycle path (sanity of the recipe)
    for name in ("accepted", "materialized", "victims_ordinary", "served", "reuse_probes",
                 "blocks_allocated"):
        assert ctr[orc.K[name]] > 0, name
    # contract traces never harm an obligated claim (I4)
    per = b.counters()
    for i in range(len(cfgs)):
        if cfgs[i]["lowering"] == 0:
            assert per[i][orc.K["harmed_obligated"]] == 0


def test_generator_is_counter_based():
    a_cfg, a_ops = gen.random_traces(3, seed=11, trace_begin=0, n_traces=64, T=64, N=1024, nthreads=1)
    b_cfg, b_ops = gen.random_traces(3, seed=11, trace_begin=32, n_traces=32, T=64, N=1024, nthreads=8)
    assert a_cfg[32:].tobytes() == b_cfg.tobytes()
    assert np.ascontiguousarray(a_ops[:, 32:]).tobytes() == b_ops.tobytes()


def test_oracle_deterministic_and_thread_independent():
    cfgs, ops = gen.random_traces(3, seed=3, trace_begin=0, n_traces=48, T=128, N=1024)
    b1 = orc.OracleBatch(cfgs, N=1024)
    b1.run(ops, nthreads=1)
    b2 = orc.OracleBatch(cfgs, N=1024)
    b2.run(ops, nthreads=8)
    assert b1.events().tobytes() == b2.events().tobytes()
    assert b1.counters().tobytes() == b2.counters().tobytes()


def test_trace_offset_equals_subset():
    """Running traces [16,32) from the full op matrix equals generating them alone."""
    cfgs, ops = gen.random_traces(3, seed=5, trace_begin=0, n_traces=32, T=96, N=1024)
    full = orc.OracleBatch(cfgs, N=1024)
    full.run(ops)
    part = orc.OracleBatch(cfgs[16:], N=1024)
    part.run(ops, trace_offset=16)
    assert (full.counters()[16:] == part.counters()).all()


def test_random_c4_small_sample_invariants():
    cfgs, ops = gen.random_traces(4, seed=1, trace_begin=0, n_traces=2, T=96, N=65536,
                                  C=16, Q=16, O=128)
    b = orc.OracleBatch(cfgs, N=65536, C=16, Q=16, O=128)
    assert b.run(ops, nthreads=2, check=False) == 0
    assert b.counters().sum() > 0


def test_random_c6_prefix_hit_invariants():
    """c6 = c3 + prefix hits (NEXT f3): I1-I10 hold with pins in play (I10:
    a pinned prefix is always fully present) and hits actually pin blocks."""
    cfgs, ops = gen.random_traces(6, seed=7, trace_begin=0, n_traces=24, T=256, N=1024)
    b = orc.OracleBatch(cfgs, N=1024)
    assert b.run(ops, nthreads=8, check=True) == 0
    ctr = b.counters().astype(np.int64).sum(0)
    assert ctr[orc.K["prefix_hits"]] > 0 and ctr[orc.K["hit_tokens"]] > 0
    per = b.counters()
    for i in range(len(cfgs)):
        if cfgs[i]["lowering"] == 0:
            assert per[i][orc.K["harmed_obligated"]] == 0
