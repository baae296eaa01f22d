"""GPU parity: the CUDA path (through the C ABI) equals the oracle bit for bit
on every event record, counter and state view, for the same seeded inputs.

Integer-only path: the bar is exact equality (no tolerance)."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2605_24259_b200 import gen
from paper_2605_24259_b200.gen import litmus
from parity_util import assert_parity, oracle_hist, run_gpu, run_ref

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_24259_b200 import build
    build.build()


def test_paper_litmus_parity_and_json():
    cfgs, ops, _ = litmus.paper_litmus()
    g = run_gpu(cfgs, ops, N=80)
    o = run_ref(cfgs, ops, N=80)
    assert_parity(g, o, what="c1")
    ev = g["events"]
    ref = ev[(ev["trace"] == 0) & (ev["type"] == orc.E_ACTIVE_REFUSED)][0]
    rendered = orc.render_refusal_json(ref, {0: "active"}, {0: "claim:resident"})
    assert rendered == json.load(open(os.path.join(GOLD, "refusal_event_P1069.json")))


def test_litmus_suite_parity():
    cfgs, ops, params = litmus.suite(range(1000))
    g = run_gpu(cfgs, ops, N=1024)
    o = run_ref(cfgs, ops, N=1024)
    assert_parity(g, o, what="c2")
    assert (g["hist"] == oracle_hist(o, ops.shape[0])).all()


def test_capacity_sweep_parity():
    cfgs, ops, _ = litmus.capacity_sweep(60, 70, range(60, 136))
    g = run_gpu(cfgs, ops, N=135)
    o = run_ref(cfgs, ops, N=135)
    assert_parity(g, o, what="sweep")


@pytest.mark.parametrize("N", [64, 100, 200, 333, 500, 1000, 1024, 1500, 3000])
def test_random_pool_sizes(N):
    """Every kernel instantiation (register-cached VPL=1/2/4/8 and streaming)
    and ragged pool sizes (U not a multiple of 4, 32 or 128)."""
    cfgs, ops = gen.random_traces(3, seed=100 + N, trace_begin=0, n_traces=300, T=160, N=N)
    rng = np.random.default_rng(N)
    cfgs["U"] = rng.integers(max(1, N // 2), N + 1, size=len(cfgs))
    g = run_gpu(cfgs, ops, N=N)
    o = run_ref(cfgs, ops, N=N)
    assert_parity(g, o, what=f"N={N}")


def test_random_c3_parity_2000_traces():
    cfgs, ops = gen.random_traces(3, seed=1, trace_begin=0, n_traces=2000, T=256, N=1024)
    g = run_gpu(cfgs, ops, N=1024)
    o = run_ref(cfgs, ops, N=1024)
    assert_parity(g, o, what="c3")
    assert (g["hist"] == oracle_hist(o, 256)).all()


def test_small_slot_limits_and_claim_slots_32():
    cfgs, ops = gen.random_traces(3, seed=9, trace_begin=0, n_traces=500, T=200, N=256,
                                  C=32, Q=32, O=128)
    g = run_gpu(cfgs, ops, N=256, C=32, Q=32, O=128)
    o = run_ref(cfgs, ops, N=256, C=32, Q=32, O=128)
    assert_parity(g, o, what="C32")


@pytest.mark.parametrize("N", [256, 1536])
def test_slot_stress_parity_all_slots(N):
    """Recipe 7 (slot stress) on the o128 builds (small pools: keys staged in
    shared memory; N > 1024: the crew kernel): claim slots up to 31, request
    slots up to 31, object slots up to 127, refusals whose blocking masks carry
    claim slots >= 16 (ballot masks, emit_lanes, mark_reclass_lanes on the
    upper claim lanes)."""
    cfgs, ops = gen.random_traces(7, seed=31 + N, trace_begin=0, n_traces=400, T=400, N=N,
                                  C=32, Q=32, O=128)
    k = ops["kind"]
    assert ops["a"][k == gen.SUBMIT].max() == 31
    assert ops["a"][(k == gen.ADMIT) | (k == gen.ADVANCE)].max() == 31
    assert max(ops["a"][k == gen.INSERT].max(), ops["b"][k == gen.ADMIT].max(),
               ops["b"][k == gen.SUBMIT].max()) >= 120
    if N > 1024:     # big pools: usable sizes well below N keep the pressure on
        cfgs["U"] = np.random.default_rng(N).integers(N // 6, N // 2, size=len(cfgs))
    g = run_gpu(cfgs, ops, N=N, C=32, Q=32, O=128)
    o = run_ref(cfgs, ops, N=N, C=32, Q=32, O=128)
    assert_parity(g, o, what=f"slot stress N={N}")
    ev = g["events"]
    masks = ev["mask"][np.isin(ev["type"], [7, 8, 9])]
    assert int(((masks >> 16) != 0).sum()) > 0
    assert (g["requests"]["status"][:, 16:] != 0).any()
    assert (g["claims"]["state"][:, 16:] != 0).any()
    assert (g["objects"]["live"][:, 64:] != 0).any()


def test_c4_full_length_parity():
    """BASELINE configs[3] shape at full length: 32 traces x 1024 steps on
    65536-block pools (the bench's c4 launch configuration: crew kernel, o128
    build), with usable sizes drawn from [12000, 65536] so that refusals,
    deferrals, insert refusals and harms occur at this size."""
    cfgs, ops = gen.random_traces(4, seed=2, trace_begin=0, n_traces=32, T=1024, N=65536,
                                  C=16, Q=16, O=128)
    rng = np.random.default_rng(5)
    cfgs["U"] = rng.integers(12000, 65537, size=len(cfgs))
    g = run_gpu(cfgs, ops, N=65536, O=128)
    o = run_ref(cfgs, ops, N=65536, O=128, nthreads=16)
    assert_parity(g, o, what="c4 full length")
    t = np.bincount(g["events"]["type"], minlength=16)
    assert t[7] > 0 and t[8] > 0 and t[9] > 0 and t[6] > 0 and t[12] > 0


def test_c4_subset_parity():
    cfgs, ops = gen.random_traces(4, seed=2, trace_begin=0, n_traces=4, T=64, N=65536,
                                  C=16, Q=16, O=128)
    g = run_gpu(cfgs, ops, N=65536, O=128)
    o = run_ref(cfgs, ops, N=65536, O=128, nthreads=4)
    assert_parity(g, o, what="c4")


def test_host_replay_equals_device_replay():
    cfgs, ops = gen.random_traces(3, seed=4, trace_begin=0, n_traces=700, T=120, N=1024)
    g1 = run_gpu(cfgs, ops, N=1024, device_ops=True, views=False)
    g2 = run_gpu(cfgs, ops, N=1024, device_ops=False, views=False)
    assert g1["events"].tobytes() == g2["events"].tobytes()
    assert (g1["counters"] == g2["counters"]).all()


@pytest.mark.parametrize("recipe", [3, 6])
def test_online_staging_api_equals_replay(recipe):
    """rkc_claim_submit / rkc_request_admit / rkc_op_stage + rkc_step_batch(None)
    give the same results as the replay of the same op stream (recipe 6: the
    prefix-hit admissions go through rkc_op_stage)."""
    from paper_2605_24259_b200 import rkc
    import torch
    cfgs, ops = gen.random_traces(recipe, seed=6, trace_begin=0, n_traces=64, T=80, N=512)
    ident = 0x1234
    pool = rkc.Pool(cfgs, 512, events_per_trace=512, pool_identity=ident)
    for s in range(ops.shape[0]):
        row = ops[s]
        sub = np.nonzero(row["kind"] == gen.SUBMIT)[0]
        adm = np.nonzero(row["kind"] == gen.ADMIT)[0]
        oth = np.nonzero((row["kind"] != gen.SUBMIT) & (row["kind"] != gen.ADMIT) & (row["kind"] != 0))[0]
        if len(sub):
            ci = np.zeros(len(sub), dtype=rkc.CLAIM_INPUT)
            ci["trace"] = sub
            ci["claim_slot"] = row["a"][sub]
            ci["object_slot"] = row["b"][sub]
            ci["mode"] = row["c"][sub] & 0x7F
            ci["footprint_blocks"], ci["required_leading_blocks"] = row["x"][sub], row["y"][sub]
            ci["duration_steps"] = row["z"][sub]
            ci["cache_identity"] = np.where(row["c"][sub] & 0x80, ident + 1, ident)
            if s % 2:
                pool.rkc_claim_submit(torch.from_numpy(ci.view(np.uint8).copy()).cuda())
            else:
                pool.rkc_claim_submit(ci)
        if len(adm):
            ri = np.zeros(len(adm), dtype=rkc.REQUEST_INPUT)
            ri["trace"] = adm
            ri["request_slot"], ri["target_object"], ri["write_admit"] = \
                row["a"][adm], row["b"][adm], row["c"][adm]
            ri["prompt_tokens"], ri["chunk_tokens"], ri["decode_tokens"] = \
                row["x"][adm], row["y"][adm], row["z"][adm]
            pool.rkc_request_admit(ri)
        if len(oth):
            to = np.zeros(len(oth), dtype=rkc.TRACE_OP)
            to["trace"] = oth
            for f in ("kind", "a", "b", "c", "x", "y", "z"):
                to[f] = row[f][oth]
            if s % 2:
                pool.rkc_op_stage(torch.from_numpy(to.view(np.uint8).copy()).cuda())
            else:
                pool.rkc_op_stage(to)
        pool.rkc_step_batch()
    torch.cuda.synchronize()
    counters, events, _ = pool.read_all()
    o = run_ref(cfgs, ops, N=512, views=False)
    assert events.tobytes() == o["events"].tobytes()
    assert (counters == o["counters"]).all()
    assert pool.rkc_staging_conflicts() == 0


def test_staging_conflict_rejected_on_host():
    from paper_2605_24259_b200 import rkc
    cfgs, _ = gen.random_traces(3, seed=0, trace_begin=0, n_traces=4, T=1, N=128)
    pool = rkc.Pool(cfgs, 128)
    to = np.zeros(2, dtype=rkc.TRACE_OP)
    to["trace"] = [1, 1]
    to["kind"] = gen.TOUCH
    with pytest.raises(rkc.RkcError) as e:
        pool.rkc_op_stage(to)
    assert e.value.status == rkc.RKC_E_INVAL


def test_telemetry_overflow_lost_and_drain():
    from paper_2605_24259_b200 import rkc
    cfgs, ops = gen.random_traces(3, seed=8, trace_begin=0, n_traces=50, T=100, N=256)
    g = run_gpu(cfgs, ops, N=256, views=False)
    pool = g["pool"]
    _, total = pool.rkc_telemetry_read()
    small = np.zeros(max(0, total - 1), dtype=rkc.EVENT)
    with pytest.raises(rkc.RkcError) as e:
        pool.rkc_telemetry_read(events_out=small)
    assert e.value.status == rkc.RKC_E_OVERFLOW
    # drain empties the buffers
    full = np.zeros(total, dtype=rkc.EVENT)
    pool.rkc_telemetry_read(events_out=full, drain=True)
    _, after = pool.rkc_telemetry_read()
    assert after == 0
    # a tiny per-trace buffer loses events and says so
    p2 = rkc.Pool(cfgs, 256, events_per_trace=4)
    import torch
    p2.rkc_step_batch(torch.from_numpy(ops.view(np.uint8).reshape(-1)).cuda(), ops.shape[0])
    st, n = p2.rkc_telemetry_read(allow_lost=True)
    assert st == rkc.RKC_E_LOST and n <= 4 * len(cfgs)
    counters = np.zeros((len(cfgs), 32), dtype=np.uint32)
    p2.rkc_telemetry_read(counters_out=counters, allow_lost=True)
    assert counters[:, 27].sum() == g["counters"][:, 27].sum()   # emitted totals still exact


def test_L6_state_injection_on_gpu():
    """L6: positions 1..59 cached, 0 missing -> leading 0; the
    claim is accepted and never materializes; probe unsatisfied."""
    from paper_2605_24259_b200 import rkc
    from paper_2605_24259_b200.gen import HARD, SUBMIT, TOUCH, make_cfg, op, pack_ops
    cfgs = np.stack([make_cfg(80)])
    pool = rkc.Pool(cfgs, 80)
    st = pool.rkc_state_export()
    blocks, objs = st["blocks"], st["objects"]
    for p in range(1, 60):
        blocks[0, p] = (1, 0, 0, p, 1000 - p)
    objs[0]["claim"] = 0xFF
    objs[0, 0]["live"], objs[0, 0]["len"] = 1, 60
    hdr = st["header"].copy()
    hdr[0]["seq_ctr"] = 2000
    pool.rkc_state_import(0, hdr, blocks, st["claims"], st["requests"], objs)
    ops = pack_ops([[op(SUBMIT, 0, 0, HARD, 60, 60, 0), op(TOUCH, 0)]])
    pool.rkc_step_batch(ops, 2)
    counters, events, _ = pool.read_all()
    st2 = pool.rkc_state_export()
    assert st2["objects"][0, 0]["leading"] == 0
    assert int((st2["blocks"][0]["res"] == 1).sum()) == 59
    assert st2["claims"][0, 0]["state"] == 1
    probe = events[events["type"] == 13][0]
    assert probe["f"][1] == 0 and probe["reason"] == 0
    # and the oracle agrees on the same injected state
    b = orc.OracleBatch(cfgs, 80)
    ob = b.export(0)
    ob["blocks"][:] = blocks[0]
    ob["objects"][:] = objs[0]
    b.import_(0, 2000, 0, ob["blocks"], ob["claims"], ob["requests"], ob["objects"])
    b.run(ops)
    assert b.events().tobytes() == events.tobytes()


def test_full_size_c3_sampled_parity():
    """BASELINE configs[2] at full size (100k traces x 256 steps, the bench
    launch configuration): a random sample of traces equals the oracle run
    on just those traces (traces are independent)."""
    import torch
    from paper_2605_24259_b200 import rkc
    n, T = 100_000, 256
    cfgs, ops = gen.random_traces(3, seed=0, trace_begin=0, n_traces=n, T=T, N=1024)
    pool = rkc.Pool(cfgs, 1024, events_per_trace=512)
    pool.rkc_step_batch(torch.from_numpy(ops.view(np.uint8).reshape(-1)).cuda(), T)
    torch.cuda.synchronize()
    counters, events, hist = pool.read_all()
    rng = np.random.default_rng(123)
    sample = np.sort(rng.choice(n, size=300, replace=False))
    sub_ops = np.ascontiguousarray(ops[:, sample])
    o = run_ref(cfgs[sample], sub_ops, N=1024, views=False)
    assert (counters[sample] == o["counters"]).all()
    idx = np.searchsorted(events["trace"], np.arange(n + 1))
    ge = np.concatenate([events[idx[t]:idx[t + 1]] for t in sample])
    oe = o["events"].copy()
    oe["trace"] = sample[oe["trace"]]
    assert ge.tobytes() == oe.tobytes()
    # whole-run invariants that hold at any size
    assert hist[48 + 26] == n * T                      # steps
    assert hist[48 + 0] == int((ops["kind"] != 0).sum())  # ops = non-NOP records
    assert (counters[:, 27] <= 512).all()


def test_histogram_shard_invariance():
    """Sum of per-shard histograms = histogram of the whole run (the
    multi-GPU allreduce contract)."""
    cfgs, ops = gen.random_traces(3, seed=12, trace_begin=0, n_traces=1000, T=128, N=1024)
    whole = run_gpu(cfgs, ops, N=1024, views=False)["hist"]
    a = run_gpu(cfgs[:400], np.ascontiguousarray(ops[:, :400]), N=1024, views=False)["hist"]
    b = run_gpu(cfgs[400:], np.ascontiguousarray(ops[:, 400:]), N=1024, views=False)["hist"]
    steps = 48 + 26
    s = a + b
    assert (np.delete(s, steps) == np.delete(whole, steps)).all()
    assert s[steps] == whole[steps]


def test_reserve_admission_parity():
    """NEXT f4 (resident-reserve admission, G34): the c8 recipe (c3 with
    admit_check = RESERVE on 40 % of the traces) and the hand-built reserve
    cases of tests/test_oracle_reserve.py, GPU = oracle bit for bit."""
    from paper_2605_24259_b200.gen import (ADMIT, ADMIT_RESERVE, ADVANCE, CONTRACT, DEMOTE, HARD,
                                           HIT_ADMIT, INSERT, SUBMIT, make_cfg, op, pack_ops)
    cfgs, ops = gen.random_traces(8, seed=17, trace_begin=0, n_traces=2000, T=256, N=1024)
    g = run_gpu(cfgs, ops, N=1024)
    o = run_ref(cfgs, ops, N=1024)
    assert_parity(g, o, what="c8")
    ev = g["events"]
    assert ((ev["type"] == orc.E_ACTIVE_REFUSED) & (ev["reason"] == orc.WHY_RESIDENT_RESERVE)).sum() > 0
    lists = [
        [op(INSERT, 0, x=40), op(SUBMIT, 0, 0, HARD, 60, 40, 0), op(ADMIT, 0, 1, 0, 656, 656, 0)],
        [op(SUBMIT, 0, 0, HARD, 60, 60, 0), op(ADMIT, 0, 1, 0, 1120, 1120, 0), op(ADVANCE, 0),
         op(INSERT, 0, x=60)],
        [op(SUBMIT, 0, 0, HARD, 50, 1, 0), op(ADMIT, 0, 1, 0, 640, 640, 0), op(DEMOTE, 0),
         op(ADVANCE, 0)],
        [op(INSERT, 0, x=30), op(SUBMIT, 0, 0, HARD, 30, 30, 0),
         op(HIT_ADMIT, 0, 0, 0, 16 * 60, 64, 0), op(ADVANCE, 0)],
    ]
    cf = np.stack([make_cfg(100, CONTRACT, ADMIT_RESERVE), make_cfg(80, CONTRACT, ADMIT_RESERVE),
                   make_cfg(80, CONTRACT, ADMIT_RESERVE, defer_budget=1),
                   make_cfg(80, CONTRACT, ADMIT_RESERVE)])
    ops2 = pack_ops(lists)
    assert_parity(run_gpu(cf, ops2, N=100), run_ref(cf, ops2, N=100), what="reserve cases")
