"""GPU tests of the C ABI's boundary behaviour (include/rkc.h): drained event
rings, host staging across calls, malformed state views, the device-side
materialization predicate of an injected state, the SPEC lifecycle accepted
-> harmed in the conformance checker, and the caller's current device."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2605_24259_b200 import gen
from parity_util import run_ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_24259_b200 import build
    build.build()


def _dev(ops):
    import torch
    return torch.from_numpy(np.ascontiguousarray(ops).view(np.uint8).reshape(-1)).cuda()


def test_drain_then_step_then_conformance():
    """A drained ring holds only later events: the emitted total stays exact
    (RKC_CTR_EVENTS), the events read after the drain are exactly the oracle's
    events of the later steps, and the pool conformance pass reports no
    spurious failure for drained traces (rkc.h, rkc_telemetry_read)."""
    import torch
    from paper_2605_24259_b200 import rkc
    cfgs, ops = gen.random_traces(3, seed=44, trace_begin=0, n_traces=600, T=200, N=1024)
    pool = rkc.Pool(cfgs, 1024, events_per_trace=1024)
    pool.rkc_step_batch(_dev(ops[:120]), 120)
    _, n1 = pool.rkc_telemetry_read()
    first = np.zeros(n1, dtype=rkc.EVENT)
    pool.rkc_telemetry_read(events_out=first, drain=True)
    pool.rkc_step_batch(_dev(ops[120:]), 80)
    torch.cuda.synchronize()
    counters, later, _ = pool.read_all()
    o = run_ref(cfgs, ops, N=1024, views=False)
    oe = o["events"]
    # (trace, step) order: the union of both reads, re-sorted, is the oracle stream
    both = np.concatenate([first, later])
    both = both[np.lexsort((both["seq"], both["step"], both["trace"]))]
    assert both.tobytes() == oe.tobytes()
    assert (later["step"] >= 120).all() and (first["step"] < 120).all()
    assert (counters == o["counters"]).all()             # RKC_CTR_EVENTS monotonic
    v, evd = pool.rkc_pool_conformance()
    v = v.cpu().numpy()
    assert (v == 0).all(), (np.nonzero(v)[0][:10], v[v != 0][:10])


def test_host_staging_duplicate_across_calls_rejected():
    """A second host-staged op for a trace in the same step, from another
    staging call, is RKC_E_INVAL with nothing staged; the step then runs the
    first op only."""
    from paper_2605_24259_b200 import rkc
    from paper_2605_24259_b200.gen import HARD, INSERT, TOUCH, make_cfg
    cfgs = np.stack([make_cfg(64), make_cfg(64)])
    pool = rkc.Pool(cfgs, 64)
    ci = np.zeros(1, dtype=rkc.CLAIM_INPUT)
    ci["trace"], ci["claim_slot"], ci["object_slot"], ci["mode"] = 0, 0, 0, HARD
    ci["footprint_blocks"], ci["required_leading_blocks"] = 8, 8
    pool.rkc_claim_submit(ci)
    to = np.zeros(2, dtype=rkc.TRACE_OP)
    to["trace"], to["kind"], to["a"], to["x"] = [1, 0], [INSERT, TOUCH], [0, 0], [8, 0]
    with pytest.raises(rkc.RkcError) as e:
        pool.rkc_op_stage(to)                       # trace 0 already staged by the submit
    assert e.value.status == rkc.RKC_E_INVAL
    pool.rkc_op_stage(to[:1])                       # trace 1 alone is fine
    pool.rkc_step_batch()
    _, ev, _ = pool.read_all()
    assert [int(x) for x in ev["type"]] == [orc.E_CLAIM_ACCEPTED]   # INSERT emits nothing
    st = pool.rkc_state_export()
    assert st["objects"][1, 0]["live"] == 1 and st["claims"][0, 0]["state"] == orc.C_ACCEPTED
    # the next step accepts a new op for trace 0 again
    pool.rkc_op_stage(to[1:])
    pool.rkc_step_batch()


def test_state_import_rejects_malformed_views():
    from paper_2605_24259_b200 import rkc
    from paper_2605_24259_b200.gen import make_cfg
    cfgs = np.stack([make_cfg(80)])
    pool = rkc.Pool(cfgs, 80, max_claims=4, max_objects=8)
    st = pool.rkc_state_export()
    base = {k: v.copy() for k, v in st.items()}

    def attempt(mutate):
        s = {k: v.copy() for k, v in base.items()}
        mutate(s)
        with pytest.raises(rkc.RkcError) as e:
            pool.rkc_state_import(0, s["header"], s["blocks"], s["claims"], s["requests"], s["objects"])
        assert e.value.status == rkc.RKC_E_INVAL

    def cached_owner_out_of_range(s):
        s["blocks"][0, 0] = (1, 9, 0, 0, 5)          # owner 9 >= O = 8
    attempt(cached_owner_out_of_range)

    def object_claim_out_of_range(s):
        s["objects"][0, 0]["live"], s["objects"][0, 0]["len"], s["objects"][0, 0]["claim"] = 1, 4, 6
    attempt(object_claim_out_of_range)              # claim 6 >= C = 4

    def cached_pos_beyond_len(s):
        s["objects"][0, 1]["live"], s["objects"][0, 1]["len"] = 1, 2
        s["blocks"][0, 3] = (1, 1, 0, 5, 7)
    attempt(cached_pos_beyond_len)

    def bad_state(s):
        s["claims"][0, 0]["state"] = 9
    attempt(bad_state)
    # nothing was written: the pool still equals its exported state
    after = pool.rkc_state_export()
    for k in ("blocks", "claims", "requests", "objects"):
        assert after[k].tobytes() == base[k].tobytes()


@pytest.mark.parametrize("N,L,gap", [(80, 60, 0), (65536, 40000, 35000), (65536, 40000, 40000)])
def test_injected_leading_prefix_computed_on_device(N, L, gap):
    """L6 and larger: an injected chain of L positions with
    position `gap` missing; the device derives leading = gap (= L when the
    gap is past the end), TOUCH reports it, and the oracle agrees."""
    from paper_2605_24259_b200 import rkc
    from paper_2605_24259_b200.gen import HARD, SUBMIT, TOUCH, make_cfg, op, pack_ops
    cfgs = np.stack([make_cfg(N)])
    pool = rkc.Pool(cfgs, N, max_objects=128)
    st = pool.rkc_state_export()
    blocks, objs = st["blocks"], st["objects"]
    rng = np.random.default_rng(L + gap)
    where = rng.permutation(N)[:L]                 # scattered block ids
    for p in range(L):
        if p != gap:
            blocks[0, where[p]] = (1, 3, 0, p, 5 * L - p)
    objs[0, 3]["live"], objs[0, 3]["len"], objs[0, 3]["claim"] = 1, L, 0xFF
    hdr = st["header"].copy()
    hdr[0]["seq_ctr"] = 6 * L
    pool.rkc_state_import(0, hdr, blocks, st["claims"], st["requests"], objs)
    assert pool.rkc_state_export()["objects"][0, 3]["leading"] == min(gap, L)
    ops = pack_ops([[op(SUBMIT, 0, 3, HARD, L, L, 0), op(TOUCH, 3)]])
    pool.rkc_step_batch(ops, 2)
    _, events, _ = pool.read_all()
    probe = events[events["type"] == orc.E_REUSE_PROBE][0]
    assert probe["f"][1] == min(gap, L)
    b = orc.OracleBatch(cfgs, N, O=128)
    ob = b.export(0)
    ob["blocks"][:] = blocks[0]
    ob["objects"][:] = objs[0]
    b.import_(0, 6 * L, 0, ob["blocks"], ob["claims"], ob["requests"], ob["objects"])
    b.run(ops)
    assert b.events().tobytes() == events.tobytes()


def test_conformance_accepts_spec_accepted_to_harmed():
    """S:68 "accepted -> harmed -> ok, claim_harmed event emitted" and S:488
    L1 "every claim_harmed event has an earlier claim_accepted": a harm
    straight from ACCEPTED passes L1 and L7; without a lowering array the
    checker does not apply I4; a harm with no acceptance still fails L1."""
    import torch
    from paper_2605_24259_b200 import rkc
    ev = np.zeros(2, dtype=rkc.EVENT)
    ev[0] = (0, 0, orc.E_CLAIM_ACCEPTED, 0, 0, 0, 0, (0, 8, 8, 0))
    ev[1] = (0, 1, orc.E_CLAIM_HARMED, 0, 0, 1, 0, (3, 8, 0, 0))
    off = torch.tensor([0, 2], dtype=torch.int32).cuda()
    e = torch.from_numpy(ev.view(np.uint8).copy()).cuda()
    fs = torch.tensor([[orc.C_HARMED]], dtype=torch.uint8).cuda()
    v, _ = rkc.rkc_conformance_check(e, off, 1, fs, 1)
    assert int(v[0]) == 0
    lo = torch.tensor([0], dtype=torch.uint8).cuda()          # contract lowering given: I4
    v, _ = rkc.rkc_conformance_check(e, off, 1, fs, 1, lo)
    assert int(v[0]) == rkc.RKC_CHECK["I4"]
    e2 = torch.from_numpy(ev[1:].view(np.uint8).copy()).cuda()
    off2 = torch.tensor([0, 1], dtype=torch.int32).cuda()
    v, _ = rkc.rkc_conformance_check(e2, off2, 1, fs, 1)
    assert int(v[0]) & rkc.RKC_CHECK["L1"]


def test_current_device_unchanged():
    import torch
    from paper_2605_24259_b200 import rkc
    from paper_2605_24259_b200.gen import make_cfg
    last = torch.cuda.device_count() - 1
    torch.cuda.set_device(0)
    pool = rkc.Pool(np.stack([make_cfg(16)]), 16, device=last)
    pool.rkc_step_batch(gen.pack_ops([[gen.op(gen.INSERT, 0, x=4)]]), 1)
    pool.read_all()
    assert torch.cuda.current_device() == 0
    pool.close()
    assert torch.cuda.current_device() == 0
