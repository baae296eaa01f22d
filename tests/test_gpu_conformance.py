"""the conformance checker (L1-L7, I4) replayed on the GPU over
the claim-level event stream.  It must pass on every stream the
oracle and the CUDA path produce, reproduce the paper's evidence numbers on
the canonical traces, and fail the right check on injected faults."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2605_24259_b200 import gen
from paper_2605_24259_b200.gen import litmus

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_24259_b200 import build
    build.build()


def _offsets(ev, n):
    return np.searchsorted(ev["trace"], np.arange(n + 1)).astype(np.uint32)


def _check_array(ev, n, final_states=None, C=16, lowering=None):
    import torch
    from paper_2605_24259_b200 import rkc
    ev = np.ascontiguousarray(ev)
    e = torch.from_numpy(ev.view(np.uint8).copy()).cuda() if len(ev) else torch.zeros(32, dtype=torch.uint8).cuda()
    o = torch.from_numpy(_offsets(ev, n)).cuda()
    fs = torch.from_numpy(np.ascontiguousarray(final_states, dtype=np.uint8)).cuda() if final_states is not None else None
    lo = torch.from_numpy(np.ascontiguousarray(lowering, dtype=np.uint8)).cuda() if lowering is not None else None
    v, evd = rkc.rkc_conformance_check(e, o, n, fs, C, lo)
    return v.cpu().numpy().astype(np.uint32), evd.cpu().numpy()


def _oracle(cfgs, ops, N, C=16):
    b = orc.OracleBatch(cfgs, N, C)
    b.run(ops, nthreads=8)
    fs = np.stack([b.export(i)["claims"]["state"] for i in range(len(cfgs))])
    return b.events(), fs, b.counters()


def test_pool_conformance_passes_on_gpu_streams():
    import torch
    from paper_2605_24259_b200 import rkc
    for cfgs, ops, N in [litmus.paper_litmus()[:2] + (80,),
                         litmus.suite(range(200))[:2] + (1024,),
                         gen.random_traces(3, 21, 0, 2000, 256, 1024) + (1024,),
                         gen.random_traces(6, 22, 0, 2000, 256, 1024) + (1024,)]:  # f3 hits
        pool = rkc.Pool(cfgs, N, events_per_trace=4 * ops.shape[0] + 64)
        pool.rkc_step_batch(torch.from_numpy(np.ascontiguousarray(ops).view(np.uint8).reshape(-1)).cuda(),
                            ops.shape[0])
        v, evd = pool.rkc_pool_conformance()
        v = v.cpu().numpy()
        assert (v == 0).all(), np.nonzero(v)[0][:10]
        counters, _, _ = pool.read_all()
        c = counters.astype(np.int64).sum(0)
        evd = evd.cpu().numpy()
        assert evd[0] == c[orc.K["accepted"]] and evd[1] == c[orc.K["materialized"]]
        assert evd[2] == c[orc.K["harmed_obligated"]] + c[orc.K["harmed_unobligated"]]
        assert evd[5] == c[orc.K["victims_ordinary"]] + c[orc.K["victims_after_release"]] + c[orc.K["victims_claimed"]]
        assert evd[6] == c[orc.K["victims_after_release"]]
        assert evd[8] == 0


def test_array_conformance_passes_on_oracle_streams():
    cfgs, ops = gen.random_traces(3, 22, 0, 1500, 200, 1024)
    ev, fs, _ = _oracle(cfgs, ops, 1024)
    v, evd = _check_array(ev, len(cfgs), fs, lowering=cfgs["lowering"])
    assert (v == 0).all()
    assert evd[8] == 0


def test_paper_evidence_on_canonical_traces():
    """L1: native 60/70/80 -> 50 victims, 0 accepted, 0 harm;
    L2: no-admit served with 50 victims; L3:
    one attributed refusal, 130/80/50; L4/L5: 50 losses after
    release, 0 harm."""
    from paper_2605_24259_b200.gen import (ADMIT, ADVANCE, CONTRACT, DEMOTE, EXPIRING, HARD, INSERT,
                                           NOP, SUBMIT, make_cfg, op, pack_ops)
    cfgs, ops, _ = litmus.paper_litmus()
    ev, fs, _ = _oracle(cfgs, ops, 80)
    per = [ev[ev["trace"] == i].copy() for i in range(3)]
    for p in per:
        p["trace"] = 0
    v, evd = _check_array(per[1], 1, fs[1:2])     # native no-admit
    assert v[0] == 0 and evd[0] == 0 and evd[2] == 0 and evd[5] == 50 and evd[7] == 1
    t0 = per[0]
    v, evd = _check_array(t0, 1, fs[0:1])          # hard claim -> refusal
    assert v[0] == 0 and evd[3] == 1 and evd[4] == 1
    ref = t0[t0["type"] == orc.E_ACTIVE_REFUSED][0]
    assert int(ref["f"][0]) + int(ref["f"][1]) == 130 and ref["f"][2] == 80 and ref["f"][3] == 50
    demote = [op(INSERT, 0, x=60), op(SUBMIT, 0, 0, HARD, 60, 60, 0), op(DEMOTE, 0),
              op(ADMIT, 0, 1, 0, 1120, 1120, 0), op(ADVANCE, 0)]
    expire = [op(INSERT, 0, x=60), op(SUBMIT, 0, 0, EXPIRING, 60, 60, 3), op(NOP), op(NOP),
              op(ADMIT, 0, 1, 0, 1120, 1120, 0), op(ADVANCE, 0)]
    cf = np.stack([make_cfg(80, CONTRACT), make_cfg(80, CONTRACT)])
    ev2, fs2, _ = _oracle(cf, pack_ops([demote, expire]), 80)
    v, evd = _check_array(ev2, 2, fs2)
    assert (v == 0).all() and evd[6] == 100 and evd[2] == 0


def _faulted(mutate):
    cfgs, ops, _ = litmus.paper_litmus()
    ev, fs, _ = _oracle(cfgs, ops, 80)
    ev = ev.copy()
    fs = fs.copy()
    ev = mutate(ev, fs)
    return _check_array(ev, 3, fs, lowering=cfgs["lowering"])[0]


def test_faults_are_caught_by_the_right_check():
    from paper_2605_24259_b200 import rkc
    K = rkc.RKC_CHECK

    def harm_before_accept(ev, fs):       # trace 2: move the harm to the front
        i2 = np.nonzero(ev["trace"] == 2)[0]
        h = i2[ev["type"][i2] == orc.E_CLAIM_HARMED][0]
        order = list(range(len(ev)))
        order.remove(h)
        order.insert(i2[0], h)
        return ev[order]
    assert _faulted(harm_before_accept)[2] & K["L1"]

    def bad_shortfall(ev, fs):
        i = np.nonzero((ev["trace"] == 0) & (ev["type"] == orc.E_ACTIVE_REFUSED))[0][0]
        ev["f"][i, 3] = 49
        return ev
    assert _faulted(bad_shortfall)[0] & K["L3"]

    def unattributed(ev, fs):
        i = np.nonzero((ev["trace"] == 0) & (ev["type"] == orc.E_ACTIVE_REFUSED))[0][0]
        ev["mask"][i] = 0
        return ev
    assert _faulted(unattributed)[0] & K["L3"]

    def denial_without_service(ev, fs):
        i = np.nonzero((ev["trace"] == 1) & (ev["type"] == orc.E_REQUEST_SERVED))[0][0]
        return np.delete(ev, i)
    assert _faulted(denial_without_service)[1] & K["L2"]

    def loss_after_release_without_release(ev, fs):
        i = np.nonzero((ev["trace"] == 1) & (ev["type"] == orc.E_VICTIMS))[0][0]
        ev["f"][i, 1] = 5
        return ev
    assert _faulted(loss_after_release_without_release)[1] & K["L45"]

    def bad_materialization(ev, fs):
        i = np.nonzero((ev["trace"] == 0) & (ev["type"] == orc.E_CLAIM_MATERIALIZED))[0][0]
        ev["f"][i, 0] = 59
        ev["f"][i, 2] = 59 * 16
        return ev
    assert _faulted(bad_materialization)[0] & K["L6"]

    def wrong_final_state(ev, fs):
        fs[0, 0] = orc.C_DEMOTED
        return ev
    assert _faulted(wrong_final_state)[0] & K["L7"]

    def contract_harm(ev, fs):            # trace 0 is under the contract lowering
        i = np.nonzero((ev["trace"] == 0) & (ev["type"] == orc.E_REUSE_PROBE))[0][0]
        ev["type"][i] = orc.E_CLAIM_HARMED
        ev["reason"][i] = 1
        ev["f"][i] = (10, 60, 60, 0)
        ev["slot"][i] = 0
        fs[0, 0] = orc.C_HARMED
        return ev
    assert _faulted(contract_harm)[0] & K["I4"]
    # and the unmodified streams pass
    assert (_faulted(lambda ev, fs: ev) == 0).all()


def test_checker_equals_cpu_reconstruction():
    """f2 parity: the GPU checker's per-trace verdicts and its
    evidence vector equal the plain CPU reconstruction (oracle/conformance.py)
    element by element -- on the GPU's own compacted streams of c3, c6 and c7
    (slot stress) pools, with and without the lowering array, and on every
    fault-injection stream (tests/test_oracle_conformance.py)."""
    import torch
    from oracle import conformance as cf
    from paper_2605_24259_b200 import rkc
    from test_oracle_conformance import faulted_streams
    for recipe, N, C, O in [(3, 1024, 16, 64), (6, 1024, 16, 64), (7, 256, 32, 128)]:
        cfgs, ops = gen.random_traces(recipe, 91, 0, 1500, 256, N, C, C, O)
        pool = rkc.Pool(cfgs, N, C, C, O, events_per_trace=4 * 256 + 64)
        pool.rkc_step_batch(torch.from_numpy(np.ascontiguousarray(ops).view(np.uint8).reshape(-1)).cuda(),
                            256)
        _, ev, _ = pool.read_all()
        fs = pool.rkc_state_export()["claims"]["state"]
        for low in (None, cfgs["lowering"]):
            vg, eg = _check_array(ev, len(cfgs), fs, C=C, lowering=low)
            vc, ec = cf.check_stream(ev, len(cfgs), C, fs, low)
            assert (vg == vc).all() and (eg == ec).all(), (recipe, low is None)
        # a stream with faults sprinkled in: the two still agree trace by trace
        bad = ev.copy()
        rng = np.random.default_rng(recipe)
        pick = rng.choice(len(bad), size=min(300, len(bad)), replace=False)
        bad["f"][pick, rng.integers(0, 4, size=len(pick))] += 1
        vg, eg = _check_array(bad, len(cfgs), fs, C=C, lowering=cfgs["lowering"])
        vc, ec = cf.check_stream(bad, len(cfgs), C, fs, cfgs["lowering"])
        assert (vg == vc).all() and (eg == ec).all() and (vc != 0).sum() > 0
    for name, ev, fs, low, check in faulted_streams():
        vg, eg = _check_array(ev, 3, fs, lowering=low)
        vc, ec = cf.check_stream(ev, 3, 16, fs, low)
        assert (vg == vc).all() and (eg == ec).all(), name
