"""Pins of the CPU conformance reconstruction (oracle/conformance.py, the
oracle of f2) against what the paper and SPEC fix:

* the evidence numbers the paper prints for the canonical traces:
  L1 native 60/70/80 -> 50 victims, 0 accepted, 0 harm; L2 no-admit served
  with 50 victims; L3 one attributed refusal with 130 resident-plus-active,
  80 usable, 50 shortfall; L4/L5 50 losses after release each, 0 harm;
* S:551 reconstruction fidelity: on every simulator trace the reconstructed
  final claim states equal the simulator's (the plain C++ oracle's, an
  independent program) -- c3, c6 prefix hits, c7 slot stress;
* SPEC's examples for the checks: harm with no acceptance fails
  L1, accepted -> harmed is legal, an illegal transition spliced in fails L7,
  two valid independent traces concatenated pass, a loss before the release
  fails L4/L5, a refusal without its blocking claim fails L3;
* every fault injection fails the check it targets and no other stream fails.
"""
import numpy as np
import pytest

from oracle import conformance as cf
from oracle import oracle as orc
from paper_2605_24259_b200 import gen
from paper_2605_24259_b200.gen import litmus


def _run(cfgs, ops, N, C=16, Q=16, O=64):
    b = orc.OracleBatch(cfgs, N, C, Q, O)
    assert b.run(ops, nthreads=8, check=True) == 0
    fs = np.stack([b.export(i)["claims"]["state"] for i in range(len(cfgs))])
    return b.events(), fs


def _one(ev, t):
    e = ev[ev["trace"] == t].copy()
    e["trace"] = 0
    return e


def test_paper_evidence_L1_L2_L3():
    cfgs, ops, _ = litmus.paper_litmus()
    ev, fs = _run(cfgs, ops, 80)
    v, e, _ = cf.check_trace(_one(ev, 1), 16, fs[1])          # native no-admit (L1, L2)
    assert v == 0
    assert (e[0], e[2], e[5], e[7]) == (0, 0, 50, 1)           # 0 accepted, 0 harm, 50 victims
    v, e, _ = cf.check_trace(_one(ev, 0), 16, fs[0], lowering=0)  # hard claim (L3, L7)
    assert v == 0 and e[0] == 1 and e[1] == 1 and e[3] == 1 and e[4] == 1
    ref = ev[(ev["trace"] == 0) & (ev["type"] == orc.E_ACTIVE_REFUSED)][0]
    assert (int(ref["f"][0]) + int(ref["f"][1]), int(ref["f"][2]), int(ref["f"][3])) == (130, 80, 50)


def test_paper_evidence_L4_L5():
    from paper_2605_24259_b200.gen import (ADMIT, ADVANCE, CONTRACT, DEMOTE, EXPIRING, HARD, INSERT,
                                           NOP, SUBMIT, make_cfg, op, pack_ops)
    demote = [op(INSERT, 0, x=60), op(SUBMIT, 0, 0, HARD, 60, 60, 0), op(DEMOTE, 0),
              op(ADMIT, 0, 1, 0, 1120, 1120, 0), op(ADVANCE, 0)]
    expire = [op(INSERT, 0, x=60), op(SUBMIT, 0, 0, EXPIRING, 60, 60, 3), op(NOP), op(NOP),
              op(ADMIT, 0, 1, 0, 1120, 1120, 0), op(ADVANCE, 0)]
    cfgs = np.stack([make_cfg(80, CONTRACT), make_cfg(80, CONTRACT)])
    ev, fs = _run(cfgs, pack_ops([demote, expire]), 80)
    for t in (0, 1):
        v, e, _ = cf.check_trace(_one(ev, t), 16, fs[t], lowering=0)
        assert v == 0 and e[6] == 50 and e[2] == 0              # 50 losses after release, 0 harm


@pytest.mark.parametrize("recipe,N,C,O", [(3, 1024, 16, 64), (6, 1024, 16, 64), (7, 256, 32, 128)])
def test_reconstruction_fidelity_S551(recipe, N, C, O):
    """The reconstruction's final claim states equal the simulator's, and the
    simulator's streams pass every check."""
    cfgs, ops = gen.random_traces(recipe, seed=77, trace_begin=0, n_traces=300, T=256, N=N,
                                  C=C, Q=C, O=O)
    ev, fs = _run(cfgs, ops, N, C, C, O)
    assert (cf.reconstruct_states(ev, len(cfgs), C) == fs).all()
    v, e = cf.check_stream(ev, len(cfgs), C, fs, cfgs["lowering"])
    assert (v == 0).all() and e[8] == 0
    assert e[0] > 0 and e[3] > 0 and e[5] > 0


def _ev(rows):
    out = np.zeros(len(rows), dtype=orc.EVENT_DTYPE)
    for i, (step, typ, slot, reason, mask, f) in enumerate(rows):
        out[i] = (0, step, typ, 0, slot, reason, mask, f)
    return out


ACC = lambda s, c, o=0, R=8: (s, orc.E_CLAIM_ACCEPTED, c, 0, 0, (o, R, R, 0))
HARM = lambda s, c: (s, orc.E_CLAIM_HARMED, c, 1, 0, (3, 8, 0, 0))


def test_spec_examples():
    # S:491 injected claim_harmed with no acceptance -> L1 fails; S:492 empty trace passes
    assert cf.check_trace(_ev([HARM(0, 0)]), 4)[0] & cf.L1
    assert cf.check_trace(_ev([]), 4)[0] == 0
    # S:68 accepted -> harmed is legal (and I4 only with a known contract lowering)
    assert cf.check_trace(_ev([ACC(0, 0), HARM(1, 0)]), 4, [orc.C_HARMED, 0, 0, 0])[0] == 0
    assert cf.check_trace(_ev([ACC(0, 0), HARM(1, 0)]), 4, lowering=0)[0] == cf.I4
    # S:67 expired -> accepted is illegal: splicing an acceptance after expiry fails L7
    exp = (1, orc.E_CLAIM_EXPIRED, 0, 0, 0, (0, 8, 0, 1))
    assert cf.check_trace(_ev([ACC(0, 0), exp, ACC(2, 0)]), 4)[0] & cf.L7
    # S:528 two valid independent traces with disjoint ids concatenated -> pass
    a = [ACC(0, 0, o=0), (1, orc.E_CLAIM_MATERIALIZED, 0, 0, 0, (8, 8, 128, 0))]
    b = [ACC(2, 1, o=1), (3, orc.E_CLAIM_DEMOTED, 1, 0, 0, (1, 8, 0, 0))]
    assert cf.check_trace(_ev(a + b), 4)[0] == 0
    # S:505 loss event before release event -> L4/L5 fails
    vic = (1, orc.E_VICTIMS, 0, 0, 0, (0, 5, 0, 5))
    dem = (2, orc.E_CLAIM_DEMOTED, 0, 0, 0, (0, 8, 0, 0))
    assert cf.check_trace(_ev([ACC(0, 0), vic, dem]), 4)[0] & cf.L45
    assert cf.check_trace(_ev([ACC(0, 0), dem, vic]), 4)[0] == 0
    # S:499 refusal missing blocking_claim_ids -> L3 fails
    ref = lambda m: (1, orc.E_ACTIVE_REFUSED, 0, orc.WHY_PROTECTED_RESIDENT, m, (60, 70, 80, 50))
    assert cf.check_trace(_ev([ACC(0, 0, R=60), ref(0)]), 4)[0] & cf.L3
    assert cf.check_trace(_ev([ACC(0, 0, R=60), ref(1)]), 4)[0] == 0
    # a harm after demotion is L4/L5 (release before loss) and an illegal transition
    assert cf.check_trace(_ev([ACC(0, 0), dem, HARM(3, 0)]), 4)[0] == cf.L45 | cf.L7


FAULTS = {}


def fault(check):
    def deco(fn):
        FAULTS[fn.__name__] = (fn, check)
        return fn
    return deco


@fault(cf.L1)
def harm_before_accept(ev, fs):
    i2 = np.nonzero(ev["trace"] == 2)[0]
    h = i2[ev["type"][i2] == orc.E_CLAIM_HARMED][0]
    order = list(range(len(ev)))
    order.remove(h)
    order.insert(i2[0], h)
    return ev[order]


@fault(cf.L3)
def bad_shortfall(ev, fs):
    i = np.nonzero((ev["trace"] == 0) & (ev["type"] == orc.E_ACTIVE_REFUSED))[0][0]
    ev["f"][i, 3] = 49
    return ev


@fault(cf.L3)
def unattributed(ev, fs):
    i = np.nonzero((ev["trace"] == 0) & (ev["type"] == orc.E_ACTIVE_REFUSED))[0][0]
    ev["mask"][i] = 0
    return ev


@fault(cf.L2)
def denial_without_service(ev, fs):
    i = np.nonzero((ev["trace"] == 1) & (ev["type"] == orc.E_REQUEST_SERVED))[0][0]
    return np.delete(ev, i)


@fault(cf.L45)
def loss_after_release_without_release(ev, fs):
    i = np.nonzero((ev["trace"] == 1) & (ev["type"] == orc.E_VICTIMS))[0][0]
    ev["f"][i, 1] = 5
    return ev


@fault(cf.L6)
def bad_materialization(ev, fs):
    i = np.nonzero((ev["trace"] == 0) & (ev["type"] == orc.E_CLAIM_MATERIALIZED))[0][0]
    ev["f"][i, 0] = 59
    ev["f"][i, 2] = 59 * 16
    return ev


@fault(cf.L7)
def wrong_final_state(ev, fs):
    fs[0, 0] = orc.C_DEMOTED
    return ev


@fault(cf.I4)
def contract_harm(ev, fs):
    i = np.nonzero((ev["trace"] == 0) & (ev["type"] == orc.E_REUSE_PROBE))[0][0]
    ev["type"][i] = orc.E_CLAIM_HARMED
    ev["reason"][i] = 1
    ev["f"][i] = (10, 60, 60, 0)
    ev["slot"][i] = 0
    fs[0, 0] = orc.C_HARMED
    return ev


def faulted_streams():
    """(name, events, final states, lowering, check) for every fault on the
    paper litmus streams, plus the unmodified streams (check 0)."""
    cfgs, ops, _ = litmus.paper_litmus()
    ev0, fs0 = _run(cfgs, ops, 80)
    out = [("clean", ev0, fs0, cfgs["lowering"], 0)]
    for name, (fn, check) in FAULTS.items():
        ev, fs = ev0.copy(), fs0.copy()
        out.append((name, fn(ev, fs), fs, cfgs["lowering"], check))
    return out


def test_faults_fail_the_right_check():
    for name, ev, fs, low, check in faulted_streams():
        v, _ = cf.check_stream(ev, 3, 16, fs, low)
        if check == 0:
            assert (v == 0).all(), name
        else:
            assert any(int(x) & check for x in v), name
