"""Pins of NEXT f4: admission under the resident reserve (admit_check =
RESERVE).  Table 5 "Resident reserve -- Resident survives; active work that
cannot fit is refused.  Modeled reserve action"; "a static
block count subtracted from usable headroom at admission; default reserve
equals the sum of accepted hard-protected footprints" (G34).

The expectations are closed forms: reserve = sum of F over live obligated
claims under the contract lowering; an admission of peak p with Alive held is
refused iff reserve + Alive + p > U, with (P, A, U, shortfall) =
(reserve, Alive + p, U, reserve + Alive + p - U) and the reserving claims as
the blocking set -- or as an ACTIVE_CAPACITY refusal with no claims when
Alive + p > U alone.
"""
import random

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2605_24259_b200.gen import (ADMIT, ADMIT_RESERVE, ADVANCE, BEST_EFFORT, COMPLETE,
                                       CONTRACT, DEMOTABLE, DEMOTE, EXPIRING, HARD, INSERT, NATIVE,
                                       NOP, OFFLOADABLE, PEAK, SOFT, SOFT_LOWERING, SUBMIT, TOUCH,
                                       make_cfg, op, pack_ops)

OBLIGATED = {HARD, DEMOTABLE, OFFLOADABLE, EXPIRING}
RESV = orc.WHY_RESIDENT_RESERVE


def _run(cfgs, lists, N, C=16):
    b = orc.OracleBatch(np.stack(cfgs), N=N, C=C)
    assert b.run(pack_ops(lists), check=True) == 0
    ev = b.events()
    idx = np.searchsorted(ev["trace"], np.arange(len(cfgs) + 1))
    return b, [ev[idx[i]:idx[i + 1]] for i in range(len(cfgs))]


def _refusals(e):
    m = np.isin(e["type"], [orc.E_ACTIVE_REFUSED, orc.E_ACTIVE_DEFERRED])
    return [(int(x["type"]), int(x["reason"]), int(x["mask"]), [int(v) for v in x["f"]])
            for x in e[m]]


def test_reserve_counts_the_footprint_not_the_cached_blocks():
    """A hard claim F = 60 on a 40-block object (materialized at R = 40): the
    boundary sees P = 40 cached protected blocks, the reserve sees F = 60.
    Peak 41 at U = 100: PEAK admits (40 + 41 <= 100), RESERVE refuses
    (60 + 41 = 101, shortfall 1); peak 40 fits both (60 + 40 = 100)."""
    pre = [op(INSERT, 0, x=40), op(SUBMIT, 0, 0, HARD, 60, 40, 0)]
    lists = [pre + [op(ADMIT, 0, 1, 0, 16 * 41, 16 * 41, 0)],
             pre + [op(ADMIT, 0, 1, 0, 16 * 41, 16 * 41, 0)],
             pre + [op(ADMIT, 0, 1, 0, 16 * 40, 16 * 40, 0)]]
    cfgs = [make_cfg(100, CONTRACT, PEAK), make_cfg(100, CONTRACT, ADMIT_RESERVE),
            make_cfg(100, CONTRACT, ADMIT_RESERVE)]
    b, evs = _run(cfgs, lists, 100)
    assert _refusals(evs[0]) == []
    assert _refusals(evs[1]) == [(orc.E_ACTIVE_REFUSED, RESV, 0b1, [60, 41, 100, 1])]
    assert _refusals(evs[2]) == []
    assert b.export(0)["claims"][0]["state"] == orc.C_MATERIALIZED
    assert b.counters()[1][orc.K["refused_protected"]] == 1


def test_reserve_protects_a_claim_before_it_materializes_P1069():
    """The paper's 60/70/80 numbers with the resident not yet cached: a hard
    claim F = R = 60 on an object that is not live yet reserves 60 blocks, so
    a 70-block active request is refused with the capacity proof of
    P:1069-1079 (60 + 70 = 130 > 80, shortfall 50), attributed to the claim;
    the PEAK boundary (P = 0) would admit it and the later insertion of the
    resident would then be refused."""
    seq = [op(SUBMIT, 0, 0, HARD, 60, 60, 0), op(ADMIT, 0, 1, 0, 1120, 1120, 0), op(ADVANCE, 0),
           op(INSERT, 0, x=60)]
    b, evs = _run([make_cfg(80, CONTRACT, ADMIT_RESERVE), make_cfg(80, CONTRACT, PEAK)],
                  [seq, seq], 80)
    assert _refusals(evs[0]) == [(orc.E_ACTIVE_REFUSED, RESV, 0b1, [60, 70, 80, 50])]
    ref = evs[0][evs[0]["type"] == orc.E_ACTIVE_REFUSED][0]
    rendered = orc.render_refusal_json(ref, {0: "active"}, {0: "claim:resident"})
    assert rendered["resident_plus_active_blocks"] == 130 and rendered["capacity_shortfall_blocks"] == 50
    assert rendered["blocking_claim_ids"] == ["claim:resident"]
    assert b.export(0)["claims"][0]["state"] == orc.C_MATERIALIZED      # the resident got its room
    assert _refusals(evs[1]) == []
    ins = evs[1][evs[1]["type"] == orc.E_RESIDENT_INSERT_REFUSED]
    assert len(ins) == 1 and b.export(1)["claims"][0]["state"] == orc.C_ACCEPTED


def test_what_does_not_reserve():
    """Non-obligated claims, released claims and non-contract lowerings hold
    no reserve; Alive + peak > U alone is ACTIVE_CAPACITY with no claims."""
    U = 64
    big = op(ADMIT, 0, 5, 0, 16 * 40, 16 * 40, 0)
    lists = [
        [op(SUBMIT, 0, 0, SOFT, 60, 1, 0), op(SUBMIT, 1, 1, BEST_EFFORT, 60, 1, 0), big],
        [op(SUBMIT, 0, 0, HARD, 60, 1, 0), op(DEMOTE, 0), big],
        [op(SUBMIT, 0, 0, EXPIRING, 60, 1, 2), op(NOP), big],           # expired at step 2
        [op(SUBMIT, 0, 0, HARD, 60, 1, 0), big],
        [op(SUBMIT, 0, 0, HARD, 60, 1, 0), big],
        [op(SUBMIT, 0, 0, HARD, 10, 1, 0), op(ADMIT, 0, 5, 0, 16 * 65, 16 * 65, 0)],
    ]
    cfgs = [make_cfg(U, CONTRACT, ADMIT_RESERVE)] * 3 + [make_cfg(U, SOFT_LOWERING, ADMIT_RESERVE),
                                                         make_cfg(U, NATIVE, ADMIT_RESERVE),
                                                         make_cfg(U, CONTRACT, ADMIT_RESERVE)]
    _, evs = _run(cfgs, lists, U)
    for i in range(5):
        assert _refusals(evs[i]) == [], i
    assert _refusals(evs[5]) == [(orc.E_ACTIVE_REFUSED, orc.WHY_ACTIVE_CAPACITY, 0, [10, 65, 64, 11])]


def test_reserve_deferral_then_admission_after_release():
    """defer_budget 1: the first admission is deferred with the reserve proof;
    a DEMOTE releases the reserve, and the retry (ADVANCE of the deferred
    request) is admitted and allocates."""
    seq = [op(SUBMIT, 0, 0, HARD, 50, 1, 0), op(ADMIT, 0, 1, 0, 16 * 40, 16 * 40, 0),
           op(DEMOTE, 0), op(ADVANCE, 0)]
    b, evs = _run([make_cfg(80, CONTRACT, ADMIT_RESERVE, defer_budget=1)], [seq], 80)
    assert _refusals(evs[0]) == [(orc.E_ACTIVE_DEFERRED, RESV, 0b1, [50, 40, 80, 10])]
    st = b.export(0)
    assert st["requests"][0]["status"] == orc.R_RUNNING and st["requests"][0]["live"] == 40


@pytest.mark.parametrize("seed", range(20))
def test_reserve_closed_form_random(seed):
    """Random claim sets (modes, footprints, demotions) followed by one
    admission: refused iff the live obligated footprints plus the peak exceed
    U, with the closed-form proof and mask."""
    rng = random.Random(seed)
    cfgs, lists, want = [], [], []
    for _ in range(200):
        U = rng.randint(16, 400)
        low = rng.choice([CONTRACT, CONTRACT, CONTRACT, SOFT_LOWERING, NATIVE])
        ops, live = [], {}
        for c in range(rng.randint(0, 6)):
            mode = rng.randrange(6)
            F = rng.randint(1, U)
            ops.append(op(SUBMIT, c, c, mode, F, 1, 50 if mode == EXPIRING else 0))
            live[c] = (mode, F)
        for c in list(live):
            if rng.random() < 0.25:
                ops.append(op(DEMOTE, c))
                del live[c]
        p = rng.randint(1, U + 20)
        ops.append(op(ADMIT, 0, 10, 0, 16 * p, 16 * p, 0))
        # the capacity rule rejects F > U at submission: never happens here (F <= U)
        res = sum(F for (m, F) in live.values() if m in OBLIGATED) if low == CONTRACT else 0
        mask = sum(1 << c for c, (m, F) in live.items() if m in OBLIGATED) if low == CONTRACT else 0
        if res + p <= U:
            w = []
        elif p <= U and res > 0:
            w = [(orc.E_ACTIVE_REFUSED, RESV, mask, [res, p, U, res + p - U])]
        else:
            w = [(orc.E_ACTIVE_REFUSED, orc.WHY_ACTIVE_CAPACITY, 0, [res, p, U, res + p - U])]
        cfgs.append(make_cfg(U, low, ADMIT_RESERVE))
        lists.append(ops)
        want.append(w)
    _, evs = _run(cfgs, lists, 400)
    for i, w in enumerate(want):
        assert _refusals(evs[i]) == w, (seed, i)


def test_reserve_never_harms_random_traces():
    """Under the contract lowering with reserve admission, random c3-like
    traces keep every invariant (I1-I10 asserted per op) and never harm an
    obligated claim (I4)."""
    from paper_2605_24259_b200 import gen
    cfgs, ops = gen.random_traces(8, seed=3, trace_begin=0, n_traces=400, T=256, N=1024)
    assert (cfgs["admit_check"] == ADMIT_RESERVE).sum() > 100
    b = orc.OracleBatch(cfgs, 1024)
    assert b.run(ops, nthreads=8, check=True) == 0
    ev = b.events()
    assert ((ev["type"] == orc.E_ACTIVE_REFUSED) & (ev["reason"] == RESV)).sum() > 0
    c = b.counters()
    assert c[cfgs["lowering"] == CONTRACT][:, orc.K["harmed_obligated"]].sum() == 0
