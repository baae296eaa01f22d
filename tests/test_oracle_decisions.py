"""Pins of the oracle's claim decision (op_submit), of `obligated(offloadable)`
(G11) and of the blocking set -- the branches the round-1
verdict found unpinned.

Each expectation is either a SPEC / paper example quoted verbatim or a closed
form of the rule the ledger reading states, evaluated here on inputs whose
outcome it fixes by hand.  Every test below fails against a plausible mutant
of `oracle/rkc_oracle.cpp` (`>=` for `>`, summing non-obligated footprints,
counting released claims, dropping `pos < F`, offloadable not obligated,
a blocking mask that lists only the first claim); the mutants tried are listed
in DESIGN.md "Oracle pins".
"""
import random

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2605_24259_b200.gen import (ADMIT, ADVANCE, BEST_EFFORT, CAPACITY, COMPLETE, CONTRACT,
                                       DEMOTABLE, DEMOTE, EXPIRING, HARD, HIT_ADMIT, ID_MISMATCH,
                                       INSERT, NATIVE, NONE, NOP, OFFLOADABLE, PEAK, RESERVE, SOFT,
                                       SOFT_LOWERING, SUBMIT, TOUCH, make_cfg, op, pack_ops)
from paper_2605_24259_b200.gen import litmus

REJ_IDENTITY, REJ_OBJECT_CLAIMED, REJ_FOOTPRINT, REJ_RESERVE = 1, 2, 3, 4
OBLIGATED = {HARD, DEMOTABLE, OFFLOADABLE, EXPIRING}          # Table 3, G11


def _run(cfgs, lists, N, C=16, Q=16, O=64):
    b = orc.OracleBatch(np.stack(cfgs), N=N, C=C, Q=Q, O=O)
    assert b.run(pack_ops(lists), check=True) == 0
    ev = b.events()
    idx = np.searchsorted(ev["trace"], np.arange(len(cfgs) + 1))
    return b, [ev[idx[i]:idx[i + 1]] for i in range(len(cfgs))]


def _decisions(e):
    """claim slot -> (event type, reason) of its accept / reject event."""
    out = {}
    for x in e:
        if int(x["type"]) in (orc.E_CLAIM_ACCEPTED, orc.E_CLAIM_REJECTED):
            out[int(x["slot"])] = (int(x["type"]), int(x["reason"]))
    return out


ACC = (orc.E_CLAIM_ACCEPTED, 0)


def REJ(reason):
    return (orc.E_CLAIM_REJECTED, reason)


# --------------------------------------------------------------------------
# 1. FOOTPRINT: S:59-61, the three submit_claim examples verbatim
# --------------------------------------------------------------------------
def test_submit_footprint_spec_examples_S59_61():
    """S:59 "footprint 60, usable 80 -> accepted"; "footprint 81,
    usable 80 -> rejected"; "footprint 80, usable 80 -> accepted"
    (boundary equality is feasible).  The rejection reason is FOOTPRINT."""
    cases = [(60, ACC), (81, REJ(REJ_FOOTPRINT)), (80, ACC)]
    cfgs = [make_cfg(80, CONTRACT) for _ in cases]
    lists = [[op(SUBMIT, 0, 0, HARD, F, F, 0)] for F, _ in cases]
    b, evs = _run(cfgs, lists, N=80)
    for i, (F, want) in enumerate(cases):
        assert _decisions(evs[i]) == {0: want}, F
        st = b.export(i)
        assert st["claims"][0]["state"] == (orc.C_ACCEPTED if want == ACC else orc.C_REFUSED)
        # a rejected claim does not bind its object (Table 2: rejected decision)
        assert st["objects"][0]["claim"] == (0 if want == ACC else 0xFF)
    ctr = b.counters()
    assert [int(c[orc.K["rejected"]]) for c in ctr] == [0, 1, 0]


@pytest.mark.parametrize("U", [1, 2, 17, 80, 1023, 1024])
def test_submit_footprint_boundary_sweep(U):
    """F <= U accepted, F = U + 1 rejected, for every mode (the CAPACITY
    rule does not depend on the mode)."""
    cfgs, lists, want = [], [], []
    for mode in range(6):
        for F in (max(1, U - 1), U, U + 1):
            cfgs.append(make_cfg(U, CONTRACT))
            lists.append([op(SUBMIT, 0, 0, mode, F, 1, 8 if mode == EXPIRING else 0)])
            want.append(ACC if F <= U else REJ(REJ_FOOTPRINT))
    _, evs = _run(cfgs, lists, N=U)
    for i, w in enumerate(want):
        assert _decisions(evs[i]) == {0: w}, (U, i)


# --------------------------------------------------------------------------
# 2. IDENTITY (P:618 salted controls give zero useful survival; G26)
# --------------------------------------------------------------------------
def test_submit_identity_mismatch_P618():
    """A claim whose cache identity differs from the pool's can never
    materialize ("salted/no-reuse controls show zero useful
    leading-prefix survival"), so it is rejected IDENTITY, before any other
    rule: an identity mismatch on an already-claimed object, or with F > U,
    still reports IDENTITY.  The object stays unbound by it."""
    U = 64
    lists = [
        # plain mismatch on a live 40-block object; then a matching claim on it is accepted
        [op(INSERT, 0, x=40), op(SUBMIT, 0, 0, HARD | ID_MISMATCH, 40, 40, 0),
         op(SUBMIT, 1, 0, HARD, 40, 40, 0)],
        # mismatch on an object already bound to a live claim -> IDENTITY, not OBJECT_CLAIMED
        [op(SUBMIT, 0, 0, HARD, 8, 8, 0), op(SUBMIT, 1, 0, SOFT | ID_MISMATCH, 8, 8, 0)],
        # mismatch with F > U -> IDENTITY, not FOOTPRINT
        [op(SUBMIT, 0, 0, HARD | ID_MISMATCH, U + 1, 1, 0)],
        # mismatch under RESERVE with an over-reserving footprint -> IDENTITY
        [op(SUBMIT, 0, 0, HARD, U, 1, 0), op(SUBMIT, 1, 1, HARD | ID_MISMATCH, 1, 1, 0)],
    ]
    cfgs = [make_cfg(U), make_cfg(U), make_cfg(U), make_cfg(U, accept_rule=RESERVE)]
    b, evs = _run(cfgs, lists, N=U)
    assert _decisions(evs[0]) == {0: REJ(REJ_IDENTITY), 1: ACC}
    assert _decisions(evs[1]) == {0: ACC, 1: REJ(REJ_IDENTITY)}
    assert _decisions(evs[2]) == {0: REJ(REJ_IDENTITY)}
    assert _decisions(evs[3]) == {0: ACC, 1: REJ(REJ_IDENTITY)}
    st = b.export(0)
    assert st["claims"][0]["state"] == orc.C_REFUSED
    assert st["claims"][1]["state"] == orc.C_MATERIALIZED     # the matching claim: L = 40 >= R
    assert st["objects"][0]["claim"] == 1


# --------------------------------------------------------------------------
# 3. OBJECT_CLAIMED (G15: one live claim per object; terminal bindings replaced)
# --------------------------------------------------------------------------
def test_submit_object_claimed_G15():
    U = 100
    lists = [
        # second live claim on the object -> OBJECT_CLAIMED, whatever its mode, even with F > U
        [op(INSERT, 0, x=30), op(SUBMIT, 0, 0, HARD, 30, 30, 0),
         op(SUBMIT, 1, 0, SOFT, 10, 10, 0), op(SUBMIT, 2, 0, BEST_EFFORT, U + 5, 1, 0),
         op(SUBMIT, 3, 1, HARD, 10, 10, 0)],
        # after DEMOTE the binding is terminal: a new claim on the object is accepted and rebinds
        [op(INSERT, 0, x=30), op(SUBMIT, 0, 0, HARD, 30, 30, 0), op(DEMOTE, 0),
         op(SUBMIT, 1, 0, DEMOTABLE, 20, 20, 0)],
        # after EXPIRY likewise (D = 2: accepted at step 1, expired at the start of step 3)
        [op(SUBMIT, 0, 0, HARD, 5, 5, 2), op(SUBMIT, 1, 0, HARD, 5, 5, 0), op(NOP),
         op(SUBMIT, 2, 0, HARD, 5, 5, 0)],
        # a REFUSED (rejected) claim never bound the object
        [op(SUBMIT, 0, 0, HARD, U + 1, 1, 0), op(SUBMIT, 1, 0, HARD, 5, 5, 0)],
        # ... and neither does a materialized claim that was then harmed (native lowering)
        [op(INSERT, 0, x=60), op(SUBMIT, 0, 0, HARD, 60, 60, 0),
         op(ADMIT, 0, 1, 0, 16 * 70, 16 * 70, 0), op(ADVANCE, 0), op(SUBMIT, 1, 0, HARD, 5, 5, 0)],
    ]
    cfgs = [make_cfg(U), make_cfg(U), make_cfg(U), make_cfg(U), make_cfg(80, NATIVE)]
    b, evs = _run(cfgs, lists, N=U)
    assert _decisions(evs[0]) == {0: ACC, 1: REJ(REJ_OBJECT_CLAIMED), 2: REJ(REJ_OBJECT_CLAIMED),
                                  3: ACC}
    assert b.export(0)["objects"][0]["claim"] == 0
    assert _decisions(evs[1]) == {0: ACC, 1: ACC}
    assert b.export(1)["objects"][0]["claim"] == 1
    assert _decisions(evs[2]) == {0: ACC, 1: REJ(REJ_OBJECT_CLAIMED), 2: ACC}
    assert len(evs[2][evs[2]["type"] == orc.E_CLAIM_EXPIRED]) == 1
    assert _decisions(evs[3]) == {0: REJ(REJ_FOOTPRINT), 1: ACC}
    assert _decisions(evs[4]) == {0: ACC, 1: ACC}
    assert b.export(4)["claims"][0]["state"] == orc.C_HARMED


# --------------------------------------------------------------------------
# 4. RESERVE (Table 5 "Resident reserve")
# --------------------------------------------------------------------------
def test_submit_reserve_worked_example_P573():
    """U = 100 under the RESERVE rule: an obligated claim is rejected iff its
    footprint plus the footprints of the LIVE OBLIGATED claims exceeds U
    ("active work that cannot fit is refused"; "default reserve
    equals the sum of accepted hard-protected footprints").  Non-obligated
    claims are never reserve-rejected and do not count; released claims do
    not count; offloadable counts (G11).  The same stream under CAPACITY
    accepts every claim (all F <= U)."""
    stream = [
        (op(SUBMIT, 0, 0, HARD, 60, 60, 0), ACC),                  # reserve 60
        (op(SUBMIT, 1, 1, SOFT, 100, 1, 0), ACC),                  # not obligated: not checked
        (op(SUBMIT, 2, 2, BEST_EFFORT, 90, 1, 0), ACC),            # not obligated: not counted
        (op(SUBMIT, 3, 3, HARD, 41, 41, 0), REJ(REJ_RESERVE)),     # 60 + 41 = 101 > 100
        (op(SUBMIT, 4, 4, DEMOTABLE, 40, 1, 0), ACC),              # 60 + 40 = 100: equality fits
        (op(SUBMIT, 5, 5, EXPIRING, 1, 1, 50), REJ(REJ_RESERVE)),  # 101
        (op(DEMOTE, 0), None),                                     # releases 60
        (op(SUBMIT, 6, 6, OFFLOADABLE, 60, 1, 0), ACC),            # 40 + 60 = 100
        (op(SUBMIT, 7, 7, HARD, 1, 1, 0), REJ(REJ_RESERVE)),       # offloadable counts: 101
        (op(SUBMIT, 8, 8, SOFT, 100, 1, 0), ACC),
    ]
    ops = [s for s, _ in stream]
    want = {i: w for i, (s, w) in enumerate(stream) if w is not None}
    want = {int(stream[i][0][1]): w for i, w in want.items()}
    b, evs = _run([make_cfg(100, accept_rule=RESERVE), make_cfg(100, accept_rule=CAPACITY)],
                  [ops, ops], N=100)
    assert _decisions(evs[0]) == want
    assert all(v == ACC for v in _decisions(evs[1]).values())
    assert len(_decisions(evs[1])) == 9


def _reserve_model(U, ops, rule):
    """Expected decisions of a SUBMIT/DEMOTE/NOP stream with no blocks
    (objects never become live, so claims only leave their live states by
    DEMOTE or expiry; G13: expired at the start of step t when d + D <= t)."""
    live = {}                                   # slot -> (mode, F, decision_step, D)
    out = {}
    for t, o in enumerate(ops):
        for c in [c for c, (m, F, d, D) in live.items() if D > 0 and d + D <= t]:
            del live[c]
        kind = o[0]
        if kind == DEMOTE:
            live.pop(o[1], None)
        elif kind == SUBMIT:
            c, mode, F, D = o[1], o[3], o[4], o[6]
            if F > U:
                out[c] = REJ(REJ_FOOTPRINT)
            elif (rule == RESERVE and mode in OBLIGATED
                  and F + sum(f for (m, f, _, _) in live.values() if m in OBLIGATED) > U):
                out[c] = REJ(REJ_RESERVE)
            else:
                out[c] = ACC
                live[c] = (mode, F, t, D)
    return out


@pytest.mark.parametrize("seed", range(30))
def test_submit_reserve_random_streams(seed):
    """Random SUBMIT / DEMOTE / NOP streams (distinct objects, so no
    OBJECT_CLAIMED) against the reserve rule evaluated on a plain dict of
    live claims."""
    rng = random.Random(seed)
    cfgs, lists, exp = [], [], []
    for _ in range(64):
        U = rng.randint(4, 200)
        ops, slot = [], 0
        for _t in range(40):
            k = rng.random()
            if k < 0.6 and slot < 32:
                mode = rng.randrange(6)
                F = rng.randint(1, U + 2)
                D = rng.randint(1, 12) if mode == EXPIRING or rng.random() < 0.3 else 0
                ops.append(op(SUBMIT, slot, slot % 64, mode, F, rng.randint(1, F), D))
                slot += 1
            elif k < 0.8 and slot:
                ops.append(op(DEMOTE, rng.randrange(slot)))
            else:
                ops.append(op(NOP))
        rule = rng.choice([RESERVE, RESERVE, CAPACITY])
        cfgs.append(make_cfg(U, accept_rule=rule))
        lists.append(ops)
        exp.append(_reserve_model(U, ops, rule))
    b, evs = _run(cfgs, lists, N=200, C=32, O=64)
    for i in range(len(cfgs)):
        assert _decisions(evs[i]) == exp[i], (seed, i)


# --------------------------------------------------------------------------
# 5. offloadable behaves exactly like hard (G11: no offload tier)
# --------------------------------------------------------------------------
def _swap_mode(ops, frm, to):
    ops = ops.copy()
    m = (ops["kind"] == SUBMIT) & ((ops["c"] & 0x7F) == frm)
    ops["c"][m] = (ops["c"][m] & 0x80) | to
    return ops


def test_offloadable_equals_hard_capacity_sweep_P988_997():
    """The capacity sweep with the hard claim made offloadable:
    served iff U >= R + A = 130, else refused with (P, A, U, shortfall) =
    (60, 70, U, 130 - U) and the claim as the blocking set; the event stream
    equals the hard run's byte for byte."""
    cfgs, ops, params = litmus.capacity_sweep()
    off = _swap_mode(ops, HARD, OFFLOADABLE)
    sub = ops["kind"] == SUBMIT
    assert (off["c"][sub] == OFFLOADABLE).sum() == (ops["c"][sub] == HARD).sum() > 0
    hb = orc.OracleBatch(cfgs, N=135)
    ob = orc.OracleBatch(cfgs, N=135)
    assert hb.run(ops, check=True) == 0 and ob.run(off, check=True) == 0
    he, oe = hb.events(), ob.events()
    assert he.tobytes() == oe.tobytes()
    idx = np.searchsorted(oe["trace"], np.arange(len(params) + 1))
    for i, p in enumerate(params):
        if p["policy"] != "hard":
            continue
        e = oe[idx[i]:idx[i + 1]]
        ref = e[e["type"] == orc.E_ACTIVE_REFUSED]
        U = p["U"]
        if U >= 130:
            assert len(ref) == 0, U
        else:
            assert len(ref) == 1 and ref[0]["mask"] == (1 if 70 <= U else 0), U  # G7
            assert list(ref[0]["f"]) == [60, 70, U, 130 - U]
        assert ob.export(i)["claims"][0]["state"] == orc.C_MATERIALIZED


def test_offloadable_equals_hard_litmus_suite():
    """Every litmus template (Appendix A closed forms, tests/test_oracle_litmus.py)
    with every hard claim made offloadable yields the identical event stream
    and counters: protected under CONTRACT, class 2 under SOFT lowering,
    obligated harm (reason 1) when lost, counted by RESERVE."""
    cfgs, ops, params = litmus.suite(range(200))
    off = _swap_mode(ops, HARD, OFFLOADABLE)
    hb = orc.OracleBatch(cfgs, N=1024)
    ob = orc.OracleBatch(cfgs, N=1024)
    assert hb.run(ops, nthreads=8, check=True) == 0
    assert ob.run(off, nthreads=8, check=True) == 0
    assert hb.events().tobytes() == ob.events().tobytes()
    assert (hb.counters() == ob.counters()).all()
    # the swap did change inputs, and some of them hit the protected / harmed paths
    assert (off["c"] != ops["c"]).any()
    assert hb.counters()[:, orc.K["refused_protected"]].sum() > 0
    assert hb.counters()[:, orc.K["harmed_obligated"]].sum() > 0


def test_offloadable_soft_lowering_harm_is_obligated():
    """C1 unsoundness with an offloadable claim: SOFT lowering
    serves the request and harms the claim, and the harm carries the
    obligated flag (reason 1) -- offloadable is obligated (G11)."""
    U, R, A = 80, 60, 70
    ops = [op(INSERT, 0, x=R), op(SUBMIT, 0, 0, OFFLOADABLE, R, R, 0),
           op(ADMIT, 0, 1, 0, 16 * A, 16 * A, 0), op(ADVANCE, 0), op(COMPLETE, 0)]
    b, evs = _run([make_cfg(U, SOFT_LOWERING)], [ops], N=U)
    h = evs[0][evs[0]["type"] == orc.E_CLAIM_HARMED]
    assert len(h) == 1 and h[0]["reason"] == 1
    assert list(h[0]["f"][:2]) == [R - (A - (U - R)), R]      # L = 10, R = 60
    assert b.counters()[0][orc.K["victims_claimed"]] == A - (U - R)


# --------------------------------------------------------------------------
# 6. Blocking set with several claims (S:385 completeness, S:392 acceptance order)
# --------------------------------------------------------------------------
def test_two_hard_claims_blocking_mask():
    """Two hard residents R0, R1 and an active request A with R0 + R1 + A > U
    and A <= U: the refusal lists both claims in acceptance order
    (S:392), P = R0 + R1 and shortfall = R0 + R1 + A - U."""
    U, R0, R1, A = 100, 30, 25, 60
    ops = [op(INSERT, 0, x=R0), op(INSERT, 1, x=R1), op(SUBMIT, 0, 0, HARD, R0, R0, 0),
           op(SUBMIT, 1, 1, HARD, R1, R1, 0), op(ADMIT, 0, 2, 0, 16 * A, 16 * A, 0)]
    _, evs = _run([make_cfg(U)], [ops], N=U)
    ref = evs[0][evs[0]["type"] == orc.E_ACTIVE_REFUSED]
    assert len(ref) == 1
    r = ref[0]
    assert r["reason"] == orc.WHY_PROTECTED_RESIDENT and r["mask"] == 0b11
    assert list(r["f"]) == [R0 + R1, A, U, R0 + R1 + A - U]
    rendered = orc.render_refusal_json(r, {0: "active"}, {0: "claim:a", 1: "claim:b"})
    assert rendered["blocking_claim_ids"] == ["claim:a", "claim:b"]
    assert rendered["resident_plus_active_blocks"] == R0 + R1 + A


def test_blocking_mask_closed_forms_sweep():
    """Sweep over (U, R_i, modes, F_i) with 3 claims on 3 objects: P counts
    only obligated claims' positions < F (G12); the mask is exactly the
    obligated live claims with F >= 1 cached position; soft / best-effort /
    demoted claims never block; the refusal reason is PROTECTED_RESIDENT iff
    A <= U and P > 0 (G7)."""
    rng = random.Random(7)
    cfgs, lists, exp = [], [], []
    for _ in range(600):
        U = rng.randint(8, 300)
        n = [rng.randint(1, max(1, U // 4)) for _ in range(3)]
        modes = [rng.choice([HARD, DEMOTABLE, OFFLOADABLE, EXPIRING, SOFT, BEST_EFFORT])
                 for _ in range(3)]
        Fs = [rng.randint(1, n[i] + 3) for i in range(3)]
        demote = [rng.random() < 0.2 for _ in range(3)]
        ops = [op(INSERT, i, x=n[i]) for i in range(3)]
        for i in range(3):
            ops.append(op(SUBMIT, i, i, modes[i], Fs[i], 1, 100 if modes[i] == EXPIRING else 0))
        for i in range(3):
            if demote[i]:
                ops.append(op(DEMOTE, i))
        A = rng.randint(1, U + 10)
        ops.append(op(ADMIT, 0, 3, 0, 16 * A, 16 * A, 0))
        prot = [0 if (demote[i] or modes[i] not in OBLIGATED) else min(Fs[i], n[i])
                for i in range(3)]
        P = sum(prot)
        mask = sum(1 << i for i in range(3) if prot[i] > 0)
        if P + A <= U:
            want = None
        elif A <= U and P > 0:
            want = (orc.WHY_PROTECTED_RESIDENT, mask, [P, A, U, P + A - U])
        else:
            want = (orc.WHY_ACTIVE_CAPACITY, 0, [P, A, U, P + A - U])
        if sum(n) > U:
            continue
        cfgs.append(make_cfg(U))
        lists.append(ops)
        exp.append(want)
    _, evs = _run(cfgs, lists, N=300)
    seen = set()
    for i, want in enumerate(exp):
        ref = evs[i][evs[i]["type"] == orc.E_ACTIVE_REFUSED]
        if want is None:
            assert len(ref) == 0, i
            continue
        assert len(ref) == 1, i
        got = (int(ref[0]["reason"]), int(ref[0]["mask"]), [int(v) for v in ref[0]["f"]])
        assert got == want, i
        seen.add((got[0], bin(got[1]).count("1")))
    # every shape was exercised: capacity refusals and masks of 1, 2 and 3 claims
    assert {(orc.WHY_ACTIVE_CAPACITY, 0), (orc.WHY_PROTECTED_RESIDENT, 1),
            (orc.WHY_PROTECTED_RESIDENT, 2), (orc.WHY_PROTECTED_RESIDENT, 3)} <= seen


def _protected_from_views(st, cfg, t):
    """Protected cached blocks per claim, recomputed from the raw state views
    (blocks, objects, claims, requests) at the start of step t's op: a cached
    block is protected iff its object's bound claim is live (accepted /
    materialized, not expiring at t), obligated, the lowering is CONTRACT,
    pos < F (G12), and no running prefix hit pins it (G29)."""
    if int(cfg["lowering"]) != CONTRACT:
        return {}
    pin = {}
    for r in st["requests"]:
        if int(r["status"]) == orc.R_RUNNING:
            pin[int(r["target"])] = max(pin.get(int(r["target"]), 0), int(r["hit"]))
    out = {}
    for b in st["blocks"]:
        if int(b["res"]) != 1:
            continue
        o = int(b["owner"])
        c = int(st["objects"][o]["claim"])
        if c == 0xFF:
            continue
        cl = st["claims"][c]
        live = int(cl["state"]) in (orc.C_ACCEPTED, orc.C_MATERIALIZED)
        if live and int(cl["D"]) > 0 and int(cl["decision_step"]) + int(cl["D"]) <= t:
            live = False                                       # expires first (G13)
        if (live and int(cl["mode"]) in OBLIGATED and int(b["pos"]) < int(cl["F"])
                and int(b["pos"]) >= pin.get(o, 0)):
            out[c] = out.get(c, 0) + 1
    return out


def _random_tiny_op(rng, U):
    k = rng.choice([INSERT, INSERT, INSERT, SUBMIT, SUBMIT, SUBMIT, ADMIT, HIT_ADMIT, ADVANCE,
                    ADVANCE, ADVANCE, COMPLETE, TOUCH, DEMOTE, NOP])
    if k == INSERT:
        return op(INSERT, rng.randrange(6), x=rng.randint(1, max(1, U // 2)))
    if k == SUBMIT:
        F = rng.randint(1, U)
        return op(SUBMIT, rng.randrange(8), rng.randrange(6),
                  rng.choice([HARD, HARD, OFFLOADABLE, DEMOTABLE, EXPIRING, SOFT, BEST_EFFORT]),
                  F, rng.randint(1, F), rng.randint(1, 30))
    if k in (ADMIT, HIT_ADMIT):
        return op(k, rng.randrange(2), rng.randrange(6), rng.randrange(2) if k == ADMIT else 0,
                  rng.randint(1, 16 * U), rng.choice([16, 32, 64]), rng.randint(0, 20))
    if k in (ADVANCE, COMPLETE):
        return op(k, rng.randrange(2))
    if k == TOUCH:
        return op(TOUCH, rng.randrange(6))
    if k == DEMOTE:
        return op(DEMOTE, rng.randrange(8))
    return op(NOP)


def test_blocking_mask_completeness_random():
    """Random tiny traces with up to 8 claims, stepped one op at a time: every
    refusal / deferral / insert refusal lists exactly the claims that hold at
    least one protected block at that moment, ascending slot ("every
    ... lists a non-empty blocking_claim_ids set", S:392 all of them), and
    its P field is their total.  Some refusals carry >= 2 blocking claims."""
    n_multi = checked = 0
    for seed in range(96):
        rng = random.Random(1000 + seed)
        U = rng.randint(6, 24)
        cfg = make_cfg(U, CONTRACT, rng.choice([PEAK, NONE]), rng.randint(0, 2), 0)
        b = orc.OracleBatch(np.stack([cfg]), N=24, C=8, Q=2, O=6)
        for t in range(200):
            rec = _random_tiny_op(rng, U)
            before = b.export(0)
            n0 = b.lib.oracle_batch_num_events(b.h)
            assert b.run(pack_ops([[rec]]), check=True) == 0
            for x in b.events()[n0:]:
                if int(x["type"]) not in (orc.E_ACTIVE_REFUSED, orc.E_ACTIVE_DEFERRED,
                                          orc.E_RESIDENT_INSERT_REFUSED):
                    continue
                prot = _protected_from_views(before, cfg, t)
                P, A = int(x["f"][0]), int(x["f"][1])
                assert P == sum(prot.values()), (seed, t)
                if A <= U and P > 0:
                    assert int(x["mask"]) == sum(1 << c for c in prot), (seed, t)
                    n_multi += len(prot) >= 2
                else:
                    assert int(x["mask"]) == 0, (seed, t)
                checked += 1
    assert checked > 50 and n_multi > 0, (checked, n_multi)
