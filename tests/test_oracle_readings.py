"""Pins of the readings DESIGN.md takes where the paper is silent (the ledger),
each against a closed form written from the reading or a property the paper
states -- so that a change of the oracle's ordering rules fails a test:

* G1 tail-first stamps: "survived positions form leading ranges"
  (the oracle's check mode asserts it as I11 after every op, on every random
  and exhaustive trace); here also explicitly after interleaved evictions.
* G10 auto-demotion: demotable claims holding protected blocks, ascending slot,
  the shortest prefix that makes P + A <= U; none when even all do not help.
* G18 event order within a step: expiries (by slot), then the op's events in
  emission order (auto-demotions before VICTIMS), then materialized / harmed
  (by slot).
"""
import random

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2605_24259_b200.gen import (ADMIT, ADVANCE, COMPLETE, CONTRACT, DEMOTABLE, DEMOTE,
                                       EXPIRING, HARD, INSERT, NATIVE, NOP, PEAK, SOFT, SUBMIT,
                                       TOUCH, make_cfg, op, pack_ops)


def _run(cfgs, lists, N, C=16):
    b = orc.OracleBatch(np.stack(cfgs), N=N, C=C)
    assert b.run(pack_ops(lists), check=True) == 0
    ev = b.events()
    idx = np.searchsorted(ev["trace"], np.arange(len(cfgs) + 1))
    return b, [ev[idx[i]:idx[i + 1]] for i in range(len(cfgs))]


def test_G1_survivors_form_leading_ranges_P615():
    """Three objects cached at different times, then an active request that
    evicts across them: every object keeps exactly a leading range of its
    positions, the oldest object losing first (tail first within each)."""
    U = 100
    seq = [op(INSERT, 0, x=30), op(INSERT, 1, x=30), op(TOUCH, 0), op(INSERT, 2, x=30),
           op(ADMIT, 0, 3, 0, 16 * 50, 16 * 50, 0), op(ADVANCE, 0)]
    b, evs = _run([make_cfg(U, NATIVE)], [seq], U)
    st = b.export(0)
    blocks, objs = st["blocks"], st["objects"]
    for o in range(3):
        pos = sorted(int(x["pos"]) for x in blocks if x["res"] == 1 and x["owner"] == o)
        assert pos == list(range(len(pos))), (o, pos)            # a leading range
        assert int(objs[o]["leading"]) == len(pos)
    # 10 free + 40 evicted: object 1 (stamped oldest: object 0 was touched) loses all
    # 30, then object 0 loses its 10 tail blocks; object 2 (newest) keeps everything
    assert [int(objs[o]["leading"]) for o in range(3)] == [20, 0, 30]


@pytest.mark.parametrize("seed", range(30))
def test_G10_auto_demotion_prefix_closed_form(seed):
    """k demotable hard-protected residents of sizes g_0..g_{k-1} (slots in
    submission order) and an active request of A blocks at U: with P = sum g,
    the oracle demotes exactly the shortest ascending-slot prefix j with
    P - (g_0 + ... + g_{j-1}) + A <= U, emitting CLAIM_DEMOTED(auto) for each
    before any VICTIMS event; if no prefix suffices it demotes none and refuses."""
    rng = random.Random(seed)
    k = rng.randint(1, 5)
    g = [rng.randint(1, 20) for _ in range(k)]
    P = sum(g)
    U = rng.randint(P + 1, P + 40)
    A = rng.randint(1, U)
    seq = []
    for i in range(k):
        seq += [op(INSERT, i, x=g[i]), op(SUBMIT, i, i, DEMOTABLE, g[i], g[i], 0)]
    seq += [op(ADMIT, 0, 10, 0, 16 * A, 16 * A, 0), op(ADVANCE, 0)]
    b, evs = _run([make_cfg(U, CONTRACT, PEAK, auto_demote=1)], [seq], U)
    e = evs[0]
    j = next((j for j in range(1, k + 1) if P - sum(g[:j]) + A <= U), None)
    if P + A <= U:
        j = 0
    dem = e[e["type"] == orc.E_CLAIM_DEMOTED]
    if j is None:
        assert len(dem) == 0 and len(e[e["type"] == orc.E_ACTIVE_REFUSED]) == 1
        return
    assert [int(x["slot"]) for x in dem] == list(range(j)), (g, U, A)
    assert all(int(x["reason"]) == 1 for x in dem)                 # auto
    assert [int(x["f"][1]) for x in dem] == g[:j]                  # protected blocks released
    vic = e[e["type"] == orc.E_VICTIMS]
    for x in vic:                                                  # demotions precede the loss
        assert all((d["step"], d["seq"]) < (x["step"], x["seq"]) for d in dem)


def test_G18_event_order_within_a_step():
    """One step in which (1) two claims expire, (2) the op is an ADVANCE
    whose allocation evicts the unprotected tail of a materialized soft
    claim's object, and (3) that claim is harmed: the events of the step are
    EXPIRED(slot 1), EXPIRED(slot 2), VICTIMS, HARMED(slot 0), with seq 0..3."""
    U = 64
    seq = [op(INSERT, 0, x=40), op(SUBMIT, 0, 0, SOFT, 40, 40, 0),
           op(INSERT, 1, x=4), op(SUBMIT, 1, 1, EXPIRING, 4, 4, 4),
           op(INSERT, 2, x=4), op(SUBMIT, 2, 2, HARD, 4, 4, 2),
           op(ADMIT, 0, 3, 0, 16 * 30, 16 * 30, 0), op(ADVANCE, 0)]
    # claim 1 (decided at step 3, D = 4) and claim 2 (step 5, D = 2) both expire at step 7
    b, evs = _run([make_cfg(U, CONTRACT, PEAK)], [seq], U)
    e = evs[0]
    last = e[e["step"] == 7]
    kinds = [(int(x["type"]), int(x["slot"])) for x in last]
    assert kinds == [(orc.E_CLAIM_EXPIRED, 1), (orc.E_CLAIM_EXPIRED, 2), (orc.E_VICTIMS, 0),
                     (orc.E_CLAIM_HARMED, 0)], kinds
    assert [int(x["seq"]) for x in last] == [0, 1, 2, 3]
    assert int(last[3]["reason"]) == 0                             # soft: not obligated
