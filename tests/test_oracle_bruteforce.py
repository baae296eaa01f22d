"""Brute-force pins of the oracle on tiny pools.

1. Victim choice (S:176, S:649(e)): for pools of <= 12 blocks, every
   allocation the oracle makes equals the exhaustive search over all legal
   victim sets of the right size, choosing the set whose sorted
   (class, key) vector is lexicographically smallest -- free blocks first
   (P:947-952), protected blocks never, then oldest stamp
   (G1), soft-priority last (G6).  Positions follow block-id order (G24).
   Blocks pinned by a running prefix hit (f3, G28) are never candidates.
2. Exhaustive tiny traces: every op sequence of length 5 over a 13-op
   alphabet on a 6-block pool, under two policies, runs with the oracle's
   debug invariants (I1-I9) on, and the event-level invariants I4-I7 hold.
"""
import itertools
import random

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2605_24259_b200.gen import (ADMIT, ADVANCE, COMPLETE, CONTRACT, DEMOTABLE, DEMOTE,
                                       EXPIRING, HARD, HIT_ADMIT, INSERT, NATIVE, NONE, NOP,
                                       OFFLOADABLE, PEAK, SOFT,
                                       SOFT_LOWERING, SUBMIT, TOUCH, BEST_EFFORT, make_cfg, op,
                                       pack_ops)

OBLIGATED = {HARD, DEMOTABLE, OFFLOADABLE, EXPIRING}


def _candidates(view, cfg):
    """(class, key) of every legal candidate block, from the state view."""
    blocks, claims, objs = view["blocks"], view["claims"], view["objects"]
    U = int(cfg["U"])
    # pinned prefix per object: the longest running prefix hit on it (f3, G28)
    pin = {}
    for r in view["requests"]:
        if int(r["status"]) == orc.R_RUNNING:
            o = int(r["target"])
            pin[o] = max(pin.get(o, 0), int(r["hit"]))
    out = {}
    for b in range(U):
        res = int(blocks[b]["res"])
        if res == 0:
            out[b] = (0, b)
            continue
        if res == 2:
            continue
        o = int(blocks[b]["owner"])
        if int(blocks[b]["pos"]) < pin.get(o, 0):
            continue                                   # pinned by a running hit: never a victim
        c = int(objs[o]["claim"])
        claimed = (c != 0xFF and int(claims[c]["state"]) in (1, 2)
                   and int(blocks[b]["pos"]) < int(claims[c]["F"]))
        mode = int(claims[c]["mode"]) if c != 0xFF else -1
        low = int(cfg["lowering"])
        if claimed and low == CONTRACT and mode in OBLIGATED:
            continue                                   # protected: never a victim
        cls = 1
        if claimed and low != NATIVE and (mode == SOFT or (low == SOFT_LOWERING and mode in OBLIGATED)):
            cls = 2
        out[b] = (cls, int(blocks[b]["seq"]))
    return out


def _exhaustive_best(cands, k):
    best, best_key = None, None
    for subset in itertools.combinations(sorted(cands), k):
        key = sorted(cands[b] for b in subset)
        if best_key is None or key < best_key:
            best, best_key = set(subset), key
    return best


def _random_tiny_ops(rng, U, T):
    ops = []
    for _ in range(T):
        k = rng.choice([INSERT, INSERT, SUBMIT, ADMIT, ADVANCE, ADVANCE, ADVANCE, COMPLETE,
                        TOUCH, DEMOTE, NOP, HIT_ADMIT])
        if k == INSERT:
            ops.append(op(INSERT, rng.randrange(4), x=rng.randint(1, U)))
        elif k == SUBMIT:
            F = rng.randint(1, U)
            ops.append(op(SUBMIT, rng.randrange(3), rng.randrange(4),
                          rng.choice([SOFT, HARD, DEMOTABLE, OFFLOADABLE, EXPIRING, BEST_EFFORT]),
                          F, rng.randint(1, F), rng.randint(1, 6)))
        elif k == ADMIT:
            ops.append(op(ADMIT, rng.randrange(2), rng.randrange(4), rng.randrange(2),
                          rng.randint(1, 16 * U), rng.choice([16, 32, 48]), rng.randint(0, 20)))
        elif k == HIT_ADMIT:
            ops.append(op(HIT_ADMIT, rng.randrange(2), rng.randrange(4), 0,
                          rng.randint(1, 16 * U), rng.choice([16, 32, 48]), rng.randint(0, 20)))
        elif k in (ADVANCE, COMPLETE):
            ops.append(op(k, rng.randrange(2)))
        elif k == TOUCH:
            ops.append(op(TOUCH, rng.randrange(4)))
        elif k == DEMOTE:
            ops.append(op(DEMOTE, rng.randrange(3)))
        else:
            ops.append(op(NOP))
    return ops


@pytest.mark.parametrize("seed", range(40))
def test_victim_choice_equals_exhaustive_search(seed):
    rng = random.Random(seed)
    U = rng.randint(3, 12)
    cfg = make_cfg(U, rng.choice([CONTRACT, CONTRACT, SOFT_LOWERING, NATIVE]),
                   rng.choice([PEAK, NONE]), rng.randint(0, 2), rng.randint(0, 1))
    ops = _random_tiny_ops(rng, U, 80)
    b = orc.OracleBatch(np.stack([cfg]), N=12, C=3, Q=2, O=4)
    checked = 0
    for s, rec in enumerate(ops):
        before = b.export(0)
        b.run(pack_ops([[rec]]), check=True)
        after = b.export(0)
        assert b.violation(0) == 0
        kind = rec[0]
        bb, ab = before["blocks"], after["blocks"]
        if kind == ADVANCE:
            r = rec[1]
            was = {i for i in range(U) if bb[i]["res"] == 2 and bb[i]["owner"] == r}
            now = {i for i in range(U) if ab[i]["res"] == 2 and ab[i]["owner"] == r}
            if not now or not (now - was):
                continue
            taken = now - was
            base = int(before["requests"][r]["live"])
        elif kind == INSERT:
            o = rec[1]
            if before["objects"][o]["live"] or not after["objects"][o]["live"]:
                continue
            taken = {i for i in range(U) if ab[i]["res"] == 1 and ab[i]["owner"] == o}
            base = 0
        else:
            continue
        # claim states at allocation time: this step's expiry and auto-demotion
        # happen before the allocation, the post-op harm pass after it
        claims = after["claims"].copy()
        for c in range(len(claims)):
            if claims[c]["state"] == orc.C_HARMED and before["claims"][c]["state"] != orc.C_HARMED:
                claims[c] = before["claims"][c]
        view = dict(before)
        view["claims"] = claims
        cands = _candidates(view, cfg)
        assert taken == _exhaustive_best(cands, len(taken)), (seed, s)
        for i, blk in enumerate(sorted(taken)):          # G24 block-id order
            assert int(ab[blk]["pos"]) == base + i
        checked += 1
    assert checked >= 1


ALPHABET = [
    op(INSERT, 0, x=2), op(INSERT, 1, x=3), op(SUBMIT, 0, 0, HARD, 2, 2, 0),
    op(SUBMIT, 1, 1, SOFT, 3, 2, 0), op(SUBMIT, 1, 1, DEMOTABLE, 3, 2, 2),
    op(ADMIT, 0, 2, 1, 48, 16, 2), op(ADMIT, 1, 3, 0, 64, 64, 0), op(ADVANCE, 0),
    op(ADVANCE, 1), op(COMPLETE, 0), op(DEMOTE, 0), op(TOUCH, 0),
    op(HIT_ADMIT, 1, 1, 0, 40, 16, 1),                      # f3: hit on object 1's prefix
]


def _event_invariants(ev, n, lowering):
    idx = np.searchsorted(ev["trace"], np.arange(n + 1))
    for i in range(n):
        e = ev[idx[i]:idx[i + 1]]
        acc, mat, released = set(), set(), set()
        for x in e:
            t, slot = int(x["type"]), int(x["slot"])
            if t == orc.E_CLAIM_ACCEPTED:
                acc.add(slot)
            elif t == orc.E_CLAIM_MATERIALIZED:
                assert slot in acc
                mat.add(slot)
            elif t in (orc.E_CLAIM_DEMOTED, orc.E_CLAIM_EXPIRED):
                assert slot in acc
                released.add(slot)
            elif t == orc.E_CLAIM_HARMED:
                assert slot in acc and slot in mat                   # I5
                assert not (lowering == CONTRACT and x["reason"] == 1)  # I4
            elif t in (orc.E_ACTIVE_REFUSED, orc.E_ACTIVE_DEFERRED, orc.E_RESIDENT_INSERT_REFUSED):
                P, A, U, short = (int(v) for v in x["f"])
                assert short == P + A - U and short > 0                  # I7
                assert (x["mask"] != 0) == (x["reason"] == orc.WHY_PROTECTED_RESIDENT)
                if x["mask"]:
                    assert all(c in acc for c in range(32) if x["mask"] >> c & 1)
            elif t == orc.E_VICTIMS:
                if x["f"][1] > 0:
                    assert released                                     # I6


@pytest.mark.parametrize("policy", ["contract", "native"])
def test_exhaustive_tiny_traces(policy):
    seqs = np.array(list(itertools.product(range(len(ALPHABET)), repeat=5)), dtype=np.int64)
    n = len(seqs)
    alpha = pack_ops([ALPHABET])[:, 0]
    ops = alpha[seqs.T]                                    # [5, n]
    if policy == "contract":
        cfg = make_cfg(6, CONTRACT, PEAK, defer_budget=1, auto_demote=1)
    else:
        cfg = make_cfg(6, NATIVE, NONE)
    cfgs = np.repeat(np.stack([cfg]), n)
    b = orc.OracleBatch(cfgs, N=6, C=2, Q=2, O=4)
    bad = b.run(np.ascontiguousarray(ops), nthreads=8, check=True)
    assert bad == 0
    _event_invariants(b.events(), n, int(cfg["lowering"]))
