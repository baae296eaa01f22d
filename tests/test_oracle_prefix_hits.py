"""Pins of the oracle's prefix-hit extension (G28-G30).

A prefix hit is the "future materialization surface" of P:303-304 used by a
live request: a request whose prompt begins with object o's content shares
the surviving leading prefix of o instead of allocating it, and
pins it while it runs (the BlockPool.touch protection of P:953).  The paper
fixes no hit arithmetic, so these pins are closed forms that follow from the
contract boundary P + A <= U once the shared blocks count as active
live KV exactly once (G29), checked against brute-force sweeps:

* hard claim R + hit request of A blocks: served iff R + A - h <= U, else
  refused with (P, A, U, shortfall) = (R, A - h, U, R + A - h - U);
* native pool: the hit saves h blocks of eviction, victims come only from
  positions >= h, leading(o) = R - max(0, A - h - (U - R));
* refcounts: pins of several requests on one object release to the longest
  remaining hit; protected blocks under a pin count in A, not in P;
* a deferral drops the hit (restart at token 0, G9).
"""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2605_24259_b200.gen import (ADMIT, ADVANCE, COMPLETE, CONTRACT, HARD, HIT_ADMIT, INSERT,
                                       NATIVE, NONE, PEAK, SUBMIT, TOUCH, make_cfg, op, pack_ops)


def _run(cfg, ops, N, **dims):
    b = orc.OracleBatch(np.stack([cfg]), N=N, **dims)
    bad = b.run(pack_ops([ops]), check=True)
    assert bad == 0 and b.violation(0) == 0
    return b


def _types(ev):
    return [orc.EVENT_NAMES[int(t)] for t in ev["type"]]


def test_hit_makes_paper_case_feasible():
    """P:281-295 / P:1069-1079: 60 protected + 70 active > 80 is refused.  If
    the active request's prompt begins with the resident object, its first
    60 blocks are the resident blocks: 60 + 70 - 60 = 70 <= 80, so it is
    served with no victim and the claim stays materialized."""
    cfg = make_cfg(80, CONTRACT, PEAK)
    ops = [op(INSERT, 0, x=60), op(SUBMIT, 0, 0, HARD, 60, 60, 0),
           op(HIT_ADMIT, 0, 0, 0, 1120, 1120, 0), op(ADVANCE, 0), op(COMPLETE, 0), op(TOUCH, 0)]
    b = _run(cfg, ops, 80)
    ev = b.events()
    assert _types(ev) == ["claim_accepted", "claim_materialized", "prefix_hit",
                          "write_admission_denied", "request_served", "reuse_probe"]
    hit = ev[ev["type"] == orc.E_PREFIX_HIT][0]
    assert list(hit["f"]) == [0, 60, 960, 60]
    ctr = b.counters()[0]
    assert ctr[orc.K["victims_ordinary"]] + ctr[orc.K["victims_claimed"]] == 0
    assert ctr[orc.K["blocks_allocated"]] == 60 + 10            # insert + exclusive tail
    assert ctr[orc.K["prefix_hits"]] == 1 and ctr[orc.K["hit_tokens"]] == 960
    st = b.export(0)
    assert st["claims"][0]["state"] == orc.C_MATERIALIZED
    assert st["claims"][0]["protected_blocks"] == 60             # pins released at completion
    assert st["header"]["alive"] == 0 and st["header"]["protected_total"] == 60


def test_pinned_protected_blocks_count_in_A_not_P():
    """G29: while the hit request runs, its 60 shared blocks are active live
    KV (A) and not protected resident KV (P): P + A stays the number of
    non-candidate blocks."""
    cfg = make_cfg(80, CONTRACT, PEAK)
    ops = [op(INSERT, 0, x=60), op(SUBMIT, 0, 0, HARD, 60, 60, 0),
           op(HIT_ADMIT, 0, 0, 0, 16 * 40 + 1, 64, 0)]
    b = _run(cfg, ops, 80)
    st = b.export(0)
    assert st["requests"][0]["hit"] == 40 and st["requests"][0]["done"] == 640
    assert st["header"]["protected_total"] == 20 and st["header"]["alive"] == 40
    assert st["claims"][0]["protected_blocks"] == 20


@pytest.mark.parametrize("seed", range(6))
def test_hard_claim_hit_boundary_closed_form(seed):
    """served iff R + A - h <= U with h = min(R, A - 1); otherwise the PEAK
    check refuses with the capacity proof (R, A - h, U, R + A - h - U)."""
    rng = np.random.default_rng(seed)
    for _ in range(40):
        R = int(rng.integers(1, 100))
        A = int(rng.integers(1, 120))
        U = int(rng.integers(R, R + A + 10))
        h = min(R, A - 1)
        cfg = make_cfg(U, CONTRACT, PEAK)
        ops = [op(INSERT, 0, x=R), op(SUBMIT, 0, 0, HARD, R, R, 0),
               op(HIT_ADMIT, 0, 0, 0, 16 * A, 16 * A, 0), op(ADVANCE, 0), op(COMPLETE, 0)]
        b = _run(cfg, ops, max(U, 1))
        ev = b.events()
        served = R + A - h <= U
        assert (orc.E_REQUEST_SERVED in ev["type"]) == served, (R, A, U)
        if not served:
            ref = ev[ev["type"] == orc.E_ACTIVE_REFUSED][0]
            assert list(ref["f"]) == [R, A - h, U, R + A - h - U]
            assert ref["reason"] == (orc.WHY_PROTECTED_RESIDENT if A - h <= U else orc.WHY_ACTIVE_CAPACITY)
        st = b.export(0)
        assert st["claims"][0]["state"] == orc.C_MATERIALIZED   # never harmed (I4)
        assert st["header"]["alive"] == 0


@pytest.mark.parametrize("seed", range(6))
def test_native_hit_saves_eviction_closed_form(seed):
    """NATIVE pool: R resident blocks, a hit request of A blocks.  Victims
    come only from the unpinned tail: v = max(0, A - h - (U - R)), and the
    resident keeps leading R - v >= h (without the hit: R - max(0, A - (U - R)))."""
    rng = np.random.default_rng(100 + seed)
    for _ in range(40):
        U = int(rng.integers(4, 200))
        R = int(rng.integers(1, U + 1))
        A = int(rng.integers(1, U + 1))
        h = min(R, A - 1)
        cfg = make_cfg(U, NATIVE, NONE)
        ops = [op(INSERT, 0, x=R), op(HIT_ADMIT, 0, 0, 0, 16 * A, 16 * A, 0), op(ADVANCE, 0),
               op(TOUCH, 0)]
        b = _run(cfg, ops, U)
        v = max(0, A - h - (U - R))
        ctr = b.counters()[0]
        assert ctr[orc.K["victims_ordinary"]] == v, (U, R, A)
        probe = b.events()[b.events()["type"] == orc.E_REUSE_PROBE][0]
        assert probe["f"][1] == R - v and R - v >= h


def test_refcounted_pins_release_to_longest_remaining_hit():
    cfg = make_cfg(64, CONTRACT, NONE)
    ops = [op(INSERT, 0, x=20), op(SUBMIT, 0, 0, HARD, 12, 12, 0),
           op(HIT_ADMIT, 0, 0, 0, 16 * 5 + 1, 16, 0), op(HIT_ADMIT, 1, 0, 0, 16 * 15 + 1, 16, 0)]
    b = orc.OracleBatch(np.stack([cfg]), N=64)
    assert b.run(pack_ops([ops]), check=True) == 0
    st = b.export(0)
    assert st["header"]["alive"] == 15                        # pin prefix 15, counted once
    assert st["header"]["protected_total"] == 0               # positions < 12 all pinned
    assert b.run(pack_ops([[op(COMPLETE, 1)]]), check=True) == 0
    st = b.export(0)
    assert st["header"]["alive"] == 5 and st["header"]["protected_total"] == 12 - 5
    assert b.run(pack_ops([[op(COMPLETE, 0)]]), check=True) == 0
    st = b.export(0)
    assert st["header"]["alive"] == 0 and st["header"]["protected_total"] == 12


def test_pinned_prefix_is_never_a_victim_under_pressure():
    """A second request needing space evicts the unpinned tail only; when the
    unpinned candidates cannot cover it, it is refused (ACTIVE_CAPACITY: no
    claim) instead of taking a pinned block."""
    U = 32
    cfg = make_cfg(U, NATIVE, PEAK)
    ops = [op(INSERT, 0, x=24), op(HIT_ADMIT, 0, 0, 0, 16 * 10 + 1, 16, 0),
           op(ADMIT, 1, 1, 0, 16 * 20, 16 * 20, 0), op(ADVANCE, 1), op(TOUCH, 0),
           op(ADMIT, 2, 2, 0, 16 * 25, 16, 0)]
    b = _run(cfg, ops, U, C=4, Q=4, O=4)
    ev = b.events()
    probe = ev[ev["type"] == orc.E_REUSE_PROBE][0]
    assert probe["f"][1] == 24 - (20 - 8)                    # 8 free, 12 from the tail, 10 pinned stay
    ref = ev[ev["type"] == orc.E_ACTIVE_REFUSED][0]
    assert ref["reason"] == orc.WHY_ACTIVE_CAPACITY and ref["mask"] == 0
    assert list(ref["f"]) == [0, 10 + 20 + 25, U, 10 + 20 + 25 - U]


def test_deferral_drops_the_hit():
    """G9 + G28: an infeasible hit admission is deferred without pinning; the
    retry re-checks the full peak and restarts at token 0 with no hit."""
    cfg = make_cfg(40, CONTRACT, PEAK, defer_budget=1)
    ops = [op(INSERT, 0, x=30), op(SUBMIT, 0, 0, HARD, 30, 30, 0),
           op(HIT_ADMIT, 0, 0, 0, 16 * 50, 64, 0)]
    b = _run(cfg, ops, 40)
    ev = b.events()
    d = ev[ev["type"] == orc.E_ACTIVE_DEFERRED][0]
    assert list(d["f"]) == [30, 50 - 30, 40, 30 + 20 - 40]
    st = b.export(0)
    assert st["requests"][0]["status"] == orc.R_DEFERRED
    assert st["requests"][0]["hit"] == 0 and st["header"]["alive"] == 0
    assert b.run(pack_ops([[op(ADVANCE, 0)]]), check=True) == 0
    ev = b.events()
    r = ev[ev["type"] == orc.E_ACTIVE_REFUSED][0]
    assert list(r["f"]) == [30, 50, 40, 40]                   # full peak, no hit


def test_hit_admit_errors():
    cfg = make_cfg(16, CONTRACT, PEAK)
    ops = [op(HIT_ADMIT, 0, 0, 1, 32, 16, 0),                 # c must be 0
           op(HIT_ADMIT, 0, 0, 0, 0, 16, 0),                  # prompt < 1
           op(HIT_ADMIT, 0, 0, 0, 32, 16, 0),                 # object not live: h = 0
           op(HIT_ADMIT, 0, 0, 0, 32, 16, 0)]                 # duplicate slot
    b = _run(cfg, ops, 16)
    ev = b.events()
    errs = ev[ev["type"] == orc.E_OP_ERROR]
    assert [int(e["reason"]) for e in errs] == [orc.ERR_INVALID_ARG, orc.ERR_INVALID_ARG,
                                                orc.ERR_DUPLICATE_SLOT]
    hit = ev[ev["type"] == orc.E_PREFIX_HIT][0]
    assert list(hit["f"]) == [0, 0, 0, 0]


def test_auto_demotion_during_hit_peak_check_then_backstop():
    """G29's reading of a PEAK check that auto-demotes the hit object's own
    claim: at HIT_ADMIT, P = 60, A = 0, need = (75-60)
    + 60 - 60 = 15 -> 75 > 70, so the demotable claim is demoted (P' = 0 fits);
    the 60 hit blocks are then pinned unprotected (A = 60).  The first chunk
    needs 15 own blocks: 0 + 60 + 15 = 75 > 70 -> refused by the per-allocation
    backstop with the capacity proof (0, 75, 70, 5), ACTIVE_CAPACITY (P = 0)."""
    cfg = make_cfg(70, CONTRACT, PEAK, defer_budget=0, auto_demote=1)
    from paper_2605_24259_b200.gen import DEMOTABLE
    ops = [op(INSERT, 0, x=60), op(SUBMIT, 0, 0, DEMOTABLE, 60, 60, 0),
           op(HIT_ADMIT, 0, 0, 0, 16 * 75, 16 * 75, 0), op(ADVANCE, 0)]
    b = _run(cfg, ops, 70)
    ev = b.events()
    assert _types(ev) == ["claim_accepted", "claim_materialized", "claim_demoted", "prefix_hit",
                          "active_request_refused"]
    assert ev[2]["reason"] == 1 and list(ev[2]["f"][:2]) == [0, 60]     # auto, 60 protected released
    assert list(ev[3]["f"]) == [0, 60, 960, 60]
    ref = ev[4]
    assert ref["reason"] == orc.WHY_ACTIVE_CAPACITY and ref["mask"] == 0
    assert list(ref["f"]) == [0, 75, 70, 5]
    st = b.export(0)
    assert st["header"]["alive"] == 0 and st["requests"][0]["hit"] == 0   # pins dropped
    assert st["claims"][0]["state"] == orc.C_DEMOTED
