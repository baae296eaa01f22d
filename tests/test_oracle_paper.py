"""Pins of the oracle against the numbers the paper prints (tests/golden/).

Every assertion here compares the oracle with a value from PAPER.md, cited.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2605_24259_b200 import gen
from paper_2605_24259_b200.gen import litmus
from paper_2605_24259_b200.gen import (ADMIT, ADVANCE, COMPLETE, CONTRACT, HARD, INSERT, NATIVE,
                                       NONE, PEAK, SUBMIT, TOUCH, make_cfg, op, pack_ops)

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PAPER = json.load(open(os.path.join(GOLD, "paper_numbers.json")))


def _events_of(ev, trace):
    return ev[ev["trace"] == trace]


def _types(ev):
    return [orc.EVENT_NAMES[int(t)] for t in ev["type"]]


def test_paper_litmus_hard_claim_refusal_json():
    """configs[0] (i): hard claim -> active refusal attributed to the claim;
    the rendered event equals the paper's JSON field for field."""
    cfgs, ops, _ = litmus.paper_litmus()
    b, bad = orc.run_oracle(cfgs, ops, N=80, check=True)
    assert bad == 0
    ev = _events_of(b.events(), 0)
    assert _types(ev) == ["claim_accepted", "claim_materialized", "active_request_refused",
                          "reuse_probe"]
    refusal = ev[ev["type"] == orc.E_ACTIVE_REFUSED][0]
    rendered = orc.render_refusal_json(refusal, {0: "active"}, {0: "claim:resident"})
    golden = json.load(open(os.path.join(GOLD, "refusal_event_P1069.json")))
    assert rendered == golden
    # the resident survives intact: TOUCH sees 60 leading blocks = 960 tokens, satisfied
    probe = ev[ev["type"] == orc.E_REUSE_PROBE][0]
    assert probe["f"][1] == 60 and probe["f"][2] == 960 and probe["reason"] == 1
    st = b.export(0)
    assert st["claims"][0]["state"] == orc.C_MATERIALIZED
    assert st["requests"][0]["status"] == orc.R_REFUSED


def test_paper_blockpool_probe_native():
    """configs[0] (ii): native 60/70/80 BlockPool probe -- 70 allocated, 50
    resident evicted, 10 remaining (Table 9); write no-admit makes
    the bulky repeat reuse 0 tokens (Table 7); L1: 50 victims, 0
    accepted, 0 harm."""
    pin = PAPER["blockpool_probe_P947_952"]
    cfgs, ops, _ = litmus.paper_litmus()
    b, bad = orc.run_oracle(cfgs, ops, N=80, check=True)
    assert bad == 0
    ctr = b.counters()[1]
    assert ctr[orc.K["blocks_allocated"]] == 60 + pin["allocated"]   # insert 60 + active 70
    assert ctr[orc.K["victims_ordinary"]] == pin["resident_evicted"]
    assert ctr[orc.K["accepted"]] == PAPER["L1_P1026_1028"]["accepted"]
    assert ctr[orc.K["harmed_obligated"]] + ctr[orc.K["harmed_unobligated"]] == 0
    ev = _events_of(b.events(), 1)
    probes = ev[ev["type"] == orc.E_REUSE_PROBE]
    assert probes[0]["f"][1] == pin["resident_remaining"]          # leading(o0) = 10
    assert probes[0]["f"][2] == 16 * pin["resident_remaining"]
    assert probes[1]["f"][2] == PAPER["write_no_admit_P862_865"]["no_admit_repeat_tokens"]
    assert "write_admission_denied" in _types(ev)


def test_paper_native_claim_made_visible():
    """configs[0] (iii): the same loss with an accepted hard claim under the
    native lowering is claim harm (Table 4): HARMED with L=10,
    R=60 and the obligated flag; the 50 victims are attributed to the claim."""
    cfgs, ops, _ = litmus.paper_litmus()
    b, _ = orc.run_oracle(cfgs, ops, N=80)
    ev = _events_of(b.events(), 2)
    harmed = ev[ev["type"] == orc.E_CLAIM_HARMED]
    assert len(harmed) == 1
    assert list(harmed[0]["f"][:2]) == [10, 60] and harmed[0]["reason"] == 1
    ctr = b.counters()[2]
    assert ctr[orc.K["victims_claimed"]] == 50 and ctr[orc.K["victims_ordinary"]] == 0


def test_write_admit_repeat_is_1120_tokens():
    """Table 7: cache-all active prefill -> immediate bulky repeat
    reusable for 1120 tokens; still 50 resident victims."""
    cfg = make_cfg(80, NATIVE)
    ops = pack_ops([[op(INSERT, 0, x=60), op(ADMIT, 0, 1, 1, 1120, 1120, 0), op(ADVANCE, 0),
                     op(COMPLETE, 0), op(TOUCH, 1), op(TOUCH, 0)]])
    b, bad = orc.run_oracle(np.stack([cfg]), ops, N=80, check=True)
    assert bad == 0
    ev = b.events()
    probes = ev[ev["type"] == orc.E_REUSE_PROBE]
    assert probes[0]["f"][2] == PAPER["write_no_admit_P862_865"]["cache_all_repeat_tokens"]
    assert probes[1]["f"][1] == 10
    assert b.counters()[0][orc.K["victims_ordinary"]] == 50


def test_chunked_prefill_accumulation_20_40_60_70():
    """Table 8: chunks of 20/20/20/10 blocks -> live 20/40/60/70;
    chunking does not bound live KV."""
    pin = PAPER["chunked_prefill_P898_901"]
    prompt = 16 * sum(pin["chunk_blocks"])
    cfg = make_cfg(200, CONTRACT, NONE)
    lives = []
    for k in range(1, 5):
        ops = pack_ops([[op(ADMIT, 0, 1, 0, prompt, 16 * 20, 0)] + [op(ADVANCE, 0)] * k])
        b, bad = orc.run_oracle(np.stack([cfg]), ops, N=200, check=True)
        assert bad == 0
        lives.append(int(b.export(0)["requests"][0]["live"]))
    assert lives == pin["live_after_chunk"]


def test_capacity_sweep_flip_at_130():
    """Capacity sweep: hard exclusion refuses below 130 usable and
    serves at >= 130 with the resident preserved; native / no-admit serve at
    every size and lose resident materialization below 130."""
    pin = PAPER["capacity_sweep_P988_997"]
    cfgs, ops, params = litmus.capacity_sweep(pin["resident"], pin["active"], range(75, 136))  # S:647 sweep 75..135
    b, bad = orc.run_oracle(cfgs, ops, N=135, check=True)
    assert bad == 0
    ev = b.events()
    flips = {}
    for i, p in enumerate(params):
        e = _events_of(ev, i)
        refused = bool((e["type"] == orc.E_ACTIVE_REFUSED).any())
        served = bool((e["type"] == orc.E_REQUEST_SERVED).any())
        probe = e[e["type"] == orc.E_REUSE_PROBE][-1]
        resident_kept = int(probe["f"][1]) == p["R"]
        assert served != refused
        if p["policy"] == "hard":
            assert resident_kept
            flips.setdefault("hard", []).append((p["U"], served))
        else:
            assert served
            assert resident_kept == (p["U"] >= pin["flip_usable"])
    hard = flips["hard"]
    assert all(s == (U >= pin["flip_usable"]) for U, s in hard)
    assert min(U for U, s in hard if s) == pin["flip_usable"]


def test_q1_predicate_fixture():
    """Table 6: naive fair share keeps 480/320/304 tokens with
    first missing 30/20/19 -> thresholded value 0; complete-prefix keeps
    640/640/0 (40/40/0) -> value 18 with span values 9+9."""
    pin = PAPER["q1_P794_799"]
    spans = [40, 40, 20]          # S:317 default spans, thresholds = full span
    values = [9, 9, 0]            # S:318; only the total 18 is the paper's

    def value(first_missing):
        tot, tokens = 0, []
        for fm, span, v in zip(first_missing, spans, values):
            L = orc.leading_of_positions(list(range(fm)), span)
            tokens.append(16 * L)
            tot += v if L >= span else 0
        return tokens, tot

    tok, v = value(pin["naive_first_missing"])
    assert tok == pin["naive_fair_share_tokens"] and v == pin["naive_value"]
    tok, v = value(pin["complete_prefix_first_missing"])
    assert tok == pin["complete_prefix_tokens"] and v == pin["complete_prefix_value"]
    # non-leading survivors do not count
    assert orc.leading_of_positions([0, 1, 2, 5, 6], 10) == 3


def test_L6_materialization_failure_state_injection():
    """L6: 59 surviving blocks, zero leading (position 0
    missing), requirement 60 -> the accepted claim does not materialize and a
    reuse probe reports leading 0, unsatisfied."""
    pin = PAPER["L6_P1047_1050"]
    cfg = make_cfg(80, CONTRACT)
    b = orc.OracleBatch(np.stack([cfg]), N=80)
    st = b.export(0)
    blocks, claims, reqs, objs = st["blocks"], st["claims"], st["requests"], st["objects"]
    for p in range(1, 60):                       # positions 1..59 cached, block id = p
        blocks[p] = (1, 0, 0, p, 1000 - p)
    objs[0]["live"], objs[0]["len"], objs[0]["claim"] = 1, 60, 0xFF
    for o in range(1, len(objs)):
        objs[o]["claim"] = 0xFF
    b.import_(0, 2000, 0, blocks, claims, reqs, objs)
    ops = pack_ops([[op(SUBMIT, 0, 0, HARD, 60, pin["required"], 0), op(TOUCH, 0)]])
    assert b.run(ops, check=True) == 0
    st = b.export(0)
    assert st["objects"][0]["leading"] == pin["leading"]
    assert int((st["blocks"]["res"] == 1).sum()) == pin["surviving"]
    assert st["claims"][0]["state"] == orc.C_ACCEPTED          # never materialized
    ev = b.events()
    probe = ev[ev["type"] == orc.E_REUSE_PROBE][0]
    assert probe["f"][1] == 0 and probe["reason"] == 0


def test_live_scheduler_one_deferral_then_refusal():
    """Table 10: with defer budget 1 the active request is
    deferred once by the gate and then refused, both attributed to the
    resident claim."""
    pin = PAPER["live_scheduler_P1103_1105"]
    cfg = make_cfg(68, CONTRACT, PEAK, defer_budget=1)
    ops = pack_ops([[op(INSERT, 0, x=40), op(SUBMIT, 0, 0, HARD, 40, 40, 0),
                     op(ADMIT, 0, 1, 1, 16 * 46, 256, 0), op(ADVANCE, 0), op(ADVANCE, 0)]])
    b, bad = orc.run_oracle(np.stack([cfg]), ops, N=68, check=True)
    assert bad == 0
    ev = b.events()
    d = ev[ev["type"] == orc.E_ACTIVE_DEFERRED]
    r = ev[ev["type"] == orc.E_ACTIVE_REFUSED]
    assert len(d) == pin["deferred"] and len(r) == pin["refused"]
    for e in (d[0], r[0]):
        assert e["mask"] == 1 and e["reason"] == orc.WHY_PROTECTED_RESIDENT
        # capacity proof 40 + 46 = 86 > 68; shortfall by the contract
        # formula P + A - U = 18 (G20: the paper prints 19)
        assert list(e["f"]) == [40, 46, 68, 18]
    # the trailing ADVANCE hits a refused request -> deterministic OP_ERROR
    err = ev[ev["type"] == orc.E_OP_ERROR]
    assert len(err) == 1 and err[0]["reason"] == orc.ERR_UNKNOWN_REQUEST


def test_L4_L5_release_before_loss_60_70_80():
    """L4/L5: after demotion or expiry, 50 block losses are
    losses after release and there is zero claim harm."""
    pin = PAPER["L4_L5_P1042_1045"]
    from paper_2605_24259_b200.gen import DEMOTE, EXPIRING, NOP
    demote = [op(INSERT, 0, x=60), op(SUBMIT, 0, 0, HARD, 60, 60, 0), op(DEMOTE, 0),
              op(ADMIT, 0, 1, 0, 1120, 1120, 0), op(ADVANCE, 0)]
    expire = [op(INSERT, 0, x=60), op(SUBMIT, 0, 0, EXPIRING, 60, 60, 3), op(NOP), op(NOP),
              op(ADMIT, 0, 1, 0, 1120, 1120, 0), op(ADVANCE, 0)]
    cfgs = np.stack([make_cfg(80, CONTRACT), make_cfg(80, CONTRACT)])
    b, bad = orc.run_oracle(cfgs, pack_ops([demote, expire]), N=80, check=True)
    assert bad == 0
    ctr = b.counters()
    ev = b.events()
    for i, release in ((0, orc.E_CLAIM_DEMOTED), (1, orc.E_CLAIM_EXPIRED)):
        assert ctr[i][orc.K["victims_after_release"]] == pin["loss_after_release"]
        assert ctr[i][orc.K["harmed_obligated"]] + ctr[i][orc.K["harmed_unobligated"]] == pin["harmed"]
        e = _events_of(ev, i)
        t_rel = int(e[e["type"] == release][0]["step"])
        t_vic = int(e[e["type"] == orc.E_VICTIMS][0]["step"])
        assert t_rel < t_vic
