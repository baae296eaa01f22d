"""Plain CPU reconstruction of the conformance checks L1-L7 (+ I4) over a
claim-level event stream -- TEST INFRASTRUCTURE (the oracle of SURVEY 8(f) f2).

Only tests/ may use this module.  It shares no code with the CUDA checker
(paper_2605_24259_b200/csrc/rkc_conformance.cu); both follow the checks as the
paper states them (sec. 5.4) and SPEC's operations:

  L1  "No accepted claim, no claim harm": every claim_harmed
      has an earlier claim_accepted of that claim.
  L2  "Write no-admit separation": a write_admission_denied is
      followed, in the same step, by the request_served of that request.
  L3  "Hard-claim infeasibility": every refusal / deferral /
      insert refusal carries the capacity proof -- shortfall = P + A - U > 0,
      the protected-resident reason iff a non-empty blocking set iff
      (A <= U and P > 0) (G7), and every blocking claim is live then.
  L45 "Demotion or expiry before loss": no harm of a claim after
      its demotion / expiry; after-release victims only once some claim was
      released.
  L6  "Materialization failure" / predicate consistency (P:1046-1050,
      P:614-616): materialized => L >= R and tokens = 16 L; harmed => L < R;
      reuse probes report tokens = 16 L and satisfied = (bound claim live and
      L >= R).
  L7  "Trace reconstruction": the replay is a legal lifecycle
      (accepted -> harmed is legal) and, when final claim states
      are given, ends in them ("reconstruction fidelity").
  I4  under the contract lowering no obligated claim is harmed (north star);
      only where the trace's lowering is given.
  LOST the trace's event buffer overflowed (passed in by the caller).

Event records follow DESIGN.md "Records" (oracle.EVENT_DTYPE).  Verdict bits
and the evidence vector follow include/rkc.h (written out again below).
"""
from __future__ import annotations

import numpy as np

from . import oracle as orc

L1, L2, L3, L45, L6, L7, I4, LOST = 0x01, 0x02, 0x04, 0x08, 0x10, 0x20, 0x40, 0x80
# evidence: accepted, materialized, harmed, refusals (incl. deferrals and insert
# refusals), attributed refusals, victims, after-release victims, write denials,
# failing traces
NEVIDENCE = 9
LIVE = (orc.C_ACCEPTED, orc.C_MATERIALIZED)
CONTRACT = 0


def check_trace(events, C: int, final_states=None, lowering=None, lost: bool = False):
    """(verdict bits, evidence[8], reconstructed claim states) of one trace's
    events in (step, seq) order."""
    st = [orc.C_EMPTY] * 32
    accepted = [False] * 32
    released = [False] * 32
    R = [0] * 32
    bound = {}                        # object slot -> claim slot of its last acceptance
    fail = 0
    any_release = False
    pending = None                    # (request slot, step) of an unanswered denial
    ev = [0] * 8
    for x in events:
        typ, slot, reason = int(x["type"]), int(x["slot"]), int(x["reason"])
        step, mask = int(x["step"]), int(x["mask"])
        f = [int(v) for v in x["f"]]
        if pending is not None:
            if not (typ == orc.E_REQUEST_SERVED and (slot, step) == pending):
                fail |= L2
            pending = None
        if typ == orc.E_CLAIM_ACCEPTED:
            if slot >= C or st[slot] != orc.C_EMPTY:
                fail |= L7
                continue
            st[slot], accepted[slot], R[slot] = orc.C_ACCEPTED, True, f[2]
            bound[f[0]] = slot
            ev[0] += 1
        elif typ == orc.E_CLAIM_REJECTED:
            if slot >= C or st[slot] != orc.C_EMPTY:
                fail |= L7
                continue
            st[slot] = orc.C_REFUSED
        elif typ == orc.E_CLAIM_MATERIALIZED:
            if slot >= C or st[slot] != orc.C_ACCEPTED:
                fail |= L7
                continue
            if f[0] < f[1] or f[2] != 16 * f[0]:
                fail |= L6
            st[slot] = orc.C_MATERIALIZED
            ev[1] += 1
        elif typ in (orc.E_CLAIM_DEMOTED, orc.E_CLAIM_EXPIRED):
            if slot >= C or st[slot] not in LIVE:
                fail |= L7
                continue
            st[slot] = orc.C_DEMOTED if typ == orc.E_CLAIM_DEMOTED else orc.C_EXPIRED
            released[slot] = True
            any_release = True
        elif typ == orc.E_CLAIM_HARMED:
            if slot >= C:
                fail |= L7
                continue
            if not accepted[slot]:
                fail |= L1
            if released[slot]:
                fail |= L45
            if st[slot] not in LIVE:
                fail |= L7
            if f[0] >= f[1]:
                fail |= L6
            if reason and lowering is not None and lowering == CONTRACT:
                fail |= I4
            st[slot] = orc.C_HARMED
            ev[2] += 1
        elif typ in (orc.E_ACTIVE_DEFERRED, orc.E_ACTIVE_REFUSED, orc.E_RESIDENT_INSERT_REFUSED):
            P, A, U, short = f
            if P + A <= U or P + A - U != short:
                fail |= L3
            resident = A <= U and P > 0    # P: protected blocks, or the reserve (f4, G34)
            resident_reason = reason in (orc.WHY_PROTECTED_RESIDENT, orc.WHY_RESIDENT_RESERVE)
            if resident_reason != resident or (mask != 0) != resident:
                fail |= L3
            for c in range(32):
                if mask >> c & 1 and (c >= C or st[c] not in LIVE):
                    fail |= L3
            ev[3] += 1
            if mask:
                ev[4] += 1
        elif typ == orc.E_WRITE_ADMISSION_DENIED:
            pending = (slot, step)
            ev[7] += 1
        elif typ == orc.E_VICTIMS:
            if f[1] > 0 and not any_release:
                fail |= L45
            ev[5] += f[0] + f[1] + f[2]
            ev[6] += f[1]
        elif typ == orc.E_REUSE_PROBE:
            if f[2] != 16 * f[1]:
                fail |= L6
            c = slot
            live = c < C and st[c] in LIVE
            satisfied = live and f[1] >= R[c]
            if (reason != 0) != satisfied:
                fail |= L6
            if f[0] >= 128 or bound.get(f[0], 0xFF) != c:
                fail |= L7                           # the probe names the bound claim
    if pending is not None:
        fail |= L2
    if final_states is not None and any(int(final_states[c]) != st[c] for c in range(C)):
        fail |= L7
    if lost:
        fail |= LOST
    return fail, ev, st[:C]


def check_stream(events, n_traces: int, C: int, final_states=None, lowering=None, lost=None):
    """Per-trace verdicts (u32[n]) and the evidence vector (int64[9]) of a
    compacted stream in (trace, step, seq) order."""
    idx = np.searchsorted(events["trace"], np.arange(n_traces + 1))
    verdict = np.zeros(n_traces, dtype=np.uint32)
    evidence = np.zeros(NEVIDENCE, dtype=np.int64)
    for t in range(n_traces):
        v, e, _ = check_trace(events[idx[t]:idx[t + 1]], C,
                              None if final_states is None else final_states[t],
                              None if lowering is None else int(lowering[t]),
                              bool(lost[t]) if lost is not None else False)
        verdict[t] = v
        evidence[:8] += e
        evidence[8] += 1 if v else 0
    return verdict, evidence


def reconstruct_states(events, n_traces: int, C: int) -> np.ndarray:
    """Final claim states of every trace as the reconstruction sees them."""
    idx = np.searchsorted(events["trace"], np.arange(n_traces + 1))
    return np.array([check_trace(events[idx[t]:idx[t + 1]], C)[2] for t in range(n_traces)],
                    dtype=np.uint8).reshape(n_traces, C)
