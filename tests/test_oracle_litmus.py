"""configs[1]: the full litmus suite (8 templates x 1000 seeds) -- the oracle
against closed forms derived from the paper's feasibility boundary
(P:504), free-first native allocation, hard exclusion
(P:567-569), leading-prefix value and the release /
harm semantics of Table 4.  SURVEY.md Appendix A."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2605_24259_b200.gen import litmus


def _split(ev, n):
    idx = np.searchsorted(ev["trace"], np.arange(n + 1))
    return [ev[idx[i]:idx[i + 1]] for i in range(n)]


def _of(e, t):
    return e[e["type"] == t]


def _probe_L(e, obj):
    p = e[(e["type"] == orc.E_REUSE_PROBE) & (e["f"][:, 0] == obj)]
    return int(p[-1]["f"][1]), int(p[-1]["reason"])


@pytest.fixture(scope="module")
def suite_run():
    cfgs, ops, params = litmus.suite(range(1000))
    b = orc.OracleBatch(cfgs, N=1024)
    bad = b.run(ops, nthreads=8, check=True)
    ev = b.events()
    return params, _split(ev, len(params)), b.counters(), b, bad


def test_no_invariant_violation(suite_run):
    params, evs, ctr, b, bad = suite_run
    assert bad == 0


def test_templates_closed_forms(suite_run):
    params, evs, ctr, b, _ = suite_run
    seen = set()
    for i, p in enumerate(params):
        e, c, t, U = evs[i], ctr[i], p["template"], p["U"]
        seen.add(t)
        harms = c[orc.K["harmed_obligated"]] + c[orc.K["harmed_unobligated"]]
        if t in ("L-ORD", "L-NOADMIT"):
            R, f, A = p["R"], p["f"], p["A"]
            free = U - f - R
            v = max(0, A - free)
            vR = max(0, A - (U - R))
            assert c[orc.K["victims_ordinary"]] == v, p
            assert c[orc.K["served"]] == 1
            L0, _ = _probe_L(e, litmus.O_RES)
            assert L0 == R - vR, p
            L1, _ = _probe_L(e, litmus.O_ACT)
            assert L1 == (A if t == "L-ORD" else 0), p
            assert (len(_of(e, orc.E_WRITE_ADMISSION_DENIED)) == 1) == (t == "L-NOADMIT")
            vic = _of(e, orc.E_VICTIMS)
            assert len(vic) == (1 if v > 0 else 0)
            if v > 0:
                assert list(vic[0]["f"]) == [v, 0, 0, A]
        elif t == "L-HARD":
            R, A, k = p["R"], p["A"], p["chunks"]
            cb = -(-A // k)
            ref = _of(e, orc.E_ACTIVE_REFUSED)
            if p["admit_check"] == 0:          # PEAK
                feasible = R + A <= U
                a_field = A
            else:                              # NONE: per-chunk backstop
                live, feasible, a_field = 0, True, 0
                while live < A:
                    need = min(cb, A - live)
                    if R + live + need > U:
                        feasible, a_field = False, live + need
                        break
                    live += need
            if feasible:
                assert len(ref) == 0 and c[orc.K["served"]] == 1, p
                assert c[orc.K["victims_claimed"]] + c[orc.K["victims_ordinary"]] == 0
            else:
                assert len(ref) == 1, p
                r = ref[0]
                resident = a_field <= U
                assert r["reason"] == (orc.WHY_PROTECTED_RESIDENT if resident else orc.WHY_ACTIVE_CAPACITY)
                assert r["mask"] == (1 if resident else 0)
                assert list(r["f"]) == [R, a_field, U, R + a_field - U], p
                assert c[orc.K["served"]] == 0
            # the resident claim is preserved either way (Table 5 row 3)
            assert b.export(i)["claims"][0]["state"] == orc.C_MATERIALIZED
            L0, sat = _probe_L(e, litmus.O_RES)
            assert L0 == R and sat == 1
            assert harms == 0
        elif t == "L-REFUSE":
            R, A, bud = p["R"], p["A"], p["b"]
            d, r = _of(e, orc.E_ACTIVE_DEFERRED), _of(e, orc.E_ACTIVE_REFUSED)
            assert len(d) == bud and len(r) == 1, p
            for x in list(d) + list(r):
                assert list(x["f"]) == [R, A, U, R + A - U] and x["mask"] == 1
            assert all(d["step"] < r[0]["step"])
        elif t == "L-SOFT":
            if p["variant"] == "a":
                S, Of, A, Rs = p["S"], p["Of"], p["A"], p["Rs"]
                free = U - S - Of
                v = max(0, A - free)
                vS = max(0, A - (U - S))
                assert c[orc.K["victims_ordinary"]] == v - vS, p
                assert c[orc.K["victims_claimed"]] == vS, p
                assert c[orc.K["harmed_unobligated"]] == (1 if S - vS < Rs else 0), p
                assert c[orc.K["harmed_obligated"]] == 0
                L0, _ = _probe_L(e, litmus.O_RES)
                assert L0 == S - vS
            else:
                R, A = p["R"], p["A"]
                vR = max(0, A - (U - R))
                # SOFT lowering protects nothing (P = 0, A <= U): the active
                # request is never refused and gets all A blocks (C1)
                assert c[orc.K["refused_protected"]] + c[orc.K["refused_capacity"]] == 0, p
                assert c[orc.K["blocks_allocated"]] == R + A, p
                assert c[orc.K["victims_claimed"]] == vR, p
                assert c[orc.K["harmed_obligated"]] == (1 if vR > 0 else 0), p
        elif t == "L-MATFAIL":
            n, eblk = p["n"], p["e"]
            L0, sat = _probe_L(e, litmus.O_RES)
            assert L0 == n - eblk and sat == 0, p
            assert c[orc.K["accepted"]] == 1 and c[orc.K["materialized"]] == 0
            assert b.export(i)["claims"][0]["state"] == orc.C_ACCEPTED
        elif t == "L-DEMOTE":
            R, A = p["R"], p["A"]
            vR = max(0, A - (U - R))
            dem = _of(e, orc.E_CLAIM_DEMOTED)
            if p["variant"] == "explicit":
                expect_demote = True
            else:
                expect_demote = R + A > U
            assert len(dem) == (1 if expect_demote else 0), p
            if expect_demote:
                assert dem[0]["reason"] == (0 if p["variant"] == "explicit" else 1)
                assert c[orc.K["victims_after_release"]] == vR, p
                vic = _of(e, orc.E_VICTIMS)
                if vR > 0:
                    assert dem[0]["step"] < vic[0]["step"] or (
                        dem[0]["step"] == vic[0]["step"] and dem[0]["seq"] < vic[0]["seq"])
            else:
                assert c[orc.K["victims_after_release"]] + c[orc.K["victims_claimed"]] == 0
            assert harms == 0
        elif t == "L-EXPIRE":
            R, A, d = p["R"], p["A"], p["d"]
            vR = max(0, A - (U - R))
            exp = _of(e, orc.E_CLAIM_EXPIRED)
            if p["variant"] == "after":
                assert len(exp) == 1 and exp[0]["step"] == 1 + d, p
                assert c[orc.K["victims_after_release"]] == vR
            else:
                expired_at_admit = 1 + d <= 2
                if not expired_at_admit and R + A > U:
                    r = _of(e, orc.E_ACTIVE_REFUSED)
                    assert len(r) == 1 and r[0]["mask"] == 1, p
                    assert c[orc.K["victims_after_release"]] == 0
                else:
                    expired_at_advance = 1 + d <= 3
                    if expired_at_advance:
                        assert c[orc.K["victims_after_release"]] == vR, p
                    else:
                        assert c[orc.K["victims_after_release"]] + c[orc.K["victims_claimed"]] == 0
            assert harms == 0
    assert seen == set(litmus.TEMPLATES)


def test_contract_never_harms_obligated(suite_run):
    """North-star invariant (I4): under the contract lowering no accepted
    obligated claim is ever harmed (Table 4 row 4 never fires)."""
    params, evs, ctr, b, _ = suite_run
    for i, p in enumerate(params):
        if b.cfgs[i]["lowering"] == 0:
            assert ctr[i][orc.K["harmed_obligated"]] == 0
