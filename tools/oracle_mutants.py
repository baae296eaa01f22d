"""Mutation check of the oracle's pins (test infrastructure, run by hand).

Applies one plausible mistake at a time to oracle/rkc_oracle.cpp, rebuilds the
oracle, runs the `-m "not gpu"` oracle pins, and reports which mutants the
pins kill.  The source file is restored after every mutant (and on any exit).

    python tools/oracle_mutants.py [-k SUBSTRING]
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "rkc_oracle.cpp")
LIB = os.path.join(ROOT, "oracle", "librkc_oracle.so")
TESTS = ["tests/test_oracle_decisions.py", "tests/test_oracle_paper.py",
         "tests/test_oracle_litmus.py", "tests/test_oracle_bruteforce.py",
         "tests/test_oracle_prefix_hits.py", "tests/test_oracle_random.py",
         "tests/test_oracle_reserve.py", "tests/test_oracle_conformance.py",
         "tests/test_oracle_readings.py"]

# (name, old, new): each `old` must occur exactly once in the oracle source
MUTANTS = [
    ("footprint >= U", "else if (F > cfg.U) rej = REJ_FOOTPRINT;",
     "else if (F >= cfg.U) rej = REJ_FOOTPRINT;"),
    ("reserve sums non-obligated", "if (live_claim(j) && obligated(clm[j].mode)) sum += clm[j].F;",
     "if (live_claim(j)) sum += clm[j].F;"),
    ("reserve counts released claims",
     "if (live_claim(j) && obligated(clm[j].mode)) sum += clm[j].F;",
     "if (clm[j].state != C_EMPTY && clm[j].state != C_REFUSED && obligated(clm[j].mode)) sum += clm[j].F;"),
    ("reserve >= U", "if (sum > cfg.U) rej = REJ_RESERVE;", "if (sum >= cfg.U) rej = REJ_RESERVE;"),
    ("reserve checks every mode",
     "else if (cfg.accept_rule == ACCEPT_RESERVE && obligated((uint8_t)mode)) {",
     "else if (cfg.accept_rule == ACCEPT_RESERVE) {"),
    ("offloadable not obligated",
     "return mode == M_HARD || mode == M_DEMOTABLE || mode == M_OFFLOADABLE || mode == M_EXPIRING;",
     "return mode == M_HARD || mode == M_DEMOTABLE || mode == M_EXPIRING;"),
    ("identity after object-claimed", "if (id_mismatch) rej = REJ_IDENTITY;",
     "if (id_mismatch && !(obj[o].claim != NO_OBJ_CLAIM && live_claim(obj[o].claim))) rej = REJ_IDENTITY;"),
    ("object-claimed ignores liveness",
     "else if (obj[o].claim != NO_OBJ_CLAIM && live_claim(obj[o].claim)) rej = REJ_OBJECT_CLAIMED;",
     "else if (obj[o].claim != NO_OBJ_CLAIM) rej = REJ_OBJECT_CLAIMED;"),
    ("rejected claim binds object", "      cl.state = C_REFUSED;\n",
     "      cl.state = C_REFUSED; obj[o].claim = c;\n"),
    ("blocking mask lists first claim only", "if (protected_of_claim(c) > 0) m |= 1u << c;",
     "if (protected_of_claim(c) > 0) { m |= 1u << c; break; }"),
    ("claim protects the whole object (no pos < F)",
     "return c != NO_OBJ_CLAIM && live_claim(c) && blk[b].pos < clm[c].F;",
     "return c != NO_OBJ_CLAIM && live_claim(c);"),
    ("mask kept when A > U", "const bool resident_cause = (A <= U) && P > 0;",
     "const bool resident_cause = P > 0;"),
    ("admission reserve counts non-obligated claims",
     "      if (live_claim(c) && obligated(clm[c].mode)) r += clm[c].F;",
     "      if (live_claim(c)) r += clm[c].F;"),
    ("admission reserve = cached protected blocks", "    const uint64_t Rv = reserve_total();",
     "    const uint64_t Rv = protected_total();"),
    ("admission reserve under every lowering", "    if (cfg.lowering != LOW_CONTRACT) return 0;\n    uint64_t r = 0;",
     "    uint64_t r = 0;"),
    ("admission reserve boundary <", "    if (Rv + A <= cfg.U) return true;", "    if (Rv + A < cfg.U) return true;"),
    ("head-first stamps on insert (G1)", "b.res = B_CACHED; b.owner = (uint8_t)o; b.pos = i; b.seq = base + (n - 1 - i);",
     "b.res = B_CACHED; b.owner = (uint8_t)o; b.pos = i; b.seq = base + i;"),
    ("head-first stamps on complete (G1)", "b.seq = base + (full - 1 - b.pos); }",
     "b.seq = base + b.pos; }"),
    ("soft claims not evicted last (G6)",
     "if (m == M_SOFT || (cfg.lowering == LOW_SOFT && obligated(m))) return 2;",
     "if (m == M_SOFT || (cfg.lowering == LOW_SOFT && obligated(m))) return 1;"),
    ("auto-demotion from the highest slot (G10)",
     "        if (live_claim(c) && clm[c].mode == M_DEMOTABLE) {\n          uint32_t pc = protected_of_claim(c);\n          if (pc > 0) { dm.push_back(c); g.push_back(pc); }",
     "        if (live_claim(c) && clm[c].mode == M_DEMOTABLE) {\n          uint32_t pc = protected_of_claim(c);\n          if (pc > 0) { dm.insert(dm.begin(), c); g.insert(g.begin(), pc); }"),
    ("shortfall off by one", "const uint32_t shortfall = (uint32_t)((uint64_t)P + A - U);",
     "const uint32_t shortfall = (uint32_t)((uint64_t)P + A - U - 1);"),
]


def main() -> int:
    sel = sys.argv[sys.argv.index("-k") + 1] if "-k" in sys.argv else ""
    orig = open(SRC).read()
    tests = [t for t in TESTS if os.path.exists(os.path.join(ROOT, t))]
    survived = []
    try:
        for name, old, new in MUTANTS:
            if sel not in name:
                continue
            assert orig.count(old) == 1, f"mutant '{name}': pattern occurs {orig.count(old)} times"
            open(SRC, "w").write(orig.replace(old, new))
            subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", SRC, "-o", LIB,
                                   "-lpthread"])
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu",
                                "-p", "no:cacheprovider", *tests], cwd=ROOT,
                               capture_output=True, text=True)
            killed = r.returncode != 0
            first = next((ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")), "")
            print(f"{'KILLED ' if killed else 'SURVIVED'} {name:48s} {first[:110]}", flush=True)
            if not killed:
                survived.append(name)
    finally:
        open(SRC, "w").write(orig)
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", SRC, "-o", LIB,
                               "-lpthread"])
    print(f"{len(survived)} survived: {survived}")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
