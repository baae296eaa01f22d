"""bench.py's roofline byte model (SURVEY.md 8(d)'s per-op table, bench.survey_bytes)
on a hand-computed four-step trace, with the replay's counters and events taken
from the oracle (CPU).  Fixes the arithmetic the bench's `roofline.achieved`
uses: N = 128 blocks, H = 256 (claim + request lanes).

  step 0  INSERT o0, 100 blocks        free-only allocation: reads N/8 = 16,
                                       writes 4*100 + 4 + 32 = 436
  step 1  ADMIT r0, 800 tokens         PEAK check passes (P = 0): writes 32
  step 2  ADVANCE r0 (50 blocks)       28 free -> evicting allocation of 50
                                       (22 victims): reads 8N + N/8 = 1040,
                                       writes 4*50 + 4 + 32 = 236; one event
  step 3  TOUCH o0                     the 22 tail positions were evicted:
                                       L = 78, reads 4N = 512, writes 4*78 = 312;
                                       one event
  every step                           reads 16 + 256 = 272 (4 steps: 1088)
  events                               2 * 32 = 64
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_survey_bytes_hand_computed():
    import bench
    from oracle import oracle as orc
    from paper_2605_24259_b200.gen import ADMIT, ADVANCE, INSERT, NATIVE, TOUCH, make_cfg, op, pack_ops
    bench.select_workload("c3")
    bench.NBLK = 128
    ops = pack_ops([[op(INSERT, 0, x=100), op(ADMIT, 0, 1, 0, 800, 800, 0), op(ADVANCE, 0),
                     op(TOUCH, 0)]])
    b = orc.OracleBatch(np.stack([make_cfg(128, NATIVE)]), N=128)
    assert b.run(ops, check=True) == 0
    ev, ctr = b.events(), b.counters()
    vic = ev[ev["type"] == orc.E_VICTIMS]
    assert len(vic) == 1 and list(vic[0]["f"]) == [22, 0, 0, 50]
    probe = ev[ev["type"] == orc.E_REUSE_PROBE]
    assert probe[0]["f"][1] == 78
    sb = bench.survey_bytes(ops, ctr, ev)
    assert sb["allocations"] == 2 and sb["evicting_selections"] == 1
    assert sb["read"] == 1088 + 16 + 1040 + 512
    assert sb["write"] == 436 + 32 + 236 + 312 + 64
    assert sb["bytes"] == 3736
