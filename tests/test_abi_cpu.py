"""CPU-only checks of the boundary: librkc.so loads, exports every symbol that
include/rkc.h declares, and the record layouts in the header have the sizes
DESIGN.md states (checked by compiling the header with the host C compiler).
No compute calls (there is no GPU here)."""
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rkc.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"RKC_API\s+[\w\s\*]+?\b(rkc_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2605_24259_b200 import build
    build.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", build.LIB], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    declared = _declared()
    assert len(declared) >= 15
    missing = [s for s in declared if s not in exported]
    assert not missing, missing


def test_binding_loads_and_matches_header():
    from paper_2605_24259_b200 import rkc
    assert rkc.rkc_abi_version() == 2
    assert set(rkc.EXPORTED_SYMBOLS) == set(_declared())


def test_record_sizes_from_header():
    prog = r"""
#include <stdio.h>
#include <stddef.h>
#include "rkc.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(rkc_op), sizeof(rkc_trace_config),
         sizeof(rkc_event), sizeof(rkc_block_view), sizeof(rkc_claim_view), sizeof(rkc_request_view),
         sizeof(rkc_object_view), sizeof(rkc_header_view), sizeof(rkc_claim_input),
         sizeof(rkc_request_input), sizeof(rkc_trace_op), sizeof(rkc_pool_config));
  printf("%zu %zu\n", offsetof(rkc_event, mask), offsetof(rkc_claim_input, cache_identity));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe])
        lines = subprocess.check_output([exe], text=True).split("\n")
    sizes = [int(v) for v in lines[0].split()]
    assert sizes == [16, 12, 32, 12, 24, 32, 12, 16, 48, 32, 20, 40]
    assert [int(v) for v in lines[1].split()] == [12, 24]
    from paper_2605_24259_b200 import rkc
    assert rkc.CLAIM_INPUT.itemsize == 48 and rkc.REQUEST_INPUT.itemsize == 32
    assert rkc.EVENT.itemsize == 32 and rkc.TRACE_OP.itemsize == 20


def test_sass_is_sm100a():
    """The step kernel is compiled for sm_100a (cuobjdump lists the arch)."""
    from paper_2605_24259_b200 import build
    build.build()
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB], text=True)
    assert "sm_100a" in out
