"""ctypes wrapper of the plain CPU oracle (rkc_oracle.cpp) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module.  It shares no code with paper_2605_24259_b200 (the product path);
the record dtypes below are written out again from DESIGN.md "Records" and
"State views".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

EVENT_DTYPE = np.dtype([("trace", "<u4"), ("step", "<u4"), ("type", "u1"), ("seq", "u1"),
                        ("slot", "u1"), ("reason", "u1"), ("mask", "<u4"), ("f", "<u4", (4,))])
BLOCK_VIEW = np.dtype([("res", "u1"), ("owner", "u1"), ("pad", "<u2"), ("pos", "<u4"),
                       ("seq", "<u4")])
CLAIM_VIEW = np.dtype([("state", "u1"), ("mode", "u1"), ("obj", "u1"), ("pad", "u1"),
                       ("F", "<u4"), ("R", "<u4"), ("D", "<u4"), ("decision_step", "<u4"),
                       ("protected_blocks", "<u4")])
REQUEST_VIEW = np.dtype([("status", "u1"), ("write_admit", "u1"), ("target", "u1"),
                         ("defer_count", "u1"), ("prompt", "<u4"), ("chunk", "<u4"),
                         ("decode", "<u4"), ("done", "<u4"), ("live", "<u4"), ("hit", "<u4"),
                         ("pad", "<u4")])
OBJECT_VIEW = np.dtype([("live", "u1"), ("claim", "u1"), ("pad", "u1", (2,)), ("len", "<u4"),
                        ("leading", "<u4")])
HEADER_VIEW = np.dtype([("seq_ctr", "<u4"), ("free_blocks", "<u4"), ("alive", "<u4"),
                        ("protected_total", "<u4")])
assert EVENT_DTYPE.itemsize == 32 and BLOCK_VIEW.itemsize == 12 and CLAIM_VIEW.itemsize == 24
assert REQUEST_VIEW.itemsize == 32 and OBJECT_VIEW.itemsize == 12 and HEADER_VIEW.itemsize == 16

NCOUNTERS = 32
COUNTER_NAMES = [
    "ops", "accepted", "rejected", "materialized", "demoted_explicit", "demoted_auto", "expired",
    "harmed_obligated", "harmed_unobligated", "admitted", "served", "deferred_protected",
    "deferred_capacity", "refused_protected", "refused_capacity", "inserted", "insert_refused",
    "write_denied", "victims_ordinary", "victims_after_release", "victims_claimed",
    "blocks_allocated", "blocks_cached", "reuse_probes", "reuse_tokens", "op_errors", "steps",
    "events", "prefix_hits", "hit_tokens", "allocations"]
K = {n: i for i, n in enumerate(COUNTER_NAMES)}

# event types
(E_CLAIM_ACCEPTED, E_CLAIM_REJECTED, E_CLAIM_MATERIALIZED, E_CLAIM_DEMOTED, E_CLAIM_EXPIRED,
 E_CLAIM_HARMED, E_ACTIVE_DEFERRED, E_ACTIVE_REFUSED, E_RESIDENT_INSERT_REFUSED,
 E_WRITE_ADMISSION_DENIED, E_REQUEST_SERVED, E_VICTIMS, E_REUSE_PROBE, E_OP_ERROR,
 E_PREFIX_HIT) = range(1, 16)
EVENT_NAMES = {1: "claim_accepted", 2: "claim_rejected", 3: "claim_materialized",
               4: "claim_demoted", 5: "claim_expired", 6: "claim_harmed",
               7: "active_request_deferred", 8: "active_request_refused",
               9: "resident_insert_refused", 10: "write_admission_denied",
               11: "request_served", 12: "victims", 13: "reuse_probe", 14: "op_error",
               15: "prefix_hit"}
# claim states / request status
C_EMPTY, C_ACCEPTED, C_MATERIALIZED, C_DEMOTED, C_EXPIRED, C_REFUSED, C_HARMED = range(7)
R_EMPTY, R_RUNNING, R_DEFERRED, R_REFUSED, R_COMPLETED = range(5)
# reasons
WHY_PROTECTED_RESIDENT, WHY_ACTIVE_CAPACITY, WHY_RESIDENT_RESERVE = 1, 2, 3
(ERR_DUPLICATE_SLOT, ERR_INVALID_ARG, ERR_ILLEGAL_TRANSITION, ERR_UNKNOWN_CLAIM,
 ERR_UNKNOWN_REQUEST, ERR_NO_CHUNKS_REMAINING, ERR_OBJECT_IN_USE, ERR_SEQ_EXHAUSTED,
 ERR_UNKNOWN_OP) = range(1, 10)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rkc_oracle.cpp")
_LIB = os.path.join(_HERE, "librkc_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (-O2, no -march=native)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", _SRC, "-o", _LIB,
                               "-lpthread"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        vp, u32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64
        lib.oracle_batch_create.restype = vp
        lib.oracle_batch_create.argtypes = [vp, u32, u32, u32, u32, u32]
        lib.oracle_batch_free.argtypes = [vp]
        lib.oracle_batch_run.restype = ctypes.c_int
        lib.oracle_batch_run.argtypes = [vp, vp, u32, u64, u64, ctypes.c_int, ctypes.c_int]
        lib.oracle_trace_violation.restype = ctypes.c_int
        lib.oracle_trace_violation.argtypes = [vp, u32]
        lib.oracle_batch_num_events.restype = u64
        lib.oracle_batch_num_events.argtypes = [vp]
        lib.oracle_batch_events.restype = u64
        lib.oracle_batch_events.argtypes = [vp, vp, u64]
        lib.oracle_batch_counters.argtypes = [vp, vp]
        lib.oracle_trace_export.argtypes = [vp, u32, vp, vp, vp, vp, vp]
        lib.oracle_trace_import.argtypes = [vp, u32, u32, u32, vp, vp, vp, vp]
        lib.oracle_leading_of_positions.restype = u32
        lib.oracle_leading_of_positions.argtypes = [vp, u32, u32]
        _lib = lib
    return _lib


class OracleBatch:
    """A batch of independent traces run by the plain CPU oracle."""

    def __init__(self, cfgs: np.ndarray, N: int, C: int = 16, Q: int = 16, O: int = 64):
        self.lib = _load()
        self.cfgs = np.ascontiguousarray(cfgs)
        assert self.cfgs.dtype.itemsize == 12
        self.n = len(self.cfgs)
        self.N, self.C, self.Q, self.O = N, C, Q, O
        self.h = self.lib.oracle_batch_create(self.cfgs.ctypes.data, self.n, N, C, Q, O)
        if not self.h:
            raise ValueError("oracle_batch_create: invalid sizes")

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.oracle_batch_free(h)
            self.h = None

    def run(self, ops: np.ndarray, nthreads: int = 1, check: bool = False,
            trace_offset: int = 0) -> int:
        """Run T lockstep steps; ops is [T, stride] (column trace_offset+i feeds trace i)."""
        ops = np.ascontiguousarray(ops)
        assert ops.dtype.itemsize == 16 and ops.ndim == 2
        T, stride = ops.shape
        return self.lib.oracle_batch_run(self.h, ops.ctypes.data, T, stride, trace_offset,
                                         nthreads, 1 if check else 0)

    def violation(self, trace: int) -> int:
        return self.lib.oracle_trace_violation(self.h, trace)

    def events(self) -> np.ndarray:
        n = self.lib.oracle_batch_num_events(self.h)
        out = np.zeros(n, dtype=EVENT_DTYPE)
        self.lib.oracle_batch_events(self.h, out.ctypes.data, n)
        return out

    def counters(self) -> np.ndarray:
        out = np.zeros((self.n, NCOUNTERS), dtype=np.uint32)
        self.lib.oracle_batch_counters(self.h, out.ctypes.data)
        return out

    def export(self, trace: int):
        hdr = np.zeros((), dtype=HEADER_VIEW)
        blocks = np.zeros(self.N, dtype=BLOCK_VIEW)
        claims = np.zeros(self.C, dtype=CLAIM_VIEW)
        reqs = np.zeros(self.Q, dtype=REQUEST_VIEW)
        objs = np.zeros(self.O, dtype=OBJECT_VIEW)
        self.lib.oracle_trace_export(self.h, trace, hdr.ctypes.data, blocks.ctypes.data,
                                     claims.ctypes.data, reqs.ctypes.data, objs.ctypes.data)
        return dict(header=hdr, blocks=blocks, claims=claims, requests=reqs, objects=objs)

    def import_(self, trace: int, seq_ctr: int, step: int, blocks, claims, reqs, objs):
        blocks = np.ascontiguousarray(blocks, dtype=BLOCK_VIEW)
        claims = np.ascontiguousarray(claims, dtype=CLAIM_VIEW)
        reqs = np.ascontiguousarray(reqs, dtype=REQUEST_VIEW)
        objs = np.ascontiguousarray(objs, dtype=OBJECT_VIEW)
        self.lib.oracle_trace_import(self.h, trace, seq_ctr, step, blocks.ctypes.data,
                                     claims.ctypes.data, reqs.ctypes.data, objs.ctypes.data)


def leading_of_positions(positions, length: int) -> int:
    """The materialization predicate alone: first missing position."""
    lib = _load()
    p = np.ascontiguousarray(np.asarray(positions, dtype=np.uint32))
    return int(lib.oracle_leading_of_positions(p.ctypes.data, len(p), length))


def run_oracle(cfgs, ops, N, C=16, Q=16, O=64, nthreads=1, check=False):
    b = OracleBatch(cfgs, N, C, Q, O)
    bad = b.run(ops, nthreads=nthreads, check=check)
    return b, bad


def render_refusal_json(ev, request_names: dict, claim_names: dict) -> dict:
    """Render an active_request_refused event in the paper's field set
    (P:1069-1079).  Used by the litmus JSON pin only."""
    mask = int(ev["mask"])
    blocking = [claim_names[c] for c in range(32) if mask >> c & 1]
    P, A, U, short = (int(v) for v in ev["f"])
    feas = ("infeasible_preserve_resident_and_active" if ev["reason"] == WHY_PROTECTED_RESIDENT
            else "infeasible_active_exceeds_reserve_headroom" if ev["reason"] == WHY_RESIDENT_RESERVE
            else "infeasible_active_exceeds_usable")
    return {
        "event": EVENT_NAMES[int(ev["type"])],
        "request_id": request_names[int(ev["slot"])],
        "blocking_claim_ids": blocking,
        "protected_resident_blocks": P,
        "active_live_blocks_required": A,
        "resident_plus_active_blocks": P + A,
        "usable_blocks": U,
        "capacity_shortfall_blocks": short,
        "feasibility": feas,
    }
