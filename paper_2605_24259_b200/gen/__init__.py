"""Seeded synthetic allocator-trace generator (input only; no method arithmetic).

This module is the ONE thing the CUDA path and the oracle share: it produces
op streams and per-trace configs.  It never simulates allocation outcomes
(see rkc_gen.cpp header).  Recipes: DESIGN.md "Input recipe".

Record layouts:
  op        16 B {u8 kind, a, b, c; u32 x, y, z}
  trace cfg 12 B {u32 U; u8 lowering, admit_check, defer_budget, auto_demote,
                  accept_rule, pad[3]}
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

OP_DTYPE = np.dtype([("kind", "u1"), ("a", "u1"), ("b", "u1"), ("c", "u1"),
                     ("x", "<u4"), ("y", "<u4"), ("z", "<u4")])
CFG_DTYPE = np.dtype([("U", "<u4"), ("lowering", "u1"), ("admit_check", "u1"),
                      ("defer_budget", "u1"), ("auto_demote", "u1"), ("accept_rule", "u1"),
                      ("pad", "u1", (3,))])
assert OP_DTYPE.itemsize == 16 and CFG_DTYPE.itemsize == 12

# op kinds
NOP, SUBMIT, ADMIT, ADVANCE, COMPLETE, INSERT, DEMOTE, TOUCH, HIT_ADMIT = range(9)
# protection modes (Table 3)
SOFT, HARD, DEMOTABLE, OFFLOADABLE, EXPIRING, BEST_EFFORT = range(6)
# policy bytes
CONTRACT, SOFT_LOWERING, NATIVE = 0, 1, 2
PEAK, NONE, ADMIT_RESERVE = 0, 1, 2     # admit_check (ADMIT_RESERVE: NEXT f4)
CAPACITY, RESERVE = 0, 1
ID_MISMATCH = 0x80

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rkc_gen.cpp")
_LIB = os.path.join(_HERE, "librkc_gen.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile librkc_gen.so in-tree (plain g++; no GPU needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", _SRC,
                               "-o", _LIB, "-lpthread"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.rkc_gen_random.restype = ctypes.c_int
        lib.rkc_gen_random.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                       ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        _lib = lib
    return _lib


def random_traces(config: int, seed: int, trace_begin: int, n_traces: int, T: int,
                  N: int, C: int = 16, Q: int = 16, O: int = 64, nthreads: int | None = None,
                  ops_out: np.ndarray | None = None):
    """Random traces of recipe `config` (3 = c3/c5, 4 = c4, 6 = c3 + prefix hits,
    7 = slot stress: every claim / request / object slot up to C, Q, O; 8 = c3 with
    resident-reserve admission (NEXT f4) on 40 % of the traces).

    Returns (cfgs[n_traces] CFG_DTYPE, ops[T, n_traces] OP_DTYPE).  ops_out
    may be a preallocated (e.g. pinned) uint8/OP_DTYPE buffer of T*n*16 bytes.
    """
    lib = _load()
    cfgs = np.zeros(n_traces, dtype=CFG_DTYPE)
    if ops_out is None:
        ops = np.zeros((T, n_traces), dtype=OP_DTYPE)
    else:
        ops = ops_out.view(OP_DTYPE).reshape(T, n_traces)
    if nthreads is None:
        nthreads = os.cpu_count() or 1
    rc = lib.rkc_gen_random(int(config), int(seed), int(trace_begin), int(n_traces), int(T),
                            int(N), int(C), int(Q), int(O), cfgs.ctypes.data, ops.ctypes.data,
                            int(nthreads))
    if rc != 0:
        raise ValueError(f"rkc_gen_random failed ({rc})")
    return cfgs, ops


def make_cfg(U: int, lowering: int = CONTRACT, admit_check: int = PEAK, defer_budget: int = 0,
             auto_demote: int = 0, accept_rule: int = CAPACITY) -> np.ndarray:
    c = np.zeros((), dtype=CFG_DTYPE)
    c["U"], c["lowering"], c["admit_check"] = U, lowering, admit_check
    c["defer_budget"], c["auto_demote"], c["accept_rule"] = defer_budget, auto_demote, accept_rule
    return c


def op(kind: int, a: int = 0, b: int = 0, c: int = 0, x: int = 0, y: int = 0, z: int = 0):
    return (kind, a, b, c, x, y, z)


def pack_ops(per_trace: list[list[tuple]], T: int | None = None) -> np.ndarray:
    """Pack per-trace op lists into the step-major [T, n] layout (NOP padded)."""
    n = len(per_trace)
    if T is None:
        T = max((len(t) for t in per_trace), default=0)
    ops = np.zeros((T, n), dtype=OP_DTYPE)
    for i, lst in enumerate(per_trace):
        for s, rec in enumerate(lst):
            ops[s, i] = rec
    return ops
