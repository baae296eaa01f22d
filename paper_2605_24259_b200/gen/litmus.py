"""Litmus trace recipes (BASELINE.json configs[0] and configs[1]) -- inputs only.

Each template builds one trace per seed with parameters drawn from a seeded
`random.Random`; it returns the parameters so tests can evaluate the closed
forms themselves.  Nothing here evaluates the method.

Slots: object 0 = resident prefix, 1 = the active request's output object,
2 = filler; claim 0 = "claim:resident"; request 0 = "active".
"""
from __future__ import annotations

import random

import numpy as np

from . import (ADMIT, ADVANCE, CAPACITY, COMPLETE, CONTRACT, DEMOTABLE, DEMOTE, EXPIRING, HARD,
               INSERT, NATIVE, NONE, NOP, PEAK, SOFT, SOFT_LOWERING, SUBMIT, TOUCH, make_cfg, op,
               pack_ops)

O_RES, O_ACT, O_FILL = 0, 1, 2
TEMPLATES = ["L-ORD", "L-NOADMIT", "L-HARD", "L-REFUSE", "L-SOFT", "L-MATFAIL", "L-DEMOTE",
             "L-EXPIRE"]


def paper_litmus():
    """configs[0]: the paper's 60/70/80 case (Table 9 P:947-959,
    refusal JSON P:1069-1079) as three traces:
      (i)   hard claim under the contract lowering -> active refusal
      (ii)  native runtime with write no-admit -> 50 resident victims
      (iii) (ii) plus an accepted hard claim, native lowering -> visible harm
    The active request is 1120 tokens = 70 blocks."""
    U, R, A = 80, 60, 70
    hard = [op(INSERT, O_RES, x=R), op(SUBMIT, 0, O_RES, HARD, R, R, 0),
            op(ADMIT, 0, O_ACT, 0, 16 * A, 16 * A, 0), op(TOUCH, O_RES)]
    native = [op(INSERT, O_RES, x=R), op(ADMIT, 0, O_ACT, 0, 16 * A, 16 * A, 0), op(ADVANCE, 0),
              op(COMPLETE, 0), op(TOUCH, O_RES), op(TOUCH, O_ACT)]
    native_claim = [op(INSERT, O_RES, x=R), op(SUBMIT, 0, O_RES, HARD, R, R, 0),
                    op(ADMIT, 0, O_ACT, 0, 16 * A, 16 * A, 0), op(ADVANCE, 0), op(COMPLETE, 0),
                    op(TOUCH, O_RES), op(TOUCH, O_ACT)]
    cfgs = np.stack([make_cfg(U, CONTRACT), make_cfg(U, NATIVE), make_cfg(U, NATIVE)])
    return cfgs, pack_ops([hard, native, native_claim]), dict(U=U, R=R, A=A)


def _sample(rng: random.Random, template: str):
    U = rng.randint(16, 1024)
    p = dict(template=template, U=U)
    if template in ("L-ORD", "L-NOADMIT"):
        R = rng.randint(1, U)
        f = rng.randint(0, U - R)
        A = rng.randint(1, U)
        p.update(R=R, f=f, A=A)
    elif template == "L-HARD":
        R = rng.randint(1, U)
        A = rng.randint(1, U + 32)
        chunks = rng.choice([1, 1, 2, 4])
        p.update(R=R, A=A, chunks=chunks, admit_check=rng.choice([PEAK, PEAK, NONE]))
    elif template == "L-REFUSE":
        A = rng.randint(1, U - 1)
        R = rng.randint(U - A + 1, U)          # R + A > U, A <= U: resident-caused
        p.update(R=R, A=A, b=rng.randint(0, 2))
    elif template == "L-SOFT":
        variant = rng.choice(["a", "b"])
        if variant == "a":
            S = rng.randint(1, U)
            Of = rng.randint(0, U - S)
            A = rng.randint(1, U)
            Rs = rng.randint(1, S)
            p.update(variant=variant, S=S, Of=Of, A=A, Rs=Rs)
        else:
            R = rng.randint(1, U)
            A = rng.randint(1, U)
            p.update(variant=variant, R=R, A=A)
    elif template == "L-MATFAIL":
        n = rng.randint(1, U - 1)
        e = rng.randint(1, n)
        p.update(n=n, e=e, A=(U - n) + e)
    elif template == "L-DEMOTE":
        R = rng.randint(1, U)
        A = rng.randint(1, U)
        p.update(R=R, A=A, variant=rng.choice(["explicit", "auto"]))
    elif template == "L-EXPIRE":
        R = rng.randint(1, U)
        A = rng.randint(1, U)
        d = rng.randint(1, 8)
        p.update(R=R, A=A, d=d, variant=rng.choice(["after", "before"]))
    return p


def _build(p):
    t = p["template"]
    U = p["U"]
    if t in ("L-ORD", "L-NOADMIT"):
        wa = 1 if t == "L-ORD" else 0
        ops = []
        if p["f"] > 0:
            ops.append(op(INSERT, O_FILL, x=p["f"]))
        ops += [op(INSERT, O_RES, x=p["R"]), op(ADMIT, 0, O_ACT, wa, 16 * p["A"], 16 * p["A"], 0),
                op(ADVANCE, 0), op(COMPLETE, 0), op(TOUCH, O_RES), op(TOUCH, O_ACT)]
        return make_cfg(U, NATIVE), ops
    if t == "L-HARD":
        A, R, k = p["A"], p["R"], p["chunks"]
        chunk_blocks = -(-A // k)
        ops = [op(INSERT, O_RES, x=R), op(SUBMIT, 0, O_RES, HARD, R, R, 0),
               op(ADMIT, 0, O_ACT, 1, 16 * A, 16 * chunk_blocks, 0)]
        ops += [op(ADVANCE, 0)] * (-(-A // chunk_blocks))
        ops += [op(COMPLETE, 0), op(TOUCH, O_RES)]
        return make_cfg(U, CONTRACT, p["admit_check"]), ops
    if t == "L-REFUSE":
        R, A, b = p["R"], p["A"], p["b"]
        ops = [op(INSERT, O_RES, x=R), op(SUBMIT, 0, O_RES, HARD, R, R, 0),
               op(ADMIT, 0, O_ACT, 1, 16 * A, 16 * A, 0)] + [op(ADVANCE, 0)] * b
        return make_cfg(U, CONTRACT, PEAK, defer_budget=b), ops
    if t == "L-SOFT":
        if p["variant"] == "a":
            S, Of, A, Rs = p["S"], p["Of"], p["A"], p["Rs"]
            ops = [op(INSERT, O_RES, x=S), op(SUBMIT, 0, O_RES, SOFT, S, Rs, 0)]
            if Of > 0:
                ops.append(op(INSERT, O_FILL, x=Of))
            ops += [op(ADMIT, 0, O_ACT, 0, 16 * A, 16 * A, 0), op(ADVANCE, 0), op(TOUCH, O_RES)]
            return make_cfg(U, CONTRACT), ops
        R, A = p["R"], p["A"]
        ops = [op(INSERT, O_RES, x=R), op(SUBMIT, 0, O_RES, HARD, R, R, 0),
               op(ADMIT, 0, O_ACT, 0, 16 * A, 16 * A, 0), op(ADVANCE, 0), op(TOUCH, O_RES)]
        return make_cfg(U, SOFT_LOWERING), ops
    if t == "L-MATFAIL":
        n, A = p["n"], p["A"]
        ops = [op(INSERT, O_RES, x=n), op(ADMIT, 0, O_ACT, 0, 16 * A, 16 * A, 0), op(ADVANCE, 0),
               op(COMPLETE, 0), op(SUBMIT, 0, O_RES, HARD, n, n, 0), op(TOUCH, O_RES)]
        return make_cfg(U, CONTRACT), ops
    if t == "L-DEMOTE":
        R, A = p["R"], p["A"]
        if p["variant"] == "explicit":
            ops = [op(INSERT, O_RES, x=R), op(SUBMIT, 0, O_RES, HARD, R, R, 0), op(DEMOTE, 0),
                   op(ADMIT, 0, O_ACT, 0, 16 * A, 16 * A, 0), op(ADVANCE, 0)]
            return make_cfg(U, CONTRACT), ops
        ops = [op(INSERT, O_RES, x=R), op(SUBMIT, 0, O_RES, DEMOTABLE, R, R, 0),
               op(ADMIT, 0, O_ACT, 0, 16 * A, 16 * A, 0), op(ADVANCE, 0)]
        return make_cfg(U, CONTRACT, auto_demote=1), ops
    if t == "L-EXPIRE":
        R, A, d = p["R"], p["A"], p["d"]
        ops = [op(INSERT, O_RES, x=R), op(SUBMIT, 0, O_RES, EXPIRING, R, R, d)]
        if p["variant"] == "after":
            ops += [op(NOP)] * (d - 1)     # claim decided at step 1; expires at step 1+d
        ops += [op(ADMIT, 0, O_ACT, 0, 16 * A, 16 * A, 0), op(ADVANCE, 0)]
        return make_cfg(U, CONTRACT), ops
    raise ValueError(t)


def suite(seeds=range(1000), templates=TEMPLATES):
    """configs[1]: every template x every seed, one trace each (T <= 16 for
    the default templates; L-HARD with chunks adds steps)."""
    params, cfgs, lists = [], [], []
    for ti, t in enumerate(templates):
        for s in seeds:
            rng = random.Random((ti + 1) * 1_000_003 + int(s))
            p = _sample(rng, t)
            p["seed"] = int(s)
            cfg, ops = _build(p)
            params.append(p)
            cfgs.append(cfg)
            lists.append(ops)
    return np.stack(cfgs), pack_ops(lists), params


def capacity_sweep(R: int = 60, A: int = 70, U_range=range(1, 136)):
    """The capacity sweep input: L-HARD and the
    native/no-admit pair over usable sizes.  Returns (cfgs, ops, params)."""
    params, cfgs, lists = [], [], []
    for U in U_range:
        for policy in ("hard", "native", "noadmit"):
            if R > U:
                continue
            if policy == "hard":
                ops = [op(INSERT, O_RES, x=R), op(SUBMIT, 0, O_RES, HARD, R, R, 0),
                       op(ADMIT, 0, O_ACT, 1, 16 * A, 16 * A, 0), op(ADVANCE, 0), op(COMPLETE, 0),
                       op(TOUCH, O_RES)]
                cfg = make_cfg(U, CONTRACT)
            else:
                wa = 1 if policy == "native" else 0
                ops = [op(INSERT, O_RES, x=R), op(SUBMIT, 0, O_RES, HARD, R, R, 0),
                       op(ADMIT, 0, O_ACT, wa, 16 * A, 16 * A, 0), op(ADVANCE, 0),
                       op(COMPLETE, 0), op(TOUCH, O_RES)]
                cfg = make_cfg(U, NATIVE)
            params.append(dict(U=U, R=R, A=A, policy=policy))
            cfgs.append(cfg)
            lists.append(ops)
    return np.stack(cfgs), pack_ops(lists), params
