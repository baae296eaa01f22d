#!/usr/bin/env python3
"""bench.py -- batched resident-KV-claim arbitration on B200 (BASELINE.json metric:
allocator events/s and traces/s at 1/2/4/8 GPUs, % of HBM roofline).

One bench step = one pass of the whole hot path over one batch:
  rkc_pool_reset -> rkc_step_batch(T=256 lockstep steps over this rank's traces, ops
  resident in HBM) -> rkc_telemetry_read (K2 event compaction + K3 outcome
  histogram, device outputs) -> NCCL allreduce of the histogram (N > 1).
Default workload (config c5 = BASELINE.json configs[4], strong scaling): 10^6 random
traces in total, 1024-block pools, T = 256 steps; rank r of N replays trace ids
[r*10^6/N, (r+1)*10^6/N).  --config c3 (100k traces per GPU, weak scaling), c4, c6.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config c3|c4|c5|c6]
Under torchrun (N > 1) every rank runs; rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "allocator events/sec and traces/sec at 1/2/4/8 B200; % of HBM roofline"
UNIT = "events/s"
SEED = 0
# workloads: the default is c5 (BASELINE.json configs[4], "1M random
# traces sharded over 1/2/4/8 B200" -- the configuration the metric "at 1/2/4/8 B200" is
# quoted on; it fits one GPU); c3 (configs[2], 100k traces per GPU, weak scaling), c4
# (configs[3]) and c6 (c3 + prefix hits) are selectable with --config
WORKLOADS = {
    "c3": dict(recipe=3, traces=100_000, nblk=1024, steps=256, C=16, Q=16, O=64, ept=512,
               desc="c3: 100k random traces per GPU, 1024-block pools (16-token blocks), T=256 "
                    "lockstep steps, mixed chunked prefill/decode, 4-16 claims",
               l2="inputs larger than L2: pool state 0.83 GB + ops 0.41 GB per GPU, no flush"),
    "c4": dict(recipe=4, traces=10_000, nblk=65536, steps=1024, C=16, Q=16, O=128, ept=1024,
               desc="c4: 10k random traces per GPU, 65536-block pools (Llama-3-8B-sized KV), "
                    "T=1024 lockstep steps, long shared prefixes, demotion/expiry churn",
               l2="inputs larger than L2: pool state 5.2 GB + ops 0.16 GB per GPU, no flush"),
    # c6 (NEXT f3): the c3 recipe with half of the admissions replaced by
    # prefix-hit admissions on a known object (shared, pinned leading prefix)
    "c6": dict(recipe=6, traces=100_000, nblk=1024, steps=256, C=16, Q=16, O=64, ept=512,
               desc="c6: c3 + prefix hits (NEXT f3): 100k random traces per GPU, 1024-block pools, "
                    "T=256 lockstep steps, half of the admissions share a known object's surviving prefix",
               l2="inputs larger than L2: pool state 0.83 GB + ops 0.41 GB per GPU, no flush"),
    # c8 (NEXT f4): the c3 recipe with admission under the resident reserve on 40 % of the traces
    "c8": dict(recipe=8, traces=100_000, nblk=1024, steps=256, C=16, Q=16, O=64, ept=512,
               desc="c8: c3 + resident-reserve admission (NEXT f4): 100k random traces per GPU, "
                    "1024-block pools, T=256 lockstep steps, admit_check PEAK/NONE/RESERVE .4/.2/.4",
               l2="inputs larger than L2: pool state 0.83 GB + ops 0.41 GB per GPU, no flush"),
    # c5 (configs[4]): 10^6 c3 traces in total, sharded over the ranks (strong scaling)
    "c5": dict(recipe=3, traces=1_000_000, nblk=1024, steps=256, C=16, Q=16, O=64, ept=512, strong=True,
               desc="c5: 10^6 random c3 traces sharded over the GPUs (1024-block pools, T=256 lockstep "
                    "steps), outcome histograms NCCL-allreduced",
               l2="inputs larger than L2: pool state 8.3 GB + ops 4.1 GB per GPU at N=1, no flush"),
}
WL = WORKLOADS["c3"]
TRACES, NBLK, TSTEPS, C, Q, O, EPT = (WL[k] for k in ("traces", "nblk", "steps", "C", "Q", "O", "ept"))


_T0 = time.time()


def _phase(what: str) -> None:
    """wall-clock progress on stderr (the JSON line stays alone on stdout)"""
    print(f"[bench {time.time() - _T0:7.1f} s] {what}", file=sys.stderr, flush=True)


def select_workload(name: str):
    global WL, TRACES, NBLK, TSTEPS, C, Q, O, EPT
    WL = WORKLOADS[name]
    TRACES, NBLK, TSTEPS, C, Q, O, EPT = (WL[k] for k in ("traces", "nblk", "steps", "C", "Q", "O", "ept"))


def shard(rank: int, world: int) -> tuple[int, int]:
    """(first trace id, trace count) of this rank (paper_2605_24259_b200/shard.py):
    weak scaling replays WL["traces"] per rank; strong scaling (c5) splits
    WL["traces"] over the ranks."""
    from paper_2605_24259_b200.shard import shard_range, weak_range
    lo, hi = (shard_range(rank, world, WL["traces"]) if WL.get("strong")
              else weak_range(rank, WL["traces"]))
    return lo, hi - lo


def scaling() -> str:
    return "strong" if WL.get("strong") else "weak"


def workload_config(n_gpus: int) -> dict:
    per = shard(0, n_gpus)[1]
    return {"workload": WL["desc"], "traces_per_gpu": per, "pool_blocks": NBLK,
            "steps_per_replay": TSTEPS,
            "global_traces": WL["traces"] if WL.get("strong") else WL["traces"] * n_gpus,
            "parallelism": f"trace-sharded x{n_gpus}", "l2": WL["l2"]}


# --------------------------------------------------------------------------
# algorithmic bytes of the lockstep step: SURVEY.md sec. 8(d) per-op table
# --------------------------------------------------------------------------
K_BLOCKS_ALLOCATED, K_ALLOCATIONS = 21, 30          # rkc.h RKC_CTR_*
H_LANES = 128 + 128                                 # claim lanes + request lanes


def survey_bytes(ops: np.ndarray, counters: np.ndarray, events: np.ndarray) -> dict:
    """Bytes one full replay must move by SURVEY.md sec. 8(d)'s per-op table
    (flat SoA layout: meta u32[N] + seq u32[N] + free bitmap N/8, header H =
    claim lanes 128 B + request lanes 128 B).  Where the table gives an upper
    bound ("<= 64") the bound is used for SUBMIT / DEMOTE and nothing for a
    NOP; where a row depends on the outcome, the outcome comes from this
    replay's own telemetry (events, counters):

      every trace-step (NOP too)   reads 16 + H
      SUBMIT / DEMOTE              writes 64
      ADMIT / HIT_ADMIT            writes 32
      ADVANCE without allocation   writes 32 (the request record; the table's
                                   need <= free row with need = 0, no bitmap read)
      allocation, need <= free     reads N/8, writes 4 need + 4 ceil(need/32) + 32
                                   (ceil(need/32) >= 1 per allocation: 4 is used)
      allocation with eviction     reads 4N + 4N + N/8, writes 4 k + 4 + 32
                                   (+ 4 n seq words for an evicting INSERT)
      COMPLETE                     reads 4N, writes 8 live (live >= blocks cached
                                   or freed, from REQUEST_SERVED / WRITE_ADMISSION_DENIED)
      TOUCH                        reads 4N, writes 4 L (L from REUSE_PROBE)
      deferral / refusal           reads 4N (release of the request's blocks: not in
                                   the table, counted like COMPLETE's scan)
      HIT_ADMIT with h > 0 (f3)    reads 4N, writes 4 h (restamp, like TOUCH)
      every event                  writes 32
    """
    T, n = ops.shape
    N = NBLK
    kind = ops["kind"]
    et = events["type"]
    cnt = {k: int((kind == k).sum()) for k in range(9)}
    n_alloc = int(counters[:, K_ALLOCATIONS].astype(np.int64).sum())
    k_all = int(counters[:, K_BLOCKS_ALLOCATED].astype(np.int64).sum())
    vic = events[et == 12]
    n_ev = len(vic)
    k_ev = int(vic["f"][:, 3].astype(np.int64).sum())
    k_ev_insert = int(vic[vic["reason"] == 1]["f"][:, 3].astype(np.int64).sum())
    n_af, k_af = n_alloc - n_ev, k_all - k_ev
    n_inserted = int(counters[:, 15].astype(np.int64).sum())
    adv_alloc = n_alloc - n_inserted
    served = events[et == 11]
    denied = events[et == 10]
    live_blocks = int(served[served["reason"] == 1]["f"][:, 1].astype(np.int64).sum()) + \
        int(denied["f"][:, 1].astype(np.int64).sum())
    probes = events[et == 13]
    L_sum = int(probes["f"][:, 1].astype(np.int64).sum())
    hits = events[et == 15]
    hits_pos = hits[hits["f"][:, 1] > 0]
    refusals = int(((et == 7) | (et == 8)).sum())
    rd = n * T * (16 + H_LANES)
    wr = 64 * (cnt[1] + cnt[6]) + 32 * (cnt[2] + cnt[8]) + 32 * max(0, cnt[3] - adv_alloc)
    rd += n_af * (N // 8)
    wr += 4 * k_af + n_af * (4 + 32)
    rd += n_ev * (8 * N + N // 8)
    wr += 4 * k_ev + n_ev * (4 + 32) + 4 * k_ev_insert
    rd += len(served) * 4 * N
    wr += 8 * live_blocks
    rd += len(probes) * 4 * N
    wr += 4 * L_sum
    rd += refusals * 4 * N
    rd += len(hits_pos) * 4 * N
    wr += 4 * int(hits_pos["f"][:, 1].astype(np.int64).sum())
    wr += 32 * len(events)
    return dict(bytes=int(rd + wr), read=int(rd), write=int(wr), allocations=n_alloc,
                evicting_selections=n_ev, events=len(events))


# --------------------------------------------------------------------------
# this layout's own byte model, reported beside it
# --------------------------------------------------------------------------
def algorithmic_bytes(ops: np.ndarray, counters: np.ndarray, events: np.ndarray) -> dict:
    """Bytes the method must move in this layout for one full replay, by what
    each op semantically reads and writes:

    every trace-step     : op 16 + hot header 64 (next expiry, U, P, Alive, free, policy)
    ADMIT                : request 32 read + 32 write
    ADVANCE              : request 32 read + 8 write (done, live)
      free-only alloc    : free bitmap N/8 read + N/8 write + 8 per block (meta, key)
      evicting alloc     : keys 4N + bitmap N/8 + claim table 32C + object table 8O
                           (victim attribution) + 12 per taken block + header write 64
    deferral / refusal   : meta scan 4N + 8 per released block + header write 64
    COMPLETE             : request 32 + target object 8 + meta scan 4N + 8 per block + header 64
    SUBMIT               : claim table 32C (duplicate, reserve rule) + object 8 + writes 40
    DEMOTE / expiry      : claim 32 read + 32 write
    claim-state change   : reclass pass meta 4N + keys 4N (accepted, demoted, expired, harmed)
    INSERT               : object 8 + claim 32 + allocation as above + header write 64
    TOUCH                : object 8 + claim 32 + meta scan 4N + key read+write 8 per leading block
    HIT_ADMIT (f3)       : request 32 read + 32 write + object table 8O + claim 32; a hit of
                           h > 0 blocks: other requests' status/hit 8Q + meta scan 4N + 8 per
                           pinned block + reclass pass 8N, and the same again when it unpins
    event                : 32 (write); counters 4 per op (reduction)
    """
    T, n = ops.shape
    kind = ops["kind"]
    N = NBLK
    et = events["type"]
    cnt = {k: int((kind == k).sum()) for k in range(9)}
    non_nop = n * T - cnt[0]
    vic = events[et == 12]
    n_evict = len(vic)
    k_evict = int(vic["f"][:, 3].astype(np.int64).sum())
    k_all = int(counters[:, 21].astype(np.int64).sum())
    k_free = max(0, k_all - k_evict)
    n_alloc_free = int((counters[:, 21] > 0).sum())  # lower bound on free-only allocations
    refusals = int(((et == 7) | (et == 8)).sum())
    served = int((et == 11).sum())
    served_blocks = int(events[et == 11]["f"][:, 1].astype(np.int64).sum())
    probes = events[et == 13]
    touch_scans = int((probes["f"][:, 1] > 0).sum())
    touch_blocks = int(probes["f"][:, 1].astype(np.int64).sum())
    claim_changes = int(((et == 1) | (et == 4) | (et == 5) | (et == 6)).sum())
    b = 0
    b += n * T * (16 + 64)
    b += cnt[2] * 64
    b += cnt[3] * 40
    b += k_free * 8 + n_alloc_free * (N // 4)
    b += n_evict * (4 * N + N // 8 + 32 * C + 8 * O + 64) + 12 * k_evict
    b += refusals * (4 * N + 64)
    b += served * (32 + 8 + 4 * N + 64) + 8 * served_blocks
    b += cnt[1] * (32 * C + 8 + 40)
    b += (cnt[6] + int((et == 5).sum())) * 64
    b += claim_changes * 8 * N
    b += cnt[5] * (8 + 32 + 64)
    b += touch_scans * 4 * N + cnt[7] * 40 + 8 * touch_blocks
    hits = events[et == 15]
    pinning = hits[hits["f"][:, 1] > 0]
    b += cnt[8] * (64 + 8 * O + 32)
    b += 2 * len(pinning) * (8 * Q + 4 * N + 8 * N) + 16 * int(pinning["f"][:, 1].astype(np.int64).sum())
    b += 32 * len(events) + 4 * non_nop
    return dict(bytes=int(b), non_nop=non_nop, evicting_selections=n_evict, events=len(events))


# --------------------------------------------------------------------------
def clocks_sampler(path: str, gpu_index: int):
    q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    try:
        return subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={q}",
                                 "--format=csv,noheader,nounits", "-lms", "100"],
                                stdout=open(path, "w"), stderr=subprocess.DEVNULL)
    except Exception:
        return None


def clocks_summary(path: str) -> dict:
    sm, mx, reasons = [], [], set()
    try:
        for line in open(path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                "sw_power_cap"), f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
    except OSError:
        pass
    if not sm:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
    return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
            "samples": len(sm)}


def load_peak() -> tuple[float, str]:
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _ncu_json() -> dict | None:
    name = "ncu_step_kernel.json" if WL is WORKLOADS["c3"] else f"ncu_step_kernel_{WL['desc'][:2]}.json"
    try:
        return json.load(open(os.path.join(ROOT, "profiles", name)))
    except Exception:
        return None


def load_traffic() -> float | None:
    """dram bytes per lockstep step from the committed ncu --set full capture of this workload."""
    d = _ncu_json()
    return float(d["dram_bytes_per_launch"]) if d and "dram_bytes_per_launch" in d else None


def issue_roofline(step_us: float, sm_mhz: float) -> dict | None:
    """Secondary roofline: the step is issue / latency bound, so report the
    warp-instruction rate of one lockstep step (instructions per step from the committed ncu
    capture, time from this run) against the issue peak 148 SMs x 4 schedulers x 1 warp
    instruction per cycle at the SM clock measured during the timed region."""
    d = _ncu_json()
    if not d or "warp_instructions_per_launch" not in d or not sm_mhz:
        return None
    achieved = d["warp_instructions_per_launch"] / (step_us * 1e-6) / 1e12
    peak = 148 * 4 * sm_mhz * 1e6 / 1e12
    return {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "T warp-inst/s",
            "frac": achieved / peak, "source": "warp instructions per step: profiles/" +
            ("ncu_step_kernel.json" if WL is WORKLOADS["c3"] else f"ncu_step_kernel_{WL['desc'][:2]}.json")}


# --------------------------------------------------------------------------
def host_info() -> dict:
    """lscpu model / sockets x cores x threads and the oracle's compiler."""
    info = {}
    try:
        out = subprocess.check_output(["lscpu"], text=True, env={**os.environ, "LC_ALL": "C"})
        kv = {ln.split(":", 1)[0].strip(): ln.split(":", 1)[1].strip() for ln in out.splitlines()
              if ":" in ln}
        info = {"cpu_model": kv.get("Model name"), "sockets": kv.get("Socket(s)"),
                "cores_per_socket": kv.get("Core(s) per socket"),
                "threads_per_core": kv.get("Thread(s) per core"), "cpus": kv.get("CPU(s)"),
                "numa_nodes": kv.get("NUMA node(s)")}
    except Exception:
        pass
    try:
        info["compiler"] = subprocess.check_output(["g++", "--version"], text=True).splitlines()[0]
    except Exception:
        info["compiler"] = None
    info["flags"] = "-O2 -std=c++17 (no -march=native)"
    return info


def _compare_chunk(b, lo: int, hi: int, g_counters, g_events, g_idx) -> tuple[int, int]:
    """(#traces whose events or counters differ, #events compared) for oracle batch b
    holding traces [lo, hi) of this rank's pool."""
    oe = b.events()
    oe["trace"] += lo                                     # oracle trace ids are batch-local
    ge = g_events[g_idx[lo]:g_idx[hi]]
    bad = set()
    if ge.tobytes() != oe.tobytes():
        oi = np.searchsorted(oe["trace"], np.arange(lo, hi + 1))
        for t in range(lo, hi):
            a = ge[g_idx[t] - g_idx[lo]:g_idx[t + 1] - g_idx[lo]]
            bb = oe[oi[t - lo]:oi[t - lo + 1]]
            if a.tobytes() != bb.tobytes():
                bad.add(t)
    cd = np.nonzero((b.counters() != g_counters[lo:hi]).any(1))[0]
    bad.update(int(lo + i) for i in cd)
    return len(bad), len(oe)


def _compare_views(pool, b, lo: int, n: int) -> bool:
    """final state views (header, blocks, claims, requests, objects) of traces
    [lo, lo + n): GPU export vs oracle export, byte for byte"""
    g = pool.rkc_state_export(lo, n)
    for i in range(n):
        o = b.export(i)
        for k in ("header", "blocks", "claims", "requests", "objects"):
            if np.ascontiguousarray(g[k][i]).tobytes() != np.ascontiguousarray(o[k]).tobytes():
                return False
    return True


def cpu_baseline(cfgs, ops, g_counters, g_events, pool, budget_s: float = 12.0,
                 single_budget_s: float = 4.0) -> tuple[dict, dict]:
    """The oracle as it stands, on the host cores, on a bounded sample of the
    same workload (the first traces of rank 0's shard): one figure on a single
    core and one on every host core (SURVEY 8(d) "Oracle timing").  Outside
    the timing, the oracle's results for the sampled traces are compared bit
    for bit with the GPU's replay of the same traces in the bench's own pool
    (events, counters, and the final state views of the first 64 traces)."""
    from oracle import oracle as orc
    try:
        os.sched_setaffinity(0, range(os.cpu_count() or 1))   # every host core for the oracle
    except Exception:
        pass
    nthreads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    g_idx = np.searchsorted(g_events["trace"], np.arange(ops.shape[1] + 1))
    checked, mism, ev_checked = 0, 0, 0
    # single core
    n1, ops1, t1 = 0, 0, 0.0
    while t1 < single_budget_s and n1 < ops.shape[1]:
        sl = slice(n1, min(n1 + 16, ops.shape[1]))
        sub = np.ascontiguousarray(ops[:, sl])
        b = orc.OracleBatch(cfgs[sl], NBLK, C, Q, O)
        t0 = time.perf_counter()
        b.run(sub, nthreads=1)
        t1 += time.perf_counter() - t0
        ops1 += int((sub["kind"] != 0).sum())
        n1 = sl.stop
    # all cores; every chunk is checked against the GPU after its timing
    chunk = max(64, 16 * nthreads) if WL["recipe"] != 4 else max(4, nthreads)
    done_traces, ops_done, t_used = 0, 0, 0.0
    views_ok = None
    while t_used < budget_s and done_traces < ops.shape[1]:
        sl = slice(done_traces, min(done_traces + chunk, ops.shape[1]))
        sub = np.ascontiguousarray(ops[:, sl])
        b = orc.OracleBatch(cfgs[sl], NBLK, C, Q, O)
        t0 = time.perf_counter()
        b.run(sub, nthreads=nthreads)
        t_used += time.perf_counter() - t0
        ops_done += int((sub["kind"] != 0).sum())
        m, ne = _compare_chunk(b, sl.start, sl.stop, g_counters, g_events, g_idx)
        mism += m
        ev_checked += ne
        checked += sl.stop - sl.start
        if views_ok is None:
            nv = min(64, sl.stop - sl.start)
            views_ok = _compare_views(pool, b, sl.start, nv)
        done_traces = sl.stop
    base = {"value": ops_done / t_used, "unit": UNIT, "cores": nthreads, "kind": "oracle",
            "sample": f"first {done_traces} traces of the {WL['desc'][:2]} workload x {TSTEPS} steps "
                      f"({ops_done} non-NOP ops) in {t_used:.1f} s, plain C++ oracle, "
                      f"{nthreads} threads, one trace per task",
            "traces_per_s": done_traces / t_used,
            "single_core": {"value": ops1 / t1, "unit": UNIT, "cores": 1,
                            "sample": f"first {n1} traces x {TSTEPS} steps ({ops1} non-NOP ops) "
                                      f"in {t1:.1f} s"},
            "host": host_info()}
    parity = {"status": "sampled-bit-exact" if mism == 0 and views_ok else "MISMATCH",
              "traces_checked": checked, "events_checked": ev_checked,
              "traces_mismatched": mism, "state_views_first_64": bool(views_ok),
              "what": "the oracle's events (trace, step, seq order), counters and final state "
                      "views vs the GPU replay of the same traces in the bench's own pool"}
    return base, parity


def run_reference(args, rank: int, world: int):
    """--impl reference: the oracle, as it stands, on the host cores (rank 0 only)."""
    if rank != 0:
        return
    from paper_2605_24259_b200 import gen
    from oracle import oracle as orc
    nthreads = os.cpu_count() or 1
    sample = max(64, 32 * nthreads) if WL["recipe"] == 3 else max(8, nthreads)
    cfgs, ops = gen.random_traces(WL["recipe"], SEED, 0, sample, TSTEPS, NBLK, C, Q, O)
    non_nop = int((ops["kind"] != 0).sum())
    times = []
    for i in range(args.warmup + args.steps):
        b = orc.OracleBatch(cfgs, NBLK, C, Q, O)
        t0 = time.perf_counter()
        b.run(ops, nthreads=nthreads)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    t = float(np.sum(times))
    value = non_nop * args.steps / t
    desc = (f"each step: the first {sample} traces of the {WL['desc'][:2]} workload x {TSTEPS} steps "
            f"({non_nop} non-NOP ops), plain C++ oracle, {nthreads} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t / args.steps,
        "higher_is_better": True, "scaling": scaling(), "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "config": workload_config(world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "traces_per_s": sample * args.steps / t,
    }), flush=True)


# --------------------------------------------------------------------------
def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def respawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: re-run this command under
    torchrun with N ranks on this node (rendezvous on 127.0.0.1), the same
    launch the driver uses; returns torchrun's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def bind_numa(gpu: int) -> dict:
    """Bind this process to the CPUs of the GPU's NUMA node (pinned host
    buffers are then allocated node-locally); returns what was found."""
    out = {"numa_node": None, "bound_cpus": None}
    try:
        bus = subprocess.check_output(["nvidia-smi", "-i", str(gpu), "--query-gpu=pci.bus_id",
                                       "--format=csv,noheader"], text=True).strip()
        dom, rest = bus.split(":", 1)
        path = f"/sys/bus/pci/devices/{dom[-4:].lower()}:{rest.lower()}/numa_node"
        node = int(open(path).read().strip())
        out["numa_node"] = node
        if node >= 0:
            cpus = set()
            for part in open(f"/sys/devices/system/node/node{node}/cpulist").read().strip().split(","):
                a, _, b = part.partition("-")
                cpus.update(range(int(a), int(b or a) + 1))
            os.sched_setaffinity(0, cpus)
            out["bound_cpus"] = len(cpus)
    except Exception:
        pass
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="rkc", choices=["rkc", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=9)  # median of 9: host-side copy noise on shared boxes
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="c5", choices=sorted(WORKLOADS))
    args = ap.parse_args()
    select_workload(args.config)
    args.warmup = max(3, args.warmup)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(respawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2605_24259_b200 import build, gen
    if rank == 0:                 # the other ranks wait at the barrier below
        build.build()
        gen.build()
    from paper_2605_24259_b200.shard import allreduce_histogram

    # one process per GPU over NCCL.  With fewer GPUs than ranks (e.g. the
    # 1-GPU lease), ranks share devices round-robin over gloo: the multi-rank
    # path runs end to end, but the numbers are time-sliced, not a scaling point.
    ndev = torch.cuda.device_count()
    oversub = world > ndev or bool(os.environ.get("RKC_BENCH_SAME_GPU"))
    gpu = local_rank % max(1, ndev)
    torch.cuda.set_device(gpu)
    dist_on = world > 1
    if dist_on:
        backend = os.environ.get("RKC_DIST_BACKEND", "gloo" if oversub else "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(backend)
        dist.barrier()
    from paper_2605_24259_b200 import rkc
    host = bind_numa(gpu)
    dev = torch.device("cuda", gpu)
    if os.environ.get("RKC_BENCH_WATCHDOG"):          # debugging: dump every stack if stuck
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["RKC_BENCH_WATCHDOG"]), exit=True)
    gloo = dist_on and dist.get_backend() == "gloo"

    def allreduce(t, op=None):
        """SUM (or `op`) over ranks; gloo reduces a host copy (no gloo CUDA path)"""
        if not dist_on:
            return t
        if gloo:
            h = t.cpu()
            if op is None:
                allreduce_histogram(h)
            else:
                dist.all_reduce(h, op=op)
            t.copy_(h)
        elif op is None:
            allreduce_histogram(t)
        else:
            dist.all_reduce(t, op=op)
        return t

    # ---- inputs: this rank's shard, generated on the host, resident in HBM ----
    global TRACES
    first, TRACES = shard(rank, world)
    _phase("start")
    cfgs, ops = gen.random_traces(WL["recipe"], SEED, first, TRACES, TSTEPS, NBLK, C, Q, O)
    non_nop = int((ops["kind"] != 0).sum())
    ops_u8 = ops.view(np.uint8).reshape(-1)
    ops_dev = torch.from_numpy(ops_u8).to(dev)
    ops_pinned = torch.empty(ops_u8.size, dtype=torch.uint8, pin_memory=True)
    ops_pinned.numpy()[:] = ops_u8
    _phase("inputs generated and staged")
    pool = rkc.Pool(cfgs, NBLK, C, Q, O, events_per_trace=EPT, device=gpu)
    stream = torch.cuda.current_stream(dev)
    ev_cap = TRACES * EPT
    events_dev = torch.empty(ev_cap * 32, dtype=torch.uint8, device=dev)
    hist_dev = torch.zeros(rkc.RKC_NHIST, dtype=torch.int64, device=dev)

    def one_step(ev_pair=None):
        pool.rkc_pool_reset(stream)
        if ev_pair is not None:
            ev_pair[0].record(stream)
        pool.rkc_step_batch(ops_dev, TSTEPS, stream)
        if ev_pair is not None:
            ev_pair[1].record(stream)
        pool.rkc_telemetry_read(events_out=events_dev, hist_out=hist_dev, stream=stream)
        allreduce(hist_dev)

    _phase("pool created")
    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()

    _phase("warm-up done")
    # ---- timed region (device events; barrier + sync both sides) ----
    clk_path = os.path.join(tempfile.gettempdir(), f"rkc_clocks_{rank}.csv")
    sampler = clocks_sampler(clk_path, gpu)
    time.sleep(0.3)
    pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
             for _ in range(args.steps)]
    launches0 = rkc.rkc_launch_count()
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for i in range(args.steps):
        one_step(pairs[i])
    stop.record(stream)
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    launches = rkc.rkc_launch_count() - launches0
    if sampler is not None:
        sampler.terminate()
        sampler.wait()
    ms = start.elapsed_time(stop)
    step_kernel_ms = sum(a.elapsed_time(b) for a, b in pairs)
    t = torch.tensor([ms, step_kernel_ms], dtype=torch.float64, device=dev)
    allreduce(t, dist.ReduceOp.MAX)
    ms, step_kernel_ms = float(t[0]), float(t[1])

    _phase("timed region done")
    # ---- e2e: the public C-ABI call with HOST buffers (pinned ops in, results out) ----
    # results land in pinned host memory (a user's choice the C ABI allows)
    counters_host = torch.zeros((TRACES, rkc.RKC_NCTR), dtype=torch.int32,
                                pin_memory=True).numpy().view(np.uint32)
    hist_host = torch.zeros(rkc.RKC_NHIST, dtype=torch.int64, pin_memory=True).numpy()
    # one untimed pass first: the library allocates its host-replay buffers on
    # first use and the pinned pages are touched once
    pool.rkc_pool_reset(stream)
    _step_host(pool, ops_pinned, stream)
    _, n_events = pool.rkc_telemetry_read(counters_out=counters_host, hist_out=hist_host,
                                          stream=stream)

    def e2e_pass(events_host=None) -> float:
        # ranks that share a GPU (oversubscribed harness) take turns: the
        # host-replay path of two contexts time-slicing one GPU is not what
        # the line reports, and was seen to stall
        turns = range(world) if oversub and dist_on else [rank]
        ms_pass = 0.0
        for r in turns:
            if dist_on:
                dist.barrier()
            if r != rank:
                continue
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pool.rkc_pool_reset(stream)
            _step_host(pool, ops_pinned, stream)
            pool.rkc_telemetry_read(counters_out=counters_host, events_out=events_host,
                                    hist_out=hist_host, stream=stream)
            if dist_on and not oversub:                    # the histogram SUM over ranks (NCCL)
                hd = torch.from_numpy(hist_host).to(dev)
                allreduce(hd)
                hist_host[:] = hd.cpu().numpy()
            e1.record(stream)
            torch.cuda.synchronize()
            ms_pass = e0.elapsed_time(e1)
        if dist_on and oversub:                            # gloo: outside the device-timed pass
            hd = torch.from_numpy(hist_host).to(dev)
            allreduce(hd)
            hist_host[:] = hd.cpu().numpy()
        te = torch.tensor([ms_pass], dtype=torch.float64, device=dev)
        allreduce(te, dist.ReduceOp.MAX)
        return float(te[0])

    e2e_all = [e2e_pass() for _ in range(max(3, args.e2e_steps))]
    e2e_ms = float(np.median(e2e_all))
    # the same with the compacted claim-level event stream read back too (the
    # paper's telemetry), when host memory allows a pinned buffer
    ev_bytes = int(n_events) * 32
    e2e_ev_ms = None
    try:
        avail = int([ln.split()[1] for ln in open("/proc/meminfo")
                     if ln.startswith("MemAvailable")][0]) * 1024
    except Exception:
        avail = 0
    if ev_bytes and ev_bytes < avail // 4:
        events_host = torch.empty(ev_bytes, dtype=torch.uint8, pin_memory=True).numpy()
        e2e_pass(events_host)                              # touch the pages once
        e2e_ev_ms = float(np.median([e2e_pass(events_host) for _ in range(5)]))
        del events_host
    # this box's pinned host->device copy bandwidth (the e2e floor is
    # h2d_bytes_per_step / h2d_gbs when the copies outrun the steps)
    probe = ops_pinned[: min(ops_pinned.numel(), 256 << 20)]
    probe_dev = torch.empty(probe.numel(), dtype=torch.uint8, device=dev)
    probe_dev.copy_(probe, non_blocking=True)
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0.record(stream)
    for _ in range(3):
        probe_dev.copy_(probe, non_blocking=True)
    h1.record(stream)
    torch.cuda.synchronize()
    h2d_gbs = 3 * probe.numel() / (h0.elapsed_time(h1) * 1e-3) / 1e9
    del probe_dev

    _phase("e2e done")
    # ---- telemetry of one replay for the algorithmic byte models (outside timing) ----
    counters, events, hist = pool.read_all()
    sb = survey_bytes(ops, counters, events)
    ab = algorithmic_bytes(ops, counters, events)
    tot = torch.tensor([non_nop, TRACES, len(events), sb["bytes"], ab["bytes"]],
                       dtype=torch.float64, device=dev)
    allreduce(tot, dist.ReduceOp.SUM)
    total_events, total_traces, total_records = float(tot[0]), float(tot[1]), float(tot[2])
    survey_total, layout_total = float(tot[3]), float(tot[4])

    clk = clocks_summary(clk_path)
    parity = None
    if rank == 0 and not args.no_cpu_baseline:
        _phase("cpu baseline + sampled parity")
        cpu, parity = cpu_baseline(cfgs, ops, counters, events, pool)
    if dist_on:
        dist.barrier()
    if rank != 0:
        if dist_on:
            dist.destroy_process_group()
        return
    peak, peak_src = load_peak()
    per_launch_ms = step_kernel_ms / (args.steps * TSTEPS)
    # every rank's lockstep step runs concurrently: bytes of all ranks / the max step time
    achieved = survey_total / TSTEPS / (per_launch_ms * 1e-3) / 1e9
    achieved_layout = layout_total / TSTEPS / (per_launch_ms * 1e-3) / 1e9
    traffic = load_traffic()
    value = total_events * args.steps / (ms * 1e-3)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": scaling(), "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": workload_config(world),
        "traces_per_s": total_traces * args.steps / (ms * 1e-3),
        "telemetry_records_per_s": total_records * args.steps / (ms * 1e-3),
        "events_per_step": total_events,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "lockstep step: rkc_light_kernel + rkc_step_kernel + rkc_step_overflow_kernel",
                     "peak_source": peak_src,
                     "byte_model": "SURVEY.md 8(d) per-op table (bench.py survey_bytes)",
                     "algorithmic_bytes_per_launch": survey_total / TSTEPS,
                     "avg_launch_us": per_launch_ms * 1e3,
                     "step_kernel_share": step_kernel_ms / ms,
                     "layout_model": {"bytes_per_launch": layout_total / TSTEPS,
                                      "achieved": achieved_layout, "frac": achieved_layout / peak,
                                      "what": "this layout's own byte model (DESIGN.md sec. 6)"}},
        "e2e": {"value": total_events / (e2e_ms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": int(ops_u8.size),
                "d2h_bytes_per_step": int(counters_host.nbytes + hist_host.nbytes),
                "ms_per_step": e2e_ms, "passes_ms": e2e_all, "stat": "median",
                "h2d_gbs_measured": h2d_gbs,
                "path": "rkc_pool_reset + rkc_step_batch(pinned host ops) + "
                        "rkc_telemetry_read(host counters + histogram)"},
        "gpu_launches": int(launches),
        "clocks": clk,
        "host": host,
    }
    if e2e_ev_ms is not None:
        out["e2e_with_events"] = {
            "value": total_events / (e2e_ev_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ev_ms,
            "h2d_bytes_per_step": int(ops_u8.size),
            "d2h_bytes_per_step": int(counters_host.nbytes + hist_host.nbytes + ev_bytes),
            "path": "as e2e, plus the compacted claim-level event stream read into pinned host memory"}
    if oversub:
        out["oversubscribed"] = (f"{world} ranks share {ndev} GPU(s) over gloo: the multi-rank "
                                 "path end to end, time-sliced, not a scaling figure")
    iss = issue_roofline(per_launch_ms * 1e3, (clk or {}).get("sm_mhz") or 0)
    if iss:
        out["roofline_issue"] = iss
    _phase("telemetry + byte model done")
    if parity is not None:
        out["cpu_baseline"] = cpu
        out["parity"] = parity["status"]
        out["parity_detail"] = parity
    print(json.dumps(out), flush=True)
    if dist_on:
        dist.destroy_process_group()


def _step_host(pool, ops_pinned, stream):
    # rkc_step_batch with a HOST (pinned) op stream: the library copies it in
    # double-buffered chunks on its copy stream, overlapped with the steps
    from paper_2605_24259_b200 import rkc
    rkc._check(rkc._lib.rkc_step_batch(pool.handle, ops_pinned.data_ptr(), TSTEPS, 0,
                                       stream.cuda_stream), "rkc_step_batch")


if __name__ == "__main__":
    main()
