// rkc_step.cu -- K1: the lockstep step kernel.
//
// One warp owns one trace (one paged KV pool) for one step:
//   a0 op fetch -> a1 expiry -> a2 claim decision | a3 feasibility (P + A <= U,
//   P:504) -> a4 claim-excluding victim selection -> a5 block updates ->
//   a6 materialization predicate (leading prefix) -> a7 lifecycle
//   -> a8 telemetry.
// Semantics: DESIGN.md sec. 1 (the same reading the oracle implements; no
// code is shared with it).
//
// Warp-level mapping: lane c holds claim slot c in registers; the object
// table (<= 128 entries) is staged in shared memory; block words are streamed
// with coalesced 16-byte loads, lane L of vector j owning blocks
// (j*32 + L)*4 .. +3.  For pools of <= 1024 blocks the selection keys of the
// whole pool stay in registers (VPL uint4 per lane) across the threshold
// search and the apply pass.
#include <cuda_runtime.h>

#include <atomic>

#include "rkc_internal.cuh"

namespace rkc {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kWarpsPerCta = 4;

struct WarpSmem {
  uint32_t obj0[128];   // object word 0 (live | claim | len)
  uint32_t lead[128];   // leading prefix per object
  uint32_t lim3[128];   // reclass: positions < lim3 become protected (class 3)
  uint32_t lim2[128];   // reclass: positions < lim2 become soft (class 2)
  uint32_t cnt3[128];   // reclass: protected blocks found per object
  uint32_t cstate[32];  // claim state / mode / F mirrors for lane-divergent lookups
  uint32_t cmode[32];
  uint32_t cF[32];
  uint32_t ctr[32];     // counter deltas of this step
  uint32_t objdirty[4];
};

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ bool obligated(uint32_t mode) {
  return mode == M_HARD || mode == M_DEMOTABLE || mode == M_OFFLOADABLE || mode == M_EXPIRING;
}
__device__ __forceinline__ bool live_state(uint32_t st) {
  return st == C_ACCEPTED || st == C_MATERIALIZED;
}
// class a live claim of `mode` gives the blocks it covers
__device__ __forceinline__ uint32_t claim_class(uint32_t mode, uint32_t lowering) {
  if (lowering == LOW_CONTRACT && obligated(mode)) return 3;
  if (lowering != LOW_NATIVE && (mode == M_SOFT || (lowering == LOW_SOFT && obligated(mode)))) return 2;
  return 1;
}
// k-th (1-based) set bit of w
__device__ __forceinline__ uint32_t nth_set_bit(uint32_t w, uint32_t r) {
  uint32_t pos = 0;
#pragma unroll
  for (int width = 16; width >= 1; width >>= 1) {
    uint32_t c = __popc(w & ((1u << width) - 1u));
    if (r > c) { r -= c; w >>= width; pos += width; }
  }
  return pos;
}
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t u = __shfl_up_sync(kFull, v, d);
    if (lane >= (uint32_t)d) v += u;
  }
  return v;
}

struct StepArgs {
  PoolDev p;
  const uint4* ops;     // [steps][num_traces]
  uint32_t step;        // global step index of this launch
};

template <int VPL>
struct Trace {
  const PoolDev p;
  WarpSmem* s;
  uint32_t t, step, lane;
  uint32_t kind, a, b, c, x, y, z;
  uint32_t h[H_NWORDS];
  // claim lane registers (lane < C)
  uint32_t cw0, cF, cR, cD, cdec, cpc;
  bool cdirty;
  bool claims_changed;
  // request a (uniform copy)
  uint32_t rq[8];
  bool rq_dirty;
  uint32_t nev;
  uint32_t rc0, rc1, rc2, rc3;  // reclass mask over objects
  uint32_t* key;
  uint32_t* meta;
  uint32_t* fbm;
  uint32_t nvec;

  __device__ Trace(const PoolDev& pd, WarpSmem* sm, uint32_t trace, uint32_t st)
      : p(pd), s(sm), t(trace), step(st), lane(lane_id()) {}

  __device__ __forceinline__ uint32_t U() const { return h[H_U]; }
  __device__ __forceinline__ uint32_t lowering() const { return h[H_POLICY] & 0xFFu; }
  __device__ __forceinline__ uint32_t admit_check() const { return (h[H_POLICY] >> 8) & 0xFFu; }
  __device__ __forceinline__ uint32_t defer_budget() const { return (h[H_POLICY] >> 16) & 0xFFu; }
  __device__ __forceinline__ uint32_t auto_demote() const { return h[H_POLICY] >> 24; }
  __device__ __forceinline__ uint32_t cstate() const { return cw0 & 0xFFu; }
  __device__ __forceinline__ uint32_t cmode() const { return (cw0 >> 8) & 0xFFu; }
  __device__ __forceinline__ uint32_t cobj() const { return (cw0 >> 16) & 0xFFu; }
  __device__ __forceinline__ void set_cstate(uint32_t st) { cw0 = (cw0 & ~0xFFu) | st; cdirty = true; }

  // ------------------------------ telemetry --------------------------------
  __device__ __forceinline__ void ctr_add(uint32_t k, uint32_t v) {
    if (lane == 0) s->ctr[k] += v;
  }
  __device__ __forceinline__ void write_event(uint32_t idx, uint32_t type, uint32_t seq, uint32_t slot,
                              uint32_t reason, uint32_t mask, uint32_t f0, uint32_t f1,
                              uint32_t f2, uint32_t f3) {
    if (idx < p.EPT) {
      uint4* e = p.ev + ((size_t)t * p.EPT + idx) * 2;
      e[0] = make_uint4(t, step, type | (seq << 8) | ((slot & 0xFFu) << 16) | (reason << 24), mask);
      e[1] = make_uint4(f0, f1, f2, f3);
    }
  }
  // uniform single event
  __device__ __forceinline__ void emit(uint32_t type, uint32_t slot, uint32_t reason, uint32_t mask,
                       uint32_t f0 = 0, uint32_t f1 = 0, uint32_t f2 = 0, uint32_t f3 = 0) {
    if (lane == 0) write_event(h[H_EVCOUNT] + nev, type, nev, slot, reason, mask, f0, f1, f2, f3);
    ++nev;
  }
  // one event per lane with pred, in lane (= slot) order
  __device__ __forceinline__ void emit_lanes(bool pred, uint32_t type, uint32_t slot, uint32_t reason,
                             uint32_t mask, uint32_t f0, uint32_t f1, uint32_t f2, uint32_t f3) {
    const uint32_t m = __ballot_sync(kFull, pred);
    if (pred) {
      const uint32_t r = __popc(m & lanemask_lt());
      write_event(h[H_EVCOUNT] + nev + r, type, nev + r, slot, reason, mask, f0, f1, f2, f3);
    }
    nev += __popc(m);
  }
  __device__ __forceinline__ void op_error(uint32_t code) {
    emit(EV_OP_ERROR, a, code, 0, kind);
    ctr_add(K_OP_ERRORS, 1);
  }

  // --------------------------- claim helpers -------------------------------
  __device__ __forceinline__ uint32_t claim_field(uint32_t v, uint32_t slot) const {
    return __shfl_sync(kFull, v, slot & 31u);
  }
  __device__ __forceinline__ void mirror_claims() {
    s->cstate[lane] = cstate();
    s->cmode[lane] = cmode();
    s->cF[lane] = cF;
    __syncwarp();
  }
  __device__ __forceinline__ void mark_reclass(uint32_t o) {
    const uint32_t bit = 1u << (o & 31u), w = o >> 5;
    rc0 |= w == 0 ? bit : 0u; rc1 |= w == 1 ? bit : 0u;
    rc2 |= w == 2 ? bit : 0u; rc3 |= w == 3 ? bit : 0u;
  }
  __device__ __forceinline__ bool in_reclass(uint32_t o) const {
    const uint32_t w = o >> 5;
    const uint32_t v = w == 0 ? rc0 : w == 1 ? rc1 : w == 2 ? rc2 : rc3;
    return (v >> (o & 31u)) & 1u;
  }
  __device__ __forceinline__ void mark_reclass_lanes(bool pred, uint32_t o) {
    const uint32_t bit = pred ? 1u << (o & 31u) : 0u, w = o >> 5;
    rc0 |= __reduce_or_sync(kFull, w == 0 ? bit : 0u);
    rc1 |= __reduce_or_sync(kFull, w == 1 ? bit : 0u);
    rc2 |= __reduce_or_sync(kFull, w == 2 ? bit : 0u);
    rc3 |= __reduce_or_sync(kFull, w == 3 ? bit : 0u);
  }
  __device__ __forceinline__ void mark_obj_dirty(uint32_t o) {
    if (lane == 0) s->objdirty[o >> 5] |= 1u << (o & 31u);
  }
  // P and the blocking set are derived from the per-claim protected counts
  __device__ __forceinline__ void refresh_protected() {
    h[H_P] = __reduce_add_sync(kFull, cpc);
    h[H_BLOCKMASK] = __ballot_sync(kFull, cpc > 0);
  }
  // class of a new cached block (o, pos) from the object's bound claim (smem)
  __device__ __forceinline__ uint32_t new_block_class(uint32_t o, uint32_t pos) const {
    const uint32_t c = obj_claim(s->obj0[o]);
    if (c >= 32 || !live_state(s->cstate[c])) return 1;
    if (pos >= s->cF[c]) return 1;
    return claim_class(s->cmode[c], lowering());
  }
  // a live bound protected claim of object o gains `added` protected blocks
  __device__ __forceinline__ void add_protected(uint32_t o, uint32_t added) {
    const uint32_t cc = obj_claim(s->obj0[o]);
    if (cc < 32 && lane == cc && live_state(cstate()) && claim_class(cmode(), lowering()) == 3) {
      cpc += added;
      cdirty = true;
    }
    refresh_protected();
  }

  // ----------------------------- block passes ------------------------------
  __device__ __forceinline__ uint4 ld_key(uint32_t j) const {
    return __ldcg(reinterpret_cast<const uint4*>(key) + j * 32 + lane);
  }
  __device__ __forceinline__ uint4 ld_meta(uint32_t j) const {
    return __ldcg(reinterpret_cast<const uint4*>(meta) + j * 32 + lane);
  }
  __device__ __forceinline__ static uint32_t el(const uint4& v, int e) {
    return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
  }
  __device__ __forceinline__ uint32_t block_of(uint32_t j, int e) const { return (j * 32 + lane) * 4 + e; }

  // set free-bitmap bits of blocks in nib (4 bits at block_of(j,0))
  __device__ __forceinline__ void fbm_set(uint32_t j, uint32_t nib) {
    if (nib) {
      const uint32_t b0 = block_of(j, 0);
      atomicOr(fbm + (b0 >> 5), nib << (b0 & 31u));
    }
  }

  // reclass pass: rewrite the class bits of every cached block whose owner is
  // marked, from the owner's bound claim; recount protected blocks.
  __device__ __forceinline__ void flush_reclass() {
    if ((rc0 | rc1 | rc2 | rc3) == 0) return;
    mirror_claims();
    for (uint32_t o = lane; o < p.O; o += 32) {
      uint32_t l3 = 0, l2 = 0;
      const uint32_t cc = obj_claim(s->obj0[o]);
      if (cc < 32 && live_state(s->cstate[cc])) {
        const uint32_t cls = claim_class(s->cmode[cc], lowering());
        if (cls == 3) l3 = s->cF[cc];
        if (cls == 2) l2 = s->cF[cc];
      }
      s->lim3[o] = l3;
      s->lim2[o] = l2;
      s->cnt3[o] = 0;
    }
    __syncwarp();
    for (uint32_t j = 0; j < nvec; ++j) {
      const uint4 mv = ld_meta(j);
      const uint4 kv = ld_key(j);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t m = el(mv, e);
        if (meta_res(m) != kResCached) continue;
        const uint32_t o = meta_owner(m);
        if (!in_reclass(o)) continue;
        const uint32_t pos = meta_pos(m);
        const uint32_t cls = pos < s->lim3[o] ? 3u : (pos < s->lim2[o] ? 2u : 1u);
        const uint32_t k0 = el(kv, e);
        const uint32_t k1 = (cls << kClassShift) | (k0 & kSeqMask);
        if (k1 != k0) key[block_of(j, e)] = k1;
        if (cls == 3) atomicAdd(&s->cnt3[o], 1u);
      }
    }
    __syncwarp();
    if (lane < p.C) {
      const uint32_t o = cobj();
      if (live_state(cstate()) && in_reclass(o)) {
        const uint32_t np = claim_class(cmode(), lowering()) == 3 ? s->cnt3[o] : 0u;
        if (np != cpc) { cpc = np; cdirty = true; }
      }
    }
    rc0 = rc1 = rc2 = rc3 = 0;
    refresh_protected();
  }

  // release request r's active blocks to FREE (deferral / refusal / no-admit)
  __device__ __forceinline__ uint32_t release_blocks(uint32_t r) {
    uint32_t freed = 0;
    for (uint32_t j = 0; j < nvec; ++j) {
      const uint4 mv = ld_meta(j);
      uint32_t nib = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t m = el(mv, e);
        if (meta_res(m) == kResActive && meta_owner(m) == r) {
          const uint32_t bb = block_of(j, e);
          meta[bb] = meta_make(kResFree, 0, 0);
          key[bb] = bb;
          nib |= 1u << e;
        }
      }
      fbm_set(j, nib);
      freed += __popc(nib);
    }
    freed = __reduce_add_sync(kFull, freed);
    h[H_FREE] += freed;
    return freed;
  }

  // ------------------------------ arbiter ----------------------------------
  // Feasibility boundary protected + active <= usable; relax by
  // auto-demotion (G10); else explicit refusal / deferral with
  // blocking-claim attribution and the capacity proof.
  // requester: request slot, or 0xFFFFFFFF for INSERT of object `a`.
  __device__ __forceinline__ bool arbitrate(uint32_t need, uint32_t requester) {
    const uint32_t Uu = U();
    uint32_t P = h[H_P];
    const uint64_t A = (uint64_t)h[H_ALIVE] + need;
    if ((uint64_t)P + A <= Uu) return true;
    if (lowering() == LOW_CONTRACT && auto_demote()) {
      const uint32_t g = (lane < p.C && live_state(cstate()) && cmode() == M_DEMOTABLE) ? cpc : 0u;
      const uint32_t S = warp_incl_scan(g);
      const bool ok = g > 0 && (uint64_t)(P - S) + A <= Uu;
      const uint32_t mk = __ballot_sync(kFull, ok);
      if (mk) {
        const uint32_t j = __ffs(mk) - 1;
        const bool dem = g > 0 && lane <= j;
        emit_lanes(dem, EV_DEMOTED, lane, 1, 0, cobj(), g, 0, 0);
        const uint32_t nd = __popc(__ballot_sync(kFull, dem));
        mark_reclass_lanes(dem, cobj());
        if (dem) { set_cstate(C_DEMOTED); cpc = 0; }
        claims_changed = true;
        refresh_protected();
        ctr_add(K_DEMOTED_AUTO, nd);
        return true;
      }
    }
    const uint32_t shortfall = (uint32_t)((uint64_t)P + A - Uu);
    const bool resident = A <= Uu && P > 0;
    const uint32_t why = resident ? WHY_PROTECTED : WHY_CAPACITY;
    const uint32_t mask = resident ? h[H_BLOCKMASK] : 0u;
    if (requester == 0xFFFFFFFFu) {
      emit(EV_INSERT_REFUSED, a, why, mask, P, (uint32_t)A, Uu, shortfall);
      ctr_add(K_INSERT_REFUSED, 1);
      return false;
    }
    // request: release its live blocks, then defer or refuse (G9)
    if (rq[RQ_LIVE] > 0) {
      release_blocks(requester);
      h[H_ALIVE] -= rq[RQ_LIVE];
    }
    rq[RQ_LIVE] = 0;
    rq[RQ_DONE] = 0;
    const uint32_t defer = rq[RQ_W0] >> 24;
    if (defer < defer_budget()) {
      rq[RQ_W0] = (rq[RQ_W0] & 0x00FFFF00u) | R_DEFERRED | ((defer + 1) << 24);
      emit(EV_DEFERRED, requester, why, mask, P, (uint32_t)A, Uu, shortfall);
      ctr_add(resident ? K_DEFERRED_PROTECTED : K_DEFERRED_CAPACITY, 1);
    } else {
      rq[RQ_W0] = (rq[RQ_W0] & 0xFFFFFF00u) | R_REFUSED;
      emit(EV_REFUSED, requester, why, mask, P, (uint32_t)A, Uu, shortfall);
      ctr_add(resident ? K_REFUSED_PROTECTED : K_REFUSED_CAPACITY, 1);
    }
    rq_dirty = true;
    return false;
  }

  // ------------------------- victim selection ------------------------------
  // k-th free block id (1-based k <= free count) from the free bitmap
  __device__ __forceinline__ uint32_t kth_free(uint32_t k) const {
    const uint32_t nw = nvec * 4;
    uint32_t acc = 0;
    for (uint32_t w0 = 0; w0 < nw; w0 += 32) {
      const uint32_t w = w0 + lane;
      const uint32_t word = w < nw ? __ldcg(fbm + w) : 0u;
      const uint32_t cnt = __popc(word);
      const uint32_t S = warp_incl_scan(cnt);
      const uint32_t tot = __shfl_sync(kFull, S, 31);
      if (acc + tot >= k) {
        const uint32_t hit = __ballot_sync(kFull, acc + S >= k);
        const uint32_t L = __ffs(hit) - 1;
        const uint32_t before = __shfl_sync(kFull, acc + S - cnt, L);
        const uint32_t wl = __shfl_sync(kFull, word, L);
        return (w0 + L) * 32 + nth_set_bit(wl, k - before);
      }
      acc += tot;
    }
    return 0xFFFFFFFFu;  // unreachable when k <= free count
  }

  template <class GetK>
  __device__ __forceinline__ uint32_t count_le(const GetK& getk, uint32_t T) const {
    uint32_t c = 0;
    if constexpr (VPL > 0) {
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const uint4 v = getk(j);
        c += (v.x <= T) + (v.y <= T) + (v.z <= T) + (v.w <= T);
      }
    } else {
      for (uint32_t j = 0; j < nvec; ++j) {
        const uint4 v = getk(j);
        c += (v.x <= T) + (v.y <= T) + (v.z <= T) + (v.w <= T);
      }
    }
    return __reduce_add_sync(kFull, c);
  }

  // threshold T with #{b : key[b] <= T} == k, k > free count (evicting case).
  template <class GetK>
  __device__ __forceinline__ uint32_t select_threshold(const GetK& getk, uint32_t k) const {
    // stats of class 1 and class 2 keys
    uint32_t c1 = 0, mn1 = kFull, mx1 = 0, mn2 = kFull, mx2 = 0;
    auto stat = [&](uint32_t kk) {
      const uint32_t cls = kk >> kClassShift;
      if (cls == 1) { ++c1; mn1 = min(mn1, kk); mx1 = max(mx1, kk); }
      else if (cls == 2 && kk != kKeyActive) { mn2 = min(mn2, kk); mx2 = max(mx2, kk); }
    };
    if constexpr (VPL > 0) {
#pragma unroll
      for (int j = 0; j < VPL; ++j) { const uint4 v = getk(j); stat(v.x); stat(v.y); stat(v.z); stat(v.w); }
    } else {
      for (uint32_t j = 0; j < nvec; ++j) { const uint4 v = getk(j); stat(v.x); stat(v.y); stat(v.z); stat(v.w); }
    }
    c1 = __reduce_add_sync(kFull, c1);
    mn1 = __reduce_min_sync(kFull, mn1);
    mx1 = __reduce_max_sync(kFull, mx1);
    mn2 = __reduce_min_sync(kFull, mn2);
    mx2 = __reduce_max_sync(kFull, mx2);
    const uint32_t fr = h[H_FREE];
    uint32_t lo, hi, clo, chi;
    if (k - fr <= c1) { lo = mn1 - 1; clo = fr; hi = mx1; chi = fr + c1; }
    else { lo = mn2 - 1; clo = fr + c1; hi = mx2; chi = count_le(getk, mx2); }
    // interpolation search on the counting function, bisection every other
    // probe once the first two probes missed (keys are unique, so the loop
    // ends with #(<= hi) == k exactly)
    for (uint32_t it = 0; chi != k; ++it) {
      const uint32_t span = hi - lo;
      uint32_t m;
      if (it < 2 || (it & 1u)) {
        m = lo + (uint32_t)(((uint64_t)(k - clo) * span) / (chi - clo));
      } else {
        m = lo + span / 2;
      }
      m = max(m, lo + 1);
      m = min(m, hi - 1);
      const uint32_t cm = count_le(getk, m);
      if (cm >= k) { hi = m; chi = cm; } else { lo = m; clo = cm; }
    }
    return hi;
  }

  // alloc(k): take the k smallest keys; positions base + rank
  // in block-id order (G24).  insert: blocks become CACHED(obj a) with tail-first
  // stamps, else ACTIVE(owner).  Returns nothing; updates counters, free
  // count, leading prefixes, victim telemetry.
  __device__ __forceinline__ void alloc(uint32_t k, uint32_t owner, bool insert, uint32_t base) {
    flush_reclass();
    mirror_claims();
    const uint32_t fr = h[H_FREE];
    uint4 kv[VPL > 0 ? VPL : 1];
    if constexpr (VPL > 0) {
      if (k > fr) {
#pragma unroll
        for (int j = 0; j < VPL; ++j) kv[j] = ld_key(j);
      }
    }
    auto getk = [&](uint32_t j) -> uint4 {
      if constexpr (VPL > 0) return kv[j];
      else return ld_key(j);
    };
    uint32_t T;
    if (k <= fr) T = kth_free(k);
    else T = select_threshold(getk, k);
    const uint32_t seq_base = h[H_SEQ];
    uint32_t ord = 0, rel = 0, clm = 0, acc = 0;
    const uint32_t lt = lanemask_lt();
    const uint32_t NV = VPL > 0 ? (uint32_t)VPL : nvec;
#pragma unroll
    for (uint32_t j = 0; j < NV; ++j) {
      uint4 v;
      if (k <= fr) {
        if (j * 128 > T) break;  // all taken blocks lie below T
        // free-only: taken = free blocks with id <= T, from the bitmap
        const uint32_t b0 = block_of(j, 0);
        const uint32_t word = __ldcg(fbm + (b0 >> 5));
        const uint32_t nib = (word >> (b0 & 31u)) & 0xFu;
        v.x = (nib & 1u) ? b0 : kKeyActive;
        v.y = (nib & 2u) ? b0 + 1 : kKeyActive;
        v.z = (nib & 4u) ? b0 + 2 : kKeyActive;
        v.w = (nib & 8u) ? b0 + 3 : kKeyActive;
      } else {
        v = getk(j);
      }
      const uint32_t tb = (v.x <= T ? 1u : 0u) | (v.y <= T ? 2u : 0u) | (v.z <= T ? 4u : 0u) |
                          (v.w <= T ? 8u : 0u);
      const uint32_t B0 = __ballot_sync(kFull, tb & 1u), B1 = __ballot_sync(kFull, tb & 2u);
      const uint32_t B2 = __ballot_sync(kFull, tb & 4u), B3 = __ballot_sync(kFull, tb & 8u);
      const uint32_t tot = __popc(B0) + __popc(B1) + __popc(B2) + __popc(B3);
      if (tot == 0) continue;
      uint32_t r = acc + __popc(B0 & lt) + __popc(B1 & lt) + __popc(B2 & lt) + __popc(B3 & lt);
      acc += tot;
      if (tb == 0) continue;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (!((tb >> e) & 1u)) continue;
        const uint32_t bb = block_of(j, e);
        const uint32_t old = el(v, e);
        const uint32_t pos = base + r;
        if (old >= (1u << kClassShift)) {
          // cached victim: attribute by its object's claim state now (Table 4)
          const uint32_t m = __ldcg(meta + bb);
          const uint32_t o = meta_owner(m);
          const uint32_t cc = obj_claim(s->obj0[o]);
          const uint32_t st = cc < 32 ? s->cstate[cc] : C_EMPTY;
          if (st == C_DEMOTED || st == C_EXPIRED) ++rel;
          else if (st == C_ACCEPTED || st == C_MATERIALIZED) ++clm;
          else ++ord;
          atomicMin(&s->lead[o], meta_pos(m));
          atomicOr(&s->objdirty[o >> 5], 1u << (o & 31u));
        }
        if (insert) {
          const uint32_t cls = new_block_class(a, pos);
          key[bb] = (cls << kClassShift) | (seq_base + (k - 1 - pos));
          meta[bb] = meta_make(kResCached, a, pos);
        } else {
          key[bb] = kKeyActive;
          meta[bb] = meta_make(kResActive, owner, pos);
        }
        ++r;
      }
    }
    // free bitmap: every free block with id <= T was taken
    {
      const uint32_t nw = nvec * 4;
      for (uint32_t w = lane; w < nw; w += 32) {
        const uint32_t lo = w * 32;
        if (lo > T) continue;
        const uint32_t off = T - lo;
        if (off >= 31) fbm[w] = 0;
        else fbm[w] = __ldcg(fbm + w) & ~((2u << off) - 1u);
      }
    }
    ord = __reduce_add_sync(kFull, ord);
    rel = __reduce_add_sync(kFull, rel);
    clm = __reduce_add_sync(kFull, clm);
    const uint32_t free_taken = k <= fr ? k : fr;
    h[H_FREE] -= free_taken;
    ctr_add(K_VICTIMS_ORDINARY, ord);
    ctr_add(K_VICTIMS_AFTER_RELEASE, rel);
    ctr_add(K_VICTIMS_CLAIMED, clm);
    ctr_add(K_BLOCKS_ALLOCATED, k);
    if (ord + rel + clm > 0) emit(EV_VICTIMS, insert ? a : owner, insert ? 1u : 0u, 0, ord, rel, clm, k);
    __syncwarp();
  }

  // ----------------------------- request io --------------------------------
  __device__ __forceinline__ void load_request(uint32_t r) {
    const uint4* src = reinterpret_cast<const uint4*>(p.req + ((size_t)t * p.Q + r) * 8);
    const uint4 v0 = __ldcg(src), v1 = __ldcg(src + 1);
    rq[0] = v0.x; rq[1] = v0.y; rq[2] = v0.z; rq[3] = v0.w;
    rq[4] = v1.x; rq[5] = v1.y; rq[6] = v1.z; rq[7] = v1.w;
    rq_dirty = false;
  }
  __device__ __forceinline__ void store_request(uint32_t r) {
    if (rq_dirty && lane == 0) {
      uint4* dst = reinterpret_cast<uint4*>(p.req + ((size_t)t * p.Q + r) * 8);
      dst[0] = make_uint4(rq[0], rq[1], rq[2], rq[3]);
      dst[1] = make_uint4(rq[4], rq[5], rq[6], rq[7]);
    }
  }
  __device__ __forceinline__ uint32_t rq_status() const { return rq[RQ_W0] & 0xFFu; }
  __device__ __forceinline__ uint32_t peak() const {
    return (uint32_t)(((uint64_t)rq[RQ_PROMPT] + rq[RQ_DECODE] + kBlockTokens - 1) / kBlockTokens);
  }

  // --------------------------------- ops -----------------------------------
  __device__ __forceinline__ void op_submit() {
    const uint32_t mode = c & 0x7Fu;
    const bool mismatch = (c & 0x80u) != 0;
    if (a >= p.C || b >= p.O || mode > M_BEST_EFFORT) return op_error(ERR_INVALID_ARG);
    if ((claim_field(cw0, a) & 0xFFu) != C_EMPTY) return op_error(ERR_DUPLICATE_SLOT);
    if (x < 1 || y < 1 || y > x || (mode == M_EXPIRING && z == 0)) return op_error(ERR_INVALID_ARG);
    const uint32_t ow = s->obj0[b];
    const uint32_t oc = obj_claim(ow);
    const uint32_t ocst = claim_field(cw0, oc < 32 ? oc : 0) & 0xFFu;
    const bool bound_live = oc < 32 && live_state(ocst);
    uint32_t rej = 0;
    if (mismatch) rej = REJ_IDENTITY;
    else if (bound_live) rej = REJ_OBJECT_CLAIMED;
    else if (x > U()) rej = REJ_FOOTPRINT;
    else if ((h[H_ACCEPT] & 0xFFu) == ACCEPT_RESERVE && obligated(mode)) {
      const uint32_t sum = __reduce_add_sync(
          kFull, (lane < p.C && live_state(cstate()) && obligated(cmode())) ? cF : 0u);
      if ((uint64_t)x + sum > U()) rej = REJ_RESERVE;
    }
    if (lane == a) {
      cw0 = (rej ? C_REFUSED : C_ACCEPTED) | (mode << 8) | (b << 16);
      cF = x; cR = y; cD = z; cdec = step; cpc = 0;
      cdirty = true;
    }
    claims_changed = true;
    if (rej) {
      emit(EV_REJECTED, a, rej, 0, b, x, y, z);
      ctr_add(K_REJECTED, 1);
    } else {
      emit(EV_ACCEPTED, a, 0, 0, b, x, y, z);
      ctr_add(K_ACCEPTED, 1);
      if (lane == 0) s->obj0[b] = obj_make(obj_live(ow), a, obj_len(ow));
      mark_obj_dirty(b);
      __syncwarp();
      if (obj_live(ow) && claim_class(mode, lowering()) != 1) mark_reclass(b);
    }
  }

  __device__ __forceinline__ void op_admit() {
    if (a >= p.Q || b >= p.O || c > 1) return op_error(ERR_INVALID_ARG);
    load_request(a);
    const uint32_t st = rq_status();
    if (st == R_RUNNING || st == R_DEFERRED) return op_error(ERR_DUPLICATE_SLOT);
    if (x < 1 || y < 1 || x > kMaxTokens || z > kMaxTokens) return op_error(ERR_INVALID_ARG);
    rq[RQ_W0] = R_RUNNING | (c << 8) | (b << 16);
    rq[RQ_PROMPT] = x; rq[RQ_CHUNK] = y; rq[RQ_DECODE] = z; rq[RQ_DONE] = 0; rq[RQ_LIVE] = 0;
    rq_dirty = true;
    ctr_add(K_ADMITTED, 1);
    if (admit_check() == ADMIT_PEAK) arbitrate(peak(), a);
    store_request(a);
  }

  __device__ __forceinline__ void op_advance() {
    if (a >= p.Q) return op_error(ERR_INVALID_ARG);
    load_request(a);
    const uint32_t st = rq_status();
    if (st != R_RUNNING && st != R_DEFERRED) return op_error(ERR_UNKNOWN_REQUEST);
    if (st == R_RUNNING && (uint64_t)rq[RQ_DONE] >= (uint64_t)rq[RQ_PROMPT] + rq[RQ_DECODE])
      return op_error(ERR_NO_CHUNKS);
    if (st == R_DEFERRED) {
      if (admit_check() == ADMIT_PEAK && !arbitrate(peak(), a)) { store_request(a); return; }
      rq[RQ_W0] = (rq[RQ_W0] & ~0xFFu) | R_RUNNING;
      rq_dirty = true;
    }
    const uint32_t done = rq[RQ_DONE];
    const uint32_t n = done < rq[RQ_PROMPT] ? min(rq[RQ_CHUNK], rq[RQ_PROMPT] - done) : 1u;
    const uint32_t need_total = (uint32_t)(((uint64_t)done + n + kBlockTokens - 1) / kBlockTokens);
    const uint32_t need = need_total > rq[RQ_LIVE] ? need_total - rq[RQ_LIVE] : 0u;
    if (need > 0) {
      if (!arbitrate(need, a)) { store_request(a); return; }
      alloc(need, a, false, rq[RQ_LIVE]);
      rq[RQ_LIVE] += need;
      h[H_ALIVE] += need;
    }
    rq[RQ_DONE] = done + n;
    rq_dirty = true;
    store_request(a);
  }

  __device__ __forceinline__ void op_complete() {
    if (a >= p.Q) return op_error(ERR_INVALID_ARG);
    load_request(a);
    if (rq_status() != R_RUNNING) return op_error(ERR_UNKNOWN_REQUEST);
    const uint32_t done = rq[RQ_DONE];
    const uint32_t full = done / kBlockTokens;
    const uint32_t o = (rq[RQ_W0] >> 16) & 0xFFu;
    const uint32_t wa = (rq[RQ_W0] >> 8) & 0xFFu;
    const uint32_t ow = s->obj0[o];
    const bool admitted = wa && !obj_live(ow);
    if (admitted && (uint64_t)h[H_SEQ] + full > kSeqLimit) return op_error(ERR_SEQ_EXHAUSTED);
    const uint32_t held = rq[RQ_LIVE];
    if (admitted) {
      mirror_claims();
      const uint32_t seq_base = h[H_SEQ];
      uint32_t freed = 0;
      for (uint32_t j = 0; j < nvec && held > 0; ++j) {
        const uint4 mv = ld_meta(j);
        uint32_t nib = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t m = el(mv, e);
          if (meta_res(m) != kResActive || meta_owner(m) != a) continue;
          const uint32_t bb = block_of(j, e);
          const uint32_t pos = meta_pos(m);
          if (pos < full) {
            const uint32_t cls = new_block_class(o, pos);
            key[bb] = (cls << kClassShift) | (seq_base + (full - 1 - pos));
            meta[bb] = meta_make(kResCached, o, pos);
          } else {
            key[bb] = bb;
            meta[bb] = meta_make(kResFree, 0, 0);
            nib |= 1u << e;
          }
        }
        fbm_set(j, nib);
        freed += __popc(nib);
      }
      h[H_FREE] += __reduce_add_sync(kFull, freed);
      h[H_SEQ] = seq_base + full;
      if (lane == 0) { s->obj0[o] = obj_make(1, obj_claim(ow), full); s->lead[o] = full; }
      mark_obj_dirty(o);
      __syncwarp();
      {
        const uint32_t cc = obj_claim(ow);
        uint32_t prot = 0;
        if (cc < 32) {
          const uint32_t Fc = claim_field(cF, cc);
          prot = min(Fc, full);
        }
        add_protected(o, prot);
      }
      ctr_add(K_BLOCKS_CACHED, full);
    } else {
      if (held > 0) release_blocks(a);
      emit(EV_WRITE_DENIED, a, wa ? 1u : 0u, 0, o, held);
      ctr_add(K_WRITE_DENIED, 1);
    }
    emit(EV_SERVED, a, admitted ? 1u : 0u, 0, done, admitted ? full : 0u, o);
    ctr_add(K_SERVED, 1);
    h[H_ALIVE] -= held;
    rq[RQ_W0] = (rq[RQ_W0] & ~0xFFu) | R_COMPLETED;
    rq[RQ_LIVE] = 0;
    rq_dirty = true;
    store_request(a);
  }

  __device__ __forceinline__ void op_insert() {
    if (a >= p.O) return op_error(ERR_INVALID_ARG);
    const uint32_t ow = s->obj0[a];
    if (obj_live(ow)) return op_error(ERR_OBJECT_IN_USE);
    if (x < 1 || x > kMaxTokens) return op_error(ERR_INVALID_ARG);
    if ((uint64_t)h[H_SEQ] + x > kSeqLimit) return op_error(ERR_SEQ_EXHAUSTED);
    if (!arbitrate(x, 0xFFFFFFFFu)) return;
    alloc(x, a, true, 0);
    h[H_SEQ] += x;
    if (lane == 0) { s->obj0[a] = obj_make(1, obj_claim(ow), x); s->lead[a] = x; }
    mark_obj_dirty(a);
    __syncwarp();
    {
      const uint32_t cc = obj_claim(ow);
      uint32_t prot = 0;
      if (cc < 32) prot = min(claim_field(cF, cc), x);
      add_protected(a, prot);
    }
    ctr_add(K_INSERTED, 1);
    ctr_add(K_BLOCKS_CACHED, x);
  }

  __device__ __forceinline__ void op_demote() {
    if (a >= p.C) return op_error(ERR_INVALID_ARG);
    const uint32_t st = claim_field(cw0, a) & 0xFFu;
    if (st == C_EMPTY) return op_error(ERR_UNKNOWN_CLAIM);
    if (!live_state(st)) return op_error(ERR_ILLEGAL_TRANSITION);
    const uint32_t o = (claim_field(cw0, a) >> 16) & 0xFFu;
    const uint32_t pc = claim_field(cpc, a);
    const uint32_t mode = (claim_field(cw0, a) >> 8) & 0xFFu;
    if (lane == a) { set_cstate(C_DEMOTED); cpc = 0; }
    claims_changed = true;
    emit(EV_DEMOTED, a, 0, 0, o, pc);
    ctr_add(K_DEMOTED_EXPLICIT, 1);
    if (claim_class(mode, lowering()) != 1) mark_reclass(o);
    refresh_protected();
  }

  __device__ __forceinline__ void op_touch() {
    if (a >= p.O) return op_error(ERR_INVALID_ARG);
    const uint32_t ow = s->obj0[a];
    const uint32_t L = obj_live(ow) ? s->lead[a] : 0u;
    if ((uint64_t)h[H_SEQ] + L > kSeqLimit) return op_error(ERR_SEQ_EXHAUSTED);
    const uint32_t seq_base = h[H_SEQ];
    if (L > 0) {
      for (uint32_t j = 0; j < nvec; ++j) {
        const uint4 mv = ld_meta(j);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t m = el(mv, e);
          if (meta_res(m) == kResCached && meta_owner(m) == a && meta_pos(m) < L) {
            const uint32_t bb = block_of(j, e);
            const uint32_t k0 = __ldcg(key + bb);
            key[bb] = (k0 & ~kSeqMask) | (seq_base + (L - 1 - meta_pos(m)));
          }
        }
      }
    }
    h[H_SEQ] = seq_base + L;
    const uint32_t cc = obj_claim(ow);
    const bool has = cc < 32;
    const uint32_t Rc = claim_field(cR, has ? cc : 0);
    const uint32_t stc = claim_field(cw0, has ? cc : 0) & 0xFFu;
    const bool sat = has && live_state(stc) && L >= Rc;
    emit(EV_REUSE_PROBE, has ? cc : 0xFFu, sat ? 1u : 0u, 0, a, L, L * kBlockTokens, has ? Rc : 0u);
    ctr_add(K_REUSE_PROBES, 1);
    ctr_add(K_REUSE_TOKENS, L * kBlockTokens);
  }

  // ------------------------------- phases ----------------------------------
  __device__ __forceinline__ void expiry() {
    const bool ex = lane < p.C && live_state(cstate()) && cD > 0 && (uint64_t)cdec + cD <= step;
    const uint32_t m = __ballot_sync(kFull, ex);
    if (!m) return;
    emit_lanes(ex, EV_EXPIRED, lane, 0, 0, cobj(), cpc, cdec, cD);
    mark_reclass_lanes(ex && claim_class(cmode(), lowering()) != 1, cobj());
    if (ex) { set_cstate(C_EXPIRED); cpc = 0; }
    claims_changed = true;
    refresh_protected();
    ctr_add(K_EXPIRED, __popc(m));
  }

  __device__ __forceinline__ void post_op() {
    mirror_claims();
    const uint32_t st = cstate();
    const bool lv = lane < p.C && live_state(st);
    uint32_t L = 0;
    bool olive = false;
    if (lv) {
      const uint32_t o = cobj();
      olive = obj_live(s->obj0[o]) != 0;
      L = olive ? s->lead[o] : 0u;
    }
    const bool mat = lv && st == C_ACCEPTED && olive && L >= cR;
    const bool harm = lv && st == C_MATERIALIZED && L < cR;
    const uint32_t mm = __ballot_sync(kFull, mat), hm = __ballot_sync(kFull, harm);
    if ((mm | hm) == 0) return;
    const bool ob = obligated(cmode());
    const bool any = mat || harm;
    // one ballot-ranked emission with per-lane type and fields
    emit_lanes(any, mat ? EV_MATERIALIZED : EV_HARMED, lane, harm ? (ob ? 1u : 0u) : 0u, 0, L, cR,
               mat ? L * kBlockTokens : h[H_P], mat ? cobj() : h[H_ALIVE]);
    mark_reclass_lanes(harm && claim_class(cmode(), lowering()) != 1, cobj());
    if (mat) set_cstate(C_MATERIALIZED);
    if (harm) { set_cstate(C_HARMED); cpc = 0; }
    claims_changed = true;
    ctr_add(K_MATERIALIZED, __popc(mm));
    ctr_add(K_HARMED_OBLIGATED, __popc(__ballot_sync(kFull, harm && ob)));
    ctr_add(K_HARMED_UNOBLIGATED, __popc(__ballot_sync(kFull, harm && !ob)));
    refresh_protected();
  }

  __device__ __forceinline__ void run(const uint4 opw) {
    kind = opw.x & 0xFFu; a = (opw.x >> 8) & 0xFFu; b = (opw.x >> 16) & 0xFFu; c = opw.x >> 24;
    x = opw.y; y = opw.z; z = opw.w;
    {
      const uint4* hp = reinterpret_cast<const uint4*>(p.hdr + (size_t)t * H_NWORDS);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 v = __ldcg(hp + i);
        h[4 * i] = v.x; h[4 * i + 1] = v.y; h[4 * i + 2] = v.z; h[4 * i + 3] = v.w;
      }
    }
    // a NOP with no expiry due changes nothing (fast path)
    if (kind == OP_NOP && step < h[H_NEXT_EXPIRY]) return;
    nvec = p.NS / 128;
    key = p.key + (size_t)t * p.NS;
    meta = p.meta + (size_t)t * p.NS;
    fbm = p.fbm + (size_t)t * (p.NS / 32);
    nev = 0;
    rc0 = rc1 = rc2 = rc3 = 0;
    claims_changed = false;
    rq_dirty = false;
    cdirty = false;
    s->ctr[lane] = 0;
    if (lane < 4) s->objdirty[lane] = 0;
    // claims -> lane registers
    cw0 = cF = cR = cD = cdec = cpc = 0;
    if (lane < p.C) {
      const uint4* cp = reinterpret_cast<const uint4*>(p.clm + ((size_t)t * p.C + lane) * 8);
      const uint4 v0 = __ldcg(cp), v1 = __ldcg(cp + 1);
      cw0 = v0.x; cF = v0.y; cR = v0.z; cD = v0.w; cdec = v1.x; cpc = v1.y;
    }
    // objects -> shared memory
    for (uint32_t o = lane; o < p.O; o += 32) {
      const uint2 w = __ldcg(reinterpret_cast<const uint2*>(p.obj) + (size_t)t * p.O + o);
      s->obj0[o] = w.x;
      s->lead[o] = w.y;
    }
    __syncwarp();
    mirror_claims();

    if (step >= h[H_NEXT_EXPIRY]) expiry();
    if (kind != OP_NOP) ctr_add(K_OPS, 1);
    switch (kind) {
      case OP_NOP: break;
      case OP_SUBMIT: op_submit(); break;
      case OP_ADMIT: op_admit(); break;
      case OP_ADVANCE: op_advance(); break;
      case OP_COMPLETE: op_complete(); break;
      case OP_INSERT: op_insert(); break;
      case OP_DEMOTE: op_demote(); break;
      case OP_TOUCH: op_touch(); break;
      default: op_error(ERR_UNKNOWN_OP); break;
    }
    flush_reclass();
    post_op();
    flush_reclass();

    // ---- write back ----
    if (claims_changed) {
      uint32_t ne = (lane < p.C && live_state(cstate()) && cD > 0)
                        ? (uint32_t)min((uint64_t)cdec + cD, (uint64_t)0xFFFFFFFFu)
                        : 0xFFFFFFFFu;
      h[H_NEXT_EXPIRY] = __reduce_min_sync(kFull, ne);
    }
    if (cdirty && lane < p.C) {
      uint4* cp = reinterpret_cast<uint4*>(p.clm + ((size_t)t * p.C + lane) * 8);
      cp[0] = make_uint4(cw0, cF, cR, cD);
      cp[1] = make_uint4(cdec, cpc, 0, 0);
    }
    __syncwarp();
    for (uint32_t o = lane; o < p.O; o += 32) {
      if ((s->objdirty[o >> 5] >> (o & 31u)) & 1u)
        reinterpret_cast<uint2*>(p.obj)[(size_t)t * p.O + o] = make_uint2(s->obj0[o], s->lead[o]);
    }
    h[H_EVCOUNT] += nev;
    if (lane == 0) {
      uint4* hp = reinterpret_cast<uint4*>(p.hdr + (size_t)t * H_NWORDS);
#pragma unroll
      for (int i = 0; i < 4; ++i) hp[i] = make_uint4(h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
    }
    const uint32_t d = s->ctr[lane];
    if (d) p.ctr[(size_t)t * K_NCTR + lane] += d;
  }
};

template <int VPL>
__global__ void __launch_bounds__(kWarpsPerCta * 32, 4)
rkc_step_kernel(StepArgs args) {
  __shared__ WarpSmem smem[kWarpsPerCta];
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t t = blockIdx.x * kWarpsPerCta + w;
  if (t >= args.p.num_traces) return;
  const uint4 opw = __ldcs(args.ops + t);
  Trace<VPL> tr(args.p, &smem[w], t, args.step);
  tr.run(opw);
}

// host launcher: one launch = one lockstep step over all traces
extern std::atomic<unsigned long long> g_launches;

cudaError_t launch_step(const PoolDev& p, const void* ops_step, uint32_t step, cudaStream_t st) {
  g_launches += 1;
  StepArgs args{p, reinterpret_cast<const uint4*>(ops_step), step};
  const uint32_t grid = (p.num_traces + kWarpsPerCta - 1) / kWarpsPerCta;
  const uint32_t vpl = p.NS / 128;
  switch (vpl) {
    case 1: rkc_step_kernel<1><<<grid, kWarpsPerCta * 32, 0, st>>>(args); break;
    case 2: rkc_step_kernel<2><<<grid, kWarpsPerCta * 32, 0, st>>>(args); break;
    case 4: rkc_step_kernel<4><<<grid, kWarpsPerCta * 32, 0, st>>>(args); break;
    case 8: rkc_step_kernel<8><<<grid, kWarpsPerCta * 32, 0, st>>>(args); break;
    default: rkc_step_kernel<0><<<grid, kWarpsPerCta * 32, 0, st>>>(args); break;
  }
  return cudaGetLastError();
}

}  // namespace rkc
