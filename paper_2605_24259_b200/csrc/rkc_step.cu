// rkc_step.cu -- K1: the lockstep step kernel.
//
// One warp owns one trace (one paged KV pool) for one step:
//   a0 op fetch -> a1 expiry -> a2 claim decision | a3 feasibility (P + A <= U,
//   P:504) -> a4 claim-excluding victim selection -> a5 block updates ->
//   a6 materialization predicate (leading prefix) -> a7 lifecycle
//   -> a8 telemetry.
// Semantics: DESIGN.md sec. 1 (the reading the oracle implements; no code is
// shared with it).
//
// Structure: the warp's uniform state (header, request,
// claim table, object table, counters) lives in shared memory; each op kind is
// a separate __noinline__ path so a warp only fetches the code of its own op
// (a monolithic inlined kernel thrashed the instruction cache, profiles/r01);
// claim / object tables are loaded only by the ops that need them; block
// words are streamed with coalesced 16-byte loads, lane L of vector j owning
// blocks (j*32 + L)*4 .. +3; the selection keys of a <= 1024-block pool are
// staged once in shared memory for the threshold search.
#include <cuda_runtime.h>

#include <atomic>

#include "rkc_internal.cuh"

namespace rkc {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kWarpsPerCta = 1;
constexpr uint32_t kStageMax = 1024;  // pools up to this size stage keys in smem

enum : uint32_t { F_CLAIMS = 1, F_OBJS = 2, F_POST = 4, F_CLAIMS_CHANGED = 8, F_HDR = 16 };

struct Warp {                  // per-warp shared memory
  uint32_t h[H_NWORDS];        // hot header
  uint32_t rq[8];              // the request record of the current op
  uint32_t nev, flags, cdirty, pad0;
  uint32_t rc[4];              // objects whose blocks need reclassing
  uint32_t objdirty[4];
  uint32_t ctr[32];            // counter deltas of this step
  uint32_t cl[32][8];          // claim records (lane c owns claim c)
  uint32_t obj0[128];          // object word 0
  uint32_t lead[128];          // leading prefix per object
  union {
    struct { uint32_t lim3[128], lim2[128], cnt3[128]; };  // reclass scratch
    uint32_t keys[kStageMax];  // staged selection keys (alloc only)
  };
};

struct Ctx {
  const PoolDev* p;
  Warp* w;
  uint32_t t, step, lane;
  __device__ uint32_t* key() const { return p->key + (size_t)t * p->NS; }
  __device__ uint32_t* meta() const { return p->meta + (size_t)t * p->NS; }
  __device__ uint32_t* fbm() const { return p->fbm + (size_t)t * (p->NS / 32); }
  __device__ uint32_t nvec() const { return p->NS / 128; }
};

struct Op { uint32_t kind, a, b, c, x, y, z; };

// ------------------------------ helpers ------------------------------------
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
__device__ __forceinline__ uint32_t nth_set_bit(uint32_t w, uint32_t r) {  // r is 1-based
  uint32_t pos = 0;
#pragma unroll
  for (int width = 16; width >= 1; width >>= 1) {
    const uint32_t c = __popc(w & ((1u << width) - 1u));
    if (r > c) { r -= c; w >>= width; pos += width; }
  }
  return pos;
}
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, uint32_t lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t u = __shfl_up_sync(kFull, v, d);
    if (lane >= (uint32_t)d) v += u;
  }
  return v;
}
__device__ __forceinline__ uint32_t el(const uint4& v, int e) {
  return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}

// uniform shared-memory scalars are written by lane 0 and published by __syncwarp
__device__ __forceinline__ void hset(const Ctx x, uint32_t i, uint32_t v) {
  __syncwarp();
  if (x.lane == 0) { x.w->h[i] = v; x.w->flags |= F_HDR; }
  __syncwarp();
}
__device__ __forceinline__ void flag_set(const Ctx x, uint32_t f) {
  if (x.lane == 0) x.w->flags |= f;
  __syncwarp();
}
__device__ __forceinline__ uint32_t lowering(const Ctx x) { return x.w->h[H_POLICY] & 0xFFu; }
__device__ __forceinline__ void ctr_add(const Ctx x, uint32_t k, uint32_t v) {
  if (x.lane == 0) x.w->ctr[k] += v;
}

// claim record accessors (slot c)
__device__ __forceinline__ uint32_t cl_state(const Warp* w, uint32_t c) { return w->cl[c][0] & 0xFFu; }
__device__ __forceinline__ uint32_t cl_mode(const Warp* w, uint32_t c) { return (w->cl[c][0] >> 8) & 0xFFu; }
__device__ __forceinline__ uint32_t cl_obj(const Warp* w, uint32_t c) { return (w->cl[c][0] >> 16) & 0xFFu; }
enum : uint32_t { CF_W0 = 0, CF_F = 1, CF_R = 2, CF_D = 3, CF_DEC = 4, CF_PC = 5 };

// ------------------------------ telemetry ----------------------------------
__device__ __forceinline__ void write_event(const Ctx x, uint32_t idx, uint32_t type, uint32_t seq,
                                            uint32_t slot, uint32_t reason, uint32_t mask,
                                            uint32_t f0, uint32_t f1, uint32_t f2, uint32_t f3) {
  if (idx < x.p->EPT) {
    uint4* e = x.p->ev + ((size_t)x.t * x.p->EPT + idx) * 2;
    e[0] = make_uint4(x.t, x.step, type | (seq << 8) | ((slot & 0xFFu) << 16) | (reason << 24), mask);
    e[1] = make_uint4(f0, f1, f2, f3);
  }
}
__device__ __noinline__ void emit(const Ctx x, uint32_t type, uint32_t slot, uint32_t reason,
                                  uint32_t mask, uint32_t f0, uint32_t f1, uint32_t f2, uint32_t f3) {
  const uint32_t n = x.w->nev;
  if (x.lane == 0) {
    write_event(x, x.w->h[H_EVCOUNT] + n, type, n, slot, reason, mask, f0, f1, f2, f3);
    x.w->nev = n + 1;
  }
  __syncwarp();
}
// one event per lane with pred, ranked by lane (= claim slot)
__device__ __forceinline__ void emit_lanes(const Ctx x, bool pred, uint32_t type, uint32_t reason,
                                           uint32_t mask, uint32_t f0, uint32_t f1, uint32_t f2,
                                           uint32_t f3) {
  const uint32_t m = __ballot_sync(kFull, pred);
  const uint32_t n = x.w->nev;
  if (pred) {
    const uint32_t r = __popc(m & lanemask_lt());
    write_event(x, x.w->h[H_EVCOUNT] + n + r, type, n + r, x.lane, reason, mask, f0, f1, f2, f3);
  }
  __syncwarp();
  if (x.lane == 0) x.w->nev = n + __popc(m);
  __syncwarp();
}
__device__ __noinline__ void op_error(const Ctx x, const Op op, uint32_t code) {
  emit(x, EV_OP_ERROR, op.a, code, 0, op.kind, 0, 0, 0);
  ctr_add(x, K_OP_ERRORS, 1);
}

// ------------------------------ lazy loads ---------------------------------
__device__ __noinline__ void need_claims(const Ctx x) {
  if (x.w->flags & F_CLAIMS) return;
  if (x.lane < x.p->C) {
    const uint4* cp = reinterpret_cast<const uint4*>(x.p->clm + ((size_t)x.t * x.p->C + x.lane) * 8);
    const uint4 v0 = __ldcg(cp), v1 = __ldcg(cp + 1);
    reinterpret_cast<uint4*>(x.w->cl[x.lane])[0] = v0;
    reinterpret_cast<uint4*>(x.w->cl[x.lane])[1] = v1;
  } else {
    reinterpret_cast<uint4*>(x.w->cl[x.lane])[0] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(x.w->cl[x.lane])[1] = make_uint4(0, 0, 0, 0);
  }
  __syncwarp();
  flag_set(x, F_CLAIMS);
}
__device__ __noinline__ void need_objs(const Ctx x) {
  if (x.w->flags & F_OBJS) return;
  const uint2* src = reinterpret_cast<const uint2*>(x.p->obj) + (size_t)x.t * x.p->O;
  for (uint32_t o = x.lane; o < x.p->O; o += 32) {
    const uint2 v = __ldcg(src + o);
    x.w->obj0[o] = v.x;
    x.w->lead[o] = v.y;
  }
  __syncwarp();
  flag_set(x, F_OBJS);
}
__device__ __forceinline__ void mark_obj_dirty(const Ctx x, uint32_t o) {
  if (x.lane == 0) x.w->objdirty[o >> 5] |= 1u << (o & 31u);
  __syncwarp();
}
__device__ __forceinline__ void mark_reclass(const Ctx x, uint32_t o) {
  if (x.lane == 0) x.w->rc[o >> 5] |= 1u << (o & 31u);
  __syncwarp();
}
__device__ __forceinline__ void mark_reclass_lanes(const Ctx x, bool pred, uint32_t o) {
  if (pred) atomicOr(&x.w->rc[o >> 5], 1u << (o & 31u));
  __syncwarp();
}
__device__ __forceinline__ bool in_reclass(const Warp* w, uint32_t o) {
  return (w->rc[o >> 5] >> (o & 31u)) & 1u;
}
// claim lane c changed: mark it for write-back
__device__ __forceinline__ void claims_dirty(const Ctx x, bool pred) {
  const uint32_t m = __ballot_sync(kFull, pred);
  if (x.lane == 0) { x.w->cdirty |= m; if (m) x.w->flags |= F_CLAIMS_CHANGED; }
  __syncwarp();
}
// P (protected_resident_kv) and the blocking set from per-claim protected counts
__device__ __forceinline__ void refresh_protected(const Ctx x) {
  const uint32_t pc = x.lane < x.p->C ? x.w->cl[x.lane][CF_PC] : 0u;
  const uint32_t P = __reduce_add_sync(kFull, pc);
  const uint32_t m = __ballot_sync(kFull, pc > 0);
  if (x.lane == 0) { x.w->h[H_P] = P; x.w->h[H_BLOCKMASK] = m; x.w->flags |= F_HDR; }
  __syncwarp();
}
// class of a new cached block (o, pos) from the object's bound claim
__device__ __forceinline__ uint32_t new_block_class(const Ctx x, uint32_t o, uint32_t pos) {
  const uint32_t c = obj_claim(x.w->obj0[o]);
  if (c >= 32 || !live_state(cl_state(x.w, c)) || pos >= x.w->cl[c][CF_F]) return 1;
  return claim_class(cl_mode(x.w, c), lowering(x));
}
// the live protected claim bound to object o gains `added` protected blocks
__device__ __forceinline__ void add_protected(const Ctx x, uint32_t o, uint32_t added) {
  const uint32_t c = obj_claim(x.w->obj0[o]);
  if (c < 32 && live_state(cl_state(x.w, c)) && claim_class(cl_mode(x.w, c), lowering(x)) == 3 &&
      added > 0) {
    if (x.lane == 0) x.w->cl[c][CF_PC] += added;
    __syncwarp();
    claims_dirty(x, x.lane == c);
    refresh_protected(x);
  }
}

// ------------------------------ block passes -------------------------------
__device__ __forceinline__ uint32_t block_of(const Ctx x, uint32_t j, int e) {
  return (j * 32 + x.lane) * 4 + e;
}
__device__ __forceinline__ void fbm_set(const Ctx x, uint32_t j, uint32_t nib) {
  if (nib) {
    const uint32_t b0 = block_of(x, j, 0);
    atomicOr(x.fbm() + (b0 >> 5), nib << (b0 & 31u));
  }
}

// reclass pass: rewrite the class bits of every cached block whose owner is
// marked, from the owner's bound claim; recount the protected blocks.
__device__ __noinline__ void flush_reclass(const Ctx x) {
  Warp* w = x.w;
  if ((w->rc[0] | w->rc[1] | w->rc[2] | w->rc[3]) == 0) return;
  need_claims(x);
  need_objs(x);
  const uint32_t low = lowering(x);
  for (uint32_t o = x.lane; o < x.p->O; o += 32) {
    uint32_t l3 = 0, l2 = 0;
    const uint32_t cc = obj_claim(w->obj0[o]);
    if (cc < 32 && live_state(cl_state(w, cc))) {
      const uint32_t cls = claim_class(cl_mode(w, cc), low);
      if (cls == 3) l3 = w->cl[cc][CF_F];
      if (cls == 2) l2 = w->cl[cc][CF_F];
    }
    w->lim3[o] = l3;
    w->lim2[o] = l2;
    w->cnt3[o] = 0;
  }
  __syncwarp();
  uint32_t* key = x.key();
  const uint4* meta4 = reinterpret_cast<const uint4*>(x.meta());
  const uint4* key4 = reinterpret_cast<const uint4*>(key);
  const uint32_t nv = x.nvec();
  for (uint32_t j = 0; j < nv; ++j) {
    const uint4 mv = __ldcg(meta4 + j * 32 + x.lane);
    bool any = false;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t m = el(mv, e);
      any |= meta_res(m) == kResCached && in_reclass(w, meta_owner(m));
    }
    if (!any) continue;
    const uint4 kv = __ldcg(key4 + j * 32 + x.lane);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t m = el(mv, e);
      if (meta_res(m) != kResCached) continue;
      const uint32_t o = meta_owner(m);
      if (!in_reclass(w, o)) continue;
      const uint32_t pos = meta_pos(m);
      const uint32_t cls = pos < w->lim3[o] ? 3u : (pos < w->lim2[o] ? 2u : 1u);
      const uint32_t k0 = el(kv, e);
      const uint32_t k1 = (cls << kClassShift) | (k0 & kSeqMask);
      if (k1 != k0) key[block_of(x, j, e)] = k1;
      if (cls == 3) atomicAdd(&w->cnt3[o], 1u);
    }
  }
  __syncwarp();
  bool ch = false;
  if (x.lane < x.p->C) {
    const uint32_t st = cl_state(w, x.lane), o = cl_obj(w, x.lane);
    if (live_state(st) && in_reclass(w, o)) {
      const uint32_t np = claim_class(cl_mode(w, x.lane), low) == 3 ? w->cnt3[o] : 0u;
      if (np != w->cl[x.lane][CF_PC]) { w->cl[x.lane][CF_PC] = np; ch = true; }
    }
  }
  __syncwarp();
  claims_dirty(x, ch);
  if (x.lane < 4) w->rc[x.lane] = 0;
  __syncwarp();
  refresh_protected(x);
}

// release request r's active blocks to FREE (deferral / refusal / no-admit)
__device__ __noinline__ void release_blocks(const Ctx x, uint32_t r) {
  uint32_t* key = x.key();
  uint32_t* meta = x.meta();
  const uint4* meta4 = reinterpret_cast<const uint4*>(meta);
  uint32_t freed = 0;
  const uint32_t nv = x.nvec();
  for (uint32_t j = 0; j < nv; ++j) {
    const uint4 mv = __ldcg(meta4 + j * 32 + x.lane);
    uint32_t nib = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t m = el(mv, e);
      if (meta_res(m) == kResActive && meta_owner(m) == r) nib |= 1u << e;
    }
    if (nib) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (!((nib >> e) & 1u)) continue;
        const uint32_t bb = block_of(x, j, e);
        meta[bb] = meta_make(kResFree, 0, 0);
        key[bb] = bb;
      }
      fbm_set(x, j, nib);
      freed += __popc(nib);
    }
  }
  freed = __reduce_add_sync(kFull, freed);
  hset(x, H_FREE, x.w->h[H_FREE] + freed);
}

// ------------------------------ arbiter ------------------------------------
// Feasibility boundary protected + active <= usable; relax by
// auto-demotion (G10); else explicit refusal / deferral with
// blocking-claim attribution and the capacity proof.
// requester: request slot (record in w->rq), or 0xFFFFFFFF for INSERT of `obj`.
__device__ __noinline__ bool arbitrate(const Ctx x, uint32_t need, uint32_t requester, uint32_t obj) {
  Warp* w = x.w;
  const uint32_t U = w->h[H_U];
  const uint32_t P = w->h[H_P];
  const uint64_t A = (uint64_t)w->h[H_ALIVE] + need;
  if ((uint64_t)P + A <= U) return true;
  const uint32_t pol = w->h[H_POLICY];
  if ((pol & 0xFFu) == LOW_CONTRACT && (pol >> 24)) {
    need_claims(x);
    const bool lc = x.lane < x.p->C;
    const uint32_t g = (lc && live_state(cl_state(w, x.lane)) && cl_mode(w, x.lane) == M_DEMOTABLE)
                           ? w->cl[x.lane][CF_PC] : 0u;
    const uint32_t S = warp_incl_scan(g, x.lane);
    const bool ok = g > 0 && (uint64_t)(P - S) + A <= U;
    const uint32_t mk = __ballot_sync(kFull, ok);
    if (mk) {
      const uint32_t j = __ffs(mk) - 1;
      const bool dem = g > 0 && x.lane <= j;
      const uint32_t o = lc ? cl_obj(w, x.lane) : 0u;
      emit_lanes(x, dem, EV_DEMOTED, 1, 0, o, g, 0, 0);
      const uint32_t nd = __popc(__ballot_sync(kFull, dem));
      mark_reclass_lanes(x, dem, o);
      if (dem) { w->cl[x.lane][0] = (w->cl[x.lane][0] & ~0xFFu) | C_DEMOTED; w->cl[x.lane][CF_PC] = 0; }
      __syncwarp();
      claims_dirty(x, dem);
      refresh_protected(x);
      ctr_add(x, K_DEMOTED_AUTO, nd);
      return true;
    }
  }
  const uint32_t shortfall = (uint32_t)((uint64_t)P + A - U);
  const bool resident = A <= U && P > 0;
  const uint32_t why = resident ? WHY_PROTECTED : WHY_CAPACITY;
  const uint32_t mask = resident ? w->h[H_BLOCKMASK] : 0u;
  if (requester == 0xFFFFFFFFu) {
    emit(x, EV_INSERT_REFUSED, obj, why, mask, P, (uint32_t)A, U, shortfall);
    ctr_add(x, K_INSERT_REFUSED, 1);
    return false;
  }
  // request: release its live blocks, then defer or refuse (G9)
  const uint32_t live = w->rq[RQ_LIVE];
  if (live > 0) {
    release_blocks(x, requester);
    hset(x, H_ALIVE, w->h[H_ALIVE] - live);
  }
  const uint32_t w0 = w->rq[RQ_W0];
  const uint32_t defer = w0 >> 24;
  const bool dfr = defer < ((pol >> 16) & 0xFFu);
  __syncwarp();
  if (x.lane == 0) {
    w->rq[RQ_LIVE] = 0;
    w->rq[RQ_DONE] = 0;
    w->rq[RQ_W0] = dfr ? ((w0 & 0x00FFFF00u) | R_DEFERRED | ((defer + 1) << 24))
                       : ((w0 & 0xFFFFFF00u) | R_REFUSED);
  }
  __syncwarp();
  if (dfr) {
    emit(x, EV_DEFERRED, requester, why, mask, P, (uint32_t)A, U, shortfall);
    ctr_add(x, resident ? K_DEFERRED_PROTECTED : K_DEFERRED_CAPACITY, 1);
  } else {
    emit(x, EV_REFUSED, requester, why, mask, P, (uint32_t)A, U, shortfall);
    ctr_add(x, resident ? K_REFUSED_PROTECTED : K_REFUSED_CAPACITY, 1);
  }
  return false;
}

// ------------------------------ victim selection ---------------------------
__device__ __forceinline__ uint4 key_vec(const Ctx x, uint32_t j, bool staged) {
  if (staged) return reinterpret_cast<const uint4*>(x.w->keys)[j * 32 + x.lane];
  return __ldcg(reinterpret_cast<const uint4*>(x.key()) + j * 32 + x.lane);
}
__device__ __noinline__ uint32_t count_le(const Ctx x, uint32_t T, bool staged) {
  uint32_t c = 0;
  const uint32_t nv = x.nvec();
  for (uint32_t j = 0; j < nv; ++j) {
    const uint4 v = key_vec(x, j, staged);
    c += (v.x <= T) + (v.y <= T) + (v.z <= T) + (v.w <= T);
  }
  return __reduce_add_sync(kFull, c);
}

// Free-only allocation (k <= free count): the k lowest-id free blocks, lane =
// free-bitmap word; positions base + rank in block-id order (G24).
__device__ __noinline__ void alloc_free(const Ctx x, uint32_t k, uint32_t owner, bool insert,
                                        uint32_t base) {
  Warp* w = x.w;
  uint32_t* fbm = x.fbm();
  uint32_t* key = x.key();
  uint32_t* meta = x.meta();
  const uint32_t nw = x.nvec() * 4;
  const uint32_t seq_base = w->h[H_SEQ];
  uint32_t l3 = 0, l2 = 0;
  if (insert) {  // class of the new cached blocks from the object's bound claim
    const uint32_t cc = obj_claim(w->obj0[owner]);
    if (cc < 32 && live_state(cl_state(w, cc))) {
      const uint32_t cls = claim_class(cl_mode(w, cc), lowering(x));
      if (cls == 3) l3 = w->cl[cc][CF_F];
      if (cls == 2) l2 = w->cl[cc][CF_F];
    }
  }
  uint32_t acc = 0;
  for (uint32_t w0 = 0; w0 < nw && acc < k; w0 += 32) {
    const uint32_t wi = w0 + x.lane;
    const uint32_t word = wi < nw ? __ldcg(fbm + wi) : 0u;
    const uint32_t c = __popc(word);
    const uint32_t S = warp_incl_scan(c, x.lane);
    const uint32_t before = acc + S - c;
    const uint32_t take = before >= k ? 0u : min(c, k - before);
    if (take > 0) {
      uint32_t tw = take == c ? word : word & ((1u << nth_set_bit(word, take + 1)) - 1u);
      fbm[wi] = word & ~tw;
      uint32_t r = before;
      while (tw) {
        const uint32_t bit = __ffs(tw) - 1;
        tw &= tw - 1;
        const uint32_t bb = wi * 32 + bit;
        const uint32_t pos = base + r++;
        if (insert) {
          const uint32_t cls = pos < l3 ? 3u : (pos < l2 ? 2u : 1u);
          key[bb] = (cls << kClassShift) | (seq_base + (k - 1 - pos));
          meta[bb] = meta_make(kResCached, owner, pos);
        } else {
          key[bb] = kKeyActive;
          meta[bb] = meta_make(kResActive, owner, pos);
        }
      }
    }
    acc += __shfl_sync(kFull, S, 31);
  }
  hset(x, H_FREE, w->h[H_FREE] - k);
  ctr_add(x, K_BLOCKS_ALLOCATED, k);
}

// Evicting allocation (k > free count): every free block plus the k - free
// smallest candidate keys.  The threshold T with #{key <= T} == k is found by
// probing the counting function: first densely from the smallest key of the
// class (victims are usually the run of oldest stamps), galloping until a
// probe overshoots, then interpolation / bisection inside the bracket (keys
// are unique, so the search ends on an exact count).
__device__ __noinline__ void alloc_evict(const Ctx x, uint32_t k, uint32_t owner, bool insert,
                                         uint32_t base) {
  Warp* w = x.w;
  need_claims(x);
  need_objs(x);
  const uint32_t fr = w->h[H_FREE];
  const uint32_t nv = x.nvec();
  const bool staged = x.p->NS <= kStageMax;
  uint32_t c1 = 0, mn1 = kFull, mn2 = kFull;
  {
    const uint4* key4 = reinterpret_cast<const uint4*>(x.key());
    for (uint32_t j = 0; j < nv; ++j) {
      const uint4 v = __ldcg(key4 + j * 32 + x.lane);
      if (staged) reinterpret_cast<uint4*>(w->keys)[j * 32 + x.lane] = v;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t kk = el(v, e);
        const uint32_t cls = kk >> kClassShift;
        c1 += cls == 1 ? 1u : 0u;
        mn1 = cls == 1 ? min(mn1, kk) : mn1;
        mn2 = cls == 2 ? min(mn2, kk) : mn2;
      }
    }
    __syncwarp();
  }
  c1 = __reduce_add_sync(kFull, c1);
  uint32_t lo, clo, top;
  if (k - fr <= c1) { lo = __reduce_min_sync(kFull, mn1) - 1; clo = fr; top = (2u << kClassShift) - 1; }
  else { lo = __reduce_min_sync(kFull, mn2) - 1; clo = fr + c1; top = (3u << kClassShift) - 1; }
  uint32_t hi = top, chi = 0;
  bool bracket = false;
  uint32_t mult = 1;
  uint32_t T;
  for (uint32_t it = 0;; ++it) {
    uint32_t m;
    if (!bracket) {
      const uint64_t d = (uint64_t)(k - clo) * mult;
      m = (uint32_t)min((uint64_t)lo + d, (uint64_t)top);
      mult = mult < (1u << 20) ? mult * 4 : mult;
    } else {
      const uint32_t span = hi - lo;
      m = (it & 1u) ? lo + (uint32_t)(((uint64_t)(k - clo) * span) / (chi - clo)) : lo + span / 2;
      m = max(m, lo + 1);
      m = min(m, hi - 1);
    }
    const uint32_t cm = count_le(x, m, staged);
    if (cm == k) { T = m; break; }
    if (cm < k) { lo = m; clo = cm; }
    else { hi = m; chi = cm; bracket = true; }
  }
  // apply: taken = {key <= T}.  Pass 1 compacts the taken blocks in block-id
  // order into a shared list (in place over the staged keys: entry i is
  // written only after vectors holding keys >= i were read); pass 2 gives
  // them positions base + i, one block per lane.  Victims are attributed by
  // their object's claim state now (Table 4); leading prefixes shrink.
  uint32_t* key = x.key();
  uint32_t* meta = x.meta();
  uint32_t* list = w->keys;
  const uint32_t seq_base = w->h[H_SEQ];
  uint32_t l3 = 0, l2 = 0;
  if (insert) {
    const uint32_t cc = obj_claim(w->obj0[owner]);
    if (cc < 32 && live_state(cl_state(w, cc))) {
      const uint32_t cls = claim_class(cl_mode(w, cc), lowering(x));
      if (cls == 3) l3 = w->cl[cc][CF_F];
      if (cls == 2) l2 = w->cl[cc][CF_F];
    }
  }
  uint32_t ord = 0, rel = 0, clm = 0;
  uint32_t listed = 0, done_pos = 0;
  auto drain = [&](uint32_t n) {
    for (uint32_t i = x.lane; i < n; i += 32) {
      const uint32_t e = list[i];
      const uint32_t bb = e & 0x7FFFFFFFu;
      const uint32_t rank = done_pos + i;
      const uint32_t pos = base + rank;
      if (e >> 31) {
        const uint32_t m = __ldcg(meta + bb);
        const uint32_t o = meta_owner(m);
        const uint32_t cc = obj_claim(w->obj0[o]);
        const uint32_t st = cc < 32 ? cl_state(w, cc) : C_EMPTY;
        if (st == C_DEMOTED || st == C_EXPIRED) ++rel;
        else if (st == C_ACCEPTED || st == C_MATERIALIZED) ++clm;
        else ++ord;
        atomicMin(&w->lead[o], meta_pos(m));
        atomicOr(&w->objdirty[o >> 5], 1u << (o & 31u));
      }
      if (insert) {
        const uint32_t cls = pos < l3 ? 3u : (pos < l2 ? 2u : 1u);
        key[bb] = (cls << kClassShift) | (seq_base + (k - 1 - pos));
        meta[bb] = meta_make(kResCached, owner, pos);
      } else {
        key[bb] = kKeyActive;
        meta[bb] = meta_make(kResActive, owner, pos);
      }
    }
    __syncwarp();
    done_pos += n;
  };
  for (uint32_t j = 0; j < nv && done_pos + listed < k; ++j) {
    const uint4 v = key_vec(x, j, staged);
    const uint32_t tb = (v.x <= T ? 1u : 0u) | (v.y <= T ? 2u : 0u) | (v.z <= T ? 4u : 0u) |
                        (v.w <= T ? 8u : 0u);
    if (!__any_sync(kFull, tb != 0)) continue;
    const uint32_t cnt = __popc(tb);
    const uint32_t S = warp_incl_scan(cnt, x.lane);
    const uint32_t tot = __shfl_sync(kFull, S, 31);
    if (!staged && listed + tot > kStageMax) { drain(listed); listed = 0; }
    uint32_t r = listed + S - cnt;
    if (tb & 1u) list[r++] = block_of(x, j, 0) | (v.x >= (1u << kClassShift) ? 0x80000000u : 0u);
    if (tb & 2u) list[r++] = block_of(x, j, 1) | (v.y >= (1u << kClassShift) ? 0x80000000u : 0u);
    if (tb & 4u) list[r++] = block_of(x, j, 2) | (v.z >= (1u << kClassShift) ? 0x80000000u : 0u);
    if (tb & 8u) list[r++] = block_of(x, j, 3) | (v.w >= (1u << kClassShift) ? 0x80000000u : 0u);
    listed += tot;
    __syncwarp();
  }
  drain(listed);
  // every free block was taken
  {
    uint32_t* fb = x.fbm();
    for (uint32_t wi = x.lane; wi < nv * 4; wi += 32) fb[wi] = 0;
  }
  ord = __reduce_add_sync(kFull, ord);
  rel = __reduce_add_sync(kFull, rel);
  clm = __reduce_add_sync(kFull, clm);
  hset(x, H_FREE, 0);
  ctr_add(x, K_VICTIMS_ORDINARY, ord);
  ctr_add(x, K_VICTIMS_AFTER_RELEASE, rel);
  ctr_add(x, K_VICTIMS_CLAIMED, clm);
  ctr_add(x, K_BLOCKS_ALLOCATED, k);
  if (ord + rel + clm > 0) {
    emit(x, EV_VICTIMS, owner, insert ? 1u : 0u, 0, ord, rel, clm, k);
    flag_set(x, F_POST);
  }
}

// alloc(k): take the k smallest (class, key) candidates.
// insert: blocks become CACHED(obj owner) with tail-first stamps, else
// ACTIVE(request owner).
__device__ __noinline__ void alloc(const Ctx x, uint32_t k, uint32_t owner, bool insert,
                                   uint32_t base) {
  flush_reclass(x);
  if (insert) { need_claims(x); need_objs(x); }
  if (k <= x.w->h[H_FREE]) alloc_free(x, k, owner, insert, base);
  else alloc_evict(x, k, owner, insert, base);
}

// ------------------------------ request io ---------------------------------
__device__ __forceinline__ void load_request(const Ctx x, uint32_t r) {
  if (x.lane < 8) x.w->rq[x.lane] = __ldcg(x.p->req + ((size_t)x.t * x.p->Q + r) * 8 + x.lane);
  __syncwarp();
}
__device__ __forceinline__ void store_request(const Ctx x, uint32_t r) {
  if (x.lane < 8) x.p->req[((size_t)x.t * x.p->Q + r) * 8 + x.lane] = x.w->rq[x.lane];
}
__device__ __forceinline__ uint32_t peak_blocks(const Warp* w) {
  return (uint32_t)(((uint64_t)w->rq[RQ_PROMPT] + w->rq[RQ_DECODE] + kBlockTokens - 1) / kBlockTokens);
}

// ------------------------------ ops ----------------------------------------
// SUBMIT: claim decision (Table 2).
__device__ __noinline__ void op_submit(const Ctx x, const Op op) {
  Warp* w = x.w;
  const uint32_t mode = op.c & 0x7Fu;
  const bool mismatch = (op.c & 0x80u) != 0;
  if (op.a >= x.p->C || op.b >= x.p->O || mode > M_BEST_EFFORT) return op_error(x, op, ERR_INVALID_ARG);
  need_claims(x);
  if (cl_state(w, op.a) != C_EMPTY) return op_error(x, op, ERR_DUPLICATE_SLOT);
  if (op.x < 1 || op.y < 1 || op.y > op.x || (mode == M_EXPIRING && op.z == 0))
    return op_error(x, op, ERR_INVALID_ARG);
  need_objs(x);
  const uint32_t ow = w->obj0[op.b];
  const uint32_t oc = obj_claim(ow);
  const bool bound_live = oc < 32 && live_state(cl_state(w, oc));
  const uint32_t U = w->h[H_U];
  uint32_t rej = 0;
  if (mismatch) rej = REJ_IDENTITY;
  else if (bound_live) rej = REJ_OBJECT_CLAIMED;
  else if (op.x > U) rej = REJ_FOOTPRINT;
  else if ((w->h[H_ACCEPT] & 0xFFu) == ACCEPT_RESERVE && obligated(mode)) {
    const bool lc = x.lane < x.p->C && live_state(cl_state(w, x.lane)) && obligated(cl_mode(w, x.lane));
    const uint32_t sum = __reduce_add_sync(kFull, lc ? w->cl[x.lane][CF_F] : 0u);
    if ((uint64_t)op.x + sum > U) rej = REJ_RESERVE;
  }
  if (x.lane == op.a) {
    uint32_t* r = w->cl[op.a];
    r[0] = (rej ? C_REFUSED : C_ACCEPTED) | (mode << 8) | (op.b << 16);
    r[CF_F] = op.x; r[CF_R] = op.y; r[CF_D] = op.z; r[CF_DEC] = x.step; r[CF_PC] = 0;
  }
  __syncwarp();
  claims_dirty(x, x.lane == op.a);
  if (rej) {
    emit(x, EV_REJECTED, op.a, rej, 0, op.b, op.x, op.y, op.z);
    ctr_add(x, K_REJECTED, 1);
    return;
  }
  emit(x, EV_ACCEPTED, op.a, 0, 0, op.b, op.x, op.y, op.z);
  ctr_add(x, K_ACCEPTED, 1);
  if (x.lane == 0) w->obj0[op.b] = obj_make(obj_live(ow), op.a, obj_len(ow));
  __syncwarp();
  mark_obj_dirty(x, op.b);
  if (obj_live(ow) && claim_class(mode, lowering(x)) != 1) mark_reclass(x, op.b);
  flag_set(x, F_POST);
}

__device__ __noinline__ void op_admit(const Ctx x, const Op op) {
  Warp* w = x.w;
  if (op.a >= x.p->Q || op.b >= x.p->O || op.c > 1) return op_error(x, op, ERR_INVALID_ARG);
  load_request(x, op.a);
  const uint32_t st = w->rq[RQ_W0] & 0xFFu;
  if (st == R_RUNNING || st == R_DEFERRED) return op_error(x, op, ERR_DUPLICATE_SLOT);
  if (op.x < 1 || op.y < 1 || op.x > kMaxTokens || op.z > kMaxTokens) return op_error(x, op, ERR_INVALID_ARG);
  if (x.lane == 0) {
    w->rq[RQ_W0] = R_RUNNING | (op.c << 8) | (op.b << 16);
    w->rq[RQ_PROMPT] = op.x; w->rq[RQ_CHUNK] = op.y; w->rq[RQ_DECODE] = op.z;
    w->rq[RQ_DONE] = 0; w->rq[RQ_LIVE] = 0;
  }
  __syncwarp();
  ctr_add(x, K_ADMITTED, 1);
  if (((w->h[H_POLICY] >> 8) & 0xFFu) == ADMIT_PEAK) arbitrate(x, peak_blocks(w), op.a, 0);
  store_request(x, op.a);
}

// ADVANCE: one prefill chunk or one decode token (G14); live KV
// accumulates as ceil(done/16) (Table 8).
__device__ __noinline__ void op_advance(const Ctx x, const Op op) {
  Warp* w = x.w;
  if (op.a >= x.p->Q) return op_error(x, op, ERR_INVALID_ARG);
  load_request(x, op.a);
  const uint32_t st = w->rq[RQ_W0] & 0xFFu;
  if (st != R_RUNNING && st != R_DEFERRED) return op_error(x, op, ERR_UNKNOWN_REQUEST);
  if (st == R_RUNNING && (uint64_t)w->rq[RQ_DONE] >= (uint64_t)w->rq[RQ_PROMPT] + w->rq[RQ_DECODE])
    return op_error(x, op, ERR_NO_CHUNKS);
  if (st == R_DEFERRED) {
    if (((w->h[H_POLICY] >> 8) & 0xFFu) == ADMIT_PEAK && !arbitrate(x, peak_blocks(w), op.a, 0)) {
      store_request(x, op.a);
      return;
    }
    if (x.lane == 0) w->rq[RQ_W0] = (w->rq[RQ_W0] & ~0xFFu) | R_RUNNING;
    __syncwarp();
  }
  const uint32_t done = w->rq[RQ_DONE], prompt = w->rq[RQ_PROMPT], live = w->rq[RQ_LIVE];
  const uint32_t n = done < prompt ? min(w->rq[RQ_CHUNK], prompt - done) : 1u;
  const uint32_t need_total = (uint32_t)(((uint64_t)done + n + kBlockTokens - 1) / kBlockTokens);
  const uint32_t need = need_total > live ? need_total - live : 0u;
  if (need > 0) {
    if (!arbitrate(x, need, op.a, 0)) { store_request(x, op.a); return; }
    alloc(x, need, op.a, false, live);
    if (x.lane == 0) w->rq[RQ_LIVE] = live + need;
    hset(x, H_ALIVE, w->h[H_ALIVE] + need);
  }
  if (x.lane == 0) w->rq[RQ_DONE] = done + n;
  __syncwarp();
  store_request(x, op.a);
}

// COMPLETE: future reusable admission is separate from active allocation
// (Table 7); only full blocks become reusable (G16).
__device__ __noinline__ void op_complete(const Ctx x, const Op op) {
  Warp* w = x.w;
  if (op.a >= x.p->Q) return op_error(x, op, ERR_INVALID_ARG);
  load_request(x, op.a);
  if ((w->rq[RQ_W0] & 0xFFu) != R_RUNNING) return op_error(x, op, ERR_UNKNOWN_REQUEST);
  need_objs(x);
  const uint32_t done = w->rq[RQ_DONE];
  const uint32_t full = done / kBlockTokens;
  const uint32_t o = (w->rq[RQ_W0] >> 16) & 0xFFu;
  const uint32_t wa = (w->rq[RQ_W0] >> 8) & 0xFFu;
  const uint32_t ow = w->obj0[o];
  const bool admitted = wa && !obj_live(ow);
  if (admitted && (uint64_t)w->h[H_SEQ] + full > kSeqLimit) return op_error(x, op, ERR_SEQ_EXHAUSTED);
  const uint32_t held = w->rq[RQ_LIVE];
  if (admitted) {
    if (obj_claim(ow) < 32) need_claims(x);
    uint32_t cls_lim3 = 0, cls_lim2 = 0;
    {
      const uint32_t cc = obj_claim(ow);
      if (cc < 32 && live_state(cl_state(w, cc))) {
        const uint32_t cls = claim_class(cl_mode(w, cc), lowering(x));
        if (cls == 3) cls_lim3 = w->cl[cc][CF_F];
        if (cls == 2) cls_lim2 = w->cl[cc][CF_F];
      }
    }
    const uint32_t seq_base = w->h[H_SEQ];
    uint32_t* key = x.key();
    uint32_t* meta = x.meta();
    const uint4* meta4 = reinterpret_cast<const uint4*>(meta);
    uint32_t freed = 0;
    const uint32_t nv = held > 0 ? x.nvec() : 0u;
    for (uint32_t j = 0; j < nv; ++j) {
      const uint4 mv = __ldcg(meta4 + j * 32 + x.lane);
      uint32_t nib = 0;
      for (int e = 0; e < 4; ++e) {
        const uint32_t m = el(mv, e);
        if (meta_res(m) != kResActive || meta_owner(m) != op.a) continue;
        const uint32_t bb = block_of(x, j, e);
        const uint32_t pos = meta_pos(m);
        if (pos < full) {
          const uint32_t cls = pos < cls_lim3 ? 3u : (pos < cls_lim2 ? 2u : 1u);
          key[bb] = (cls << kClassShift) | (seq_base + (full - 1 - pos));
          meta[bb] = meta_make(kResCached, o, pos);
        } else {
          key[bb] = bb;
          meta[bb] = meta_make(kResFree, 0, 0);
          nib |= 1u << e;
        }
      }
      fbm_set(x, j, nib);
      freed += __popc(nib);
    }
    freed = __reduce_add_sync(kFull, freed);
    hset(x, H_FREE, w->h[H_FREE] + freed);
    hset(x, H_SEQ, seq_base + full);
    if (x.lane == 0) { w->obj0[o] = obj_make(1, obj_claim(ow), full); w->lead[o] = full; }
    __syncwarp();
    mark_obj_dirty(x, o);
    add_protected(x, o, min(cls_lim3, full));
    ctr_add(x, K_BLOCKS_CACHED, full);
    flag_set(x, F_POST);
  } else {
    if (held > 0) release_blocks(x, op.a);
    emit(x, EV_WRITE_DENIED, op.a, wa ? 1u : 0u, 0, o, held, 0, 0);
    ctr_add(x, K_WRITE_DENIED, 1);
  }
  emit(x, EV_SERVED, op.a, admitted ? 1u : 0u, 0, done, admitted ? full : 0u, o, 0);
  ctr_add(x, K_SERVED, 1);
  hset(x, H_ALIVE, w->h[H_ALIVE] - held);
  if (x.lane == 0) { w->rq[RQ_W0] = (w->rq[RQ_W0] & ~0xFFu) | R_COMPLETED; w->rq[RQ_LIVE] = 0; }
  __syncwarp();
  store_request(x, op.a);
}

// INSERT: resident insertion through the ordinary allocation path (G17).
__device__ __noinline__ void op_insert(const Ctx x, const Op op) {
  Warp* w = x.w;
  if (op.a >= x.p->O) return op_error(x, op, ERR_INVALID_ARG);
  need_objs(x);
  const uint32_t ow = w->obj0[op.a];
  if (obj_live(ow)) return op_error(x, op, ERR_OBJECT_IN_USE);
  if (op.x < 1 || op.x > kMaxTokens) return op_error(x, op, ERR_INVALID_ARG);
  if ((uint64_t)w->h[H_SEQ] + op.x > kSeqLimit) return op_error(x, op, ERR_SEQ_EXHAUSTED);
  if (!arbitrate(x, op.x, 0xFFFFFFFFu, op.a)) return;
  alloc(x, op.x, op.a, true, 0);
  hset(x, H_SEQ, w->h[H_SEQ] + op.x);
  if (x.lane == 0) { w->obj0[op.a] = obj_make(1, obj_claim(ow), op.x); w->lead[op.a] = op.x; }
  __syncwarp();
  mark_obj_dirty(x, op.a);
  {
    const uint32_t cc = obj_claim(ow);
    if (cc < 32) add_protected(x, op.a, min(w->cl[cc][CF_F], op.x));
  }
  ctr_add(x, K_INSERTED, 1);
  ctr_add(x, K_BLOCKS_CACHED, op.x);
  flag_set(x, F_POST);
}

// DEMOTE: claim_demoted before post-release block loss (Table 4).
__device__ __noinline__ void op_demote(const Ctx x, const Op op) {
  Warp* w = x.w;
  if (op.a >= x.p->C) return op_error(x, op, ERR_INVALID_ARG);
  need_claims(x);
  const uint32_t st = cl_state(w, op.a);
  if (st == C_EMPTY) return op_error(x, op, ERR_UNKNOWN_CLAIM);
  if (!live_state(st)) return op_error(x, op, ERR_ILLEGAL_TRANSITION);
  const uint32_t o = cl_obj(w, op.a), pc = w->cl[op.a][CF_PC], mode = cl_mode(w, op.a);
  if (x.lane == 0) { w->cl[op.a][0] = (w->cl[op.a][0] & ~0xFFu) | C_DEMOTED; w->cl[op.a][CF_PC] = 0; }
  __syncwarp();
  claims_dirty(x, x.lane == op.a);
  emit(x, EV_DEMOTED, op.a, 0, 0, o, pc, 0, 0);
  ctr_add(x, K_DEMOTED_EXPLICIT, 1);
  if (claim_class(mode, lowering(x)) != 1) mark_reclass(x, o);
  refresh_protected(x);
}

// TOUCH: reuse probe of the materialization surface;
// restamps the leading prefix tail-first (G23).
__device__ __noinline__ void op_touch(const Ctx x, const Op op) {
  Warp* w = x.w;
  if (op.a >= x.p->O) return op_error(x, op, ERR_INVALID_ARG);
  need_objs(x);
  const uint32_t ow = w->obj0[op.a];
  const uint32_t L = obj_live(ow) ? w->lead[op.a] : 0u;
  if ((uint64_t)w->h[H_SEQ] + L > kSeqLimit) return op_error(x, op, ERR_SEQ_EXHAUSTED);
  const uint32_t seq_base = w->h[H_SEQ];
  if (L > 0) {
    uint32_t* key = x.key();
    const uint4* meta4 = reinterpret_cast<const uint4*>(x.meta());
    const uint32_t nv = x.nvec();
    for (uint32_t j = 0; j < nv; ++j) {
      const uint4 mv = __ldcg(meta4 + j * 32 + x.lane);
      for (int e = 0; e < 4; ++e) {
        const uint32_t m = el(mv, e);
        if (meta_res(m) == kResCached && meta_owner(m) == op.a && meta_pos(m) < L) {
          const uint32_t bb = block_of(x, j, e);
          key[bb] = (__ldcg(key + bb) & ~kSeqMask) | (seq_base + (L - 1 - meta_pos(m)));
        }
      }
    }
    hset(x, H_SEQ, seq_base + L);
  }
  const uint32_t cc = obj_claim(ow);
  const bool has = cc < 32;
  if (has) need_claims(x);
  const uint32_t Rc = has ? w->cl[cc][CF_R] : 0u;
  const bool sat = has && live_state(cl_state(w, cc)) && L >= Rc;
  emit(x, EV_REUSE_PROBE, has ? cc : 0xFFu, sat ? 1u : 0u, 0, op.a, L, L * kBlockTokens, Rc);
  ctr_add(x, K_REUSE_PROBES, 1);
  ctr_add(x, K_REUSE_TOKENS, L * kBlockTokens);
}

// ------------------------------ phases -------------------------------------
// expiry: "Runtime responsibility ends at expiry" (Table 3; G13)
__device__ __noinline__ void expiry(const Ctx x) {
  need_claims(x);
  Warp* w = x.w;
  const bool lc = x.lane < x.p->C;
  const uint32_t* r = w->cl[x.lane];
  const bool ex = lc && live_state(r[0] & 0xFFu) && r[CF_D] > 0 &&
                  (uint64_t)r[CF_DEC] + r[CF_D] <= x.step;
  const uint32_t m = __ballot_sync(kFull, ex);
  if (x.lane == 0) w->flags |= F_CLAIMS_CHANGED;  // next expiry is recomputed
  __syncwarp();
  if (!m) return;
  const uint32_t o = (r[0] >> 16) & 0xFFu;
  emit_lanes(x, ex, EV_EXPIRED, 0, 0, o, r[CF_PC], r[CF_DEC], r[CF_D]);
  mark_reclass_lanes(x, ex && claim_class((r[0] >> 8) & 0xFFu, lowering(x)) != 1, o);
  if (ex) { w->cl[x.lane][0] = (r[0] & ~0xFFu) | C_EXPIRED; w->cl[x.lane][CF_PC] = 0; }
  __syncwarp();
  claims_dirty(x, ex);
  refresh_protected(x);
  ctr_add(x, K_EXPIRED, __popc(m));
}

// post-op predicate pass: accepted -> materialized when leading >= R
// (P:1038-1041); materialized -> harmed when the predicate breaks without a
// prior release (Table 4, G5)
__device__ __noinline__ void post_op(const Ctx x) {
  need_claims(x);
  need_objs(x);
  Warp* w = x.w;
  const bool lc = x.lane < x.p->C;
  const uint32_t w0 = w->cl[x.lane][0];
  const uint32_t st = w0 & 0xFFu, mode = (w0 >> 8) & 0xFFu, o = (w0 >> 16) & 0xFFu;
  const uint32_t R = w->cl[x.lane][CF_R];
  const bool lv = lc && live_state(st);
  const bool olive = lv && obj_live(w->obj0[o]);
  const uint32_t L = olive ? w->lead[o] : 0u;
  const bool mat = lv && st == C_ACCEPTED && olive && L >= R;
  const bool harm = lv && st == C_MATERIALIZED && L < R;
  const uint32_t mm = __ballot_sync(kFull, mat), hm = __ballot_sync(kFull, harm);
  if ((mm | hm) == 0) return;
  const bool ob = obligated(mode);
  emit_lanes(x, mat || harm, mat ? EV_MATERIALIZED : EV_HARMED, harm ? (ob ? 1u : 0u) : 0u, 0, L, R,
             mat ? L * kBlockTokens : w->h[H_P], mat ? o : w->h[H_ALIVE]);
  mark_reclass_lanes(x, harm && claim_class(mode, lowering(x)) != 1, o);
  if (mat) w->cl[x.lane][0] = (w0 & ~0xFFu) | C_MATERIALIZED;
  if (harm) { w->cl[x.lane][0] = (w0 & ~0xFFu) | C_HARMED; w->cl[x.lane][CF_PC] = 0; }
  __syncwarp();
  claims_dirty(x, mat || harm);
  ctr_add(x, K_MATERIALIZED, __popc(mm));
  ctr_add(x, K_HARMED_OBLIGATED, __popc(__ballot_sync(kFull, harm && ob)));
  ctr_add(x, K_HARMED_UNOBLIGATED, __popc(__ballot_sync(kFull, harm && !ob)));
  refresh_protected(x);
}

__device__ __noinline__ void finish(const Ctx x) {
  Warp* w = x.w;
  flush_reclass(x);
  if (w->flags & F_POST) {
    post_op(x);
    flush_reclass(x);
  }
  if (w->flags & F_CLAIMS_CHANGED) {
    const uint32_t* r = w->cl[x.lane];
    const uint32_t ne = (x.lane < x.p->C && live_state(r[0] & 0xFFu) && r[CF_D] > 0)
                            ? (uint32_t)min((uint64_t)r[CF_DEC] + r[CF_D], (uint64_t)0xFFFFFFFFu)
                            : 0xFFFFFFFFu;
    const uint32_t m = __reduce_min_sync(kFull, ne);
    if (x.lane == 0) { w->h[H_NEXT_EXPIRY] = m; w->flags |= F_HDR; }
    __syncwarp();
  }
  // write back dirty claims and objects
  if ((w->cdirty >> x.lane) & 1u) {
    uint4* cp = reinterpret_cast<uint4*>(x.p->clm + ((size_t)x.t * x.p->C + x.lane) * 8);
    cp[0] = reinterpret_cast<const uint4*>(w->cl[x.lane])[0];
    cp[1] = reinterpret_cast<const uint4*>(w->cl[x.lane])[1];
  }
  if (w->objdirty[0] | w->objdirty[1] | w->objdirty[2] | w->objdirty[3]) {
    uint2* dst = reinterpret_cast<uint2*>(x.p->obj) + (size_t)x.t * x.p->O;
    for (uint32_t o = x.lane; o < x.p->O; o += 32)
      if ((w->objdirty[o >> 5] >> (o & 31u)) & 1u) dst[o] = make_uint2(w->obj0[o], w->lead[o]);
  }
  if (w->nev) {
    if (x.lane == 0) { w->h[H_EVCOUNT] += w->nev; w->flags |= F_HDR; }
    __syncwarp();
  }
  if (w->flags & F_HDR) {
    if (x.lane < H_NWORDS) x.p->hdr[(size_t)x.t * H_NWORDS + x.lane] = w->h[x.lane];
  }
  __syncwarp();
  const uint32_t d = w->ctr[x.lane];
  if (d) x.p->ctr[(size_t)x.t * K_NCTR + x.lane] += d;
}

struct StepArgs {
  PoolDev p;
  const uint4* ops;     // this step's row: [num_traces]
  uint32_t step;        // global step index of this launch
};

// op kind -> dispatch bucket: heavy block-scanning ops first, cheap ones last
// (so the tail of a launch is short work), one bucket per code path so the
// warps resident on an SM fetch the same instructions.
__device__ __forceinline__ uint32_t bucket_of(uint32_t kind) {
  switch (kind) {
    case OP_ADVANCE: return 0;
    case OP_INSERT: return 1;
    case OP_COMPLETE: return 2;
    case OP_TOUCH: return 3;
    case OP_SUBMIT: return 4;
    case OP_ADMIT: return 5;
    case OP_DEMOTE: return 6;
    default: return 7;  // NOP and unknown kinds
  }
}

__global__ void __launch_bounds__(256) rkc_classify_kernel(const __grid_constant__ StepArgs args) {
  const PoolDev& p = args.p;
  uint32_t* cnt = p.bcnt + (args.step & 1u) * 8;
  if (blockIdx.x == 0 && threadIdx.x < 8) p.bcnt[((args.step + 1u) & 1u) * 8 + threadIdx.x] = 0;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x; base < p.num_traces; base += stride) {
    const uint32_t t = base + threadIdx.x;
    const bool valid = t < p.num_traces;
    const uint32_t kind = valid ? (__ldcs(&args.ops[t].x) & 0xFFu) : 0u;
    const uint32_t bk = valid ? bucket_of(kind) : 8u;
    const uint32_t grp = __match_any_sync(kFull, bk);
    const uint32_t leader = __ffs(grp) - 1;
    uint32_t off = 0;
    if (lane == leader && valid) off = atomicAdd(cnt + bk, __popc(grp));
    off = __shfl_sync(kFull, off, leader);
    if (valid) p.perm[(size_t)bk * p.num_traces + off + __popc(grp & lanemask_lt())] = t;
  }
}

__global__ void __launch_bounds__(kWarpsPerCta * 32, 32)
rkc_step_kernel(const __grid_constant__ StepArgs args) {
  __shared__ Warp smem[kWarpsPerCta];
  const uint32_t lane = threadIdx.x & 31u;
  // CTA i -> the i-th trace of the op-kind bucketed order of this step
  uint32_t t;
  {
    const uint32_t* cnt = args.p.bcnt + (args.step & 1u) * 8;
    const uint32_t i = blockIdx.x;
    uint32_t acc = 0, bk = 8, off = 0;
#pragma unroll
    for (uint32_t q = 0; q < 8; ++q) {
      const uint32_t c = cnt[q];
      if (bk == 8 && i < acc + c) { bk = q; off = i - acc; }
      acc += c;
    }
    if (bk == 8) return;
    t = __ldcg(args.p.perm + (size_t)bk * args.p.num_traces + off);
  }
  const uint4 opw = __ldcs(args.ops + t);
  // hot header: lanes 0..15 hold one word each
  const uint32_t hw = lane < H_NWORDS ? __ldcg(args.p.hdr + (size_t)t * H_NWORDS + lane) : 0u;
  const uint32_t next_exp = __shfl_sync(kFull, hw, H_NEXT_EXPIRY);
  const uint32_t kind = opw.x & 0xFFu;
  // a NOP with no expiry due changes nothing (fast path)
  if (kind == OP_NOP && args.step < next_exp) return;
  Warp* w = &smem[0];
  if (lane < H_NWORDS) w->h[lane] = hw;
  w->ctr[lane] = 0;
  if (lane < 4) { w->rc[lane] = 0; w->objdirty[lane] = 0; }
  if (lane == 0) { w->nev = 0; w->flags = 0; w->cdirty = 0; }
  __syncwarp();
  Ctx x{&args.p, w, t, args.step, lane};
  Op op{kind, (opw.x >> 8) & 0xFFu, (opw.x >> 16) & 0xFFu, opw.x >> 24, opw.y, opw.z, opw.w};
  if (args.step >= next_exp) expiry(x);
  if (kind != OP_NOP) ctr_add(x, K_OPS, 1);
  switch (kind) {
    case OP_NOP: break;
    case OP_SUBMIT: op_submit(x, op); break;
    case OP_ADMIT: op_admit(x, op); break;
    case OP_ADVANCE: op_advance(x, op); break;
    case OP_COMPLETE: op_complete(x, op); break;
    case OP_INSERT: op_insert(x, op); break;
    case OP_DEMOTE: op_demote(x, op); break;
    case OP_TOUCH: op_touch(x, op); break;
    default: op_error(x, op, ERR_UNKNOWN_OP); break;
  }
  __syncwarp();
  finish(x);
}

extern std::atomic<unsigned long long> g_launches;

// host launcher: one launch = one lockstep step over all traces
cudaError_t launch_step(const PoolDev& p, const void* ops_step, uint32_t step, cudaStream_t st) {
  g_launches += 1;
  g_launches += 1;
  StepArgs args{p, reinterpret_cast<const uint4*>(ops_step), step};
  const uint32_t cgrid = (p.num_traces + 255) / 256 < 148 * 8 ? (p.num_traces + 255) / 256 : 148 * 8;
  rkc_classify_kernel<<<cgrid, 256, 0, st>>>(args);
  rkc_step_kernel<<<p.num_traces, kWarpsPerCta * 32, 0, st>>>(args);
  return cudaGetLastError();
}

}  // namespace rkc
