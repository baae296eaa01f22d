// rkc_step_impl.cuh -- K0 light pass + K1 lockstep step kernel.
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
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

#include "rkc_internal.cuh"

namespace rkc {
namespace RKC_STEP_NS {

constexpr unsigned kFull = 0xFFFFFFFFu;
#ifndef RKC_WARPS_PER_CTA
#define RKC_WARPS_PER_CTA 1
#endif
// independent warps per CTA, each its own trace (1 measured best: a CTA of
// several warps holds its slot until its slowest trace is done)
constexpr int kWarpsPerCta = RKC_WARPS_PER_CTA;
constexpr uint32_t kStageMax = 1024;  // pools up to this size stage keys in smem
// Pool-size class of this build (see rkc_step_*.cu): small pools (NS <=
// kStageMax) stage their keys in shared memory and keep the block-scan loops
// rolled (instruction cache); big pools stream their block words with
// unrolled loops (loads in flight).
#ifndef RKC_BIG
#error "compile through rkc_step_{small,big}_o{64,128}.cu"
#endif
constexpr bool kBig = RKC_BIG;
// Big pools run one CTA of kCrew warps per trace: warp 0 (the leader) runs the
// op path exactly as in the small build; its block passes are split into
// contiguous vector slices, one per warp of the crew (section "crew" below).
#ifndef RKC_CREW
#define RKC_CREW 8
#endif
constexpr uint32_t kCrew = kBig ? RKC_CREW : 1;
#ifndef RKC_CREW_UNROLL
#define RKC_CREW_UNROLL 2
#endif
constexpr int kCrewUnroll = RKC_CREW_UNROLL;  // block vectors in flight per lane in a crew pass
// Object slots held in shared memory.  This file is compiled twice
// (rkc_step_o64.cu / rkc_step_o128.cu): pools with O <= 64 run the 64-slot
// build, whose 6 KB warp state fits 32 resident CTAs per SM instead of 30.
#ifndef RKC_OMAX
#error "compile through rkc_step_o64.cu / rkc_step_o128.cu"
#endif
constexpr uint32_t kObjMax = RKC_OMAX;

#ifndef RKC_HDR_ALWAYS
#define RKC_HDR_ALWAYS 1   // round 2: c5 -0.5 %
#endif
#ifndef RKC_FINISH_VEC
#define RKC_FINISH_VEC 1   // round 2: c5 -1.4 %
#endif
#ifndef RKC_RC_REGS
#define RKC_RC_REGS 1   // round 2: c5 -1.0 %, c3 -1.6 %
#endif
#ifndef RKC_LIST_BITS
#define RKC_LIST_BITS 1   // round 2: c5 -0.8 %
#endif
#ifndef RKC_LIGHT_FA_FAST
#define RKC_LIGHT_FA_FAST 1   // round 2: c3 -0.7 %, c5 -0.3 %
#endif
#ifndef RKC_LIGHT_RANKED
#define RKC_LIGHT_RANKED 1   // free-only takes: one rank per lane instead of a bit loop per word
#endif
#ifndef RKC_LIGHT_MIN_CTAS
#define RKC_LIGHT_MIN_CTAS 10   // 48 registers: 10 light CTAs per SM
#endif
enum : uint32_t { F_CLAIMS = 1, F_OBJS = 2, F_POST = 4, F_CLAIMS_CHANGED = 8, F_HDR = 16, F_RQ = 32,
                  F_RC = 64 /* some object is marked for the reclass pass (S.rc) */ };
#ifndef RKC_RC_FLAG
#define RKC_RC_FLAG 1   // round 2: one flag test instead of four words (-0.7 % per c5 step)
#endif

struct alignas(16) Warp {      // the warp's shared memory (one warp per CTA)
  // per-trace base pointers and pool dims, set at kernel entry
  uint32_t* key;
  uint32_t* meta;
  uint32_t* fbm;
  uint32_t* clm;
  uint32_t* req;
  uint2* obj;
  uint32_t* ctrp;
  uint32_t* hdrp;
  uint4* ev;
  uint32_t t, step, nv, NS, C, Q, O, EPT;
  uint32_t h[H_NWORDS];        // hot header
  uint32_t rq[8];              // the request record of the current op
  alignas(16) uint32_t nev;    // {nev, flags, cdirty, pad0}: one 16-B load in finish()
  uint32_t flags, cdirty, pad0;
  uint32_t rc[4];              // objects whose blocks need reclassing
  alignas(16) uint32_t objdirty[4];
  uint32_t ctr[32];            // counter deltas of this step
  alignas(16) uint32_t cl[32][8];  // claim records (lane c owns claim c)
  uint32_t obj0[kObjMax];      // object word 0
  uint32_t lead[kObjMax];      // leading prefix per object
#if RKC_BIG
  uint32_t job[8];             // crew job: kind, arguments
  uint32_t red[kCrew][4];      // crew partial results, one row per warp
#endif
  union alignas(16) {
    struct { uint32_t lim3[128], lim2[128], cnt3[128]; };  // reclass scratch
    uint32_t keys[kStageMax];  // staged selection keys (alloc only)
  };
};

static_assert(offsetof(Warp, cl) % 16 == 0, "uint4 access to claim rows");
static_assert(offsetof(Warp, nev) % 16 == 0 && offsetof(Warp, flags) == offsetof(Warp, nev) + 4 &&
              offsetof(Warp, cdirty) == offsetof(Warp, nev) + 8, "one 16-B load of {nev, flags, cdirty}");
static_assert(offsetof(Warp, objdirty) % 16 == 0, "one 16-B load of objdirty");
static_assert(offsetof(Warp, keys) % 16 == 0, "uint4 access to staged keys");
__shared__ Warp S_[kWarpsPerCta];
#define S (S_[kWarpsPerCta == 1 ? 0u : (threadIdx.x >> 5)])

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// Programmatic dependent launch: one step = light pass -> step kernel ->
// overflow kernel -> next light pass, each launched with programmatic stream
// serialisation, so a kernel is launched as its predecessor's last CTAs exit
// instead of after the full kernel boundary; it waits for the predecessor's
// completion and memory (griddepcontrol.wait) before touching trace state.
// (An explicit early trigger at CTA start measured slower: the successor's
// CTAs then sit in SM slots the predecessor's tail could use.)
__device__ __forceinline__ void pdl_wait() {
#ifndef RKC_NO_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

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
__device__ __forceinline__ void hset(uint32_t i, uint32_t v) {
  __syncwarp();
  if (lane_id() == 0) { S.h[i] = v; if (!RKC_HDR_ALWAYS) S.flags |= F_HDR; }
  __syncwarp();
}
__device__ __forceinline__ void flag_set(uint32_t f) {
  if (lane_id() == 0) S.flags |= f;
  __syncwarp();
}
__device__ __forceinline__ uint32_t lowering() { return S.h[H_POLICY] & 0xFFu; }
__device__ __forceinline__ void ctr_add(uint32_t k, uint32_t v) {
  if (lane_id() == 0) S.ctr[k] += v;
}

// claim record accessors (slot c)
__device__ __forceinline__ uint32_t cl_state(uint32_t c) { return S.cl[c][0] & 0xFFu; }
__device__ __forceinline__ uint32_t cl_mode(uint32_t c) { return (S.cl[c][0] >> 8) & 0xFFu; }
__device__ __forceinline__ uint32_t cl_obj(uint32_t c) { return (S.cl[c][0] >> 16) & 0xFFu; }
enum : uint32_t { CF_W0 = 0, CF_F = 1, CF_R = 2, CF_D = 3, CF_DEC = 4, CF_PC = 5 };

// 16-B store with an L2 evict_last cache policy
__device__ __forceinline__ void st_evict_last(uint4* p, const uint4 v) {
  asm volatile(
      "{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
      "st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, pol;\n\t}" ::"l"(p),
      "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
      : "memory");
}
// ------------------------------ telemetry ----------------------------------
__device__ __forceinline__ void write_event(uint32_t idx, uint32_t type, uint32_t seq,
                                            uint32_t slot, uint32_t reason, uint32_t mask,
                                            uint32_t f0, uint32_t f1, uint32_t f2, uint32_t f3) {
  if (idx < S.EPT) {
    uint4* e = S.ev + (size_t)idx * 2;
    e[0] = make_uint4(S.t, S.step, type | (seq << 8) | ((slot & 0xFFu) << 16) | (reason << 24), mask);
    e[1] = make_uint4(f0, f1, f2, f3);
  }
}
#ifndef RKC_EMIT_INLINE
#define RKC_EMIT_INLINE 1
#endif
#if RKC_EMIT_INLINE
__device__ __forceinline__ void emit(uint32_t type, uint32_t slot, uint32_t reason,
#else
__device__ __noinline__ void emit(uint32_t type, uint32_t slot, uint32_t reason,
#endif
                                  uint32_t mask, uint32_t f0, uint32_t f1, uint32_t f2, uint32_t f3) {
  const uint32_t n = S.nev;
  if (lane_id() == 0) {
    write_event(S.h[H_EVCOUNT] + n, type, n, slot, reason, mask, f0, f1, f2, f3);
    S.nev = n + 1;
  }
  __syncwarp();
}
// one event per lane with pred, ranked by lane (= claim slot)
__device__ __forceinline__ void emit_lanes(bool pred, uint32_t type, uint32_t reason,
                                           uint32_t mask, uint32_t f0, uint32_t f1, uint32_t f2,
                                           uint32_t f3) {
  const uint32_t m = __ballot_sync(kFull, pred);
  const uint32_t n = S.nev;
  if (pred) {
    const uint32_t r = __popc(m & lanemask_lt());
    write_event(S.h[H_EVCOUNT] + n + r, type, n + r, lane_id(), reason, mask, f0, f1, f2, f3);
  }
  __syncwarp();
  if (lane_id() == 0) S.nev = n + __popc(m);
  __syncwarp();
}
__device__ __noinline__ void op_error(const Op op, uint32_t code) {
  emit(EV_OP_ERROR, op.a, code, 0, op.kind, 0, 0, 0);
  ctr_add(K_OP_ERRORS, 1);
}

// ------------------------------ lazy loads ---------------------------------
// claim and object tables: both loads are issued before either is consumed
__device__ __forceinline__ void need_tables(bool claims, bool objs) {
  claims = claims && !(S.flags & F_CLAIMS);
  objs = objs && !(S.flags & F_OBJS);
  if (!claims && !objs) return;
  const uint32_t lane = lane_id();
  uint4 c0 = make_uint4(0, 0, 0, 0), c1 = make_uint4(0, 0, 0, 0);
  uint2 ov[4] = {make_uint2(0, 0), make_uint2(0, 0), make_uint2(0, 0), make_uint2(0, 0)};
  if (claims && lane < S.C) {
    const uint4* cp = reinterpret_cast<const uint4*>(S.clm + lane * 8);
    c0 = __ldcg(cp);
    c1 = __ldcg(cp + 1);
  }
  if (objs) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t o = lane + 32 * i;
      if (o < S.O) ov[i] = __ldcg(S.obj + o);
    }
  }
  if (claims) {
    reinterpret_cast<uint4*>(S.cl[lane])[0] = c0;
    reinterpret_cast<uint4*>(S.cl[lane])[1] = c1;
  }
  if (objs) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t o = lane + 32 * i;
      if (o < S.O) { S.obj0[o] = ov[i].x; S.lead[o] = ov[i].y; }
    }
  }
  __syncwarp();
  if (lane == 0) S.flags |= (claims ? F_CLAIMS : 0u) | (objs ? F_OBJS : 0u);
  __syncwarp();
}
#ifndef RKC_NEED_INLINE_CHECK
#define RKC_NEED_INLINE_CHECK 1
#endif
#if RKC_NEED_INLINE_CHECK
// the loaded-already test inline at every call site, the loads out of line
__device__ __noinline__ void load_claims() { need_tables(true, false); }
__device__ __noinline__ void load_objs() { need_tables(false, true); }
__device__ __noinline__ void load_both() { need_tables(true, true); }
__device__ __forceinline__ void need_claims() { if (!(S.flags & F_CLAIMS)) load_claims(); }
__device__ __forceinline__ void need_objs() { if (!(S.flags & F_OBJS)) load_objs(); }
__device__ __forceinline__ void need_both() {
  const uint32_t f = S.flags & (F_CLAIMS | F_OBJS);
  if (f == (F_CLAIMS | F_OBJS)) return;
  if (f == F_CLAIMS) load_objs();
  else if (f == F_OBJS) load_claims();
  else load_both();
}
#else
__device__ __noinline__ void need_claims() { need_tables(true, false); }
__device__ __noinline__ void need_objs() { need_tables(false, true); }
__device__ __noinline__ void need_both() { need_tables(true, true); }
#endif
// pull one trace's block array into L2 ahead of a scan (one 128-B line per lane-iteration)
__device__ __forceinline__ void prefetch_blocks(const uint32_t* base) {
  for (uint32_t l = lane_id(); l < S.NS / 32; l += 32)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(base + l * 32));
}
__device__ __forceinline__ void mark_obj_dirty(uint32_t o) {
  if (lane_id() == 0) S.objdirty[o >> 5] |= 1u << (o & 31u);
  __syncwarp();
}
__device__ __forceinline__ void mark_reclass(uint32_t o) {
  if (lane_id() == 0) { S.rc[o >> 5] |= 1u << (o & 31u); if (RKC_RC_FLAG) S.flags |= F_RC; }
  __syncwarp();
}
__device__ __forceinline__ void mark_reclass_lanes(bool pred, uint32_t o) {
  if (pred) atomicOr(&S.rc[o >> 5], 1u << (o & 31u));
  if (RKC_RC_FLAG) {
    const bool any = __any_sync(kFull, pred);
    __syncwarp();
    if (any && lane_id() == 0) S.flags |= F_RC;
  }
  __syncwarp();
}
__device__ __forceinline__ bool in_reclass(uint32_t o) {
  return (S.rc[o >> 5] >> (o & 31u)) & 1u;
}
// claim lane c changed: mark it for write-back
__device__ __forceinline__ void claims_dirty(bool pred) {
  const uint32_t m = __ballot_sync(kFull, pred);
  if (lane_id() == 0) { S.cdirty |= m; if (m) S.flags |= F_CLAIMS_CHANGED; }
  __syncwarp();
}
// P (protected_resident_kv) and the blocking set from per-claim protected counts
__device__ __forceinline__ void refresh_protected() {
  const uint32_t pc = lane_id() < S.C ? S.cl[lane_id()][CF_PC] : 0u;
  const uint32_t P = __reduce_add_sync(kFull, pc);
  const uint32_t m = __ballot_sync(kFull, pc > 0);
  if (lane_id() == 0) { S.h[H_P] = P; S.h[H_BLOCKMASK] = m; if (!RKC_HDR_ALWAYS) S.flags |= F_HDR; }
  __syncwarp();
}
// class of a new cached block (o, pos) from the object's bound claim
__device__ __forceinline__ uint32_t new_block_class(uint32_t o, uint32_t pos) {
  const uint32_t c = obj_claim(S.obj0[o]);
  if (c >= 32 || !live_state(cl_state(c)) || pos >= S.cl[c][CF_F]) return 1;
  return claim_class(cl_mode(c), lowering());
}
// the live protected claim bound to object o gains `added` protected blocks
__device__ __forceinline__ void add_protected(uint32_t o, uint32_t added) {
  const uint32_t c = obj_claim(S.obj0[o]);
  if (c < 32 && live_state(cl_state(c)) && claim_class(cl_mode(c), lowering()) == 3 &&
      added > 0) {
    if (lane_id() == 0) S.cl[c][CF_PC] += added;
    __syncwarp();
    claims_dirty(lane_id() == c);
    refresh_protected();
  }
}

// ------------------------------ block passes -------------------------------
template <int U, class F>
__device__ __forceinline__ void for_vec(uint32_t nv, F&& f) {
#pragma unroll U
  for (uint32_t j = 0; j < nv; ++j) f(j);
}
// small pools: the block meta words, all loads in flight at once, into the
// staging buffer (the scans then run rolled over shared memory)
__device__ __forceinline__ const uint4* stage_meta() {
  const uint4* meta4 = reinterpret_cast<const uint4*>(S.meta);
  uint4* st = reinterpret_cast<uint4*>(S.keys);
  const uint32_t nv = S.nv, lane = lane_id();
  uint4 mv[kStageMax / 128];
#pragma unroll
  for (uint32_t j = 0; j < kStageMax / 128; ++j)
    if (j < nv) mv[j] = __ldcg(meta4 + j * 32 + lane);
#pragma unroll
  for (uint32_t j = 0; j < kStageMax / 128; ++j)
    if (j < nv) st[j * 32 + lane] = mv[j];
  __syncwarp();
  return st;
}
__device__ __forceinline__ uint32_t block_of(uint32_t j, int e) {
  return (j * 32 + lane_id()) * 4 + e;
}
__device__ __forceinline__ void fbm_set(uint32_t j, uint32_t nib) {
  if (nib) {
    const uint32_t b0 = block_of(j, 0);
    atomicOr(S.fbm + (b0 >> 5), nib << (b0 & 31u));
  }
}

// ------------------------------ crew (big pools) ----------------------------
// Warp w of the CTA owns block vectors [nv*w/kCrew, nv*(w+1)/kCrew) (block-id
// order is preserved across warps).  The leader posts a job in S.job and all
// warps run their slice between two named barriers; per-warp results land in
// S.red[w].  Helpers (warps 1..) loop on jobs until JOB_EXIT.
#if RKC_BIG
enum : uint32_t { JOB_EXIT = 0, JOB_STATS, JOB_COUNT, JOB_MIN2, JOB_APPLY, JOB_RELEASE,
                  JOB_COMPLETE, JOB_TOUCH, JOB_RECLASS, JOB_FREE_COUNT, JOB_FREE_TAKE };

__device__ __forceinline__ void crew_bar() {
  asm volatile("bar.sync 1, %0;" ::"r"(kCrew * 32) : "memory");
}
__device__ __forceinline__ uint32_t crew_j0(uint32_t w) { return S.nv * w / kCrew; }

// L2 prefetch of the line RKC_CREW_PF vectors ahead in a crew pass (one
// prefetch per 128-B line: lanes 0, 8, 16, 24); no registers held
#ifndef RKC_CREW_PF
#define RKC_CREW_PF 4   // round 2: c4 702 -> 494 us per lockstep step
#endif
__device__ __forceinline__ void crew_pf(const uint4* base, uint32_t j, uint32_t j1) {
  if (RKC_CREW_PF > 0 && (lane_id() & 7u) == 0 && j + RKC_CREW_PF < j1)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (j + RKC_CREW_PF) * 32 + lane_id()));
}
// one job's slice for warp w (lane = lane_id()); arguments in S.job[1..7]
__device__ __noinline__ void crew_work(uint32_t kind, uint32_t w) {
  const uint32_t lane = lane_id();
  const uint32_t j0 = crew_j0(w), j1 = crew_j0(w + 1);
  uint32_t* key = S.key;
  uint32_t* meta = S.meta;
  const uint4* key4 = reinterpret_cast<const uint4*>(key);
  const uint4* meta4 = reinterpret_cast<const uint4*>(meta);
  constexpr uint32_t kC1 = 1u << kClassShift;
  uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
  switch (kind) {
    case JOB_STATS: {  // class-1 count, smallest non-free key - 2^30 (see alloc_evict)
      uint32_t md = kFull;
#pragma unroll(kCrewUnroll)
      for (uint32_t j = j0; j < j1; ++j) {
        crew_pf(key4, j, j1);
        const uint4 v = __ldcg(key4 + j * 32 + lane);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t d = el(v, e) - kC1;
          r0 += d < kC1 ? 1u : 0u;
          md = min(md, d);
        }
      }
      r0 = __reduce_add_sync(kFull, r0);
      r1 = __reduce_min_sync(kFull, md);
      break;
    }
    case JOB_COUNT: {  // #{key <= T}
      const uint32_t T = S.job[1];
#pragma unroll(kCrewUnroll)
      for (uint32_t j = j0; j < j1; ++j) {
        crew_pf(key4, j, j1);
        const uint4 v = __ldcg(key4 + j * 32 + lane);
        r0 += (v.x <= T) + (v.y <= T) + (v.z <= T) + (v.w <= T);
      }
      r0 = __reduce_add_sync(kFull, r0);
      break;
    }
    case JOB_MIN2: {  // smallest class-2 key - 2^31
      constexpr uint32_t kC2 = 2u << kClassShift;
      uint32_t m2 = kFull;
#pragma unroll(kCrewUnroll)
      for (uint32_t j = j0; j < j1; ++j) {
        crew_pf(key4, j, j1);
        const uint4 v = __ldcg(key4 + j * 32 + lane);
        m2 = min(min(m2, v.x - kC2), min(v.y - kC2, min(v.z - kC2, v.w - kC2)));
      }
      r0 = __reduce_min_sync(kFull, m2);
      break;
    }
    case JOB_APPLY: {  // take {key <= T}: ranks continue from the warps before (counts at T in red[.][0])
      const uint32_t T = S.job[1], base = S.job[2], owner = S.job[3] & 0x7FFFFFFFu;
      const bool insert = S.job[3] >> 31;
      const uint32_t k = S.job[4], l3 = S.job[5], l2 = S.job[6], seq_base = S.job[7];
      uint32_t rank = 0;
      for (uint32_t v = 0; v < w; ++v) rank += S.red[v][0];
      const uint32_t end = rank + S.red[w][0];
      for (uint32_t j = j0; j < j1 && rank < end; ++j) {
        crew_pf(key4, j, j1);
        const uint4 v = __ldcg(key4 + j * 32 + lane);
        const uint32_t tb = (v.x <= T ? 1u : 0u) | (v.y <= T ? 2u : 0u) | (v.z <= T ? 4u : 0u) |
                            (v.w <= T ? 8u : 0u);
        if (!__any_sync(kFull, tb != 0)) continue;
        const uint32_t cnt = __popc(tb);
        const uint32_t Sc = warp_incl_scan(cnt, lane);
        uint32_t r = rank + Sc - cnt;
        // the vector's meta words in one 16-B load (not one dependent load per victim)
        const bool anyv = (tb & 1u && v.x >= kC1) || (tb & 2u && v.y >= kC1) || (tb & 4u && v.z >= kC1) ||
                          (tb & 8u && v.w >= kC1);
        const uint4 mvv = anyv ? __ldcg(meta4 + j * 32 + lane) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (!((tb >> e) & 1u)) continue;
          const uint32_t bb = block_of(j, e);
          const uint32_t pos = base + r++;
          if (el(v, e) >= kC1) {  // a victim: attributed by its object's claim now (Table 4)
            const uint32_t m = el(mvv, e);
            const uint32_t o = meta_owner(m);
            const uint32_t cc = obj_claim(S.obj0[o]);
            const uint32_t st = cc < 32 ? cl_state(cc) : C_EMPTY;
            if (st == C_DEMOTED || st == C_EXPIRED) ++r2;
            else if (st == C_ACCEPTED || st == C_MATERIALIZED) ++r3;
            else ++r1;
            atomicMin(&S.lead[o], meta_pos(m));
            atomicOr(&S.objdirty[o >> 5], 1u << (o & 31u));
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
        rank += __shfl_sync(kFull, Sc, 31);
      }
      for (uint32_t wi = j0 * 4 + lane; wi < j1 * 4; wi += 32) S.fbm[wi] = 0;  // every free block was taken
      r1 = __reduce_add_sync(kFull, r1);
      r2 = __reduce_add_sync(kFull, r2);
      r3 = __reduce_add_sync(kFull, r3);
      break;
    }
    case JOB_RELEASE: {  // request S.job[1]'s active blocks -> FREE
      const uint32_t rq = S.job[1];
#pragma unroll(kCrewUnroll)
      for (uint32_t j = j0; j < j1; ++j) {
        crew_pf(meta4, j, j1);
        const uint4 mv = __ldcg(meta4 + j * 32 + lane);
        uint32_t nib = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t m = el(mv, e);
          if (meta_res(m) == kResActive && meta_owner(m) == rq) nib |= 1u << e;
        }
        if (nib) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (!((nib >> e) & 1u)) continue;
            const uint32_t bb = block_of(j, e);
            meta[bb] = meta_make(kResFree, 0, 0);
            key[bb] = bb;
          }
          fbm_set(j, nib);
          r0 += __popc(nib);
        }
      }
      r0 = __reduce_add_sync(kFull, r0);
      break;
    }
    case JOB_COMPLETE: {  // request a's blocks: full ones -> CACHED(o) tail-first stamps, rest -> FREE
      const uint32_t a = S.job[1], full = S.job[2], o = S.job[3], lim3 = S.job[4], lim2 = S.job[5];
      const uint32_t seq_base = S.job[6];
#pragma unroll(kCrewUnroll)
      for (uint32_t j = j0; j < j1; ++j) {
        crew_pf(meta4, j, j1);
        const uint4 mv = __ldcg(meta4 + j * 32 + lane);
        uint32_t nib = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t m = el(mv, e);
          if (meta_res(m) != kResActive || meta_owner(m) != a) continue;
          const uint32_t bb = block_of(j, e);
          const uint32_t pos = meta_pos(m);
          if (pos < full) {
            const uint32_t cls = pos < lim3 ? 3u : (pos < lim2 ? 2u : 1u);
            key[bb] = (cls << kClassShift) | (seq_base + (full - 1 - pos));
            meta[bb] = meta_make(kResCached, o, pos);
          } else {
            key[bb] = bb;
            meta[bb] = meta_make(kResFree, 0, 0);
            nib |= 1u << e;
          }
        }
        fbm_set(j, nib);
        r0 += __popc(nib);
      }
      r0 = __reduce_add_sync(kFull, r0);
      break;
    }
    case JOB_TOUCH: {  // restamp object S.job[1]'s leading prefix [0, L) tail-first
      const uint32_t ob = S.job[1], L = S.job[2], seq_base = S.job[3];
#pragma unroll(kCrewUnroll)
      for (uint32_t j = j0; j < j1; ++j) {
        crew_pf(meta4, j, j1);
        const uint4 mv = __ldcg(meta4 + j * 32 + lane);
        // matching blocks: the key vector read back in one 16-B load
        uint32_t hit = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t m = el(mv, e);
          hit |= (meta_res(m) == kResCached && meta_owner(m) == ob && meta_pos(m) < L) ? 1u << e : 0u;
        }
        if (hit) {
          const uint4 kv = __ldcg(key4 + j * 32 + lane);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if ((hit >> e) & 1u)
              key[block_of(j, e)] = (el(kv, e) & ~kSeqMask) | (seq_base + (L - 1 - meta_pos(el(mv, e))));
        }
      }
      break;
    }
    case JOB_RECLASS: {  // class bits of the marked objects' cached blocks (S.lim3 / S.lim2 / S.cnt3)
#pragma unroll(kCrewUnroll)
      for (uint32_t j = j0; j < j1; ++j) {
        crew_pf(meta4, j, j1);
        const uint4 mv = __ldcg(meta4 + j * 32 + lane);
        bool any = false;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t m = el(mv, e);
          any |= meta_res(m) == kResCached && in_reclass(meta_owner(m));
        }
        if (!any) continue;
        const uint4 kv = __ldcg(key4 + j * 32 + lane);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t m = el(mv, e);
          if (meta_res(m) != kResCached) continue;
          const uint32_t o = meta_owner(m);
          if (!in_reclass(o)) continue;
          const uint32_t pos = meta_pos(m);
          const bool pin = meta_pinned(m);  // shared by a running hit: class 3, not protected (G29)
          const uint32_t cls = (pin || pos < S.lim3[o]) ? 3u : (pos < S.lim2[o] ? 2u : 1u);
          const uint32_t k0 = el(kv, e);
          const uint32_t k1 = (cls << kClassShift) | (k0 & kSeqMask);
          if (k1 != k0) key[block_of(j, e)] = k1;
          if (cls == 3 && !pin) atomicAdd(&S.cnt3[o], 1u);
        }
      }
      break;
    }
    case JOB_FREE_COUNT: {  // free blocks in the slice's bitmap words
      for (uint32_t wi = j0 * 4 + lane; wi < j1 * 4; wi += 32) r0 += __popc(__ldcg(S.fbm + wi));
      r0 = __reduce_add_sync(kFull, r0);
      break;
    }
    case JOB_FREE_TAKE: {  // the k lowest-id free blocks: ranks continue from the warps before
      const uint32_t k = S.job[1], owner = S.job[2] & 0x7FFFFFFFu, base = S.job[3];
      const bool insert = S.job[2] >> 31;
      const uint32_t l3 = S.job[4], l2 = S.job[5], seq_base = S.job[6];
      uint32_t acc = 0;
      for (uint32_t v = 0; v < w; ++v) acc += S.red[v][0];
      for (uint32_t w0 = j0 * 4; w0 < j1 * 4 && acc < k; w0 += 32) {
        const uint32_t wi = w0 + lane;
        const uint32_t word = wi < j1 * 4 ? __ldcg(S.fbm + wi) : 0u;
        const uint32_t c = __popc(word);
        const uint32_t Sc = warp_incl_scan(c, lane);
        const uint32_t before = acc + Sc - c;
        const uint32_t take = before >= k ? 0u : min(c, k - before);
        if (take > 0) {
          uint32_t tw = take == c ? word : word & ((1u << nth_set_bit(word, take + 1)) - 1u);
          S.fbm[wi] = word & ~tw;
          for (uint32_t r = before; tw; tw &= tw - 1, ++r) {
            const uint32_t bb = wi * 32 + __ffs(tw) - 1;
            const uint32_t pos = base + r;
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
        acc += __shfl_sync(kFull, Sc, 31);
      }
      break;
    }
    default:
      break;
  }
  if (lane == 0) { S.red[w][0] = (kind == JOB_APPLY || kind == JOB_FREE_TAKE) ? S.red[w][0] : r0; S.red[w][1] = r1; S.red[w][2] = r2; S.red[w][3] = r3; }
}

// leader: run a job (arguments already in S.job[1..]) across the crew
__device__ __noinline__ void crew_run(uint32_t kind) {
  __syncwarp();
  if (lane_id() == 0) S.job[0] = kind;
  crew_bar();  // start: the helpers read the job
  crew_work(kind, 0);
  crew_bar();  // end: every partial result is in S.red
}
__device__ __forceinline__ uint32_t crew_sum(uint32_t c) {
  uint32_t s = 0;
#pragma unroll
  for (uint32_t w = 0; w < kCrew; ++w) s += S.red[w][c];
  return s;
}
__device__ __forceinline__ uint32_t crew_min(uint32_t c) {
  uint32_t s = kFull;
#pragma unroll
  for (uint32_t w = 0; w < kCrew; ++w) s = min(s, S.red[w][c]);
  return s;
}
__device__ __forceinline__ void job_args(uint32_t a1, uint32_t a2 = 0, uint32_t a3 = 0, uint32_t a4 = 0,
                                         uint32_t a5 = 0, uint32_t a6 = 0, uint32_t a7 = 0) {
  if (lane_id() == 0) {
    S.job[1] = a1; S.job[2] = a2; S.job[3] = a3; S.job[4] = a4; S.job[5] = a5; S.job[6] = a6; S.job[7] = a7;
  }
}
__device__ __noinline__ void crew_helper() {
  const uint32_t w = threadIdx.x >> 5;
  for (;;) {
    crew_bar();
    const uint32_t kind = S.job[0];
    if (kind == JOB_EXIT) return;
    crew_work(kind, w);
    crew_bar();
  }
}
__device__ __forceinline__ void crew_exit() {
  __syncwarp();
  if (lane_id() == 0) S.job[0] = JOB_EXIT;
  crew_bar();
}
#else
__device__ __forceinline__ void crew_exit() {}
#endif

// reclass pass: rewrite the class bits of every cached block whose owner is
// marked, from the owner's bound claim; recount the protected blocks.
#ifndef RKC_RECLASS_INLINE
#define RKC_RECLASS_INLINE 0
#endif
#if RKC_RECLASS_INLINE
#define RKC_RECLASS_ATTR __forceinline__
#else
#define RKC_RECLASS_ATTR __noinline__
#endif
template <bool big>
__device__ RKC_RECLASS_ATTR void flush_reclass_pass() {
  if (!big) prefetch_blocks(S.meta);
  need_both();
  const uint32_t low = lowering();
  for (uint32_t o = lane_id(); o < S.O; o += 32) {
    uint32_t l3 = 0, l2 = 0;
    const uint32_t cc = obj_claim(S.obj0[o]);
    if (cc < 32 && live_state(cl_state(cc))) {
      const uint32_t cls = claim_class(cl_mode(cc), low);
      if (cls == 3) l3 = S.cl[cc][CF_F];
      if (cls == 2) l2 = S.cl[cc][CF_F];
    }
    S.lim3[o] = l3;
    S.lim2[o] = l2;
    S.cnt3[o] = 0;
  }
  __syncwarp();
  uint32_t* key = S.key;
  const uint4* meta4 = reinterpret_cast<const uint4*>(S.meta);
  const uint4* key4 = reinterpret_cast<const uint4*>(key);
  const uint32_t nv = S.nv;
  // one vector of block words per lane-step: rolled for staged-size pools
  // (instruction cache), unrolled for big ones (loads in flight); each
  // variant is its own function so the small-pool path stays compact
#if RKC_RC_REGS
  // the marked-object bitmap in registers (was one shared-memory load per element)
  const uint32_t rcw0 = S.rc[0], rcw1 = S.rc[1], rcw2 = S.rc[2], rcw3 = S.rc[3];
  auto in_rc = [&](uint32_t o) -> bool {
    const uint32_t w = kObjMax <= 64 ? (o < 32 ? rcw0 : rcw1)
                                     : (o < 64 ? (o < 32 ? rcw0 : rcw1) : (o < 96 ? rcw2 : rcw3));
    return (w >> (o & 31u)) & 1u;
  };
#else
  auto in_rc = [&](uint32_t o) -> bool { return in_reclass(o); };
#endif
  auto vec_pass = [&](uint32_t j) {
    const uint4 mv = __ldcg(meta4 + j * 32 + lane_id());
    bool any = false;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t m = el(mv, e);
      any |= meta_res(m) == kResCached && in_rc(meta_owner(m));
    }
    if (!any) return;
    const uint4 kv = __ldcg(key4 + j * 32 + lane_id());
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t m = el(mv, e);
      if (meta_res(m) != kResCached) continue;
      const uint32_t o = meta_owner(m);
      if (!in_rc(o)) continue;
      const uint32_t pos = meta_pos(m);
      const bool pin = meta_pinned(m);  // shared by a running hit: class 3, not protected (G29)
      const uint32_t cls = (pin || pos < S.lim3[o]) ? 3u : (pos < S.lim2[o] ? 2u : 1u);
      const uint32_t k0 = el(kv, e);
      const uint32_t k1 = (cls << kClassShift) | (k0 & kSeqMask);
      if (k1 != k0) key[block_of(j, e)] = k1;
      if (cls == 3 && !pin) atomicAdd(&S.cnt3[o], 1u);
    }
  };
#if RKC_BIG
  if constexpr (big) crew_run(JOB_RECLASS);
  else
#endif
    for_vec<big ? 4 : 1>(nv, vec_pass);
  __syncwarp();
  bool ch = false;
  if (lane_id() < S.C) {
    const uint32_t st = cl_state(lane_id()), o = cl_obj(lane_id());
    if (live_state(st) && in_reclass(o)) {
      const uint32_t np = claim_class(cl_mode(lane_id()), low) == 3 ? S.cnt3[o] : 0u;
      if (np != S.cl[lane_id()][CF_PC]) { S.cl[lane_id()][CF_PC] = np; ch = true; }
    }
  }
  __syncwarp();
  claims_dirty(ch);
  if (lane_id() < 4) S.rc[lane_id()] = 0;
  if (RKC_RC_FLAG && lane_id() == 0) S.flags &= ~F_RC;
  __syncwarp();
  refresh_protected();
}
__device__ __forceinline__ void flush_reclass() {
  if (RKC_RC_FLAG ? (S.flags & F_RC) != 0 : (S.rc[0] | S.rc[1] | S.rc[2] | S.rc[3]) != 0) {
    flush_reclass_pass<kBig>();
  }
}

// release request r's active blocks to FREE (deferral / refusal / no-admit)
template <bool big>
__device__ __noinline__ void release_blocks_t(uint32_t r) {
#if RKC_BIG
  if constexpr (big) {
    job_args(r);
    crew_run(JOB_RELEASE);
    hset(H_FREE, S.h[H_FREE] + crew_sum(0));
    return;
  }
#endif
  uint32_t* key = S.key;
  uint32_t* meta = S.meta;
  const uint4* meta4 = stage_meta();
  uint32_t freed = 0;
  const uint32_t nv = S.nv;
  // one vector of block words per lane-step: rolled for staged-size pools
  // (instruction cache), unrolled for big ones (loads in flight); each
  // variant is its own function so the small-pool path stays compact
  auto vec_pass = [&](uint32_t j) {
    const uint4 mv = meta4[j * 32 + lane_id()];
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
        const uint32_t bb = block_of(j, e);
        meta[bb] = meta_make(kResFree, 0, 0);
        key[bb] = bb;
      }
      fbm_set(j, nib);
      freed += __popc(nib);
    }
  };
  for_vec<big ? 4 : 1>(nv, vec_pass);
  freed = __reduce_add_sync(kFull, freed);
  hset(H_FREE, S.h[H_FREE] + freed);
}

__device__ __forceinline__ void release_blocks(uint32_t r) {
  release_blocks_t<kBig>(r);
}

// ------------------------------ prefix hits (NEXT f3) ----------------------
// pin_prefix(o): the longest hit on object o among running requests other
// than `self` (their records are in HBM; the op's own one is in S.rq) -- the
// refcount of block (o, p) is #{running r : target r = o, hit r > p} (G28)
__device__ __noinline__ uint32_t pin_prefix(uint32_t o, uint32_t self) {
  uint32_t h = 0;
  if (lane_id() < S.Q && lane_id() != self) {
    const uint32_t w0 = __ldcg(S.req + lane_id() * 8 + RQ_W0);
    const uint32_t hq = __ldcg(S.req + lane_id() * 8 + RQ_HIT);
    if ((w0 & 0xFFu) == R_RUNNING && ((w0 >> 16) & 0xFFu) == o) h = hq;
  }
  return __reduce_max_sync(kFull, h);
}
// pin (class 3, restamped tail-first, G30) or unpin (class from the bound
// claim's limits l3 / l2, stamp kept) the cached blocks (o, [lo, hi))
template <bool big>
__device__ __noinline__ void pin_pass_t(uint32_t o, uint32_t lo, uint32_t hi, bool pin,
                                        uint32_t seq_base, uint32_t l3, uint32_t l2) {
  uint32_t* key = S.key;
  uint32_t* meta = S.meta;
  const uint4* meta4 = reinterpret_cast<const uint4*>(meta);  // rare op: streamed, not staged
  auto vec_pass = [&](uint32_t j) {
    const uint4 mv = __ldcg(meta4 + j * 32 + lane_id());
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t m = el(mv, e);
      if (meta_res(m) != kResCached || meta_owner(m) != o) continue;
      const uint32_t pos = meta_pos(m);
      if (pos < lo || pos >= hi) continue;
      const uint32_t bb = block_of(j, e);
      if (pin) {
        meta[bb] = m | kMetaPin;
        key[bb] = (3u << kClassShift) | (seq_base + (hi - 1 - pos));
      } else {
        meta[bb] = m & ~kMetaPin;
        const uint32_t cls = pos < l3 ? 3u : (pos < l2 ? 2u : 1u);
        key[bb] = (cls << kClassShift) | (__ldcg(key + bb) & kSeqMask);
      }
    }
  };
  for_vec<big ? 4 : 1>(S.nv, vec_pass);
  __syncwarp();
}
// the live claim bound to object o: its class-3 (protected) and class-2
// (soft) footprint limits, 0 if none
__device__ __forceinline__ void class_limits(uint32_t o, uint32_t& l3, uint32_t& l2) {
  l3 = 0; l2 = 0;
  const uint32_t cc = obj_claim(S.obj0[o]);
  if (cc < 32 && live_state(cl_state(cc))) {
    const uint32_t cls = claim_class(cl_mode(cc), lowering());
    if (cls == 3) l3 = S.cl[cc][CF_F];
    if (cls == 2) l2 = S.cl[cc][CF_F];
  }
}
// the protected count of o's claim changes by d blocks (pins moved them in or out of P, G29)
// (out of line: measured better for the instruction-cache footprint of both
// the c3 and the c6 replay, profiles/r01/f3/README.md)
__device__ __noinline__ void protected_delta(uint32_t o, int32_t d) {
  if (d == 0) return;
  const uint32_t cc = obj_claim(S.obj0[o]);
  if (lane_id() == 0) S.cl[cc][CF_PC] += (uint32_t)d;
  __syncwarp();
  claims_dirty(lane_id() == cc);
  refresh_protected();
}
// request r (record in S.rq) drops its prefix-hit references: positions of
// its target past the longest remaining hit are unpinned; A shrinks by them
__device__ __noinline__ void unpin_request(uint32_t r) {
  const uint32_t h = S.rq[RQ_HIT];
  if (h == 0) return;
  const uint32_t o = (S.rq[RQ_W0] >> 16) & 0xFFu;
  const uint32_t m2 = pin_prefix(o, r);
  __syncwarp();
  if (lane_id() == 0) S.rq[RQ_HIT] = 0;
  __syncwarp();
  if (m2 >= h) return;
  need_both();
  uint32_t l3, l2;
  class_limits(o, l3, l2);
  pin_pass_t<kBig>(o, m2, h, false, 0, l3, l2);
  hset(H_ALIVE, S.h[H_ALIVE] - (h - m2));
  const uint32_t top = min(h, l3);  // unpinned positions the claim protects again
  protected_delta(o, top > m2 ? (int32_t)(top - m2) : 0);
}
// request r (record in S.rq) gives up all its KV: own blocks to FREE (A
// shrinks by them) and its prefix-hit pins (deferral, refusal, no-admit
// completion; G9, G28)
__device__ __noinline__ void drop_request_kv(uint32_t r) {
  const uint32_t live = S.rq[RQ_LIVE];
  if (live > 0) {
    release_blocks(r);
    hset(H_ALIVE, S.h[H_ALIVE] - live);
  }
  unpin_request(r);
}

// ------------------------------ arbiter ------------------------------------
// The explicit active-side action on an infeasible boundary: an insert
// refusal (G17), or the request's deferral / refusal (G9), with the capacity
// proof (P, A, U, shortfall = P + A - U) and the blocking claims.
__device__ __noinline__ bool infeasible(uint32_t why, uint32_t mask, uint32_t P, uint64_t A,
                                        uint32_t requester, uint32_t obj) {
  const uint32_t U = S.h[H_U];
  const uint32_t pol = S.h[H_POLICY];
  const uint32_t shortfall = (uint32_t)((uint64_t)P + A - U);
  const bool resident = why != WHY_CAPACITY;
  if (requester == 0xFFFFFFFFu) {
    emit(EV_INSERT_REFUSED, obj, why, mask, P, (uint32_t)A, U, shortfall);
    ctr_add(K_INSERT_REFUSED, 1);
    return false;
  }
  // request: release its live blocks, then defer or refuse (G9)
  drop_request_kv(requester);
  const uint32_t w0 = S.rq[RQ_W0];
  const uint32_t defer = w0 >> 24;
  const bool dfr = defer < ((pol >> 16) & 0xFFu);
  __syncwarp();
  if (lane_id() == 0) {
    S.rq[RQ_LIVE] = 0;
    S.rq[RQ_DONE] = 0;
    S.rq[RQ_W0] = dfr ? ((w0 & 0x00FFFF00u) | R_DEFERRED | ((defer + 1) << 24))
                       : ((w0 & 0xFFFFFF00u) | R_REFUSED);
  }
  __syncwarp();
  if (dfr) {
    emit(EV_DEFERRED, requester, why, mask, P, (uint32_t)A, U, shortfall);
    ctr_add(resident ? K_DEFERRED_PROTECTED : K_DEFERRED_CAPACITY, 1);
  } else {
    emit(EV_REFUSED, requester, why, mask, P, (uint32_t)A, U, shortfall);
    ctr_add(resident ? K_REFUSED_PROTECTED : K_REFUSED_CAPACITY, 1);
  }
  return false;
}

// Admission under the resident reserve (admit_check = RESERVE, NEXT f4, G34;
// Table 5 "Resident reserve"): reserve = F summed over the
// live obligated claims under the contract lowering (lane = claim slot);
// the request is admitted iff reserve + Alive + need <= U, else deferred or
// refused with the reserving claims as the blocking set.  No auto-demotion.
__device__ __noinline__ bool admit_reserve(uint32_t need, uint32_t requester) {
  need_claims();
  const uint32_t U = S.h[H_U];
  const bool res = lowering() == LOW_CONTRACT && lane_id() < S.C &&
                   live_state(cl_state(lane_id())) && obligated(cl_mode(lane_id()));
  const uint32_t Rv = __reduce_add_sync(kFull, res ? S.cl[lane_id()][CF_F] : 0u);
  const uint32_t mask = __ballot_sync(kFull, res);
  const uint64_t A = (uint64_t)S.h[H_ALIVE] + need;
  if ((uint64_t)Rv + A <= U) return true;
  const bool resident = A <= U && Rv > 0;
  return infeasible(resident ? WHY_RESERVE : WHY_CAPACITY, resident ? mask : 0u, Rv, A, requester, 0);
}

// Feasibility boundary protected + active <= usable; relax by
// auto-demotion (G10); else explicit refusal / deferral with
// blocking-claim attribution and the capacity proof.
// requester: request slot (record in S.rq), or 0xFFFFFFFF for INSERT of `obj`.
__device__ __noinline__ bool arbitrate_slow(uint32_t need, uint32_t requester, uint32_t obj) {
    const uint32_t U = S.h[H_U];
  const uint32_t P = S.h[H_P];
  const uint64_t A = (uint64_t)S.h[H_ALIVE] + need;
  if ((uint64_t)P + A <= U) return true;
  const uint32_t pol = S.h[H_POLICY];
  if ((pol & 0xFFu) == LOW_CONTRACT && (pol >> 24)) {
    need_claims();
    const bool lc = lane_id() < S.C;
    const uint32_t g = (lc && live_state(cl_state(lane_id())) && cl_mode(lane_id()) == M_DEMOTABLE)
                           ? S.cl[lane_id()][CF_PC] : 0u;
    const uint32_t Sg = warp_incl_scan(g, lane_id());
    const bool ok = g > 0 && (uint64_t)(P - Sg) + A <= U;
    const uint32_t mk = __ballot_sync(kFull, ok);
    if (mk) {
      const uint32_t j = __ffs(mk) - 1;
      const bool dem = g > 0 && lane_id() <= j;
      const uint32_t o = lc ? cl_obj(lane_id()) : 0u;
      emit_lanes(dem, EV_DEMOTED, 1, 0, o, g, 0, 0);
      const uint32_t nd = __popc(__ballot_sync(kFull, dem));
      mark_reclass_lanes(dem, o);
      if (dem) { S.cl[lane_id()][0] = (S.cl[lane_id()][0] & ~0xFFu) | C_DEMOTED; S.cl[lane_id()][CF_PC] = 0; }
      __syncwarp();
      claims_dirty(dem);
      refresh_protected();
      ctr_add(K_DEMOTED_AUTO, nd);
      return true;
    }
  }
  const bool resident = A <= U && P > 0;
  return infeasible(resident ? WHY_PROTECTED : WHY_CAPACITY, resident ? S.h[H_BLOCKMASK] : 0u, P, A,
                    requester, obj);
}
#ifndef RKC_ARB_FAST
#define RKC_ARB_FAST 1   // round 2: -1.2 % per c5 step
#endif
// the feasible case (P + A <= U) decided inline; everything else out of line
__device__ __forceinline__ bool arbitrate(uint32_t need, uint32_t requester, uint32_t obj) {
  if (RKC_ARB_FAST && (uint64_t)S.h[H_P] + S.h[H_ALIVE] + need <= S.h[H_U]) return true;
  return arbitrate_slow(need, requester, obj);
}

// ------------------------------ victim selection ---------------------------
#ifndef RKC_COUNT_UNROLL
#define RKC_COUNT_UNROLL 1
#endif
constexpr int kCountUnroll = RKC_COUNT_UNROLL;
__device__ __forceinline__ uint4 key_vec(uint32_t j, bool staged) {
  if (staged) return reinterpret_cast<const uint4*>(S.keys)[j * 32 + lane_id()];
  return __ldcg(reinterpret_cast<const uint4*>(S.key) + j * 32 + lane_id());
}
#ifndef RKC_COUNT_INLINE
#define RKC_COUNT_INLINE 1   // round 2: inlined into the search loop (-2 % per c5 step)
#endif
#if RKC_COUNT_INLINE
#define RKC_COUNT_ATTR __forceinline__
#else
#define RKC_COUNT_ATTR __noinline__
#endif
template <bool staged>
__device__ RKC_COUNT_ATTR uint32_t count_le(uint32_t T) {
#if RKC_BIG
  if constexpr (!staged) {
    job_args(T);
    crew_run(JOB_COUNT);
    return crew_sum(0);
  }
#endif
  uint32_t c = 0;
  const uint32_t nv = S.nv;
  // staged counting is called ~3.5 times per eviction: unrolling it costs a
  // few hundred bytes of code against the loop overhead of every probe
#pragma unroll(staged ? kCountUnroll : 4)
  for (uint32_t j = 0; j < nv; ++j) {
    const uint4 v = key_vec(j, staged);
    c += (v.x <= T) + (v.y <= T) + (v.z <= T) + (v.w <= T);
  }
  return __reduce_add_sync(kFull, c);
}

// Staged pools (round 2): the counting probe also records which of the lane's
// 32 staged keys are <= T (bit 4j + e for block (j*32 + lane)*4 + e), so the
// probe that hits the exact count hands the taken set to the apply step
// without a second pass over the keys.
#ifndef RKC_CTR_LANES
#define RKC_CTR_LANES 0
#endif
#ifndef RKC_SPREAD_FILL
#define RKC_SPREAD_FILL 0
#endif
#ifndef RKC_MASK_APPLY
#define RKC_MASK_APPLY 1
#endif
__device__ __forceinline__ uint32_t count_mask(uint32_t T, uint32_t& M) {
  const uint32_t nv = S.nv;
  uint32_t mk = 0;
#pragma unroll 1
  for (uint32_t j = 0; j < nv; ++j) {
    const uint4 v = reinterpret_cast<const uint4*>(S.keys)[j * 32 + lane_id()];
    const uint32_t nib = (v.x <= T ? 1u : 0u) | (v.y <= T ? 2u : 0u) | (v.z <= T ? 4u : 0u) |
                         (v.w <= T ? 8u : 0u);
    mk |= nib << (4 * j);
  }
  M = mk;
  return __reduce_add_sync(kFull, __popc(mk));
}

// smallest class-2 (soft) key: d2 = key - 2^31 maps class 2 to [0, 2^30) below
// every other class (rare path: class 1 cannot cover the shortfall)
template <bool staged>
__device__ __noinline__ uint32_t min_class2() {
  constexpr uint32_t kC2 = 2u << kClassShift;
#if RKC_BIG
  if constexpr (!staged) {
    crew_run(JOB_MIN2);
    return crew_min(0) + kC2;
  }
#endif
  uint32_t m2 = kFull;
  const uint32_t nv = S.nv;
#pragma unroll(staged ? 1 : 4)
  for (uint32_t j = 0; j < nv; ++j) {
    const uint4 v = key_vec(j, staged);
    m2 = min(min(m2, v.x - kC2), min(v.y - kC2, min(v.z - kC2, v.w - kC2)));
  }
  return __reduce_min_sync(kFull, m2) + kC2;
}

// Free-only allocation (k <= free count): the k lowest-id free blocks, lane =
// free-bitmap word; positions base + rank in block-id order (G24).
__device__ __noinline__ void alloc_free(uint32_t k, uint32_t owner, bool insert,
                                        uint32_t base) {
    uint32_t* fbm = S.fbm;
  uint32_t* key = S.key;
  uint32_t* meta = S.meta;
  const uint32_t nw = S.nv * 4;
  const uint32_t seq_base = S.h[H_SEQ];
  uint32_t l3 = 0, l2 = 0;
  if (insert) {  // class of the new cached blocks from the object's bound claim
    const uint32_t cc = obj_claim(S.obj0[owner]);
    if (cc < 32 && live_state(cl_state(cc))) {
      const uint32_t cls = claim_class(cl_mode(cc), lowering());
      if (cls == 3) l3 = S.cl[cc][CF_F];
      if (cls == 2) l2 = S.cl[cc][CF_F];
    }
  }
#if RKC_BIG
  crew_run(JOB_FREE_COUNT);
  job_args(k, owner | (insert ? 0x80000000u : 0u), base, l3, l2, seq_base);
  crew_run(JOB_FREE_TAKE);
  hset(H_FREE, S.h[H_FREE] - k);
  ctr_add(K_BLOCKS_ALLOCATED, k);
  ctr_add(K_ALLOCATIONS, 1);
  return;
#endif
  uint32_t acc = 0;
  for (uint32_t w0 = 0; w0 < nw && acc < k; w0 += 32) {
    const uint32_t wi = w0 + lane_id();
    const uint32_t word = wi < nw ? __ldcg(fbm + wi) : 0u;
    const uint32_t c = __popc(word);
    const uint32_t Sc = warp_incl_scan(c, lane_id());
    const uint32_t before = acc + Sc - c;
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
    acc += __shfl_sync(kFull, Sc, 31);
  }
  hset(H_FREE, S.h[H_FREE] - k);
  ctr_add(K_BLOCKS_ALLOCATED, k);
  ctr_add(K_ALLOCATIONS, 1);
}

// Evicting allocation (k > free count): every free block plus the k - free
// smallest candidate keys.  The threshold T with #{key <= T} == k is found by
// probing the counting function: first densely from the smallest key of the
// class (victims are usually the run of oldest stamps), galloping until a
// probe overshoots, then interpolation / bisection inside the bracket (keys
// are unique, so the search ends on an exact count).
#ifndef RKC_EVICT_INLINE
#define RKC_EVICT_INLINE 1   // round 2: -1.9 % per c5 step
#endif
#if RKC_EVICT_INLINE
#define RKC_EVICT_ATTR __forceinline__
#else
#define RKC_EVICT_ATTR __noinline__
#endif
template <bool staged>
__device__ RKC_EVICT_ATTR void alloc_evict(uint32_t k, uint32_t owner, bool insert, uint32_t base) {
  const uint32_t fr = S.h[H_FREE];
  const uint32_t nv = S.nv;
  const uint32_t lane = lane_id();
  const uint4* key4 = reinterpret_cast<const uint4*>(S.key);
  // one stats pass: d = key - 2^30 maps class 1 to [0, 2^30) and every free
  // key above all others, so min(d) is the smallest non-free key and
  // #{d < 2^30} the class-1 count (the class-2 minimum is needed only when
  // class 1 cannot cover the shortfall: a second pass then)
  constexpr uint32_t kC1 = 1u << kClassShift;
  uint32_t c1 = 0, md = kFull;
  auto stat = [&](const uint4& v) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t d = el(v, e) - kC1;
      c1 += d < kC1 ? 1u : 0u;
      md = min(md, d);
    }
  };
  uint4 kv[kStageMax / 128];
  if (staged) {
    // issue every key load and the claim / object table loads together
#pragma unroll
    for (uint32_t j = 0; j < kStageMax / 128; ++j)
      if (j < nv) kv[j] = __ldcg(key4 + j * 32 + lane);
    need_tables(true, true);
#pragma unroll
    for (uint32_t j = 0; j < kStageMax / 128; ++j) {
      if (j < nv) {
        reinterpret_cast<uint4*>(S.keys)[j * 32 + lane] = kv[j];
        stat(kv[j]);
      }
    }
    __syncwarp();
  } else {
    need_both();
#if RKC_BIG
    crew_run(JOB_STATS);
    c1 = lane_id() == 0 ? crew_sum(0) : 0u;  // summed over the warp below
    md = crew_min(1);
#else
    for (uint32_t j = 0; j < nv; ++j) stat(__ldcg(key4 + j * 32 + lane));
#endif
  }
  c1 = __reduce_add_sync(kFull, c1);
  uint32_t lo, clo, top;
  if (k - fr <= c1) {
    lo = __reduce_min_sync(kFull, md) + kC1 - 1; clo = fr; top = (2u << kClassShift) - 1;
  } else {  // the soft class is reached: smallest class-2 key
    lo = min_class2<staged>() - 1; clo = fr + c1; top = (3u << kClassShift) - 1;
  }
  uint32_t hi = top, chi = 0;
  bool bracket = false;
  uint32_t mult = 1;
  uint32_t T;
  // big pools: every probe is a crew pass over the whole pool, so the search
  // extrapolates the density seen so far (secant from the smallest key, 5/4
  // overshoot to bracket) and interpolates first once bracketed; the result
  // is the same set {key <= T} whatever the probe sequence (keys are unique)
  const uint32_t lo0 = lo, clo0 = clo;
  uint32_t bi = 0, last_d = 0;
  uint32_t M = 0;  // staged: this lane's taken keys at the last probe (count_mask)
#ifndef RKC_PROBE_REG
#define RKC_PROBE_REG 1   // round 2: the first probe from the staging registers
#endif
  // staged, class-1 case: the first (dense) probe counted from the key
  // registers of the staging load (no shared-memory pass)
  uint32_t pre_cm = 0xFFFFFFFFu;
  if constexpr (staged && RKC_MASK_APPLY && RKC_PROBE_REG) {
    if (k - fr <= c1) {
      const uint32_t m0 = (uint32_t)min((uint64_t)lo + (k - clo), (uint64_t)top);
      uint32_t mk = 0;
#pragma unroll
      for (uint32_t j = 0; j < kStageMax / 128; ++j) {
        if (j < nv) {
          const uint4 v = kv[j];
          mk |= ((v.x <= m0 ? 1u : 0u) | (v.y <= m0 ? 2u : 0u) | (v.z <= m0 ? 4u : 0u) |
                 (v.w <= m0 ? 8u : 0u)) << (4 * j);
        }
      }
      M = mk;
      pre_cm = __reduce_add_sync(kFull, __popc(mk));
    }
  }
  for (uint32_t it = 0;; ++it) {
    uint32_t m;
    if (!bracket) {
      if (!staged && it > 0 && clo > clo0) {
        // secant step, but never less than twice the last step (no creeping)
        // fp32 estimate (the probe position only steers the search; the
        // taken set {key <= T} is the same for any probe sequence)
        const float df = fminf((float)(k - clo) * (float)(lo - lo0) * 1.25f / (float)(clo - clo0), 4.0e9f);
        uint64_t d = (uint64_t)__float2uint_rz(df) + 1;
        d = max(d, 2 * (uint64_t)last_d);
        last_d = (uint32_t)min(d, (uint64_t)0xFFFFFFFFu);
        m = (uint32_t)min((uint64_t)lo + d, (uint64_t)top);
      } else {
        const uint64_t d = (uint64_t)(k - clo) * mult;
        m = (uint32_t)min((uint64_t)lo + d, (uint64_t)top);
        mult = mult < (1u << 20) ? mult * 4 : mult;
        last_d = (uint32_t)min(d, (uint64_t)0xFFFFFFFFu);
      }
    } else {
      const uint32_t span = hi - lo;
      const bool interp = staged ? (it & 1u) != 0 : (bi++ & 1u) == 0;
      m = interp ? lo + __float2uint_rz(fminf((float)(k - clo) * (float)span / (float)(chi - clo), (float)span))
                 : lo + span / 2;
      m = max(m, lo + 1);
      m = min(m, hi - 1);
    }
    const uint32_t cm = (staged && RKC_MASK_APPLY)
                            ? ((it == 0 && pre_cm != 0xFFFFFFFFu) ? pre_cm : count_mask(m, M))
                            : count_le<staged>(m);
    if (cm == k) { T = m; break; }
    if (cm < k) { lo = m; clo = cm; }
    else { hi = m; chi = cm; bracket = true; }
  }
  // apply: taken = {key <= T}.  Pass 1 compacts the taken blocks in block-id
  // order into a shared list (in place over the staged keys: entry i is
  // written only after vectors holding keys >= i were read); pass 2 gives
  // them positions base + i, one block per lane.  Victims are attributed by
  // their object's claim state now (Table 4); leading prefixes shrink.
  uint32_t* key = S.key;
  uint32_t* meta = S.meta;
  uint32_t* list = S.keys;
  const uint32_t seq_base = S.h[H_SEQ];
  uint32_t l3 = 0, l2 = 0;
  if (insert) {
    const uint32_t cc = obj_claim(S.obj0[owner]);
    if (cc < 32 && live_state(cl_state(cc))) {
      const uint32_t cls = claim_class(cl_mode(cc), lowering());
      if (cls == 3) l3 = S.cl[cc][CF_F];
      if (cls == 2) l2 = S.cl[cc][CF_F];
    }
  }
  uint32_t ord = 0, rel = 0, clm = 0;
#if RKC_BIG
  if constexpr (!staged) {  // each crew warp takes its slice's keys <= T (ranks from the last count)
    job_args(T, base, owner | (insert ? 0x80000000u : 0u), k, l3, l2, seq_base);
    crew_run(JOB_APPLY);
    if (lane_id() == 0) { ord = crew_sum(1); rel = crew_sum(2); clm = crew_sum(3); }
  } else
#endif
  if constexpr (staged && RKC_MASK_APPLY) {
    // ranks in block-id order (G24): vector j, then lane, then element.  Per
    // vector, the lanes' taken counts (<= 4 each, <= 128 per vector) are
    // scanned as bytes of two words (even / odd vectors) in one warp scan.
    const uint32_t lane = lane_id();
    uint32_t x = M - ((M >> 1) & 0x55555555u);
    x = (x & 0x33333333u) + ((x >> 2) & 0x33333333u);  // nibble j: taken keys of vector j
    const uint32_t A = x & 0x0F0F0F0Fu, B = (x >> 4) & 0x0F0F0F0Fu;
    uint32_t Ai = A, Bi = B;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t ua = __shfl_up_sync(kFull, Ai, d), ub = __shfl_up_sync(kFull, Bi, d);
      if (lane >= (uint32_t)d) { Ai += ua; Bi += ub; }
    }
    const uint32_t At = __shfl_sync(kFull, Ai, 31), Bt = __shfl_sync(kFull, Bi, 31);
    const uint32_t Ae = Ai - A, Be = Bi - B;
    // the taken blocks' meta lines, pulled into L2 now: the list build below
    // covers the HBM part of the victims' meta gather latency
#pragma unroll 1
    for (uint32_t j = 0; j < nv; ++j)
      if ((M >> (4 * j)) & 15u)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const uint4*>(meta) + j * 32 + lane));
    __syncwarp();  // every lane's last probe has read the staged keys the list overwrites
#if RKC_LIST_BITS
    // one iteration per taken key of this lane (not per vector): the rank
    // base of vector j is the byte sum of the totals of vectors < j (dp4a)
#pragma unroll 1
    for (uint32_t mm = M; mm; mm &= mm - 1) {
      const uint32_t bit = __ffs(mm) - 1, j = bit >> 2, e = bit & 3u;
      const uint32_t na = (j + 1) >> 1, nb = j >> 1;  // even / odd vectors below j
      const uint32_t ma = na >= 4 ? 0xFFFFFFFFu : (1u << (8 * na)) - 1u;
      const uint32_t mb = nb >= 4 ? 0xFFFFFFFFu : (1u << (8 * nb)) - 1u;
      const uint32_t vbj = (uint32_t)__dp4a(At & ma, 0x01010101u, 0u) + (uint32_t)__dp4a(Bt & mb, 0x01010101u, 0u);
      const uint32_t ex = (((j & 1u) ? Be : Ae) >> (8 * (j >> 1))) & 0xFFu;
      const uint32_t within = __popc((M >> (4 * j)) & ((1u << e) - 1u));
      list[vbj + ex + within] = block_of(j, e);
    }
#else
    uint32_t vb = 0;
#pragma unroll 1
    for (uint32_t j = 0; j < nv; ++j) {
      const uint32_t sh = 8 * (j >> 1);
      uint32_t nib = (M >> (4 * j)) & 15u;
      uint32_t r = vb + ((((j & 1u) ? Be : Ae) >> sh) & 0xFFu);
      while (nib) {
        list[r++] = block_of(j, __ffs(nib) - 1);
        nib &= nib - 1;
      }
      vb += (((j & 1u) ? Bt : At) >> sh) & 0xFFu;
    }
#endif
    __syncwarp();
    // one taken block per lane: FREE ones (meta residency FREE) are just
    // taken; cached ones are victims, attributed by their object's claim
#pragma unroll 1
    for (uint32_t i = lane; i < k; i += 32) {
      const uint32_t bb = list[i];
      const uint32_t pos = base + i;
      const uint32_t m = __ldcg(meta + bb);
      if (meta_res(m) == kResCached) {
        const uint32_t o = meta_owner(m);
        const uint32_t cc = obj_claim(S.obj0[o]);
        const uint32_t st = cc < 32 ? cl_state(cc) : C_EMPTY;
        if (st == C_DEMOTED || st == C_EXPIRED) ++rel;
        else if (st == C_ACCEPTED || st == C_MATERIALIZED) ++clm;
        else ++ord;
        atomicMin(&S.lead[o], meta_pos(m));
        atomicOr(&S.objdirty[o >> 5], 1u << (o & 31u));
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
    if (lane < nv * 4) S.fbm[lane] = 0;  // every free block was taken
  } else {
    uint32_t listed = 0, done_pos = 0;
    auto drain = [&](uint32_t n) {
#pragma unroll 1
      for (uint32_t i = lane_id(); i < n; i += 32) {
        const uint32_t e = list[i];
        const uint32_t bb = e & 0x7FFFFFFFu;
        const uint32_t rank = done_pos + i;
        const uint32_t pos = base + rank;
        if (e >> 31) {
          const uint32_t m = __ldcg(meta + bb);
          const uint32_t o = meta_owner(m);
          const uint32_t cc = obj_claim(S.obj0[o]);
          const uint32_t st = cc < 32 ? cl_state(cc) : C_EMPTY;
          if (st == C_DEMOTED || st == C_EXPIRED) ++rel;
          else if (st == C_ACCEPTED || st == C_MATERIALIZED) ++clm;
          else ++ord;
          atomicMin(&S.lead[o], meta_pos(m));
          atomicOr(&S.objdirty[o >> 5], 1u << (o & 31u));
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
#pragma unroll(staged ? 1 : 4)
    for (uint32_t j = 0; j < nv && done_pos + listed < k; ++j) {
      const uint4 v = key_vec(j, staged);
      const uint32_t tb = (v.x <= T ? 1u : 0u) | (v.y <= T ? 2u : 0u) | (v.z <= T ? 4u : 0u) |
                          (v.w <= T ? 8u : 0u);
      if (!__any_sync(kFull, tb != 0)) continue;
      const uint32_t cnt = __popc(tb);
      const uint32_t Sc = warp_incl_scan(cnt, lane_id());
      const uint32_t tot = __shfl_sync(kFull, Sc, 31);
      if (!staged && listed + tot > kStageMax) { drain(listed); listed = 0; }
      uint32_t r = listed + Sc - cnt;
      if (tb & 1u) list[r++] = block_of(j, 0) | (v.x >= (1u << kClassShift) ? 0x80000000u : 0u);
      if (tb & 2u) list[r++] = block_of(j, 1) | (v.y >= (1u << kClassShift) ? 0x80000000u : 0u);
      if (tb & 4u) list[r++] = block_of(j, 2) | (v.z >= (1u << kClassShift) ? 0x80000000u : 0u);
      if (tb & 8u) list[r++] = block_of(j, 3) | (v.w >= (1u << kClassShift) ? 0x80000000u : 0u);
      listed += tot;
      __syncwarp();
    }
    drain(listed);
    // every free block was taken (staged pools have at most 32 bitmap words:
    // one store per lane)
    {
      uint32_t* fb = S.fbm;
      if (staged) {
        if (lane_id() < nv * 4) fb[lane_id()] = 0;
      } else {
        for (uint32_t wi = lane_id(); wi < nv * 4; wi += 32) fb[wi] = 0;
      }
    }
  }
  ord = __reduce_add_sync(kFull, ord);
  rel = __reduce_add_sync(kFull, rel);
  clm = __reduce_add_sync(kFull, clm);
  hset(H_FREE, 0);
#if RKC_CTR_LANES
  {  // the five counters of an evicting allocation, one lane per counter word
    const uint32_t l = lane_id();
    const uint32_t add = l == K_VICTIMS_ORDINARY ? ord : l == K_VICTIMS_AFTER_RELEASE ? rel :
                         l == K_VICTIMS_CLAIMED ? clm : l == K_BLOCKS_ALLOCATED ? k :
                         l == K_ALLOCATIONS ? 1u : 0u;
    S.ctr[l] += add;
    __syncwarp();
  }
#else
  ctr_add(K_VICTIMS_ORDINARY, ord);
  ctr_add(K_VICTIMS_AFTER_RELEASE, rel);
  ctr_add(K_VICTIMS_CLAIMED, clm);
  ctr_add(K_BLOCKS_ALLOCATED, k);
  ctr_add(K_ALLOCATIONS, 1);
#endif
  if (ord + rel + clm > 0) {
    emit(EV_VICTIMS, owner, insert ? 1u : 0u, 0, ord, rel, clm, k);
    flag_set(F_POST);
  }
}

// alloc(k): take the k smallest (class, key) candidates.
// insert: blocks become CACHED(obj owner) with tail-first stamps, else
// ACTIVE(request owner).
#ifndef RKC_ALLOC_INLINE
#define RKC_ALLOC_INLINE 1   // round 2: -0.6 % per c5 step
#endif
#if RKC_ALLOC_INLINE
__device__ __forceinline__ void alloc(uint32_t k, uint32_t owner, bool insert,
#else
__device__ __noinline__ void alloc(uint32_t k, uint32_t owner, bool insert,
#endif
                                   uint32_t base) {
  flush_reclass();
  if (insert) need_both();
  if (k <= S.h[H_FREE]) alloc_free(k, owner, insert, base);
  else alloc_evict<!kBig>(k, owner, insert, base);
}

// ------------------------------ request io ---------------------------------
__device__ __forceinline__ void load_request(uint32_t r) {
  if (S.flags & F_RQ) return;  // prefetched by the kernel prologue (r == op.a)
  if (lane_id() < 8) S.rq[lane_id()] = __ldcg(S.req + r * 8 + lane_id());
  __syncwarp();
}
__device__ __forceinline__ void store_request(uint32_t r) {
  if (lane_id() < 8) S.req[r * 8 + lane_id()] = S.rq[lane_id()];
}
__device__ __forceinline__ uint32_t peak_blocks() {
  return (uint32_t)(((uint64_t)S.rq[RQ_PROMPT] + S.rq[RQ_DECODE] + kBlockTokens - 1) / kBlockTokens);
}

#ifndef RKC_OPS_INLINE
#define RKC_OPS_INLINE 0
#endif
#if RKC_OPS_INLINE
#define RKC_OP_ATTR __forceinline__
#else
#define RKC_OP_ATTR __noinline__
#endif
#ifndef RKC_POST_INLINE
#define RKC_POST_INLINE 1   // round 2: -0.8 % per c5 step
#endif
#if RKC_POST_INLINE
#define RKC_POST_ATTR __forceinline__
#else
#define RKC_POST_ATTR __noinline__
#endif
// ------------------------------ ops ----------------------------------------
// SUBMIT: claim decision (Table 2).
__device__ RKC_OP_ATTR void op_submit(const Op op) {
    const uint32_t mode = op.c & 0x7Fu;
  const bool mismatch = (op.c & 0x80u) != 0;
  if (op.a >= S.C || op.b >= S.O || mode > M_BEST_EFFORT) return op_error(op, ERR_INVALID_ARG);
  need_claims();
  if (cl_state(op.a) != C_EMPTY) return op_error(op, ERR_DUPLICATE_SLOT);
  if (op.x < 1 || op.y < 1 || op.y > op.x || (mode == M_EXPIRING && op.z == 0))
    return op_error(op, ERR_INVALID_ARG);
  need_objs();
  const uint32_t ow = S.obj0[op.b];
  const uint32_t oc = obj_claim(ow);
  const bool bound_live = oc < 32 && live_state(cl_state(oc));
  const uint32_t U = S.h[H_U];
  uint32_t rej = 0;
  if (mismatch) rej = REJ_IDENTITY;
  else if (bound_live) rej = REJ_OBJECT_CLAIMED;
  else if (op.x > U) rej = REJ_FOOTPRINT;
  else if ((S.h[H_ACCEPT] & 0xFFu) == ACCEPT_RESERVE && obligated(mode)) {
    const bool lc = lane_id() < S.C && live_state(cl_state(lane_id())) && obligated(cl_mode(lane_id()));
    const uint32_t sum = __reduce_add_sync(kFull, lc ? S.cl[lane_id()][CF_F] : 0u);
    if ((uint64_t)op.x + sum > U) rej = REJ_RESERVE;
  }
  __syncwarp();  // every lane has read the claim table (write-after-read in the warp)
  if (lane_id() == op.a) {
    uint32_t* r = S.cl[op.a];
    r[0] = (rej ? C_REFUSED : C_ACCEPTED) | (mode << 8) | (op.b << 16);
    r[CF_F] = op.x; r[CF_R] = op.y; r[CF_D] = op.z; r[CF_DEC] = S.step; r[CF_PC] = 0;
  }
  __syncwarp();
  claims_dirty(lane_id() == op.a);
  if (rej) {
    emit(EV_REJECTED, op.a, rej, 0, op.b, op.x, op.y, op.z);
    ctr_add(K_REJECTED, 1);
    return;
  }
  emit(EV_ACCEPTED, op.a, 0, 0, op.b, op.x, op.y, op.z);
  ctr_add(K_ACCEPTED, 1);
  if (lane_id() == 0) S.obj0[op.b] = obj_make(obj_live(ow), op.a, obj_len(ow));
  __syncwarp();
  mark_obj_dirty(op.b);
  if (obj_live(ow) && claim_class(mode, lowering()) != 1) mark_reclass(op.b);
  flag_set(F_POST);
}

__device__ RKC_OP_ATTR void op_admit(const Op op) {
    if (op.a >= S.Q || op.b >= S.O || op.c > 1) return op_error(op, ERR_INVALID_ARG);
  load_request(op.a);
  const uint32_t st = S.rq[RQ_W0] & 0xFFu;
  if (st == R_RUNNING || st == R_DEFERRED) return op_error(op, ERR_DUPLICATE_SLOT);
  if (op.x < 1 || op.y < 1 || op.x > kMaxTokens || op.z > kMaxTokens) return op_error(op, ERR_INVALID_ARG);
  __syncwarp();  // every lane has read the request status (write-after-read in the warp)
  if (lane_id() == 0) {
    S.rq[RQ_W0] = R_RUNNING | (op.c << 8) | (op.b << 16);
    S.rq[RQ_PROMPT] = op.x; S.rq[RQ_CHUNK] = op.y; S.rq[RQ_DECODE] = op.z;
    S.rq[RQ_DONE] = 0; S.rq[RQ_LIVE] = 0; S.rq[RQ_HIT] = 0;
  }
  __syncwarp();
  ctr_add(K_ADMITTED, 1);
  const uint32_t chk = (S.h[H_POLICY] >> 8) & 0xFFu;
  if (chk == ADMIT_PEAK) arbitrate(peak_blocks(), op.a, 0);
  else if (chk == ADMIT_RESERVE) admit_reserve(peak_blocks(), op.a);
  store_request(op.a);
}

// HIT_ADMIT (NEXT f3, G28-G30): admission through a prefix hit on
// object b -- the surviving leading prefix, capped so
// one prompt token is computed, is shared and pinned instead of allocated;
// the PEAK check asks for the exclusive peak plus the newly pinned blocks
// that were candidates (pinned blocks are active live KV, counted once).
__device__ RKC_OP_ATTR void op_hit_admit(const Op op) {
  if (op.a >= S.Q || op.b >= S.O || op.c != 0) return op_error(op, ERR_INVALID_ARG);
  load_request(op.a);
  const uint32_t st = S.rq[RQ_W0] & 0xFFu;
  if (st == R_RUNNING || st == R_DEFERRED) return op_error(op, ERR_DUPLICATE_SLOT);
  if (op.x < 1 || op.y < 1 || op.x > kMaxTokens || op.z > kMaxTokens) return op_error(op, ERR_INVALID_ARG);
  need_both();
  const uint32_t o = op.b;
  const uint32_t ow = S.obj0[o];
  const uint32_t L = obj_live(ow) ? S.lead[o] : 0u;
  const uint32_t h = min(L, (op.x - 1) / kBlockTokens);
  if ((uint64_t)S.h[H_SEQ] + h > kSeqLimit) return op_error(op, ERR_SEQ_EXHAUSTED);
  __syncwarp();  // write-after-read in the warp
  if (lane_id() == 0) {
    S.rq[RQ_W0] = R_RUNNING | (o << 16);
    S.rq[RQ_PROMPT] = op.x; S.rq[RQ_CHUNK] = op.y; S.rq[RQ_DECODE] = op.z;
    S.rq[RQ_DONE] = 0; S.rq[RQ_LIVE] = 0; S.rq[RQ_HIT] = 0;
  }
  __syncwarp();
  ctr_add(K_ADMITTED, 1);
  const uint32_t m = h > 0 ? pin_prefix(o, op.a) : 0u;
  const uint32_t newpin = h > m ? h - m : 0u;
  if (((S.h[H_POLICY] >> 8) & 0xFFu) == ADMIT_PEAK) {
    uint32_t l3, l2;
    class_limits(o, l3, l2);
    const uint32_t top = min(h, l3);
    const uint32_t newprot = top > m ? top - m : 0u;
    if (!arbitrate(peak_blocks() - h + newpin - newprot, op.a, 0)) {
      store_request(op.a);
      return;
    }
  } else if (((S.h[H_POLICY] >> 8) & 0xFFu) == ADMIT_RESERVE) {
    if (!admit_reserve(peak_blocks() - h, op.a)) {  // f4: the exclusive part of the peak (G34)
      store_request(op.a);
      return;
    }
  }
  if (h > 0) {
    const uint32_t seq_base = S.h[H_SEQ];
    pin_pass_t<kBig>(o, 0, h, true, seq_base, 0, 0);
    hset(H_SEQ, seq_base + h);
    hset(H_ALIVE, S.h[H_ALIVE] + newpin);
    // the claim's protected count loses the newly pinned positions (the
    // arbitration above may have demoted it: limits are read again)
    uint32_t l3, l2;
    class_limits(o, l3, l2);
    const uint32_t top = min(h, l3);
    protected_delta(o, top > m ? -(int32_t)(top - m) : 0);
  }
  if (lane_id() == 0) { S.rq[RQ_HIT] = h; S.rq[RQ_DONE] = h * kBlockTokens; }
  __syncwarp();
  emit(EV_PREFIX_HIT, op.a, 0, 0, o, h, h * kBlockTokens, L);
  ctr_add(K_PREFIX_HITS, 1);
  ctr_add(K_HIT_TOKENS, h * kBlockTokens);
  store_request(op.a);
}

// ADVANCE: one prefill chunk or one decode token (G14); live KV
// accumulates as ceil(done/16) (Table 8).
#ifndef RKC_ADVANCE_INLINE
#define RKC_ADVANCE_INLINE 1   // round 2: -1.4 % per c5 step
#endif
#if RKC_ADVANCE_INLINE
__device__ __forceinline__ void op_advance(const Op op) {
#else
__device__ __noinline__ void op_advance(const Op op) {
#endif
    if (op.a >= S.Q) return op_error(op, ERR_INVALID_ARG);
  load_request(op.a);
  const uint32_t st = S.rq[RQ_W0] & 0xFFu;
  if (st != R_RUNNING && st != R_DEFERRED) return op_error(op, ERR_UNKNOWN_REQUEST);
  if (st == R_RUNNING && (uint64_t)S.rq[RQ_DONE] >= (uint64_t)S.rq[RQ_PROMPT] + S.rq[RQ_DECODE])
    return op_error(op, ERR_NO_CHUNKS);
  if (st == R_DEFERRED) {
    const uint32_t chk = (S.h[H_POLICY] >> 8) & 0xFFu;
    if ((chk == ADMIT_PEAK && !arbitrate(peak_blocks(), op.a, 0)) ||
        (chk == ADMIT_RESERVE && !admit_reserve(peak_blocks(), op.a))) {
      store_request(op.a);
      return;
    }
    __syncwarp();  // write-after-read in the warp
    if (lane_id() == 0) S.rq[RQ_W0] = (S.rq[RQ_W0] & ~0xFFu) | R_RUNNING;
    __syncwarp();
  }
  const uint32_t done = S.rq[RQ_DONE], prompt = S.rq[RQ_PROMPT], live = S.rq[RQ_LIVE];
  const uint32_t n = done < prompt ? min(S.rq[RQ_CHUNK], prompt - done) : 1u;
  const uint32_t need_total = (uint32_t)(((uint64_t)done + n + kBlockTokens - 1) / kBlockTokens);
  const uint32_t held = live + S.rq[RQ_HIT];  // own blocks + shared hit prefix (f3)
  const uint32_t need = need_total > held ? need_total - held : 0u;
  if (need > 0) {
    if (!arbitrate(need, op.a, 0)) { store_request(op.a); return; }
    alloc(need, op.a, false, live);
    if (lane_id() == 0) S.rq[RQ_LIVE] = live + need;
    hset(H_ALIVE, S.h[H_ALIVE] + need);
  }
  __syncwarp();  // write-after-read in the warp (no block needed: no sync since the reads)
  if (lane_id() == 0) S.rq[RQ_DONE] = done + n;
  __syncwarp();
  store_request(op.a);
}

// COMPLETE: future reusable admission is separate from active allocation
// (Table 7); only full blocks become reusable (G16).
template <bool big>
#ifndef RKC_COMPLETE_INLINE
#define RKC_COMPLETE_INLINE 0
#endif
#if RKC_COMPLETE_INLINE
__device__ __forceinline__ void op_complete(const Op op) {
#else
__device__ RKC_OP_ATTR void op_complete(const Op op) {
#endif
    if (op.a >= S.Q) return op_error(op, ERR_INVALID_ARG);
  load_request(op.a);
  if ((S.rq[RQ_W0] & 0xFFu) != R_RUNNING) return op_error(op, ERR_UNKNOWN_REQUEST);
  need_objs();
  const uint32_t done = S.rq[RQ_DONE];
  const uint32_t full = done / kBlockTokens;
  const uint32_t o = (S.rq[RQ_W0] >> 16) & 0xFFu;
  const uint32_t wa = (S.rq[RQ_W0] >> 8) & 0xFFu;
  const uint32_t ow = S.obj0[o];
  const bool admitted = wa && !obj_live(ow);
  if (admitted && (uint64_t)S.h[H_SEQ] + full > kSeqLimit) return op_error(op, ERR_SEQ_EXHAUSTED);
  const uint32_t held = S.rq[RQ_LIVE];
  if (admitted) {
    if (obj_claim(ow) < 32) need_claims();
    uint32_t cls_lim3 = 0, cls_lim2 = 0;
    {
      const uint32_t cc = obj_claim(ow);
      if (cc < 32 && live_state(cl_state(cc))) {
        const uint32_t cls = claim_class(cl_mode(cc), lowering());
        if (cls == 3) cls_lim3 = S.cl[cc][CF_F];
        if (cls == 2) cls_lim2 = S.cl[cc][CF_F];
      }
    }
    const uint32_t seq_base = S.h[H_SEQ];
    uint32_t* key = S.key;
    uint32_t* meta = S.meta;
    uint32_t freed = 0;
    const uint32_t nv = held > 0 ? S.nv : 0u;
    const uint4* meta4 = (big || nv == 0) ? reinterpret_cast<const uint4*>(meta) : stage_meta();
    // small pools: one staged vector of block words per lane-step, rolled
    // (instruction cache); big pools run the crew job below
    auto vec_pass = [&](uint32_t j) {
      const uint4 mv = meta4[j * 32 + lane_id()];
      uint32_t nib = 0;
      for (int e = 0; e < 4; ++e) {
        const uint32_t m = el(mv, e);
        if (meta_res(m) != kResActive || meta_owner(m) != op.a) continue;
        const uint32_t bb = block_of(j, e);
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
      fbm_set(j, nib);
      freed += __popc(nib);
    };
#if RKC_BIG
    if constexpr (big) {
      if (nv) {
        job_args(op.a, full, o, cls_lim3, cls_lim2, seq_base);
        crew_run(JOB_COMPLETE);
        freed = lane_id() == 0 ? crew_sum(0) : 0u;
      }
    } else
#endif
      for_vec<big ? 4 : 1>(nv, vec_pass);
    freed = __reduce_add_sync(kFull, freed);
    hset(H_FREE, S.h[H_FREE] + freed);
    hset(H_SEQ, seq_base + full);
    if (lane_id() == 0) { S.obj0[o] = obj_make(1, obj_claim(ow), full); S.lead[o] = full; }
    __syncwarp();
    mark_obj_dirty(o);
    add_protected(o, min(cls_lim3, full));
    ctr_add(K_BLOCKS_CACHED, full);
    flag_set(F_POST);
    hset(H_ALIVE, S.h[H_ALIVE] - held);
  } else {
    drop_request_kv(op.a);
    emit(EV_WRITE_DENIED, op.a, wa ? 1u : 0u, 0, o, held, 0, 0);
    ctr_add(K_WRITE_DENIED, 1);
  }
  emit(EV_SERVED, op.a, admitted ? 1u : 0u, 0, done, admitted ? full : 0u, o, 0);
  ctr_add(K_SERVED, 1);
  if (lane_id() == 0) { S.rq[RQ_W0] = (S.rq[RQ_W0] & ~0xFFu) | R_COMPLETED; S.rq[RQ_LIVE] = 0; }
  __syncwarp();
  store_request(op.a);
}

// INSERT: resident insertion through the ordinary allocation path (G17).
__device__ RKC_OP_ATTR void op_insert(const Op op) {
    if (op.a >= S.O) return op_error(op, ERR_INVALID_ARG);
  need_objs();
  const uint32_t ow = S.obj0[op.a];
  if (obj_live(ow)) return op_error(op, ERR_OBJECT_IN_USE);
  if (op.x < 1 || op.x > kMaxTokens) return op_error(op, ERR_INVALID_ARG);
  if ((uint64_t)S.h[H_SEQ] + op.x > kSeqLimit) return op_error(op, ERR_SEQ_EXHAUSTED);
  if (!arbitrate(op.x, 0xFFFFFFFFu, op.a)) return;
  alloc(op.x, op.a, true, 0);
  hset(H_SEQ, S.h[H_SEQ] + op.x);
  if (lane_id() == 0) { S.obj0[op.a] = obj_make(1, obj_claim(ow), op.x); S.lead[op.a] = op.x; }
  __syncwarp();
  mark_obj_dirty(op.a);
  {
    const uint32_t cc = obj_claim(ow);
    if (cc < 32) add_protected(op.a, min(S.cl[cc][CF_F], op.x));
  }
  ctr_add(K_INSERTED, 1);
  ctr_add(K_BLOCKS_CACHED, op.x);
  flag_set(F_POST);
}

// DEMOTE: claim_demoted before post-release block loss (Table 4).
__device__ RKC_OP_ATTR void op_demote(const Op op) {
    if (op.a >= S.C) return op_error(op, ERR_INVALID_ARG);
  need_claims();
  const uint32_t st = cl_state(op.a);
  if (st == C_EMPTY) return op_error(op, ERR_UNKNOWN_CLAIM);
  if (!live_state(st)) return op_error(op, ERR_ILLEGAL_TRANSITION);
  const uint32_t o = cl_obj(op.a), pc = S.cl[op.a][CF_PC], mode = cl_mode(op.a);
  __syncwarp();  // write-after-read in the warp
  if (lane_id() == 0) { S.cl[op.a][0] = (S.cl[op.a][0] & ~0xFFu) | C_DEMOTED; S.cl[op.a][CF_PC] = 0; }
  __syncwarp();
  claims_dirty(lane_id() == op.a);
  emit(EV_DEMOTED, op.a, 0, 0, o, pc, 0, 0);
  ctr_add(K_DEMOTED_EXPLICIT, 1);
  if (claim_class(mode, lowering()) != 1) mark_reclass(o);
  refresh_protected();
}

// TOUCH: reuse probe of the materialization surface;
// restamps the leading prefix tail-first (G23).
template <bool big>
#ifndef RKC_TOUCH_INLINE
#define RKC_TOUCH_INLINE 0
#endif
#if RKC_TOUCH_INLINE
__device__ __forceinline__ void op_touch(const Op op) {
#else
__device__ RKC_OP_ATTR void op_touch(const Op op) {
#endif
    if (op.a >= S.O) return op_error(op, ERR_INVALID_ARG);
  need_objs();
  const uint32_t ow = S.obj0[op.a];
  const uint32_t L = obj_live(ow) ? S.lead[op.a] : 0u;
  if ((uint64_t)S.h[H_SEQ] + L > kSeqLimit) return op_error(op, ERR_SEQ_EXHAUSTED);
  const uint32_t seq_base = S.h[H_SEQ];
  if (L > 0) {
    uint32_t* key = S.key;
    const uint32_t nv = S.nv;
    const uint4* meta4 = big ? reinterpret_cast<const uint4*>(S.meta) : stage_meta();
    // the class bits of the restamped blocks follow from the object's bound
    // claim (the invariant the reclass pass maintains; a pending reclass of
    // this object rewrites them to the same value), so no key is read back
    uint32_t l3 = 0, l2 = 0;
    if (!big) {
      const uint32_t cc = obj_claim(ow);
      if (cc < 32) need_claims();
      if (cc < 32 && live_state(cl_state(cc))) {
        const uint32_t cls = claim_class(cl_mode(cc), lowering());
        if (cls == 3) l3 = S.cl[cc][CF_F];
        if (cls == 2) l2 = S.cl[cc][CF_F];
      }
    }
    // small pools: one staged vector per lane-step, rolled; big: the crew job
    auto vec_pass = [&](uint32_t j) {
      const uint4 mv = meta4[j * 32 + lane_id()];
      for (int e = 0; e < 4; ++e) {
        const uint32_t m = el(mv, e);
        if (meta_res(m) == kResCached && meta_owner(m) == op.a && meta_pos(m) < L) {
          const uint32_t pos = meta_pos(m);
          const uint32_t cls = (meta_pinned(m) || pos < l3) ? 3u : (pos < l2 ? 2u : 1u);
          key[block_of(j, e)] = (cls << kClassShift) | (seq_base + (L - 1 - pos));
        }
      }
    };
#if RKC_BIG
    if constexpr (big) {
      job_args(op.a, L, seq_base);
      crew_run(JOB_TOUCH);
    } else
#endif
      for_vec<big ? 4 : 1>(nv, vec_pass);
    hset(H_SEQ, seq_base + L);
  }
  const uint32_t cc = obj_claim(ow);
  const bool has = cc < 32;
  if (has) need_claims();
  const uint32_t Rc = has ? S.cl[cc][CF_R] : 0u;
  const bool sat = has && live_state(cl_state(cc)) && L >= Rc;
  emit(EV_REUSE_PROBE, has ? cc : 0xFFu, sat ? 1u : 0u, 0, op.a, L, L * kBlockTokens, Rc);
  ctr_add(K_REUSE_PROBES, 1);
  ctr_add(K_REUSE_TOKENS, L * kBlockTokens);
}

// ------------------------------ phases -------------------------------------
// expiry: "Runtime responsibility ends at expiry" (Table 3; G13)
__device__ __noinline__ void expiry() {
  need_claims();
    const bool lc = lane_id() < S.C;
  const uint32_t* r = S.cl[lane_id()];
  const bool ex = lc && live_state(r[0] & 0xFFu) && r[CF_D] > 0 &&
                  (uint64_t)r[CF_DEC] + r[CF_D] <= S.step;
  const uint32_t m = __ballot_sync(kFull, ex);
  if (lane_id() == 0) S.flags |= F_CLAIMS_CHANGED;  // next expiry is recomputed
  __syncwarp();
  if (!m) return;
  const uint32_t o = (r[0] >> 16) & 0xFFu;
  emit_lanes(ex, EV_EXPIRED, 0, 0, o, r[CF_PC], r[CF_DEC], r[CF_D]);
  mark_reclass_lanes(ex && claim_class((r[0] >> 8) & 0xFFu, lowering()) != 1, o);
  if (ex) { S.cl[lane_id()][0] = (r[0] & ~0xFFu) | C_EXPIRED; S.cl[lane_id()][CF_PC] = 0; }
  __syncwarp();
  claims_dirty(ex);
  refresh_protected();
  ctr_add(K_EXPIRED, __popc(m));
}

// post-op predicate pass: accepted -> materialized when leading >= R
// (P:1038-1041); materialized -> harmed when the predicate breaks without a
// prior release (Table 4, G5)
__device__ RKC_POST_ATTR void post_op() {
  need_both();
    const bool lc = lane_id() < S.C;
  const uint32_t w0 = S.cl[lane_id()][0];
  const uint32_t st = w0 & 0xFFu, mode = (w0 >> 8) & 0xFFu, o = (w0 >> 16) & 0xFFu;
  const uint32_t R = S.cl[lane_id()][CF_R];
  const bool lv = lc && live_state(st);
  const bool olive = lv && obj_live(S.obj0[o]);
  const uint32_t L = olive ? S.lead[o] : 0u;
  const bool mat = lv && st == C_ACCEPTED && olive && L >= R;
  const bool harm = lv && st == C_MATERIALIZED && L < R;
  const uint32_t mm = __ballot_sync(kFull, mat), hm = __ballot_sync(kFull, harm);
  if ((mm | hm) == 0) return;
  const bool ob = obligated(mode);
  emit_lanes(mat || harm, mat ? EV_MATERIALIZED : EV_HARMED, harm ? (ob ? 1u : 0u) : 0u, 0, L, R,
             mat ? L * kBlockTokens : S.h[H_P], mat ? o : S.h[H_ALIVE]);
  mark_reclass_lanes(harm && claim_class(mode, lowering()) != 1, o);
  if (mat) S.cl[lane_id()][0] = (w0 & ~0xFFu) | C_MATERIALIZED;
  if (harm) { S.cl[lane_id()][0] = (w0 & ~0xFFu) | C_HARMED; S.cl[lane_id()][CF_PC] = 0; }
  __syncwarp();
  claims_dirty(mat || harm);
  ctr_add(K_MATERIALIZED, __popc(mm));
  ctr_add(K_HARMED_OBLIGATED, __popc(__ballot_sync(kFull, harm && ob)));
  ctr_add(K_HARMED_UNOBLIGATED, __popc(__ballot_sync(kFull, harm && !ob)));
  refresh_protected();
}

#ifndef RKC_FINISH_INLINE
#define RKC_FINISH_INLINE 1   // round 2 (with RKC_NEED_INLINE_CHECK and RKC_EMIT_INLINE: -2.9 % per c5 step)
#endif
#if RKC_FINISH_INLINE
__device__ __forceinline__ void finish() {
#else
__device__ __noinline__ void finish() {
#endif
    flush_reclass();
  if (S.flags & F_POST) {
    post_op();
    flush_reclass();
  }
#if RKC_FINISH_VEC
  // the bookkeeping words in two 16-B loads ({nev, flags, cdirty}, objdirty[4]):
  // one round trip instead of one per test below
  __syncwarp();
  const uint4 nf = *reinterpret_cast<const uint4*>(&S.nev);
  const uint4 od = *reinterpret_cast<const uint4*>(S.objdirty);
  // (RKC_HDR_ALWAYS: the hot header is written back by every heavy item -- it
  // changes in almost all of them, and an unchanged one is rewritten as read)
  bool hdr = RKC_HDR_ALWAYS || (nf.y & F_HDR) != 0;
  if (nf.y & F_CLAIMS_CHANGED) {
    const uint32_t* r = S.cl[lane_id()];
    const uint32_t ne = (lane_id() < S.C && live_state(r[0] & 0xFFu) && r[CF_D] > 0)
                            ? (uint32_t)min((uint64_t)r[CF_DEC] + r[CF_D], (uint64_t)0xFFFFFFFFu)
                            : 0xFFFFFFFFu;
    const uint32_t m = __reduce_min_sync(kFull, ne);
    if (lane_id() == 0) S.h[H_NEXT_EXPIRY] = m;
    hdr = true;
  }
  if ((nf.z >> lane_id()) & 1u) {
    uint4* cp = reinterpret_cast<uint4*>(S.clm + lane_id() * 8);
    cp[0] = reinterpret_cast<const uint4*>(S.cl[lane_id()])[0];
    cp[1] = reinterpret_cast<const uint4*>(S.cl[lane_id()])[1];
  }
  if (od.x | od.y | od.z | od.w) {
    uint2* dst = S.obj;
    const uint32_t O = S.O;
#pragma unroll
    for (uint32_t q = 0; q < kObjMax / 32; ++q) {
      const uint32_t o = q * 32 + lane_id();
      const uint32_t w = q == 0 ? od.x : q == 1 ? od.y : q == 2 ? od.z : od.w;
      if (o < O && ((w >> lane_id()) & 1u)) dst[o] = make_uint2(S.obj0[o], S.lead[o]);
    }
  }
  if (nf.x) {
    if (lane_id() == 0) S.h[H_EVCOUNT] += nf.x;
    hdr = true;
  }
  __syncwarp();
  if (hdr && lane_id() < H_HOT) S.hdrp[lane_id()] = S.h[lane_id()];
  const uint32_t d = S.ctr[lane_id()];
  if (d) atomicAdd(S.ctrp + lane_id(), d);  // fire-and-forget reduction, no round trip
#else
  if (S.flags & F_CLAIMS_CHANGED) {
    const uint32_t* r = S.cl[lane_id()];
    const uint32_t ne = (lane_id() < S.C && live_state(r[0] & 0xFFu) && r[CF_D] > 0)
                            ? (uint32_t)min((uint64_t)r[CF_DEC] + r[CF_D], (uint64_t)0xFFFFFFFFu)
                            : 0xFFFFFFFFu;
    const uint32_t m = __reduce_min_sync(kFull, ne);
    __syncwarp();  // write-after-read of S.flags in the warp
    if (lane_id() == 0) { S.h[H_NEXT_EXPIRY] = m; S.flags |= F_HDR; }
    __syncwarp();
  }
  // write back dirty claims and objects
  if ((S.cdirty >> lane_id()) & 1u) {
    uint4* cp = reinterpret_cast<uint4*>(S.clm + lane_id() * 8);
    cp[0] = reinterpret_cast<const uint4*>(S.cl[lane_id()])[0];
    cp[1] = reinterpret_cast<const uint4*>(S.cl[lane_id()])[1];
  }
  if (S.objdirty[0] | S.objdirty[1] | S.objdirty[2] | S.objdirty[3]) {
    uint2* dst = S.obj;
    for (uint32_t o = lane_id(); o < S.O; o += 32)
      if ((S.objdirty[o >> 5] >> (o & 31u)) & 1u) dst[o] = make_uint2(S.obj0[o], S.lead[o]);
  }
  if (S.nev) {
    if (lane_id() == 0) { S.h[H_EVCOUNT] += S.nev; S.flags |= F_HDR; }
    __syncwarp();
  }
  if (S.flags & F_HDR) {
    if (lane_id() < H_HOT) S.hdrp[lane_id()] = S.h[lane_id()];
  }
  __syncwarp();
  const uint32_t d = S.ctr[lane_id()];
  if (d) atomicAdd(S.ctrp + lane_id(), d);  // fire-and-forget reduction, no round trip
#endif
}

struct StepArgs {
  PoolDev p;
  const uint4* ops;     // this step's row: [num_traces]
  uint32_t step;        // global step index of this launch
  uint32_t main_items;  // small pools: items of the one-warp step grid (the rest: overflow kernel)
  unsigned long long* host_heavy;  // mapped host ring [64]: (tag << 32) | heavy count, or null
  uint32_t tag_hi;      // batch epoch << 16 (the low 16 bits of the tag: the step)
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
    case OP_HIT_ADMIT: return 5;
    case OP_DEMOTE: return 6;
    default: return 7;  // NOP and unknown kinds
  }
}

// K0: light pass, one thread per trace.  Completes the ops that provably
// change nothing but a request record and a counter -- a NOP with no expiry
// due, an ADVANCE that needs no new block (decode within the last block, or a
// chunk that fits the blocks already held), an ADMIT whose PEAK check passes --
// with the exact effects the warp path would have (no events, no block, claim,
// object or header change).  Every other trace is bucketed by op kind for the
// warp-per-trace step kernel, heavy block-scanning kinds first.

#ifndef RKC_LIGHT_THREADS
#define RKC_LIGHT_THREADS 128
#endif
constexpr uint32_t kLightThreads = RKC_LIGHT_THREADS;

// heavy-trace ticket: op (4 words), hot header words 0..11 (word 10 <- the trace id)
constexpr uint32_t kTicketWords = 16u;
__global__ void __launch_bounds__(kLightThreads, RKC_LIGHT_MIN_CTAS) rkc_light_kernel(const __grid_constant__ StepArgs args) {
  const PoolDev& p = args.p;
  const uint32_t step = args.step;
  uint32_t* cnt = p.bcnt + (step & 1u) * 8;
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x < 8) p.bcnt[(((step + 1u) & 1u) * 8 + threadIdx.x)] = 0;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t stride = gridDim.x * blockDim.x;
  __shared__ uint32_t s_cnt[8], s_base[8];
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t base = blockIdx.x * blockDim.x; base < p.num_traces; base += stride) {
    const uint32_t t = base + threadIdx.x;
    const bool valid = t < p.num_traces;
    bool heavy = false, fa = false;
    uint32_t kind = 0, fa_need = 0, fa_live = 0, fa_owner = 0;
    uint4 opw = make_uint4(0, 0, 0, 0), hv0 = opw, hv1 = opw, hv2 = opw;
    if (valid) {
      // level 1: the op and the trace's hot header (independent of the op)
      opw = __ldcs(args.ops + t);
      const uint32_t* h = p.hdr + (size_t)t * H_NWORDS;
      hv0 = __ldcg(reinterpret_cast<const uint4*>(h));      // U, policy, accept, seq
      hv1 = __ldcg(reinterpret_cast<const uint4*>(h) + 1);  // free, alive, P, mask
      hv2 = __ldcg(reinterpret_cast<const uint4*>(h) + 2);  // next expiry, event count
      const uint32_t nexp = hv2.x;
      kind = opw.x & 0xFFu;
      const uint32_t a = (opw.x >> 8) & 0xFFu;
      heavy = true;
      if (kind == OP_NOP) {
        heavy = step >= nexp;
      } else if (kind == OP_ADVANCE && a < p.Q) {
        // level 2: the request record and (speculatively) the free bitmap
        uint32_t* rq = p.req + ((size_t)t * p.Q + a) * 8;
        const uint4 r0 = __ldcg(reinterpret_cast<const uint4*>(rq));
        const uint4 r1 = __ldcg(reinterpret_cast<const uint4*>(rq + 4));
        const bool small = p.NS <= 1024;  // one bitmap word per lane
        const uint32_t status = r0.x & 0xFFu, prompt = r0.y, chunk = r0.z, decode = r0.w;
        const uint32_t done = r1.x, live = r1.y, held = r1.y + r1.z;  // own + shared hit blocks
        if (step < nexp && status == R_RUNNING && (uint64_t)done < (uint64_t)prompt + decode) {
          const uint32_t n = done < prompt ? min(chunk, prompt - done) : 1u;
          const uint64_t need_total = ((uint64_t)done + n + kBlockTokens - 1) / kBlockTokens;
          if (need_total <= held) {
            rq[RQ_DONE] = done + n;
            atomicAdd(p.ctr + (size_t)t * K_NCTR + K_OPS, 1u);
            heavy = false;
          } else if (small) {
            // a feasible allocation served entirely from free blocks: the
            // `need` lowest-id free blocks get positions live.. (G24); no
            // victim, no event, no claim or object change
            const uint32_t need = (uint32_t)(need_total - held);
            if ((uint64_t)hv1.z + hv1.y + need <= hv0.x && need <= hv1.x) {
              fa = true;  // the blocks are taken warp-cooperatively below
              fa_need = need;
              fa_live = live;
              fa_owner = a;
              uint32_t* hw = const_cast<uint32_t*>(h);
              hw[H_FREE] = hv1.x - need;
              hw[H_ALIVE] = hv1.y + need;
              rq[RQ_LIVE] = live + need;
              rq[RQ_DONE] = done + n;
              atomicAdd(p.ctr + (size_t)t * K_NCTR + K_OPS, 1u);
              atomicAdd(p.ctr + (size_t)t * K_NCTR + K_BLOCKS_ALLOCATED, need);
              atomicAdd(p.ctr + (size_t)t * K_NCTR + K_ALLOCATIONS, 1u);
              heavy = false;
            }
          }
        }
      } else if (kind == OP_ADMIT && a < p.Q && ((opw.x >> 16) & 0xFFu) < p.O && (opw.x >> 24) <= 1 &&
                 opw.y >= 1 && opw.z >= 1 && opw.y <= kMaxTokens && opw.w <= kMaxTokens) {
        uint32_t* rq = p.req + ((size_t)t * p.Q + a) * 8;
        const uint32_t status = __ldcg(rq) & 0xFFu;
        if (step < nexp && status != R_RUNNING && status != R_DEFERRED) {
          const uint64_t peak = ((uint64_t)opw.y + opw.w + kBlockTokens - 1) / kBlockTokens;
          const uint32_t chk = (hv0.y >> 8) & 0xFFu;  // RESERVE admissions take the warp path
          if (chk == ADMIT_NONE || (chk == ADMIT_PEAK && (uint64_t)hv1.z + hv1.y + peak <= hv0.x)) {
            reinterpret_cast<uint4*>(rq)[0] =
                make_uint4(R_RUNNING | ((opw.x >> 24) << 8) | (((opw.x >> 16) & 0xFFu) << 16), opw.y,
                           opw.z, opw.w);
            reinterpret_cast<uint4*>(rq)[1] = make_uint4(0, 0, 0, 0);  // done, live, hit
            atomicAdd(p.ctr + (size_t)t * K_NCTR + K_OPS, 1u);
            atomicAdd(p.ctr + (size_t)t * K_NCTR + K_ADMITTED, 1u);
            heavy = false;
          }
        }
      }
    }
    // free-only allocations, one trace at a time across the warp (lane = free
    // bitmap word): the `need` lowest-id free blocks, positions live.. in
    // block-id order (G24)
    // (the bitmap words of up to 8 traces are loaded before any is consumed)
    for (uint32_t fm = __ballot_sync(kFull, fa); fm;) {
      uint32_t words[8], srcs[8], nb = 0;
#pragma unroll
      for (uint32_t q = 0; q < 8; ++q) {
        srcs[q] = fm ? __ffs(fm) - 1 : 0u;
        words[q] = 0;
        if (fm) {
          const uint32_t tq = __shfl_sync(kFull, t, srcs[q]);
          if (lane < p.NS / 32) words[q] = __ldcg(p.fbm + (size_t)tq * (p.NS / 32) + lane);
          fm &= fm - 1;
          nb = q + 1;
        }
      }
#pragma unroll
      for (uint32_t q = 0; q < 8; ++q) {
      if (q >= nb) break;
      const uint32_t src = srcs[q];
      const uint32_t tt = __shfl_sync(kFull, t, src), need = __shfl_sync(kFull, fa_need, src);
      const uint32_t live = __shfl_sync(kFull, fa_live, src), owner = __shfl_sync(kFull, fa_owner, src);
      uint32_t* fbm = p.fbm + (size_t)tt * (p.NS / 32);
      const uint32_t word = words[q];
#if RKC_LIGHT_FA_FAST
      {  // the lowest non-empty bitmap word holds all `need` blocks (pools filling: the free
         // blocks are a run at the end of the pool): no scan, no search
        const uint32_t fl = __ffs(__ballot_sync(kFull, word != 0)) - 1;
        const uint32_t wf = __shfl_sync(kFull, word, fl & 31u);
        const uint32_t cf = __popc(wf);
        if (cf >= need) {
          if (lane == fl) fbm[lane] = need == cf ? 0u : wf & ~((1u << nth_set_bit(wf, need + 1)) - 1u);
          if (lane < need) {
            const uint32_t b = fl * 32 + nth_set_bit(wf, lane + 1);
            p.meta[(size_t)tt * p.NS + b] = meta_make(kResActive, owner, live + lane);
            p.key[(size_t)tt * p.NS + b] = kKeyActive;
          }
          continue;
        }
      }
#endif
      const uint32_t c = __popc(word);
      const uint32_t incl = warp_incl_scan(c, lane);
      const uint32_t before = incl - c;
      const uint32_t take = before >= need ? 0u : min(c, need - before);
      if (take > 0) {
        const uint32_t tw = take == c ? word : word & ((1u << nth_set_bit(word, take + 1)) - 1u);
        fbm[lane] = word & ~tw;
      }
#if RKC_LIGHT_RANKED
      // rank-parallel: rank r (block at position live + r) goes to lane r % 32;
      // its bitmap word is the first whose inclusive count exceeds r (the taken
      // blocks of one allocation are usually a run inside one or two words)
      uint32_t* key = p.key + (size_t)tt * p.NS;
      uint32_t* meta = p.meta + (size_t)tt * p.NS;
      for (uint32_t r0 = 0; r0 < need; r0 += 32) {
        const uint32_t r = r0 + lane;
        uint32_t sl = 0;
#pragma unroll
        for (uint32_t b = 16; b >= 1; b >>= 1)
          if (__shfl_sync(kFull, incl, sl + b - 1) <= r) sl += b;
        const uint32_t ws = __shfl_sync(kFull, word, sl & 31u), bs = __shfl_sync(kFull, before, sl & 31u);
        if (r < need) {
          const uint32_t b = sl * 32 + nth_set_bit(ws, r - bs + 1);
          meta[b] = meta_make(kResActive, owner, live + r);
          key[b] = kKeyActive;
        }
      }
#else
      if (take > 0) {
        uint32_t tw = take == c ? word : word & ((1u << nth_set_bit(word, take + 1)) - 1u);
        uint32_t* key = p.key + (size_t)tt * p.NS;
        uint32_t* meta = p.meta + (size_t)tt * p.NS;
        for (uint32_t r = live + before; tw; tw &= tw - 1, ++r) {
          const uint32_t b = lane * 32 + __ffs(tw) - 1;
          meta[b] = meta_make(kResActive, owner, r);
          key[b] = kKeyActive;
        }
      }
#endif
      }
    }
    // bucket ranks: warp match -> CTA shared counts -> one global atomic per bucket per CTA
    const uint32_t bk = heavy ? bucket_of(kind) : 8u;
    const uint32_t grp = __match_any_sync(kFull, bk);
    const uint32_t leader = __ffs(grp) - 1;
    uint32_t off = 0;
    if (lane == leader && heavy) off = atomicAdd(&s_cnt[bk], __popc(grp));
    off = __shfl_sync(kFull, off, leader);
    __syncthreads();
    if (threadIdx.x < 8) {
      const uint32_t c = s_cnt[threadIdx.x];
      s_base[threadIdx.x] = c ? atomicAdd(cnt + threadIdx.x, c) : 0u;
      s_cnt[threadIdx.x] = 0;
    }
    __syncthreads();
    const uint32_t cbase = heavy ? s_base[bk] : 0u;
    if (heavy) {  // the ticket: op, header words 0..11 (word 10 <- the trace id)[, request]
      uint4* tk = reinterpret_cast<uint4*>(p.perm) +
                  (kTicketWords / 4) * ((size_t)bk * p.num_traces + cbase + off + __popc(grp & lanemask_lt()));
      // tickets are read back by the step kernel right after this pass: keep
      // them in L2 ahead of the streamed op / header / request lines
      st_evict_last(tk + 0, opw);
      st_evict_last(tk + 1, hv0);
      st_evict_last(tk + 2, hv1);
      st_evict_last(tk + 3, make_uint4(hv2.x, hv2.y, t, 0u));
    }
  }
}


// the step's per-bucket heavy counts (read-only in this kernel and written by
// the previous one: the L1 path serves every CTA of an SM after the first)
__device__ __forceinline__ void bucket_counts(const StepArgs& args, uint32_t (&cnt)[8]) {
  const uint4* cnt4 = reinterpret_cast<const uint4*>(args.p.bcnt + (args.step & 1u) * 8);
  const uint4 ca = __ldg(cnt4), cb = __ldg(cnt4 + 1);
  cnt[0] = ca.x; cnt[1] = ca.y; cnt[2] = ca.z; cnt[3] = ca.w;
  cnt[4] = cb.x; cnt[5] = cb.y; cnt[6] = cb.z; cnt[7] = cb.w;
}
// bucketed item i of this step -> its ticket (false past the heavy count)
__device__ __forceinline__ bool item_ticket(const StepArgs& args, const uint32_t (&cnt)[8], uint32_t i,
                                            const uint32_t*& tk) {
  uint32_t acc = 0, bk = 8, off = 0;
#pragma unroll
  for (uint32_t q = 0; q < 8; ++q) {
    const uint32_t c = cnt[q];
    if (bk == 8 && i < acc + c) { bk = q; off = i - acc; }
    acc += c;
  }
  if (bk == 8) return false;
  tk = args.p.perm + ((size_t)bk * args.p.num_traces + off) * kTicketWords;
  return true;
}
__device__ __forceinline__ bool item_trace(const StepArgs& args, uint32_t i, const uint32_t*& tk) {
  uint32_t cnt[8];
  bucket_counts(args, cnt);
  return item_ticket(args, cnt, i, tk);
}

// one heavy trace-step from its ticket (written by the light pass: the op in
// words 0..3, hot header words 0..11 in 4..15, the trace id in place of the
// unused header word 10): op, trace id, header word `lane` (< 10) and the next
// expiry step -- the warp's whole op path
__device__ __forceinline__ void run_item_body(const StepArgs& args, const uint4 opw, const uint32_t t,
                                                const uint32_t hw, const uint32_t next_exp) {
  const uint32_t lane = threadIdx.x & 31u;
  const PoolDev& p = args.p;
  const uint32_t kind = opw.x & 0xFFu, a = (opw.x >> 8) & 0xFFu;
  // Issue every load this op is known to need before waiting on any of them:
  // hot header (lanes 0..15), the request record, the claim / object tables.
  const bool rq_op = (kind == OP_ADMIT || kind == OP_ADVANCE || kind == OP_COMPLETE ||
                      kind == OP_HIT_ADMIT) && a < p.Q;
  const bool want_cl = kind == OP_SUBMIT || kind == OP_DEMOTE || kind == OP_TOUCH ||
                       kind == OP_COMPLETE || kind == OP_INSERT || kind == OP_HIT_ADMIT;
  const bool want_ob = kind == OP_SUBMIT || kind == OP_INSERT || kind == OP_COMPLETE ||
                       kind == OP_TOUCH || kind == OP_HIT_ADMIT;
  uint32_t rqv = 0;
  if (rq_op && lane < 8) rqv = __ldcg(p.req + ((size_t)t * p.Q + a) * 8 + lane);
  uint4 c0 = make_uint4(0, 0, 0, 0), c1 = make_uint4(0, 0, 0, 0);
  if (want_cl && lane < p.C) {
    const uint4* cp = reinterpret_cast<const uint4*>(p.clm + ((size_t)t * p.C + lane) * 8);
    c0 = __ldcg(cp);
    c1 = __ldcg(cp + 1);
  }
  uint2 ov[4];
  const uint2* obase = reinterpret_cast<const uint2*>(p.obj) + (size_t)t * p.O;
  if (want_ob) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i < p.O) ov[i] = __ldcg(obase + lane + 32 * i);
  }
  // small pools: one 128-B line of the block words per lane (NS <= 1024); big
  // pools: the crew streams the block words itself
  if (!kBig && lane < p.NS / 32) {
    const bool scan = kind == OP_COMPLETE || kind == OP_TOUCH;  // these ops scan the block words
    const bool sel = kind == OP_ADVANCE || kind == OP_INSERT;   // heavy ones allocate: keys next
    if (scan) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.meta + (size_t)t * p.NS + lane * 32));
    if (sel) asm volatile("prefetch.global.L2 [%0];" ::"l"(p.key + (size_t)t * p.NS + lane * 32));
  }
  // a NOP with no expiry due changes nothing (fast path)
  if (kind == OP_NOP && args.step < next_exp) {
    crew_exit();
    return;
  }
  if (lane < H_NWORDS) S.h[lane] = hw;
  S.ctr[lane] = (lane == K_OPS && kind != OP_NOP) ? 1u : 0u;  // the op counts itself
  if (lane < 4) { S.rc[lane] = 0; S.objdirty[lane] = 0; }
  if (lane < 8) S.rq[lane] = rqv;
  if (want_cl) {
    reinterpret_cast<uint4*>(S.cl[lane])[0] = c0;
    reinterpret_cast<uint4*>(S.cl[lane])[1] = c1;
  }
  if (want_ob) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane + 32 * i < p.O) { S.obj0[lane + 32 * i] = ov[i].x; S.lead[lane + 32 * i] = ov[i].y; }
  }
  if (lane == 0) {
    S.nev = 0; S.cdirty = 0;
    S.flags = (want_cl ? F_CLAIMS : 0u) | (want_ob ? F_OBJS : 0u) | (rq_op ? F_RQ : 0u);
    S.t = t; S.step = args.step;
    S.NS = p.NS; S.nv = p.NS / 128; S.C = p.C; S.Q = p.Q; S.O = p.O; S.EPT = p.EPT;
    S.key = p.key + (size_t)t * p.NS;
    S.meta = p.meta + (size_t)t * p.NS;
    S.fbm = p.fbm + (size_t)t * (p.NS / 32);
    S.clm = p.clm + (size_t)t * p.C * 8;
    S.req = p.req + (size_t)t * p.Q * 8;
    S.obj = reinterpret_cast<uint2*>(p.obj) + (size_t)t * p.O;
    S.ctrp = p.ctr + (size_t)t * K_NCTR;
    S.hdrp = p.hdr + (size_t)t * H_NWORDS;
    S.ev = p.ev + (size_t)t * p.EPT * 2;
  }
  __syncwarp();
  Op op{kind, a, (opw.x >> 16) & 0xFFu, opw.x >> 24, opw.y, opw.z, opw.w};
  if (args.step >= next_exp) expiry();
  switch (kind) {
    case OP_NOP: break;
    case OP_SUBMIT: op_submit(op); break;
    case OP_ADMIT: op_admit(op); break;
    case OP_ADVANCE: op_advance(op); break;
    case OP_COMPLETE: op_complete<kBig>(op); break;
    case OP_INSERT: op_insert(op); break;
    case OP_DEMOTE: op_demote(op); break;
    case OP_TOUCH: op_touch<kBig>(op); break;
    case OP_HIT_ADMIT: op_hit_admit(op); break;
    default: op_error(op, ERR_UNKNOWN_OP); break;
  }
  __syncwarp();
  finish();
  crew_exit();
}

__device__ __forceinline__ void run_item(const StepArgs& args, const uint32_t* tk) {
#if RKC_BIG
  if (threadIdx.x >= 32) {  // crew helpers: block-pass slices until the leader is done
    crew_helper();
    return;
  }
#endif
  const uint32_t lane = threadIdx.x & 31u;
  // the op (words 0..3) and words 12..15 {next expiry, event count, trace, -}
  // as warp-uniform 16-B loads, header words 0..9 one per lane: independent
  // loads, no shuffles
  const uint4* tk4 = reinterpret_cast<const uint4*>(tk);
  const uint4 opw = __ldg(tk4);
  const uint4 tail = __ldg(tk4 + 3);
  const uint32_t hw = lane < 10 ? __ldg(tk + 4 + lane) : 0u;
  run_item_body(args, opw, tail.z, hw, tail.x);
}

// K1: warp w of CTA b -> the (b * kWarpsPerCta + w)-th trace of the op-kind
// bucketed order.  Small pools launch CTAs for the first kMainItems(T) items
// only (the heavy share of a step is about half); the rest, if any, run on
// the overflow kernel below.
#ifndef RKC_BIG_MIN_CTAS
#define RKC_BIG_MIN_CTAS (32 / (kCrew))
#endif
// resident CTAs per SM the register budget is sized for (small pools: 32 one-warp
// CTAs = 64 registers; big pools: crews of kCrew warps)
#ifndef RKC_SMALL_MIN_CTAS
#define RKC_SMALL_MIN_CTAS (32 / kWarpsPerCta)
#endif
constexpr int kMinCtas = kBig ? RKC_BIG_MIN_CTAS : RKC_SMALL_MIN_CTAS;
__global__ void __launch_bounds__(kWarpsPerCta * kCrew * 32, kMinCtas)
rkc_step_kernel(const __grid_constant__ StepArgs args) {
  pdl_wait();
  const uint32_t* tk;
  if (args.host_heavy && blockIdx.x == 0 && threadIdx.x == 0) {
    // this step's heavy count, published to the host (which sizes the step
    // grid a few steps ahead from it: rkc_abi.cu grid pacing)
    uint32_t cnt[8];
    bucket_counts(args, cnt);
    uint32_t H = 0;
#pragma unroll
    for (uint32_t q = 0; q < 8; ++q) H += cnt[q];
    volatile unsigned long long* slot = args.host_heavy + (args.step & 63u);
    *slot = ((unsigned long long)(args.tag_hi | (args.step & 0xFFFFu)) << 32) | H;
    __threadfence_system();
  }
#if !RKC_BIG && RKC_SPREAD_FILL
  // While pools fill, most of the grid finds no item (H heavy items, G CTAs):
  // those empty CTAs would queue behind the last real one as a dispatch-bound
  // tail.  When H < 3/4 G the items are spread evenly over the grid (CTA b
  // takes item floor(b H / G) if it is the first CTA mapping to it), so the
  // empty CTAs retire between the busy ones; items stay in bucket order.
  // (Spreading at the steady state, H ~ G, measured 2.5 % slower.)
  uint32_t cnt[8];
  bucket_counts(args, cnt);
  uint32_t H = 0;
#pragma unroll
  for (uint32_t q = 0; q < 8; ++q) H += cnt[q];
  const uint32_t G = gridDim.x, b = blockIdx.x;
  uint32_t i = b;
  if ((uint64_t)H * 4 < (uint64_t)G * 3) {
    const uint64_t x = (uint64_t)b * H;
    i = (uint32_t)((double)x / (double)G);
    while ((uint64_t)(i + 1) * G <= x) ++i;   // exact floor(b H / G)
    while ((uint64_t)i * G > x) --i;
    if (b > 0 && (uint64_t)(b - 1) * H >= (uint64_t)i * G) return;  // not the first CTA of item i
  }
  if (!item_ticket(args, cnt, i, tk)) return;
  run_item(args, tk);
#else
  if (!item_trace(args, blockIdx.x * kWarpsPerCta + (kWarpsPerCta == 1 ? 0u : (threadIdx.x >> 5)), tk)) return;
  run_item(args, tk);
#endif
}

#if !RKC_BIG
#ifndef RKC_MAIN_SIXTEENTHS
#define RKC_MAIN_SIXTEENTHS 9
#endif
__host__ __device__ constexpr uint32_t kMainItems(uint32_t T) {  // RKC_MAIN_SIXTEENTHS/16 of T
  return (uint32_t)(((uint64_t)T * RKC_MAIN_SIXTEENTHS + 15) / 16);
}
// items [kMainItems(T), heavy count), if any: a grid of 1/16 of the remaining
// slots (at least 592 CTAs) loops over them, at most 16 items per warp -- a
// step with more heavy traces than the main grid slows down gradually
#ifndef RKC_OVF_MAX_CTAS
#define RKC_OVF_MAX_CTAS (148u * 16u)
#endif
__host__ __device__ constexpr uint32_t kOverflowCtas(uint32_t T, uint32_t main) {
  // capped: every overflow CTA is dispatched every step even when no item
  // overflows (~0.5 ns each), and c5 would otherwise launch 27k of them
  return (T - main) / 16 > 592
             ? ((T - main) / 16 < (uint32_t)(RKC_OVF_MAX_CTAS) ? (T - main) / 16
                                                               : (uint32_t)(RKC_OVF_MAX_CTAS))
             : 592;
}
__global__ void __launch_bounds__(32) rkc_step_overflow_kernel(const __grid_constant__ StepArgs args) {
  pdl_wait();
  for (uint32_t i = args.main_items + blockIdx.x;; i += gridDim.x) {
    const uint32_t* tk;
    if (!item_trace(args, i, tk)) return;
    run_item(args, tk);
    __syncwarp();
  }
}
#endif

template <class Kernel>
static cudaError_t launch_pdl(Kernel kernel, uint32_t grid, uint32_t block, cudaStream_t st,
                              const StepArgs& args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args);
}

// host launcher: one launch = one lockstep step over all traces
// main_items: the one-warp step grid of a small pool (0: the default
// kMainItems(T)); host_heavy: where the step kernel publishes the heavy count
cudaError_t launch_step(const PoolDev& p, const void* ops_step, uint32_t step, cudaStream_t st,
                        uint32_t main_items, unsigned long long* host_heavy, uint32_t tag_hi) {
#if RKC_BIG
  const uint32_t main = p.num_traces;
#else
  const uint32_t main = main_items ? (main_items < p.num_traces ? main_items : p.num_traces)
                                   : kMainItems(p.num_traces);
#endif
  StepArgs args{p, reinterpret_cast<const uint4*>(ops_step), step, main, host_heavy, tag_hi};
  const uint32_t lct = (p.num_traces + kLightThreads - 1) / kLightThreads;
// one light thread per trace (round 2: the former cap of 16 CTAs per SM, i.e. 3.3 traces per
// thread at c5, measured 1 % slower per lockstep step: profiles/r02/experiments.md)
#ifndef RKC_LIGHT_MAX_CTAS
#define RKC_LIGHT_MAX_CTAS 0x7FFFFFFF
#endif
  const uint32_t cgrid = lct < (uint32_t)(RKC_LIGHT_MAX_CTAS) ? lct : (uint32_t)(RKC_LIGHT_MAX_CTAS);
  cudaError_t e = launch_pdl(rkc_light_kernel, cgrid, kLightThreads, st, args);
#if RKC_BIG
  if (e == cudaSuccess)
    e = launch_pdl(rkc_step_kernel, (p.num_traces + kWarpsPerCta - 1) / kWarpsPerCta, kWarpsPerCta * kCrew * 32, st, args);
#else
  if (e == cudaSuccess)
    e = launch_pdl(rkc_step_kernel, (main + kWarpsPerCta - 1) / kWarpsPerCta, kWarpsPerCta * 32, st, args);
  if (e == cudaSuccess) e = launch_pdl(rkc_step_overflow_kernel, kOverflowCtas(p.num_traces, main), 32, st, args);
#endif
  return e;
}

}  // namespace RKC_STEP_NS
}  // namespace rkc
