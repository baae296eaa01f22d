// rkc_conformance.cu -- SURVEY 8(f) f2: conformance checks L1-L7 over the
// claim-level event stream, one thread per trace
// replaying its events in (step, seq) order and reconstructing every claim's
// lifecycle (L7, "an external observer can reconstruct acceptance,
// materialization, active conflict, blocking claims, and final outcome").
//
// Checks (a set bit in the per-trace verdict = the check FAILED):
//   L1  every claim_harmed follows a claim_accepted of that claim ("no
//       accepted claim, no claim harm"; "every claim_harmed
//       event has an earlier claim_accepted for the same claim_id")
//   L2  write no-admit is separate from allocation: every
//       write_admission_denied is followed in the same step by
//       request_served of the same request
//   L3  every refusal / deferral / insert refusal carries a consistent
//       capacity proof: shortfall = P + A - U > 0; reason protected-resident
//       <=> non-empty blocking mask <=> (A <= U and P > 0); every blocking
//       claim is live at that point
//   L45 release before loss: no claim_harmed of a claim after its
//       claim_demoted / claim_expired; after-release victims only once some
//       claim was released
//   L6  predicate consistency: materialized => L >= R and tokens = 16 L;
//       harmed => L < R; reuse probes report tokens = 16 L and
//       satisfied = (bound claim live and L >= R)
//   L7  lifecycle legality of the reconstruction (S:44 transitions, including
//       accepted -> harmed) and, when the final claim states are given,
//       equality with them
//   I4  under the contract lowering no obligated claim is harmed (north star);
//       checked only where the trace's lowering is known
// A drained pool ring holds only the events after the drain: the checks then
// start from "unknown" claim states and verify what the remaining events
// determine (no final-state comparison).
//   LOST the trace's event ring overflowed (checks ran on a prefix)
#include <cuda_runtime.h>

#include <atomic>

#include "../../include/rkc.h"
#include "rkc_internal.cuh"

namespace rkc {

extern std::atomic<unsigned long long> g_launches;

namespace {

struct EvIn {  // events of one trace: either a compacted array or a pool ring
  const uint4* base;
  uint32_t n;
};

constexpr uint8_t kUnknown = 0xFE;    // claim state before a drained ring's first event
constexpr uint32_t kNoLowering = 0xFF;  // lowering not given: I4 is not checked

__device__ __forceinline__ bool live_or_unknown(uint8_t s) {
  return s == C_ACCEPTED || s == C_MATERIALIZED || s == kUnknown;
}

__device__ uint32_t check_trace(const EvIn in, const uint8_t* final_states, uint32_t C,
                                uint32_t lowering, bool lost, bool partial,
                                unsigned long long* ev_sum) {
  uint8_t st[32];      // reconstructed claim states
  uint8_t rel[32];     // released (demoted / expired) before
  uint8_t acc[32];     // accepted at some point
  uint32_t R[32];      // claim threshold (from the accept record)
  uint8_t oc[128];     // object -> bound claim (0xFF none)
  // (a drained ring's claims may have been accepted before the drain)
  for (int i = 0; i < 32; ++i) { st[i] = partial ? kUnknown : 0; rel[i] = 0; acc[i] = partial; R[i] = 0; }
  for (int i = 0; i < 128; ++i) oc[i] = 0xFF;
  uint32_t fail = 0;
  bool any_release = partial;
  uint32_t pending_denied = 0xFFFFFFFFu, pending_step = 0;
  uint64_t e_acc = 0, e_mat = 0, e_harm = 0, e_ref = 0, e_att = 0, e_vic = 0, e_rel = 0, e_den = 0;
  for (uint32_t i = 0; i < in.n; ++i) {
    const uint4 a = in.base[2 * i], f = in.base[2 * i + 1];
    const uint32_t type = a.z & 0xFFu, slot = (a.z >> 16) & 0xFFu, reason = a.z >> 24;
    const uint32_t step = a.y, mask = a.w;
    if (pending_denied != 0xFFFFFFFFu) {  // a denial must be followed by the service
      if (!(type == EV_SERVED && slot == pending_denied && step == pending_step)) fail |= RKC_CHECK_L2;
      pending_denied = 0xFFFFFFFFu;
    }
    switch (type) {
      case EV_ACCEPTED:
        if (slot >= C || (st[slot] != C_EMPTY && st[slot] != kUnknown)) { fail |= RKC_CHECK_L7; break; }
        st[slot] = C_ACCEPTED;
        acc[slot] = 1;
        R[slot] = f.z;
        if (f.x < 128) oc[f.x] = (uint8_t)slot;
        ++e_acc;
        break;
      case EV_REJECTED:
        if (slot >= C || (st[slot] != C_EMPTY && st[slot] != kUnknown)) { fail |= RKC_CHECK_L7; break; }
        st[slot] = C_REFUSED;
        break;
      case EV_MATERIALIZED:
        if (slot >= C || (st[slot] != C_ACCEPTED && st[slot] != kUnknown)) { fail |= RKC_CHECK_L7; break; }
        if (f.x < f.y || f.z != f.x * kBlockTokens) fail |= RKC_CHECK_L6;
        st[slot] = C_MATERIALIZED;
        ++e_mat;
        break;
      case EV_DEMOTED:
      case EV_EXPIRED:
        if (slot >= C || !live_or_unknown(st[slot])) {
          fail |= RKC_CHECK_L7;
          break;
        }
        st[slot] = type == EV_DEMOTED ? C_DEMOTED : C_EXPIRED;
        rel[slot] = 1;
        any_release = true;
        break;
      case EV_HARMED:
        if (slot >= C) { fail |= RKC_CHECK_L7; break; }
        if (!acc[slot] && st[slot] != kUnknown) fail |= RKC_CHECK_L1;
        if (rel[slot]) fail |= RKC_CHECK_L45;
        if (!live_or_unknown(st[slot])) fail |= RKC_CHECK_L7;
        if (f.x >= f.y) fail |= RKC_CHECK_L6;
        if (reason && lowering == LOW_CONTRACT) fail |= RKC_CHECK_I4;
        st[slot] = C_HARMED;
        ++e_harm;
        break;
      case EV_DEFERRED:
      case EV_REFUSED:
      case EV_INSERT_REFUSED: {
        const uint64_t P = f.x, A = f.y, U = f.z;
        if (P + A <= U || P + A - U != f.w) fail |= RKC_CHECK_L3;
        const bool resident = A <= U && P > 0;  // P: protected blocks, or the reserve (f4)
        const bool resident_reason = reason == WHY_PROTECTED || reason == WHY_RESERVE;
        if (resident_reason != resident || (mask != 0) != resident) fail |= RKC_CHECK_L3;
        for (uint32_t c = 0; c < 32; ++c)
          if ((mask >> c) & 1u) {
            if (c >= C || !live_or_unknown(st[c])) fail |= RKC_CHECK_L3;
          }
        ++e_ref;
        if (mask) ++e_att;
        break;
      }
      case EV_WRITE_DENIED:
        pending_denied = slot;
        pending_step = step;
        ++e_den;
        break;
      case EV_VICTIMS:
        if (f.y > 0 && !any_release) fail |= RKC_CHECK_L45;
        e_vic += (uint64_t)f.x + f.y + f.z;
        e_rel += f.y;
        break;
      case EV_REUSE_PROBE: {
        if (f.z != f.y * kBlockTokens) fail |= RKC_CHECK_L6;
        const uint32_t c = slot;
        // what a drained ring cannot know: the bound claim and its threshold
        const bool known = !partial || (f.x < 128 && oc[f.x] != 0xFF);
        if (known) {
          const bool live = c < C && (st[c] == C_ACCEPTED || st[c] == C_MATERIALIZED);
          const bool sat = live && f.y >= R[c];
          if ((reason != 0) != sat) fail |= RKC_CHECK_L6;
          if (f.x >= 128 || oc[f.x] != c) fail |= RKC_CHECK_L7;  // probe names the bound claim
        }
        break;
      }
      default:
        break;
    }
  }
  if (pending_denied != 0xFFFFFFFFu) fail |= RKC_CHECK_L2;
  if (final_states) {
    for (uint32_t c = 0; c < C; ++c)
      if (final_states[c] != st[c]) fail |= RKC_CHECK_L7;
  }
  if (lost) fail |= RKC_CHECK_LOST;
  if (ev_sum) {
    atomicAdd(ev_sum + 0, (unsigned long long)e_acc);
    atomicAdd(ev_sum + 1, (unsigned long long)e_mat);
    atomicAdd(ev_sum + 2, (unsigned long long)e_harm);
    atomicAdd(ev_sum + 3, (unsigned long long)e_ref);
    atomicAdd(ev_sum + 4, (unsigned long long)e_att);
    atomicAdd(ev_sum + 5, (unsigned long long)e_vic);
    atomicAdd(ev_sum + 6, (unsigned long long)e_rel);
    atomicAdd(ev_sum + 7, (unsigned long long)e_den);
  }
  return fail;
}

__global__ void conformance_array_kernel(const uint4* ev, const uint32_t* offsets, uint32_t T,
                                         const uint8_t* final_states, uint32_t C,
                                         const uint8_t* lowering, uint32_t* verdict,
                                         unsigned long long* evidence) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    const uint32_t b = offsets[t], e = offsets[t + 1];
    EvIn in{ev + (size_t)b * 2, e - b};
    verdict[t] = check_trace(in, final_states ? final_states + (size_t)t * C : nullptr, C,
                             lowering ? lowering[t] : kNoLowering, false, false, evidence);
    if (evidence) {
      const uint32_t f = verdict[t];
      if (f) atomicAdd(evidence + 8, 1ull);
    }
  }
}

__global__ void conformance_pool_kernel(PoolDev p, uint32_t* verdict, unsigned long long* evidence) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < p.num_traces; t += gridDim.x * blockDim.x) {
    const uint32_t ev = p.hdr[(size_t)t * H_NWORDS + H_EVCOUNT];
    EvIn in{p.ev + (size_t)t * p.EPT * 2, ev < p.EPT ? ev : p.EPT};
    uint8_t fs[32];
    for (uint32_t c = 0; c < p.C; ++c) fs[c] = (uint8_t)(p.clm[((size_t)t * p.C + c) * 8] & 0xFFu);
    const uint32_t low = p.hdr[(size_t)t * H_NWORDS + H_POLICY] & 0xFFu;
    // a drained or overflowed ring cannot be compared with the final states
    const bool drained = p.hdr[(size_t)t * H_NWORDS + H_EVDRAINED] != 0;
    const bool complete = ev <= p.EPT && !drained;
    verdict[t] = check_trace(in, complete ? fs : nullptr, p.C, low, ev > p.EPT, drained, evidence);
    if (evidence && verdict[t]) atomicAdd(evidence + 8, 1ull);
  }
}

}  // namespace

cudaError_t launch_conformance_array(const void* events, const uint32_t* offsets, uint32_t T,
                                     const uint8_t* final_states, uint32_t C, const uint8_t* lowering,
                                     uint32_t* verdict, unsigned long long* evidence, cudaStream_t st) {
  g_launches += 1;
  const uint32_t grid = (T + 127) / 128 < 148 * 16 ? (T + 127) / 128 : 148 * 16;
  conformance_array_kernel<<<grid > 0 ? grid : 1, 128, 0, st>>>(
      reinterpret_cast<const uint4*>(events), offsets, T, final_states, C, lowering, verdict, evidence);
  return cudaGetLastError();
}

cudaError_t launch_conformance_pool(const PoolDev& p, uint32_t* verdict, unsigned long long* evidence,
                                    cudaStream_t st) {
  g_launches += 1;
  const uint32_t grid = (p.num_traces + 127) / 128 < 148 * 16 ? (p.num_traces + 127) / 128 : 148 * 16;
  conformance_pool_kernel<<<grid, 128, 0, st>>>(p, verdict, evidence);
  return cudaGetLastError();
}

}  // namespace rkc
