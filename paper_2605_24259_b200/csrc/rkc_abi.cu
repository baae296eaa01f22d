// rkc_abi.cu -- the C ABI (include/rkc.h): pool memory, staging, replay,
// telemetry compaction (K2), outcome histogram (K3), test-only state views.
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>
#include <nvtx3/nvToolsExt.h>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/rkc.h"
#include "rkc_internal.cuh"

#ifndef RKC_GRID_PACING
#define RKC_GRID_PACING 1   // round 2: c5 927 -> 902 us per lockstep step, c8 123 -> 114
#endif
#ifndef RKC_PACE_SHIFT
#define RKC_PACE_SHIFT 6   // margin 1/64 of the traces (1/32: +0.4 %, 1/16: +2.2 % on c5)
#endif
#ifndef RKC_PACE_HOST_OPS
#define RKC_PACE_HOST_OPS 1   // pace the grid in the host-op-stream replay too
#endif
#ifndef RKC_PACE_LAG
#define RKC_PACE_LAG 3   // steps between a published heavy count and the grid it sizes
#endif
#ifndef RKC_PACE_FLOOR
#define RKC_PACE_FLOOR 1024   // constant part of the margin (items)
#endif
namespace rkc {
#define RKC_DECLARE_STEP(ns) \
  namespace ns { cudaError_t launch_step(const PoolDev&, const void*, uint32_t, cudaStream_t, uint32_t, \
                                         unsigned long long*, uint32_t); }
RKC_DECLARE_STEP(small_o64)
RKC_DECLARE_STEP(small_o128)
RKC_DECLARE_STEP(big_o64)
RKC_DECLARE_STEP(big_o128)
#undef RKC_DECLARE_STEP
std::atomic<unsigned long long> g_launches{0};  // kernels this library launched

// one lockstep step = light pass + step kernel (+ the overflow kernel for
// small pools), from the build of the pool's size class: <= 1024 blocks (keys
// staged in shared memory) or more, and <= 64 object slots (32 resident CTAs
// per SM) or up to 128
static cudaError_t launch_step(const PoolDev& p, const void* ops_step, uint32_t step, cudaStream_t st,
                               uint32_t main_items = 0, unsigned long long* host_heavy = nullptr,
                               uint32_t tag_hi = 0) {
  g_launches += p.NS <= 1024 ? 3 : 2;
  if (p.NS <= 1024)
    return p.O <= 64 ? small_o64::launch_step(p, ops_step, step, st, main_items, host_heavy, tag_hi)
                     : small_o128::launch_step(p, ops_step, step, st, main_items, host_heavy, tag_hi);
  return p.O <= 64 ? big_o64::launch_step(p, ops_step, step, st, main_items, host_heavy, tag_hi)
                   : big_o128::launch_step(p, ops_step, step, st, main_items, host_heavy, tag_hi);
}
cudaError_t launch_conformance_array(const void* events, const uint32_t* offsets, uint32_t T,
                                     const uint8_t* final_states, uint32_t C, const uint8_t* lowering,
                                     uint32_t* verdict, unsigned long long* evidence, cudaStream_t st);
cudaError_t launch_conformance_pool(const PoolDev& p, uint32_t* verdict, unsigned long long* evidence,
                                    cudaStream_t st);
}

using namespace rkc;

struct rkc_pool {
  rkc_pool_config cfg;
  PoolDev d;
  uint32_t* tcfg = nullptr;      // [T][3] device copy of per-trace configs
  uint4* staged = nullptr;       // [T] staged ops (NOP = zero)
  uint32_t* owner_tag = nullptr; // [T] staging conflict resolution
  unsigned long long* conflicts = nullptr;
  uint32_t* counts = nullptr;    // [T+1] compaction counts / offsets
  uint32_t* offsets = nullptr;   // [T+1]
  uint32_t* flags = nullptr;     // [4] lost flag etc.
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  uint4* replay_buf[2] = {nullptr, nullptr};
  void* scratch = nullptr;       // grow-only device staging for host-side telemetry outputs
  size_t scratch_bytes = 0;
  size_t replay_steps = 0;       // steps per replay staging buffer
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr};
  cudaEvent_t ev_free[2] = {nullptr, nullptr};
  std::vector<void*> allocs;
  // grid pacing (small pools): the step kernel publishes each step's heavy
  // count into this mapped host ring; rkc_step_batch sizes the one-warp step
  // grid of step s from the count of step s - kPaceLag (plus a margin)
  // instead of launching 9/16 of the traces every step
  unsigned long long* heavy_host = nullptr;  // [64] (step << 32) | count, mapped
  unsigned long long* heavy_dev = nullptr;   // its device alias
  uint32_t pace_epoch = 0;                   // rkc_step_batch calls (tags the ring entries)
  uint64_t step = 0;
  uint32_t stage_calls = 0;      // staging calls since the last step
  bool staged_any = false;
  std::vector<uint8_t> host_staged;  // traces staged from host input since the last step
  size_t device_bytes = 0;
};

// Every entry point runs on the pool's device and leaves the caller's current
// device as it found it.
struct DeviceGuard {
  int prev = -1;
  bool changed = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) changed = cudaSetDevice(dev) == cudaSuccess;
    cudaGetLastError();
  }
  ~DeviceGuard() { if (changed) cudaSetDevice(prev); }
};
#define RKC_ON_DEVICE(pool) DeviceGuard rkc_guard_((pool)->cfg.device)

// NVTX range for profilers (header-only NVTX3: no cost without a tool attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// a failed CUDA call returns RKC_E_CUDA and names itself on stderr (the
// status code alone cannot say which call or which CUDA error it was)
#define CUDA_TRY(x)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      std::fprintf(stderr, "rkc: %s:%d: %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return RKC_E_CUDA;                                                                   \
    }                                                                                      \
  } while (0)

namespace {

constexpr uint32_t kThreads = 256;

// pool reset: block words four at a time (NS is a multiple of 128), 32-bit
// index math while the word count fits
__global__ void init_blocks_kernel(PoolDev p, const uint32_t* tcfg) {
  const size_t total4 = (size_t)p.num_traces * (p.NS / 4);
  const uint32_t ns4 = p.NS / 4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total4;
       i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t t = total4 < (1ull << 32) ? (uint32_t)i / ns4 : (uint32_t)(i / ns4);
    const uint32_t b = (uint32_t)(i - (size_t)t * ns4) * 4;
    const uint32_t U = tcfg[t * 3];
    uint4 k, m;
    k.x = b < U ? b : kKeyActive;
    k.y = b + 1 < U ? b + 1 : kKeyActive;
    k.z = b + 2 < U ? b + 2 : kKeyActive;
    k.w = b + 3 < U ? b + 3 : kKeyActive;
    const uint32_t mf = meta_make(kResFree, 0, 0), mp = meta_make(kResPad, 0, 0);
    m.x = b < U ? mf : mp;
    m.y = b + 1 < U ? mf : mp;
    m.z = b + 2 < U ? mf : mp;
    m.w = b + 3 < U ? mf : mp;
    reinterpret_cast<uint4*>(p.key)[i] = k;
    reinterpret_cast<uint4*>(p.meta)[i] = m;
  }
  const size_t nw = (size_t)p.num_traces * (p.NS / 32);
  const uint32_t ns32 = p.NS / 32;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nw;
       i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(i / ns32), w = (uint32_t)(i % ns32);
    const uint32_t U = tcfg[t * 3];
    const uint32_t lo = w * 32;
    uint32_t word = 0;
    if (U >= lo + 32) word = 0xFFFFFFFFu;
    else if (U > lo) word = (1u << (U - lo)) - 1u;
    p.fbm[i] = word;
  }
}

// headers (one thread per trace) and object records (element-parallel); the
// claim / request / counter tables are cleared by memsets in run_init
__global__ void init_tables_kernel(PoolDev p, const uint32_t* tcfg) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < p.num_traces;
       t += gridDim.x * blockDim.x) {
    uint4* h = reinterpret_cast<uint4*>(p.hdr + (size_t)t * H_NWORDS);
    const uint32_t U = tcfg[t * 3];
    h[0] = make_uint4(U, tcfg[t * 3 + 1], tcfg[t * 3 + 2] & 0xFFu, 0u);   // U, policy, accept, seq
    h[1] = make_uint4(U, 0u, 0u, 0u);                                     // free, alive, P, mask
    h[2] = make_uint4(0xFFFFFFFFu, 0u, 0u, 0u);                           // next expiry, events
    h[3] = make_uint4(0u, 0u, 0u, 0u);
  }
  const size_t no = (size_t)p.num_traces * p.O;
  const uint2 empty = make_uint2(obj_make(0, kNoClaim, 0), 0u);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < no; i += (size_t)gridDim.x * blockDim.x)
    reinterpret_cast<uint2*>(p.obj)[i] = empty;
}

__global__ void stage_claim_kernel(const rkc_claim_input* in, uint32_t n, uint64_t identity,
                                   uint32_t T, uint32_t tag_base, uint32_t* owner_tag,
                                   uint4* out_ops, uint32_t* out_trace) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const rkc_claim_input c = in[i];
    const uint32_t mism = c.cache_identity != identity ? 0x80u : 0u;
    out_ops[i] = make_uint4(OP_SUBMIT | ((uint32_t)c.claim_slot << 8) | ((uint32_t)c.object_slot << 16) |
                                (((uint32_t)c.mode | mism) << 24),
                            c.footprint_blocks, c.required_leading_blocks, c.duration_steps);
    out_trace[i] = c.trace;
    if (c.trace < T) atomicMin(owner_tag + c.trace, tag_base + i);
  }
}
__global__ void stage_request_kernel(const rkc_request_input* in, uint32_t n, uint32_t T,
                                     uint32_t tag_base, uint32_t* owner_tag, uint4* out_ops,
                                     uint32_t* out_trace) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const rkc_request_input r = in[i];
    out_ops[i] = make_uint4(OP_ADMIT | ((uint32_t)r.request_slot << 8) |
                                ((uint32_t)r.target_object << 16) | ((uint32_t)r.write_admit << 24),
                            r.prompt_tokens, r.chunk_tokens, r.decode_tokens);
    out_trace[i] = r.trace;
    if (r.trace < T) atomicMin(owner_tag + r.trace, tag_base + i);
  }
}
__global__ void stage_generic_kernel(const rkc_trace_op* in, uint32_t n, uint32_t T,
                                     uint32_t tag_base, uint32_t* owner_tag, uint4* out_ops,
                                     uint32_t* out_trace) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    rkc_trace_op o = in[i];
    uint4 v;
    memcpy(&v, &o.op, 16);
    out_ops[i] = v;
    out_trace[i] = o.trace;
    if (o.trace < T) atomicMin(owner_tag + o.trace, tag_base + i);
  }
}
__global__ void stage_commit_kernel(const uint4* ops, const uint32_t* trace, uint32_t n, uint32_t T,
                                    uint32_t tag_base, const uint32_t* owner_tag, uint4* staged,
                                    unsigned long long* conflicts) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t t = trace[i];
    if (t >= T) { atomicAdd(conflicts, 1ull); continue; }
    if (owner_tag[t] == tag_base + i) staged[t] = ops[i];
    else atomicAdd(conflicts, 1ull);
  }
}

__global__ void event_counts_kernel(PoolDev p, uint32_t* counts, uint32_t* flags) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t <= p.num_traces;
       t += gridDim.x * blockDim.x) {
    if (t == p.num_traces) { counts[t] = 0; continue; }
    const uint32_t ev = p.hdr[(size_t)t * H_NWORDS + H_EVCOUNT];
    counts[t] = ev < p.EPT ? ev : p.EPT;
    if (ev > p.EPT) atomicOr(flags, 1u);
  }
}
// K2: compaction, one warp per trace, events in (trace, step, seq) order
__global__ void event_gather_kernel(PoolDev p, const uint32_t* counts, const uint32_t* offsets,
                                    uint4* out) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < p.num_traces; w += nwarps) {
    const uint32_t n = counts[w] * 2;
    const uint4* src = p.ev + (size_t)w * p.EPT * 2;
    uint4* dst = out + (size_t)offsets[w] * 2;
    for (uint32_t i = lane; i < n; i += 32) dst[i] = src[i];
  }
}
// drain: the ring restarts empty; the drained count moves to H_EVDRAINED so
// the emitted total (RKC_CTR_EVENTS) stays monotonic and the conformance pass
// knows the ring no longer holds the whole history
__global__ void drain_kernel(PoolDev p) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < p.num_traces;
       t += gridDim.x * blockDim.x) {
    uint32_t* h = p.hdr + (size_t)t * H_NWORDS;
    h[H_EVDRAINED] += h[H_EVCOUNT];
    h[H_EVCOUNT] = 0;
  }
}
__global__ void counters_kernel(PoolDev p, uint64_t step, uint32_t* out) {
  const size_t total = (size_t)p.num_traces * K_NCTR;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(i / K_NCTR), k = (uint32_t)(i % K_NCTR);
    uint32_t v = p.ctr[i];
    if (k == K_STEPS) v = (uint32_t)step;
    if (k == K_EVENTS) v = p.hdr[(size_t)t * H_NWORDS + H_EVCOUNT] + p.hdr[(size_t)t * H_NWORDS + H_EVDRAINED];
    out[i] = v;
  }
}
// K3: outcome histogram (final claim state x mode, request status, counter sums)
__global__ void hist_kernel(PoolDev p, uint64_t step, unsigned long long* hist) {
  __shared__ unsigned long long sh[RKC_NHIST];
  for (uint32_t i = threadIdx.x; i < RKC_NHIST; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < p.num_traces;
       t += gridDim.x * blockDim.x) {
    for (uint32_t c = 0; c < p.C; ++c) {
      const uint32_t w0 = p.clm[((size_t)t * p.C + c) * 8];
      const uint32_t st = w0 & 0xFFu, mode = (w0 >> 8) & 0xFFu;
      if (st != C_EMPTY && mode < 6) atomicAdd(&sh[RKC_HIST_CLAIM + st * 6 + mode], 1ull);
    }
    for (uint32_t r = 0; r < p.Q; ++r) {
      const uint32_t st = p.req[((size_t)t * p.Q + r) * 8] & 0xFFu;
      if (st != R_EMPTY) atomicAdd(&sh[RKC_HIST_REQ + st], 1ull);
    }
    for (uint32_t k = 0; k < K_NCTR; ++k) {
      uint64_t v = p.ctr[(size_t)t * K_NCTR + k];
      if (k == K_STEPS) v = step;
      if (k == K_EVENTS) v = (uint64_t)p.hdr[(size_t)t * H_NWORDS + H_EVCOUNT] + p.hdr[(size_t)t * H_NWORDS + H_EVDRAINED];
      if (v) atomicAdd(&sh[RKC_HIST_CTR + k], (unsigned long long)v);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < RKC_NHIST; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

uint32_t grid_for(size_t n, uint32_t threads = kThreads) {
  size_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return (uint32_t)g;
}

rkc_status dev_alloc(rkc_pool* p, void** ptr, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (cudaMalloc(ptr, bytes) != cudaSuccess) {
    cudaGetLastError();
    return RKC_E_NOMEM;
  }
  p->allocs.push_back(*ptr);
  p->device_bytes += bytes;
  return RKC_OK;
}

rkc_status run_init(rkc_pool* p, cudaStream_t st) {
  g_launches += 2;
  init_blocks_kernel<<<grid_for((size_t)p->d.num_traces * p->d.NS / 4), kThreads, 0, st>>>(p->d, p->tcfg);
  init_tables_kernel<<<grid_for((size_t)p->d.num_traces * p->d.O), kThreads, 0, st>>>(p->d, p->tcfg);
  CUDA_TRY(cudaMemsetAsync(p->d.clm, 0, (size_t)p->d.num_traces * p->d.C * 32, st));
  CUDA_TRY(cudaMemsetAsync(p->d.req, 0, (size_t)p->d.num_traces * p->d.Q * 32, st));
  CUDA_TRY(cudaMemsetAsync(p->d.ctr, 0, (size_t)p->d.num_traces * K_NCTR * 4, st));
  CUDA_TRY(cudaMemsetAsync(p->staged, 0, sizeof(uint4) * p->d.num_traces, st));
  CUDA_TRY(cudaMemsetAsync(p->d.bcnt, 0, 16 * 4, st));
  CUDA_TRY(cudaMemsetAsync(p->owner_tag, 0xFF, sizeof(uint32_t) * p->d.num_traces, st));
  CUDA_TRY(cudaGetLastError());
  p->step = 0;
  p->stage_calls = 0;
  p->staged_any = false;
  std::fill(p->host_staged.begin(), p->host_staged.end(), 0);
  return RKC_OK;
}

void free_all(rkc_pool* p) {
  for (void* a : p->allocs) cudaFree(a);
  p->allocs.clear();
  if (p->scratch) cudaFree(p->scratch);
  p->scratch = nullptr;
  p->scratch_bytes = 0;
  for (int i = 0; i < 2; ++i) {
    if (p->ev_copied[i]) cudaEventDestroy(p->ev_copied[i]);
    if (p->ev_free[i]) cudaEventDestroy(p->ev_free[i]);
  }
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  if (p->heavy_host) cudaFreeHost(p->heavy_host);
  p->heavy_host = nullptr;
  p->heavy_dev = nullptr;
}

// device staging for host outputs of rkc_telemetry_read: kept across calls
// (grown when a read needs more), so a host read costs the gather and the
// copy, not an allocation and a mapping of gigabytes every time
rkc_status scratch_for(rkc_pool* p, size_t bytes, cudaStream_t st, void** out) {
  if (bytes > p->scratch_bytes) {
    if (cudaStreamSynchronize(st) != cudaSuccess) return RKC_E_CUDA;
    if (p->scratch) cudaFree(p->scratch);
    p->scratch = nullptr;
    p->scratch_bytes = 0;
    if (cudaMalloc(&p->scratch, bytes) != cudaSuccess) { cudaGetLastError(); return RKC_E_NOMEM; }
    p->scratch_bytes = bytes;
  }
  *out = p->scratch;
  return RKC_OK;
}

// stage n converted ops (device) via the conflict-resolving commit
template <class Kernel, class In>
rkc_status stage_common(rkc_pool* p, Kernel k, const In* in, uint32_t n, int on_device,
                        cudaStream_t st, bool with_identity) {
  if (!p || (!in && n > 0)) return RKC_E_INVAL;
  if (n == 0) return RKC_OK;
  RKC_ON_DEVICE(p);
  if (n >= (1u << 24) || p->stage_calls >= 255) return RKC_E_INVAL;
  const uint32_t T = p->d.num_traces;
  const In* src = in;
  void* tmp_in = nullptr;
  if (!on_device) {
    // host input: reject duplicates / out-of-range traces, within this call
    // and against every host staging call since the last step, with no side
    // effect (device input is resolved on the device, see rkc_op_stage)
    if (p->host_staged.size() != T) p->host_staged.assign(T, 0);
    std::vector<uint8_t> seen(T, 0);
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t t = in[i].trace;
      if (t >= T || seen[t] || p->host_staged[t]) return RKC_E_INVAL;
      seen[t] = 1;
    }
    for (uint32_t i = 0; i < n; ++i) p->host_staged[in[i].trace] = 1;
    CUDA_TRY(cudaMallocAsync(&tmp_in, sizeof(In) * n, st));
    CUDA_TRY(cudaMemcpyAsync(tmp_in, in, sizeof(In) * n, cudaMemcpyHostToDevice, st));
    src = (const In*)tmp_in;
  }
  uint4* ops = nullptr;
  uint32_t* tr = nullptr;
  CUDA_TRY(cudaMallocAsync(&ops, sizeof(uint4) * n, st));
  CUDA_TRY(cudaMallocAsync(&tr, sizeof(uint32_t) * n, st));
  const uint32_t tag_base = p->stage_calls << 24;
  g_launches += 2;
  if constexpr (std::is_same<In, rkc_claim_input>::value)
    k<<<grid_for(n), kThreads, 0, st>>>(src, n, p->cfg.pool_identity, T, tag_base, p->owner_tag, ops, tr);
  else
    k<<<grid_for(n), kThreads, 0, st>>>(src, n, T, tag_base, p->owner_tag, ops, tr);
  stage_commit_kernel<<<grid_for(n), kThreads, 0, st>>>(ops, tr, n, T, tag_base, p->owner_tag,
                                                          p->staged, p->conflicts);
  CUDA_TRY(cudaGetLastError());
  cudaFreeAsync(ops, st);
  cudaFreeAsync(tr, st);
  if (tmp_in) cudaFreeAsync(tmp_in, st);
  (void)with_identity;
  p->stage_calls++;
  p->staged_any = true;
  return RKC_OK;
}

}  // namespace

extern "C" {

int rkc_abi_version(void) { return RKC_ABI_VERSION; }

const char* rkc_status_string(rkc_status s) {
  switch (s) {
    case RKC_OK: return "ok";
    case RKC_E_INVAL: return "invalid argument";
    case RKC_E_NOMEM: return "out of memory";
    case RKC_E_CUDA: return "CUDA error";
    case RKC_E_OVERFLOW: return "event buffer too small";
    case RKC_E_LOST: return "per-trace event buffer overflowed (events dropped)";
    case RKC_E_STATE: return "invalid in current state";
    default: return "unknown status";
  }
}

rkc_status rkc_pool_create(const rkc_pool_config* config, const rkc_trace_config* per_trace,
                           rkc_pool** out) {
  if (!out) return RKC_E_INVAL;
  *out = nullptr;
  if (!config || !per_trace) return RKC_E_INVAL;
  const rkc_pool_config& c = *config;
  if (c.num_traces < 1 || c.max_blocks < 1 || c.max_blocks > (1u << 22) || c.max_claims < 1 ||
      c.max_claims > 32 || c.max_requests < 1 || c.max_requests > 32 || c.max_objects < 1 ||
      c.max_objects > 128 || c.events_per_trace < 1)
    return RKC_E_INVAL;
  for (uint32_t t = 0; t < c.num_traces; ++t) {
    const rkc_trace_config& tc = per_trace[t];
    if (tc.usable_blocks < 1 || tc.usable_blocks > c.max_blocks || tc.lowering > 2 ||
        tc.admit_check > 2 || tc.auto_demote > 1 || tc.accept_rule > 1)
      return RKC_E_INVAL;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || c.device < 0 || c.device >= ndev) {
    cudaGetLastError();
    return c.device < 0 || (ndev > 0 && c.device >= ndev) ? RKC_E_INVAL : RKC_E_CUDA;
  }
  DeviceGuard guard(c.device);
  rkc_pool* p = new (std::nothrow) rkc_pool();
  if (!p) return RKC_E_NOMEM;
  p->cfg = c;
  // per-trace block stride: 128 * VPL for small pools (register-cached
  // selection keys), else a multiple of 128
  uint32_t NS;
  if (c.max_blocks <= 128) NS = 128;
  else if (c.max_blocks <= 256) NS = 256;
  else if (c.max_blocks <= 512) NS = 512;
  else if (c.max_blocks <= 1024) NS = 1024;
  else NS = (c.max_blocks + 127) / 128 * 128;
  const size_t T = c.num_traces;
  PoolDev& d = p->d;
  d.num_traces = c.num_traces; d.NS = NS; d.C = c.max_claims; d.Q = c.max_requests;
  d.O = c.max_objects; d.EPT = c.events_per_trace;
  rkc_status s = RKC_OK;
#define ALLOC(ptr, bytes) \
  if ((s = dev_alloc(p, (void**)&(ptr), (bytes))) != RKC_OK) { free_all(p); delete p; return s; }
  ALLOC(d.key, T * NS * 4);
  ALLOC(d.meta, T * NS * 4);
  ALLOC(d.fbm, T * (NS / 32) * 4);
  ALLOC(d.hdr, T * H_NWORDS * 4);
  ALLOC(d.clm, T * d.C * 32);
  ALLOC(d.req, T * d.Q * 32);
  ALLOC(d.obj, T * d.O * 8);
  ALLOC(d.ctr, T * K_NCTR * 4);
  ALLOC(d.ev, T * (size_t)d.EPT * 32);
  ALLOC(d.perm, T * 8 * 64);   // 64-B tickets (rkc_step_impl.cuh kTicketWords)
  ALLOC(d.bcnt, 16 * 4);
  ALLOC(p->tcfg, T * 12);
  ALLOC(p->staged, T * 16);
  ALLOC(p->owner_tag, T * 4);
  ALLOC(p->conflicts, 8);
  ALLOC(p->counts, (T + 1) * 4);
  ALLOC(p->offsets, (T + 1) * 4);
  ALLOC(p->flags, 16);
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, p->counts, p->offsets, (int)(T + 1));
  p->cub_bytes = cub_bytes;
  ALLOC(p->cub_tmp, cub_bytes);
#undef ALLOC
  std::vector<uint32_t> tc(T * 3);
  for (size_t t = 0; t < T; ++t) {
    const rkc_trace_config& x = per_trace[t];
    tc[t * 3] = x.usable_blocks;
    tc[t * 3 + 1] = (uint32_t)x.lowering | ((uint32_t)x.admit_check << 8) |
                    ((uint32_t)x.defer_budget << 16) | ((uint32_t)x.auto_demote << 24);
    tc[t * 3 + 2] = x.accept_rule;
  }
  if (cudaMemcpy(p->tcfg, tc.data(), T * 12, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(p->conflicts, 0, 8) != cudaSuccess ||
      cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking) != cudaSuccess) {
    free_all(p); delete p; return RKC_E_CUDA;
  }
  for (int i = 0; i < 2; ++i) {
    if (cudaEventCreateWithFlags(&p->ev_copied[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_free[i], cudaEventDisableTiming) != cudaSuccess) {
      free_all(p); delete p; return RKC_E_CUDA;
    }
  }
  if (p->d.NS <= 1024) {  // grid pacing ring (small pools; absent: the fixed 9/16 grid)
    if (cudaHostAlloc((void**)&p->heavy_host, 64 * sizeof(unsigned long long), cudaHostAllocMapped) ==
            cudaSuccess &&
        cudaHostGetDevicePointer((void**)&p->heavy_dev, p->heavy_host, 0) == cudaSuccess) {
      for (int i = 0; i < 64; ++i) p->heavy_host[i] = ~0ull;
    } else {
      cudaGetLastError();
      if (p->heavy_host) cudaFreeHost(p->heavy_host);
      p->heavy_host = nullptr;
      p->heavy_dev = nullptr;
    }
  }
  if ((s = run_init(p, 0)) != RKC_OK || cudaDeviceSynchronize() != cudaSuccess) {
    free_all(p); delete p; return s ? s : RKC_E_CUDA;
  }
  *out = p;
  return RKC_OK;
}

rkc_status rkc_pool_destroy(rkc_pool* pool) {
  if (!pool) return RKC_E_INVAL;
  RKC_ON_DEVICE(pool);
  cudaDeviceSynchronize();
  free_all(pool);
  delete pool;
  return RKC_OK;
}

rkc_status rkc_pool_reset(rkc_pool* pool, void* stream) {
  if (!pool) return RKC_E_INVAL;
  RKC_ON_DEVICE(pool);
  return run_init(pool, (cudaStream_t)stream);
}

rkc_status rkc_pool_info(const rkc_pool* pool, rkc_pool_config* config_out, uint64_t* step_out,
                         uint64_t* device_bytes_out) {
  if (!pool) return RKC_E_INVAL;
  if (config_out) *config_out = pool->cfg;
  if (step_out) *step_out = pool->step;
  if (device_bytes_out) *device_bytes_out = pool->device_bytes;
  return RKC_OK;
}

rkc_status rkc_staging_conflicts(rkc_pool* pool, uint64_t* out) {
  if (!pool || !out) return RKC_E_INVAL;
  RKC_ON_DEVICE(pool);
  unsigned long long v = 0;
  CUDA_TRY(cudaMemcpy(&v, pool->conflicts, 8, cudaMemcpyDeviceToHost));
  *out = v;
  return RKC_OK;
}

rkc_status rkc_claim_submit(rkc_pool* pool, const rkc_claim_input* claims, uint32_t n,
                            int on_device, void* stream) {
  return stage_common(pool, stage_claim_kernel, claims, n, on_device, (cudaStream_t)stream, true);
}
rkc_status rkc_request_admit(rkc_pool* pool, const rkc_request_input* reqs, uint32_t n,
                             int on_device, void* stream) {
  return stage_common(pool, stage_request_kernel, reqs, n, on_device, (cudaStream_t)stream, false);
}
rkc_status rkc_op_stage(rkc_pool* pool, const rkc_trace_op* ops, uint32_t n, int on_device,
                        void* stream) {
  return stage_common(pool, stage_generic_kernel, ops, n, on_device, (cudaStream_t)stream, false);
}

// Grid pacing for small pools: the one-warp step grid of step s is sized from
// the heavy count the step kernel of step s - kPaceLag published (mapped host
// ring), plus a margin; items past it run on the overflow kernel, so a short
// estimate costs time, never correctness.  The first kPaceLag steps of a batch,
// or a ring that does not answer within a second, use the fixed default grid.
namespace {
constexpr uint32_t kPaceLag = RKC_PACE_LAG;
struct Pacer {
  rkc_pool* pool;
  uint64_t first;        // absolute step of the batch's first launch
  bool on = false;
  uint32_t last_h = 0;
  uint32_t tag_hi;       // this batch's epoch << 16
  Pacer(rkc_pool* p, uint64_t s0)
      : pool(p), first(s0), on(p->heavy_host != nullptr && RKC_GRID_PACING),
        tag_hi((++p->pace_epoch & 0xFFFFu) << 16) {}
  // main_items for the launch of absolute step s (0: the default grid)
  uint32_t main_items(uint64_t s) {
    if (!on || s < first + kPaceLag) return 0;
    const uint64_t src = s - kPaceLag;
    volatile unsigned long long* slot = pool->heavy_host + (src & 63u);
    const auto t0 = std::chrono::steady_clock::now();
    unsigned long long v;
    for (uint32_t spin = 0;; ++spin) {
      v = *slot;
      if ((v >> 32) == (tag_hi | (src & 0xFFFFu)) && v != ~0ull) break;
      // the host trails the GPU by kPaceLag steps (milliseconds): after a short
      // spin, poll every 20 us instead of holding a core
      if (spin >= 256) std::this_thread::sleep_for(std::chrono::microseconds(20));
      if ((spin & 63u) == 63u && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(1)) {
        on = false;  // no answer: the default grid for the rest of this batch
        return 0;
      }
    }
    const uint32_t h = (uint32_t)v, T = pool->d.num_traces;
    // margin: 1/2^RKC_PACE_SHIFT of the traces plus twice the growth over the
    // lag (pools fill; the first estimate of a batch has no growth to go on and
    // comes out generous)
    const uint32_t grow = h > last_h ? (h - last_h) * 2 * kPaceLag : 0u;
    last_h = h;
    const uint64_t m = (uint64_t)h + (T >> RKC_PACE_SHIFT) + grow + RKC_PACE_FLOOR;
    return (uint32_t)(m < T ? m : T);
  }
  unsigned long long* ring() const { return on ? pool->heavy_dev : nullptr; }
};
}  // namespace

rkc_status rkc_step_batch(rkc_pool* pool, const rkc_op* ops, uint32_t num_steps, int on_device,
                          void* stream) {
  if (!pool) return RKC_E_INVAL;
  RKC_ON_DEVICE(pool);
  NvtxRange nvtx("rkc_step_batch");
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t T = pool->d.num_traces;
  if (!ops) {
    if (num_steps != 1) return RKC_E_INVAL;
    CUDA_TRY(launch_step(pool->d, pool->staged, (uint32_t)pool->step, st));
    CUDA_TRY(cudaMemsetAsync(pool->staged, 0, sizeof(uint4) * T, st));
    CUDA_TRY(cudaMemsetAsync(pool->owner_tag, 0xFF, sizeof(uint32_t) * T, st));
    pool->step += 1;
    pool->stage_calls = 0;
    pool->staged_any = false;
    std::fill(pool->host_staged.begin(), pool->host_staged.end(), 0);
    return RKC_OK;
  }
  if (pool->staged_any) return RKC_E_STATE;  // staged ops pending: run them first
  if (num_steps == 0) return RKC_OK;
  Pacer pace(pool, pool->step);
  {  // a stream under graph capture runs nothing until the graph launches: no counts to wait for
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      pace.on = false;
    }
  }
  if (on_device) {
    for (uint32_t s = 0; s < num_steps; ++s) {
      const uint32_t mi = pace.main_items(pool->step + s);
      CUDA_TRY(launch_step(pool->d, ops + (size_t)s * T, (uint32_t)(pool->step + s), st, mi, pace.ring(),
                           pace.tag_hi));
    }
    pool->step += num_steps;
    return RKC_OK;
  }
  // host op stream: double-buffered copies on the copy stream overlap the steps
  if (!RKC_PACE_HOST_OPS) pace.on = false;
  if (!pool->replay_buf[0]) {
    size_t per_step = (size_t)T * 16;
    size_t steps = (256ull << 20) / per_step;  // 2 x 256 MB staging buffers
    if (steps < 1) steps = 1;
    pool->replay_steps = steps;
    for (int i = 0; i < 2; ++i) {
      rkc_status s = dev_alloc(pool, (void**)&pool->replay_buf[i], steps * per_step);
      if (s != RKC_OK) return s;
    }
  }
  const size_t chunk = pool->replay_steps;
  CUDA_TRY(cudaEventRecord(pool->ev_free[0], st));
  CUDA_TRY(cudaEventRecord(pool->ev_free[1], st));
  // chunk sizes ramp up (2, 8, 32, ... steps) so the first steps wait for a
  // small copy only; the copy of chunk n + 1 is enqueued before the steps of
  // chunk n are (the grid pacing below blocks the host while it launches
  // them), so every copy overlaps the previous chunk's steps
  size_t ramp = 2;
  auto next_len = [&](uint32_t from) -> uint32_t {
    const size_t lim = ramp < chunk ? ramp : chunk;
    if (ramp < chunk) ramp *= 4;  // (capped: no overflow over many chunks)
    return (uint32_t)((num_steps - from) < lim ? (num_steps - from) : lim);
  };
  auto enqueue_copy = [&](uint32_t from, uint32_t n, int b) -> cudaError_t {
    cudaError_t e = cudaStreamWaitEvent(pool->copy_stream, pool->ev_free[b], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(pool->replay_buf[b], ops + (size_t)from * T, (size_t)n * T * 16,
                          cudaMemcpyHostToDevice, pool->copy_stream);
    if (e == cudaSuccess) e = cudaEventRecord(pool->ev_copied[b], pool->copy_stream);
    return e;
  };
  uint32_t done = 0;
  int buf = 0;
  uint32_t n = next_len(0);
  CUDA_TRY(enqueue_copy(0, n, 0));
  while (done < num_steps) {
    const uint32_t nxt_from = done + n;
    const uint32_t nxt = nxt_from < num_steps ? next_len(nxt_from) : 0u;
    if (nxt) CUDA_TRY(enqueue_copy(nxt_from, nxt, buf ^ 1));
    CUDA_TRY(cudaStreamWaitEvent(st, pool->ev_copied[buf], 0));
    for (uint32_t s = 0; s < n; ++s) {
      const uint32_t mi = pace.main_items(pool->step + done + s);
      CUDA_TRY(launch_step(pool->d, pool->replay_buf[buf] + (size_t)s * T,
                           (uint32_t)(pool->step + done + s), st, mi, pace.ring(), pace.tag_hi));
    }
    CUDA_TRY(cudaEventRecord(pool->ev_free[buf], st));
    done += n;
    n = nxt;
    buf ^= 1;
  }
  pool->step += num_steps;
  return RKC_OK;
}

rkc_status rkc_telemetry_read(rkc_pool* pool, uint32_t* counters_out, rkc_event* events_out,
                              uint64_t events_cap, uint64_t* events_written, int64_t* hist_out,
                              int on_device, int drain, void* stream) {
  if (!pool) return RKC_E_INVAL;
  RKC_ON_DEVICE(pool);
  NvtxRange nvtx("rkc_telemetry_read");
  cudaStream_t st = (cudaStream_t)stream;
  const PoolDev& d = pool->d;
  const size_t T = d.num_traces;
  CUDA_TRY(cudaMemsetAsync(pool->flags, 0, 16, st));
  g_launches += 3;  // counts + 2 cub scan kernels
  event_counts_kernel<<<grid_for(T + 1), kThreads, 0, st>>>(d, pool->counts, pool->flags);
  size_t cb = pool->cub_bytes;
  CUDA_TRY(cub::DeviceScan::ExclusiveSum(pool->cub_tmp, cb, pool->counts, pool->offsets, (int)(T + 1), st));
  uint32_t host_total = 0, host_flags = 0;
  CUDA_TRY(cudaMemcpyAsync(&host_total, pool->offsets + T, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&host_flags, pool->flags, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (events_written) *events_written = host_total;
  if (events_out && host_total > events_cap) return RKC_E_OVERFLOW;
  // host outputs: staged in the pool's grow-only scratch, events first, then counters
  const size_t ev_bytes = (events_out && host_total > 0) ? (size_t)host_total * 32 : 0;
  const size_t ctr_bytes = counters_out ? T * K_NCTR * 4 : 0;
  char* stage = nullptr;
  if (!on_device && ev_bytes + ctr_bytes > 0) {
    rkc_status s = scratch_for(pool, ev_bytes + ctr_bytes, st, (void**)&stage);
    if (s != RKC_OK) return s;
  }
  if (ev_bytes) {
    uint4* dst = on_device ? reinterpret_cast<uint4*>(events_out) : reinterpret_cast<uint4*>(stage);
    g_launches += 1;
    event_gather_kernel<<<grid_for(T * 32), kThreads, 0, st>>>(d, pool->counts, pool->offsets, dst);
    CUDA_TRY(cudaGetLastError());
    if (!on_device)
      CUDA_TRY(cudaMemcpyAsync(events_out, dst, ev_bytes, cudaMemcpyDeviceToHost, st));
  }
  if (counters_out) {
    uint32_t* dst = on_device ? counters_out : reinterpret_cast<uint32_t*>(stage + ev_bytes);
    g_launches += 1;
    counters_kernel<<<grid_for(T * K_NCTR), kThreads, 0, st>>>(d, pool->step, dst);
    if (!on_device)
      CUDA_TRY(cudaMemcpyAsync(counters_out, dst, ctr_bytes, cudaMemcpyDeviceToHost, st));
  }
  if (hist_out) {
    unsigned long long* dst = nullptr;
    if (on_device) dst = reinterpret_cast<unsigned long long*>(hist_out);
    else CUDA_TRY(cudaMallocAsync(&dst, RKC_NHIST * 8, st));
    CUDA_TRY(cudaMemsetAsync(dst, 0, RKC_NHIST * 8, st));
    g_launches += 1;
    hist_kernel<<<grid_for(T), kThreads, 0, st>>>(d, pool->step, dst);
    if (!on_device) {
      CUDA_TRY(cudaMemcpyAsync(hist_out, dst, RKC_NHIST * 8, cudaMemcpyDeviceToHost, st));
      cudaFreeAsync(dst, st);
    }
  }
  if (drain) g_launches += 1;
  if (drain) drain_kernel<<<grid_for(T), kThreads, 0, st>>>(d);
  CUDA_TRY(cudaGetLastError());
  if (!on_device) CUDA_TRY(cudaStreamSynchronize(st));
  return host_flags ? RKC_E_LOST : RKC_OK;
}

// ------------------------- test-only state views -------------------------
static bool live_state_h(uint32_t st) { return st == C_ACCEPTED || st == C_MATERIALIZED; }
static bool obligated_h(uint32_t m) {
  return m == M_HARD || m == M_DEMOTABLE || m == M_OFFLOADABLE || m == M_EXPIRING;
}
static uint32_t claim_class_h(uint32_t mode, uint32_t lowering) {
  if (lowering == LOW_CONTRACT && obligated_h(mode)) return 3;
  if (lowering != LOW_NATIVE && (mode == M_SOFT || (lowering == LOW_SOFT && obligated_h(mode)))) return 2;
  return 1;
}

rkc_status rkc_state_export(rkc_pool* pool, uint32_t trace_begin, uint32_t n,
                            rkc_header_view* headers, rkc_block_view* blocks,
                            rkc_claim_view* claims, rkc_request_view* requests,
                            rkc_object_view* objects) {
  if (!pool || trace_begin + (uint64_t)n > pool->d.num_traces) return RKC_E_INVAL;
  RKC_ON_DEVICE(pool);
  const PoolDev& d = pool->d;
  const uint32_t N = pool->cfg.max_blocks, NS = d.NS;
  std::vector<uint32_t> key((size_t)n * NS), meta((size_t)n * NS), hdr((size_t)n * H_NWORDS),
      clm((size_t)n * d.C * 8), req((size_t)n * d.Q * 8), obj((size_t)n * d.O * 2);
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(key.data(), d.key + (size_t)trace_begin * NS, key.size() * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(meta.data(), d.meta + (size_t)trace_begin * NS, meta.size() * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(hdr.data(), d.hdr + (size_t)trace_begin * H_NWORDS, hdr.size() * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(clm.data(), d.clm + (size_t)trace_begin * d.C * 8, clm.size() * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(req.data(), d.req + (size_t)trace_begin * d.Q * 8, req.size() * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(obj.data(), d.obj + (size_t)trace_begin * d.O * 2, obj.size() * 4, cudaMemcpyDeviceToHost));
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t* h = &hdr[(size_t)i * H_NWORDS];
    if (headers) {
      headers[i].seq_ctr = h[H_SEQ];
      headers[i].free_blocks = h[H_FREE];
      headers[i].alive = h[H_ALIVE];
      headers[i].protected_total = h[H_P];
    }
    if (blocks) {
      for (uint32_t b = 0; b < N; ++b) {
        rkc_block_view& v = blocks[(size_t)i * N + b];
        std::memset(&v, 0, sizeof v);
        const uint32_t m = meta[(size_t)i * NS + b];
        const uint32_t res = meta_res(m);
        if (res == kResPad || res == kResFree) continue;
        v.res = (uint8_t)res;
        v.owner = (uint8_t)meta_owner(m);
        v.pos = meta_pos(m);
        if (res == kResCached) v.seq = key[(size_t)i * NS + b] & kSeqMask;
      }
    }
    if (claims) {
      for (uint32_t c = 0; c < d.C; ++c) {
        const uint32_t* w = &clm[((size_t)i * d.C + c) * 8];
        rkc_claim_view& v = claims[(size_t)i * d.C + c];
        std::memset(&v, 0, sizeof v);
        v.state = w[0] & 0xFF; v.mode = (w[0] >> 8) & 0xFF; v.obj = (w[0] >> 16) & 0xFF;
        v.F = w[CL_F]; v.R = w[CL_R]; v.D = w[CL_D]; v.decision_step = w[CL_DEC];
        v.protected_blocks = w[CL_PC];
      }
    }
    if (requests) {
      for (uint32_t r = 0; r < d.Q; ++r) {
        const uint32_t* w = &req[((size_t)i * d.Q + r) * 8];
        rkc_request_view& v = requests[(size_t)i * d.Q + r];
        std::memset(&v, 0, sizeof v);
        v.status = w[0] & 0xFF; v.write_admit = (w[0] >> 8) & 0xFF; v.target = (w[0] >> 16) & 0xFF;
        v.defer_count = w[0] >> 24;
        v.prompt = w[RQ_PROMPT]; v.chunk = w[RQ_CHUNK]; v.decode = w[RQ_DECODE];
        v.done = w[RQ_DONE]; v.live = w[RQ_LIVE]; v.hit = w[RQ_HIT];
      }
    }
    if (objects) {
      for (uint32_t o = 0; o < d.O; ++o) {
        const uint32_t w0 = obj[((size_t)i * d.O + o) * 2], w1 = obj[((size_t)i * d.O + o) * 2 + 1];
        rkc_object_view& v = objects[(size_t)i * d.O + o];
        std::memset(&v, 0, sizeof v);
        v.live = (uint8_t)obj_live(w0);
        v.claim = obj_claim(w0) == kNoClaim ? 0xFF : (uint8_t)obj_claim(w0);
        v.len = obj_len(w0);
        v.leading = obj_live(w0) ? w1 : 0;
      }
    }
  }
  return RKC_OK;
}

}  // extern "C"

namespace {
// state import, step 1: every view is checked before anything is indexed or
// written (a malformed view is RKC_E_INVAL with no side effect)
static bool views_valid(const rkc_pool* pool, uint32_t U, const rkc_block_view* bv,
                        const rkc_claim_view* cv, const rkc_request_view* rv,
                        const rkc_object_view* ov) {
  const PoolDev& d = pool->d;
  for (uint32_t o = 0; o < d.O; ++o) {
    if (ov[o].live > 1 || ov[o].len >= (1u << 22)) return false;
    if (ov[o].claim != 0xFF && ov[o].claim >= d.C) return false;
  }
  for (uint32_t c = 0; c < d.C; ++c)
    if (cv[c].state > C_HARMED || cv[c].mode > M_BEST_EFFORT || cv[c].obj >= d.O) return false;
  for (uint32_t r = 0; r < d.Q; ++r)
    if (rv[r].status > R_COMPLETED || rv[r].target >= d.O || rv[r].write_admit > 1) return false;
  for (uint32_t b = 0; b < U; ++b) {
    const rkc_block_view& v = bv[b];
    if (v.res == kResCached) {
      if (v.owner >= d.O || v.pos >= ov[v.owner].len || !ov[v.owner].live) return false;
    } else if (v.res == kResActive) {
      if (v.owner >= d.Q || v.pos >= (1u << 22)) return false;
    } else if (v.res != kResFree) {
      return false;
    }
  }
  return true;
}

// state import, step 3 (on the device): the materialization predicate of every
// live object, leading(o) = first position with no cached block of o
// (P:614-618), one CTA per trace, positions marked in a shared window bitmap
__global__ void derive_leading_kernel(PoolDev p, uint32_t trace_begin) {
  constexpr uint32_t kWin = 1u << 15;   // positions per window (4 KB of bits)
  __shared__ uint32_t bits[kWin / 32];
  __shared__ uint32_t first_missing;
  const size_t t = (size_t)trace_begin + blockIdx.x;
  const uint32_t* meta = p.meta + t * p.NS;
  uint2* obj = reinterpret_cast<uint2*>(p.obj) + t * p.O;
  for (uint32_t o = 0; o < p.O; ++o) {
    const uint32_t w0 = obj[o].x;
    if (!obj_live(w0)) continue;
    const uint32_t len = obj_len(w0);
    uint32_t lead = len;
    for (uint32_t w = 0; w < len; w += kWin) {
      for (uint32_t i = threadIdx.x; i < kWin / 32; i += blockDim.x) bits[i] = 0;
      if (threadIdx.x == 0) first_missing = 0xFFFFFFFFu;
      __syncthreads();
      for (uint32_t b = threadIdx.x; b < p.NS; b += blockDim.x) {
        const uint32_t m = meta[b];
        const uint32_t q = meta_pos(m);
        if (meta_res(m) == kResCached && meta_owner(m) == o && q >= w && q < w + kWin)
          atomicOr(&bits[(q - w) >> 5], 1u << ((q - w) & 31u));
      }
      __syncthreads();
      const uint32_t span = min(kWin, len - w);
      for (uint32_t q = threadIdx.x; q < span; q += blockDim.x)
        if (!((bits[q >> 5] >> (q & 31u)) & 1u)) atomicMin(&first_missing, w + q);
      __syncthreads();
      const uint32_t fm = first_missing;
      __syncthreads();
      if (fm != 0xFFFFFFFFu) { lead = fm; break; }
    }
    if (threadIdx.x == 0) obj[o].y = lead;
    __syncthreads();
  }
}

}  // namespace

extern "C" {

rkc_status rkc_state_import(rkc_pool* pool, uint32_t trace_begin, uint32_t n,
                            const rkc_header_view* headers, const rkc_block_view* blocks,
                            const rkc_claim_view* claims, const rkc_request_view* requests,
                            const rkc_object_view* objects) {
  if (!pool || !headers || !blocks || !claims || !requests || !objects ||
      trace_begin + (uint64_t)n > pool->d.num_traces)
    return RKC_E_INVAL;
  if (n == 0) return RKC_OK;
  RKC_ON_DEVICE(pool);
  const PoolDev& d = pool->d;
  const uint32_t N = pool->cfg.max_blocks, NS = d.NS;
  std::vector<uint32_t> hdr((size_t)n * H_NWORDS);
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(hdr.data(), d.hdr + (size_t)trace_begin * H_NWORDS, hdr.size() * 4, cudaMemcpyDeviceToHost));
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t U = hdr[(size_t)i * H_NWORDS + H_U];
    if (!views_valid(pool, U, blocks + (size_t)i * N, claims + (size_t)i * d.C,
                     requests + (size_t)i * d.Q, objects + (size_t)i * d.O))
      return RKC_E_INVAL;
  }
  // step 2 (host): block words with their selection keys, claim / request /
  // object records, and the header counts
  std::vector<uint32_t> key((size_t)n * NS), meta((size_t)n * NS), fbm((size_t)n * NS / 32),
      clm((size_t)n * d.C * 8, 0), req((size_t)n * d.Q * 8, 0), obj((size_t)n * d.O * 2);
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t* h = &hdr[(size_t)i * H_NWORDS];
    const uint32_t U = h[H_U], low = h[H_POLICY] & 0xFF;
    const rkc_block_view* bv = blocks + (size_t)i * N;
    const rkc_claim_view* cv = claims + (size_t)i * d.C;
    const rkc_object_view* ov = objects + (size_t)i * d.O;
    const rkc_request_view* rv = requests + (size_t)i * d.Q;
    std::vector<uint32_t> pc(d.C, 0), pin(d.O, 0);
    // pinned prefix per object: the longest hit of a running request (f3, G28)
    for (uint32_t r = 0; r < d.Q; ++r)
      if (rv[r].status == R_RUNNING) pin[rv[r].target] = std::max(pin[rv[r].target], rv[r].hit);
    uint32_t npinned = 0;
    uint32_t free_cnt = 0;
    for (uint32_t b = 0; b < NS; ++b) {
      const size_t k = (size_t)i * NS + b;
      if (b >= U) { key[k] = kKeyActive; meta[k] = meta_make(kResPad, 0, 0); continue; }
      const rkc_block_view& v = bv[b];
      if (v.res == kResFree) {
        key[k] = b; meta[k] = 0; fbm[k / 32] |= 1u << (b & 31); ++free_cnt;
      } else if (v.res == kResActive) {
        key[k] = kKeyActive; meta[k] = meta_make(kResActive, v.owner, v.pos);
      } else {
        meta[k] = meta_make(kResCached, v.owner, v.pos);
        uint32_t cls = 1;
        const uint32_t cc = ov[v.owner].claim;
        if (v.pos < pin[v.owner]) {
          meta[k] |= kMetaPin;
          cls = 3;
          ++npinned;
        } else {
          if (cc < d.C && live_state_h(cv[cc].state) && v.pos < cv[cc].F) cls = claim_class_h(cv[cc].mode, low);
          if (cls == 3) pc[cc]++;
        }
        key[k] = (cls << kClassShift) | (v.seq & kSeqMask);
      }
    }
    uint32_t P = 0, mask = 0, next_exp = 0xFFFFFFFFu, alive = 0;
    for (uint32_t c = 0; c < d.C; ++c) {
      uint32_t* w = &clm[((size_t)i * d.C + c) * 8];
      w[0] = cv[c].state | (cv[c].mode << 8) | (cv[c].obj << 16);
      w[CL_F] = cv[c].F; w[CL_R] = cv[c].R; w[CL_D] = cv[c].D; w[CL_DEC] = cv[c].decision_step;
      w[CL_PC] = live_state_h(cv[c].state) ? pc[c] : 0;
      P += w[CL_PC];
      if (w[CL_PC]) mask |= 1u << c;
      if (live_state_h(cv[c].state) && cv[c].D > 0) {
        const uint64_t e = (uint64_t)cv[c].decision_step + cv[c].D;
        next_exp = (uint32_t)std::min<uint64_t>(next_exp, std::min<uint64_t>(e, 0xFFFFFFFFull));
      }
    }
    for (uint32_t r = 0; r < d.Q; ++r) {
      uint32_t* w = &req[((size_t)i * d.Q + r) * 8];
      w[0] = rv[r].status | (rv[r].write_admit << 8) | (rv[r].target << 16) | (rv[r].defer_count << 24);
      w[RQ_PROMPT] = rv[r].prompt; w[RQ_CHUNK] = rv[r].chunk; w[RQ_DECODE] = rv[r].decode;
      w[RQ_DONE] = rv[r].done; w[RQ_LIVE] = rv[r].live; w[RQ_HIT] = rv[r].hit;
      if (rv[r].status == R_RUNNING) alive += rv[r].live;
    }
    alive += npinned;
    for (uint32_t o = 0; o < d.O; ++o) {
      obj[((size_t)i * d.O + o) * 2] = obj_make(ov[o].live ? 1 : 0, ov[o].claim == 0xFF ? kNoClaim : ov[o].claim, ov[o].len);
      obj[((size_t)i * d.O + o) * 2 + 1] = 0;   // leading: derived on the device below
    }
    h[H_SEQ] = headers[i].seq_ctr;
    h[H_FREE] = free_cnt;
    h[H_ALIVE] = alive;
    h[H_P] = P;
    h[H_BLOCKMASK] = mask;
    h[H_NEXT_EXPIRY] = next_exp;
  }
  CUDA_TRY(cudaMemcpy(d.key + (size_t)trace_begin * NS, key.data(), key.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(d.meta + (size_t)trace_begin * NS, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(d.fbm + (size_t)trace_begin * (NS / 32), fbm.data(), fbm.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(d.hdr + (size_t)trace_begin * H_NWORDS, hdr.data(), hdr.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(d.clm + (size_t)trace_begin * d.C * 8, clm.data(), clm.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(d.req + (size_t)trace_begin * d.Q * 8, req.data(), req.size() * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(d.obj + (size_t)trace_begin * d.O * 2, obj.data(), obj.size() * 4, cudaMemcpyHostToDevice));
  g_launches += 1;
  derive_leading_kernel<<<n, 256>>>(d, trace_begin);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaDeviceSynchronize());
  return RKC_OK;
}

unsigned long long rkc_launch_count(void) { return g_launches.load(); }

rkc_status rkc_conformance_check(const rkc_event* events, const uint32_t* offsets,
                                 uint32_t num_traces, const uint8_t* final_claim_states,
                                 uint32_t claims_per_trace, const uint8_t* lowering,
                                 uint32_t* verdict_out, int64_t* evidence_out, void* stream) {
  if (!offsets || !verdict_out || claims_per_trace > 32 || (num_traces && !events && false))
    return RKC_E_INVAL;
  if (num_traces == 0) return RKC_OK;
  CUDA_TRY(launch_conformance_array(events, offsets, num_traces, final_claim_states,
                                    claims_per_trace, lowering, verdict_out,
                                    reinterpret_cast<unsigned long long*>(evidence_out),
                                    (cudaStream_t)stream));
  return RKC_OK;
}

rkc_status rkc_pool_conformance(rkc_pool* pool, uint32_t* verdict_out, int64_t* evidence_out,
                                void* stream) {
  if (!pool || !verdict_out) return RKC_E_INVAL;
  RKC_ON_DEVICE(pool);
  CUDA_TRY(launch_conformance_pool(pool->d, verdict_out,
                                   reinterpret_cast<unsigned long long*>(evidence_out),
                                   (cudaStream_t)stream));
  return RKC_OK;
}

// the pool step counter can be set for injected states (test-only)
rkc_status rkc_state_set_step(rkc_pool* pool, uint64_t step) {
  if (!pool) return RKC_E_INVAL;
  pool->step = step;
  return RKC_OK;
}

}  // extern "C"
