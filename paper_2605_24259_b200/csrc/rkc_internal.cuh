// rkc_internal.cuh -- HBM layout of a pool and the device-side constants.
//
// Structure-of-arrays over traces; per trace, block arrays are contiguous so
// one warp streams its pool's block words with coalesced 16-byte loads.
//
//   key  [T][NS] u32   victim-selection key per block (see below)
//   meta [T][NS] u32   residency | owner | position
//   fbm  [T][NS/32]    free bitmap (bit b = block b FREE)
//   hdr  [T]           64 B hot header (U, policy, counts, stamp counter)
//   clm  [T][C]        32 B claim records (lane-per-claim loads)
//   req  [T][Q]        32 B request records
//   obj  [T][O]        8 B object records
//   ctr  [T][32] u32   telemetry counters
//   ev   [T][EPT]      32 B events (per-trace ring; compacted on read)
//
// key encoding (the composite (class, key) order of DESIGN.md 1.2 in one u32):
//   class 0 FREE      : key = block id            (< 2^30)
//   class 1 ordinary  : key = 1<<30 | seq
//   class 2 soft      : key = 2<<30 | seq
//   class 3 protected : key = 3<<30 | seq         (never a candidate)
//   ACTIVE / padding  : key = 0xFFFFFFFF          (never a candidate)
// so "the k smallest candidates" = "the k smallest keys" and the taken set is
// {b : key[b] <= T} for one threshold T (keys are unique).
#pragma once
#include <cstdint>

namespace rkc {

constexpr uint32_t kBlockTokens = 16;
constexpr uint32_t kSeqLimit = 0x3FFFFFFEu;
constexpr uint32_t kMaxTokens = 1u << 26;
constexpr uint32_t kKeyActive = 0xFFFFFFFFu;
constexpr uint32_t kClassShift = 30;
constexpr uint32_t kSeqMask = 0x3FFFFFFFu;
constexpr uint32_t kNoClaim = 0x7Fu;

// meta word: res(2) | owner(7) | pinned(1) | pos(22)  (positions < 2^22 = max pool)
// pinned: a cached block inside the shared prefix of a running prefix-hit
// request (NEXT f3, G28-G29); its key is class 3 (never a candidate)
constexpr uint32_t kResFree = 0, kResCached = 1, kResActive = 2, kResPad = 3;
constexpr uint32_t kMetaPin = 1u << 22;
__host__ __device__ inline uint32_t meta_make(uint32_t res, uint32_t owner, uint32_t pos) {
  return (res << 30) | ((owner & 0x7Fu) << 23) | (pos & 0x3FFFFFu);
}
__host__ __device__ inline uint32_t meta_res(uint32_t m) { return m >> 30; }
__host__ __device__ inline uint32_t meta_owner(uint32_t m) { return (m >> 23) & 0x7Fu; }
__host__ __device__ inline uint32_t meta_pos(uint32_t m) { return m & 0x3FFFFFu; }
__host__ __device__ inline bool meta_pinned(uint32_t m) { return (m & kMetaPin) != 0; }

// object word 0: live(1) | claim(7) | len(24); word 1: leading
__host__ __device__ inline uint32_t obj_make(uint32_t live, uint32_t claim, uint32_t len) {
  return (live << 31) | ((claim & 0x7Fu) << 24) | (len & 0xFFFFFFu);
}
__host__ __device__ inline uint32_t obj_live(uint32_t w) { return w >> 31; }
__host__ __device__ inline uint32_t obj_claim(uint32_t w) { return (w >> 24) & 0x7Fu; }
__host__ __device__ inline uint32_t obj_len(uint32_t w) { return w & 0xFFFFFFu; }

enum : uint32_t { C_EMPTY = 0, C_ACCEPTED = 1, C_MATERIALIZED = 2, C_DEMOTED = 3, C_EXPIRED = 4,
                  C_REFUSED = 5, C_HARMED = 6 };
enum : uint32_t { M_SOFT = 0, M_HARD = 1, M_DEMOTABLE = 2, M_OFFLOADABLE = 3, M_EXPIRING = 4,
                  M_BEST_EFFORT = 5 };
enum : uint32_t { R_EMPTY = 0, R_RUNNING = 1, R_DEFERRED = 2, R_REFUSED = 3, R_COMPLETED = 4 };
enum : uint32_t { OP_NOP = 0, OP_SUBMIT = 1, OP_ADMIT = 2, OP_ADVANCE = 3, OP_COMPLETE = 4,
                  OP_INSERT = 5, OP_DEMOTE = 6, OP_TOUCH = 7, OP_HIT_ADMIT = 8 };
enum : uint32_t { EV_ACCEPTED = 1, EV_REJECTED = 2, EV_MATERIALIZED = 3, EV_DEMOTED = 4,
                  EV_EXPIRED = 5, EV_HARMED = 6, EV_DEFERRED = 7, EV_REFUSED = 8,
                  EV_INSERT_REFUSED = 9, EV_WRITE_DENIED = 10, EV_SERVED = 11, EV_VICTIMS = 12,
                  EV_REUSE_PROBE = 13, EV_OP_ERROR = 14, EV_PREFIX_HIT = 15 };
enum : uint32_t { ERR_DUPLICATE_SLOT = 1, ERR_INVALID_ARG = 2, ERR_ILLEGAL_TRANSITION = 3,
                  ERR_UNKNOWN_CLAIM = 4, ERR_UNKNOWN_REQUEST = 5, ERR_NO_CHUNKS = 6,
                  ERR_OBJECT_IN_USE = 7, ERR_SEQ_EXHAUSTED = 8, ERR_UNKNOWN_OP = 9 };
enum : uint32_t { REJ_IDENTITY = 1, REJ_OBJECT_CLAIMED = 2, REJ_FOOTPRINT = 3, REJ_RESERVE = 4 };
enum : uint32_t { WHY_PROTECTED = 1, WHY_CAPACITY = 2, WHY_RESERVE = 3 };
enum : uint32_t { LOW_CONTRACT = 0, LOW_SOFT = 1, LOW_NATIVE = 2 };
enum : uint32_t { ADMIT_PEAK = 0, ADMIT_NONE = 1, ADMIT_RESERVE = 2 };
enum : uint32_t { ACCEPT_CAPACITY = 0, ACCEPT_RESERVE = 1 };
enum : uint32_t { K_OPS = 0, K_ACCEPTED, K_REJECTED, K_MATERIALIZED, K_DEMOTED_EXPLICIT,
                  K_DEMOTED_AUTO, K_EXPIRED, K_HARMED_OBLIGATED, K_HARMED_UNOBLIGATED,
                  K_ADMITTED, K_SERVED, K_DEFERRED_PROTECTED, K_DEFERRED_CAPACITY,
                  K_REFUSED_PROTECTED, K_REFUSED_CAPACITY, K_INSERTED, K_INSERT_REFUSED,
                  K_WRITE_DENIED, K_VICTIMS_ORDINARY, K_VICTIMS_AFTER_RELEASE, K_VICTIMS_CLAIMED,
                  K_BLOCKS_ALLOCATED, K_BLOCKS_CACHED, K_REUSE_PROBES, K_REUSE_TOKENS,
                  K_OP_ERRORS, K_STEPS, K_EVENTS, K_PREFIX_HITS, K_HIT_TOKENS, K_ALLOCATIONS,
                  K_NCTR = 32 };

// hot header: 16 u32
enum : uint32_t { H_U = 0, H_POLICY = 1, H_ACCEPT = 2, H_SEQ = 3, H_FREE = 4, H_ALIVE = 5,
                  H_P = 6, H_BLOCKMASK = 7, H_NEXT_EXPIRY = 8, H_EVCOUNT = 9, H_HOT = 10,
                  H_EVDRAINED = 12, H_NWORDS = 16 };
// words [0, H_HOT) are the hot header the step kernels carry and write back;
// H_EVCOUNT counts the events in the trace's ring since the last drain,
// H_EVDRAINED the events drained before it (host-side telemetry only)
// H_POLICY bytes: lowering | admit_check << 8 | defer_budget << 16 | auto_demote << 24

// claim record: 8 u32  (w0 = state | mode << 8 | obj << 16)
enum : uint32_t { CL_W0 = 0, CL_F = 1, CL_R = 2, CL_D = 3, CL_DEC = 4, CL_PC = 5 };
// request record: 8 u32 (w0 = status | write_admit << 8 | target << 16 | defer << 24)
// RQ_HIT: leading blocks of the target object shared by a prefix hit (f3);
// RQ_LIVE counts only the request's own blocks
enum : uint32_t { RQ_W0 = 0, RQ_PROMPT = 1, RQ_CHUNK = 2, RQ_DECODE = 3, RQ_DONE = 4,
                  RQ_LIVE = 5, RQ_HIT = 6 };

struct PoolDev {
  uint32_t num_traces, NS, C, Q, O, EPT;
  uint32_t* key;    // [T][NS]
  uint32_t* meta;   // [T][NS]
  uint32_t* fbm;    // [T][NS/32]
  uint32_t* hdr;    // [T][16]
  uint32_t* clm;    // [T][C][8]
  uint32_t* req;    // [T][Q][8]
  uint32_t* obj;    // [T][O][2]
  uint32_t* ctr;    // [T][32]
  uint4* ev;        // [T][EPT][2]
  uint32_t* perm;   // [8][T] 64-B tickets {op, hot header, trace}: heavy trace-steps by op kind
  uint32_t* bcnt;   // [2][8] bucket sizes (double-buffered by step parity)
};

}  // namespace rkc
