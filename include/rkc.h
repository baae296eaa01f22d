/*
 * rkc.h -- C ABI of the B200-native batched resident-KV-claim arbiter
 * (arxiv/paper_2605_24259, "Resident KV Claims").
 *
 * One pool = many independent paged-KV allocator traces (one KV block pool
 * each) replayed in lockstep on one GPU.  One step applies one op per
 * trace and runs, per trace: expiry -> op (claim decision, feasibility check
 * P + A <= U, claim-excluding victim selection, block updates) -> post-op
 * materialization predicate and lifecycle transitions, with claim-level
 * telemetry.  The operations follow the paper's proposed
 * runtime surface (runtime surface table) and claim schema (Table 2,
 * P:376-391).
 *
 * Conventions
 *  - All functions return rkc_status: 0 on success, < 0 on an API error.  An
 *    API error has no side effects on pool state.
 *  - Per-op CONTRACT errors are not API errors: they leave that trace
 *    unchanged and emit an OP_ERROR event.
 *  - Device work is stream-ordered and asynchronous on the cudaStream_t
 *    argument (passed as void*; NULL = legacy default stream).  Pointers
 *    flagged on_device=1 are device pointers that must stay valid until the
 *    stream reaches the call; on_device=0 means host memory, and the call
 *    copies it (pinned memory makes that copy asynchronous).
 *  - A pool handle is used by one host thread at a time.
 *  - Ownership: the library owns all pool state (device memory it allocates
 *    with cudaMalloc on config.device, freed by rkc_pool_destroy).  Caller
 *    buffers are caller-owned.
 *  - Record layouts are little-endian, packed, and documented in DESIGN.md
 *    sec. 1.5 ("Records") and 1.5 ("State views").
 */
#ifndef RKC_H_
#define RKC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RKC_ABI_VERSION 2

#if defined(__GNUC__)
#define RKC_API __attribute__((visibility("default")))
#else
#define RKC_API
#endif

typedef int32_t rkc_status;
#define RKC_OK 0
#define RKC_E_INVAL (-1)     /* bad handle, size, pointer or enum value        */
#define RKC_E_NOMEM (-2)     /* device or host allocation failed               */
#define RKC_E_CUDA (-3)      /* a CUDA runtime call failed                     */
#define RKC_E_OVERFLOW (-4)  /* caller event buffer too small (nothing copied) */
#define RKC_E_LOST (-5)      /* a per-trace event buffer overflowed: events were
                                dropped (counted in counter RKC_CTR_EVENTS)     */
#define RKC_E_STATE (-6)     /* call not valid in the pool's current state     */

/* ---- vocabulary ------------------------------------- */
/* protection modes, Table 3 */
enum { RKC_MODE_SOFT = 0, RKC_MODE_HARD = 1, RKC_MODE_DEMOTABLE = 2, RKC_MODE_OFFLOADABLE = 3,
       RKC_MODE_EXPIRING = 4, RKC_MODE_BEST_EFFORT = 5 };
/* claim states, Table 2; EMPTY = slot never submitted */
enum { RKC_CLAIM_EMPTY = 0, RKC_CLAIM_ACCEPTED = 1, RKC_CLAIM_MATERIALIZED = 2,
       RKC_CLAIM_DEMOTED = 3, RKC_CLAIM_EXPIRED = 4, RKC_CLAIM_REFUSED = 5, RKC_CLAIM_HARMED = 6 };
enum { RKC_REQ_EMPTY = 0, RKC_REQ_RUNNING = 1, RKC_REQ_DEFERRED = 2, RKC_REQ_REFUSED = 3,
       RKC_REQ_COMPLETED = 4 };
/* op kinds */
enum { RKC_OP_NOP = 0, RKC_OP_SUBMIT = 1, RKC_OP_ADMIT = 2, RKC_OP_ADVANCE = 3,
       RKC_OP_COMPLETE = 4, RKC_OP_INSERT = 5, RKC_OP_DEMOTE = 6, RKC_OP_TOUCH = 7,
       /* NEXT f3 (G28-G30): admission of a request whose
        * prompt begins with object b's content.  a = request, b = object,
        * c = 0, x/y/z = prompt/chunk/decode tokens.  The surviving leading
        * prefix h = min(leading(b), (x-1)/16) is shared (pinned while the
        * request runs: counted once in A, never a victim) instead of
        * allocated; the request starts at 16h tokens and does not write back. */
       RKC_OP_HIT_ADMIT = 8 };
#define RKC_SUBMIT_ID_MISMATCH 0x80  /* flag in rkc_op.c of a SUBMIT */
/* event types (ClaimEvent; Table 4 telemetry) */
enum { RKC_EV_CLAIM_ACCEPTED = 1, RKC_EV_CLAIM_REJECTED = 2, RKC_EV_CLAIM_MATERIALIZED = 3,
       RKC_EV_CLAIM_DEMOTED = 4, RKC_EV_CLAIM_EXPIRED = 5, RKC_EV_CLAIM_HARMED = 6,
       RKC_EV_ACTIVE_DEFERRED = 7, RKC_EV_ACTIVE_REFUSED = 8, RKC_EV_RESIDENT_INSERT_REFUSED = 9,
       RKC_EV_WRITE_ADMISSION_DENIED = 10, RKC_EV_REQUEST_SERVED = 11, RKC_EV_VICTIMS = 12,
       RKC_EV_REUSE_PROBE = 13, RKC_EV_OP_ERROR = 14,
       RKC_EV_PREFIX_HIT = 15 /* slot = request; f = {object, h, 16h tokens, leading} */ };
/* refusal reasons (G7) and OP_ERROR codes */
enum { RKC_WHY_PROTECTED_RESIDENT = 1, RKC_WHY_ACTIVE_CAPACITY = 2,
       RKC_WHY_RESIDENT_RESERVE = 3 /* admission under the resident reserve (f4) */ };
enum { RKC_ERR_DUPLICATE_SLOT = 1, RKC_ERR_INVALID_ARG = 2, RKC_ERR_ILLEGAL_TRANSITION = 3,
       RKC_ERR_UNKNOWN_CLAIM = 4, RKC_ERR_UNKNOWN_REQUEST = 5, RKC_ERR_NO_CHUNKS_REMAINING = 6,
       RKC_ERR_OBJECT_IN_USE = 7, RKC_ERR_SEQ_EXHAUSTED = 8, RKC_ERR_UNKNOWN_OP = 9 };
/* policy bytes */
enum { RKC_LOWER_CONTRACT = 0, RKC_LOWER_SOFT = 1, RKC_LOWER_NATIVE = 2 };
enum { RKC_ADMIT_PEAK = 0, RKC_ADMIT_NONE = 1, RKC_ADMIT_RESERVE = 2 /* NEXT f4: resident reserve */ };
enum { RKC_ACCEPT_CAPACITY = 0, RKC_ACCEPT_RESERVE = 1 };

#define RKC_NCTR 32    /* per-trace u32 counters */
enum { RKC_CTR_OPS = 0, RKC_CTR_ACCEPTED, RKC_CTR_REJECTED, RKC_CTR_MATERIALIZED,
       RKC_CTR_DEMOTED_EXPLICIT, RKC_CTR_DEMOTED_AUTO, RKC_CTR_EXPIRED,
       RKC_CTR_HARMED_OBLIGATED, RKC_CTR_HARMED_UNOBLIGATED, RKC_CTR_ADMITTED, RKC_CTR_SERVED,
       RKC_CTR_DEFERRED_PROTECTED, RKC_CTR_DEFERRED_CAPACITY, RKC_CTR_REFUSED_PROTECTED,
       RKC_CTR_REFUSED_CAPACITY, RKC_CTR_INSERTED, RKC_CTR_INSERT_REFUSED, RKC_CTR_WRITE_DENIED,
       RKC_CTR_VICTIMS_ORDINARY, RKC_CTR_VICTIMS_AFTER_RELEASE, RKC_CTR_VICTIMS_CLAIMED,
       RKC_CTR_BLOCKS_ALLOCATED, RKC_CTR_BLOCKS_CACHED, RKC_CTR_REUSE_PROBES,
       RKC_CTR_REUSE_TOKENS, RKC_CTR_OP_ERRORS, RKC_CTR_STEPS, RKC_CTR_EVENTS,
       RKC_CTR_PREFIX_HITS, RKC_CTR_HIT_TOKENS /* f3 */,
       RKC_CTR_ALLOCATIONS /* successful allocations (free-only or evicting) */ };
/* outcome histogram (int64[RKC_NHIST]):
 *   [0, 42)   final claim state (7) x mode (6): index state*6 + mode
 *   [42, 47)  final request status (5)
 *   [48, 80)  sum over traces of each counter
 *   rest 0 */
#define RKC_NHIST 128
#define RKC_HIST_CLAIM 0
#define RKC_HIST_REQ 42
#define RKC_HIST_CTR 48

/* ---- records ----------------------------------------------------------- */
#pragma pack(push, 1)
/* one op for one trace at one step (16 B). a = primary slot (claim for
 * SUBMIT/DEMOTE, request for ADMIT/ADVANCE/COMPLETE, object for INSERT/TOUCH);
 * field meaning per kind in DESIGN.md sec. 1.4. */
typedef struct { uint8_t kind, a, b, c; uint32_t x, y, z; } rkc_op;
/* per-trace config (12 B): usable blocks U and policy */
typedef struct {
  uint32_t usable_blocks;
  uint8_t lowering;      /* RKC_LOWER_*                                        */
  uint8_t admit_check;   /* RKC_ADMIT_* (G8)                                   */
  uint8_t defer_budget;  /* deferrals before refusal (G9)         */
  uint8_t auto_demote;   /* relax action before refusal (G10)       */
  uint8_t accept_rule;   /* RKC_ACCEPT_* (G3; reserve P:573-574)               */
  uint8_t pad[3];
} rkc_trace_config;
/* telemetry record (32 B) */
typedef struct {
  uint32_t trace, step;
  uint8_t type, seq, slot, reason;
  uint32_t mask;         /* blocking claim slots (refusal / deferral)          */
  uint32_t f[4];
} rkc_event;
/* state views (test-only export/import) */
typedef struct { uint8_t res, owner; uint16_t pad; uint32_t pos, seq; } rkc_block_view;
typedef struct { uint8_t state, mode, obj, pad; uint32_t F, R, D, decision_step,
                 protected_blocks; } rkc_claim_view;
typedef struct { uint8_t status, write_admit, target, defer_count;
                 uint32_t prompt, chunk, decode, done, live,
                 hit /* shared prefix blocks (f3); live = own blocks */, pad; } rkc_request_view;
typedef struct { uint8_t live, claim, pad[2]; uint32_t len, leading; } rkc_object_view;
typedef struct { uint32_t seq_ctr, free_blocks, alive, protected_total; } rkc_header_view;
#pragma pack(pop)

/* claim submission (ResidentClaimInput, Table 2) */
typedef struct {
  uint32_t trace;
  uint8_t claim_slot, object_slot, mode, pad;
  uint32_t footprint_blocks;         /* F >= 1                  */
  uint32_t required_leading_blocks;  /* R, 1 <= R <= F            */
  uint32_t duration_steps;           /* D, 0 = none                   */
  uint64_t cache_identity;           /* compared with the pool identity (G26) */
  uint64_t claim_id, owner_scope;    /* opaque, telemetry naming only         */
} rkc_claim_input;
/* active request admission (active live footprint estimate P:1213-1214;
 * future reusable admission decision P:1219-1220) */
typedef struct {
  uint32_t trace;
  uint8_t request_slot, target_object, write_admit, pad;
  uint32_t prompt_tokens, chunk_tokens, decode_tokens;
  uint64_t request_id;               /* opaque, telemetry naming only         */
} rkc_request_input;
/* one staged op for an arbitrary trace */
typedef struct { uint32_t trace; rkc_op op; } rkc_trace_op;

/* pool configuration */
typedef struct {
  uint32_t num_traces;
  uint32_t max_blocks;        /* N: per-trace capacity, 1 <= U <= N <= 2^22   */
  uint32_t max_claims;        /* C <= 32                                        */
  uint32_t max_requests;      /* Q <= 32                                        */
  uint32_t max_objects;       /* O <= 128                                       */
  uint32_t events_per_trace;  /* per-trace telemetry buffer capacity            */
  uint64_t pool_identity;     /* CacheIdentity hash of the pool     */
  int32_t device;             /* CUDA device ordinal                            */
  uint32_t flags;             /* reserved, 0                                    */
} rkc_pool_config;

typedef struct rkc_pool rkc_pool;   /* opaque, library-owned */

RKC_API int rkc_abi_version(void);
RKC_API const char* rkc_status_string(rkc_status s);

/* Create a pool: allocates and initialises every trace (all blocks FREE, no
 * claims / requests / objects, step 0).  The pool carries the runtime
 * surface's "Usable KV capacity and headroom" (runtime-surface table: per
 * trace U = usable_kv of the boundary) and the "Cache-equivalence
 * identity" claims are compared against (G26).
 * per_trace: host array of config->num_traces configs (U, policy bytes),
 * read during the call only; the library owns every device buffer it
 * allocates until rkc_pool_destroy.  Errors (no side effects): RKC_E_INVAL on
 * out-of-range sizes or policy bytes, RKC_E_NOMEM, RKC_E_CUDA.  On error *out
 * is NULL.  The caller's current CUDA device is left unchanged. */
RKC_API rkc_status rkc_pool_create(const rkc_pool_config* config, const rkc_trace_config* per_trace,
                           rkc_pool** out);
RKC_API rkc_status rkc_pool_destroy(rkc_pool* pool);
/* Re-initialise every trace to its created state (stream-ordered). */
RKC_API rkc_status rkc_pool_reset(rkc_pool* pool, void* stream);
/* Pool sizes and the step counter (host, synchronous). */
RKC_API rkc_status rkc_pool_info(const rkc_pool* pool, rkc_pool_config* config_out, uint64_t* step_out,
                         uint64_t* device_bytes_out);

/* Stage SUBMIT ops (claim decision) for the next single step.  A
 * trace may receive at most one staged op per step; with host input, a
 * second one for the same trace -- in this call or in any host staging call
 * since the last step -- is RKC_E_INVAL with nothing staged (device input:
 * see rkc_op_stage).  Identity mismatch is folded into the op (G26). */
RKC_API rkc_status rkc_claim_submit(rkc_pool* pool, const rkc_claim_input* claims, uint32_t n,
                            int on_device, void* stream);
/* Stage ADMIT ops: active request admission with the runtime surface's
 * "Active live footprint estimate -- how much KV the active request must hold
 * while being served" (runtime-surface table), checked at admission against
 * the boundary P:504 under admit_check=PEAK (G8), and the "Future reusable
 * admission decision" write_admit.  Host or device
 * input array of n records; same staging rules and errors as
 * rkc_claim_submit. */
RKC_API rkc_status rkc_request_admit(rkc_pool* pool, const rkc_request_input* reqs, uint32_t n,
                             int on_device, void* stream);
/* Stage arbitrary ops (ADVANCE / COMPLETE / INSERT / DEMOTE / TOUCH / ...).
 * on_device=1: conflicts for one trace are resolved on the device -- the op
 * of the earliest staging call, then the lowest input index, wins; the others
 * are dropped and counted (rkc_staging_conflicts).  At most 255 staging calls
 * and 2^24 inputs per call between two steps. */
RKC_API rkc_status rkc_op_stage(rkc_pool* pool, const rkc_trace_op* ops, uint32_t n, int on_device,
                        void* stream);

/* Run num_steps lockstep steps.  One step per trace is the phase order
 * expiry -> op -> post-op materialization pass around the
 * feasibility boundary "protected_resident_kv + active_live_kv <= usable_kv"
 * (sec. 3.4): when it holds the op is served with ordinary
 * (claim-excluding) eviction; when it does not, "the runtime must choose an
 * explicit action and should report that action at the claim level"
 * -- auto-demotion, deferral or refusal with blocking-claim
 * attribution.
 *   ops == NULL : num_steps must be 1; runs the staged slot, then clears it.
 *   ops != NULL : replay mode; ops is [num_steps][num_traces] rkc_op
 *                 (step-major).  on_device=0: host memory (copied through a
 *                 device staging buffer, pinned host memory overlaps the copy
 *                 with the steps).
 * Every step is one light pass over all traces plus a step grid over the
 * traces whose op needs a warp (pools of <= 1024 blocks: sized by the host
 * from the heavy count the step published three steps earlier, read from a
 * mapped pinned ring -- so in replay mode the call returns only when the
 * device is about three steps from the end of the batch; a stream under graph
 * capture, or a count that does not arrive within a second, falls back to the
 * fixed 9/16 grid).  Results never depend on the grid: items past it run on
 * an overflow kernel.  Errors: RKC_E_INVAL (NULL pool, num_steps != 1 with
 * ops == NULL), RKC_E_STATE (staged ops pending), RKC_E_CUDA (the failing
 * call is named on stderr). */
RKC_API rkc_status rkc_step_batch(rkc_pool* pool, const rkc_op* ops, uint32_t num_steps, int on_device,
                          void* stream);

/* Telemetry read.
 *   counters_out: [num_traces][RKC_NCTR] u32 or NULL
 *   events_out:   events in (trace, step, seq) order, capacity events_cap, or
 *                 NULL (then only *events_written = total is reported)
 *   hist_out:     int64[RKC_NHIST] outcome histogram or NULL
 *   on_device:    outputs are device pointers (else host; the call then
 *                 synchronises the stream)
 *   drain:        empty the per-trace event rings after a successful read;
 *                 later reads return only events emitted after the drain
 *                 (RKC_CTR_EVENTS stays the emitted total since creation /
 *                 reset, and rkc_pool_conformance then checks the drained
 *                 traces from "unknown" claim states, without the
 *                 final-state comparison)
 * RKC_E_OVERFLOW: events_cap < total -- nothing copied, *events_written =
 * total.  RKC_E_LOST: some trace overflowed events_per_trace (outputs are
 * still written; the counter RKC_CTR_EVENTS holds the emitted total).
 * Outputs are caller-owned; the call runs on the pool's device (the caller's
 * current device is left unchanged) and is bracketed by an NVTX range, as is
 * rkc_step_batch. */
RKC_API rkc_status rkc_telemetry_read(rkc_pool* pool, uint32_t* counters_out, rkc_event* events_out,
                              uint64_t events_cap, uint64_t* events_written, int64_t* hist_out,
                              int on_device, int drain, void* stream);

/* Test-only neutral state views of traces [trace_begin, trace_begin+n)
 * (host buffers; synchronous).  blocks: [n][max_blocks], claims [n][C],
 * requests [n][Q], objects [n][O], headers [n]. */
RKC_API rkc_status rkc_state_export(rkc_pool* pool, uint32_t trace_begin, uint32_t n,
                            rkc_header_view* headers, rkc_block_view* blocks,
                            rkc_claim_view* claims, rkc_request_view* requests,
                            rkc_object_view* objects);
/* Test-only state injection (e.g. the L6 fixture): derived
 * device state (keys, protected counts, free bitmap, header counts) is
 * recomputed from the views, and the leading prefix of every live object
 * (the materialization predicate) by a kernel on the device.
 * seq_ctr per trace from headers[i].seq_ctr.  Every view is validated first
 * (states / modes / statuses in range, owner < O or Q, claim < C or 0xFF,
 * cached pos < len of a live object): RKC_E_INVAL with nothing written. */
RKC_API rkc_status rkc_state_import(rkc_pool* pool, uint32_t trace_begin, uint32_t n,
                            const rkc_header_view* headers, const rkc_block_view* blocks,
                            const rkc_claim_view* claims, const rkc_request_view* requests,
                            const rkc_object_view* objects);

/* ---- conformance ---------------------------
 * Per-trace replay of the claim-level event stream reconstructing every
 * claim's lifecycle.  verdict bit set = check FAILED for that trace. */
#define RKC_CHECK_L1 0x01u   /* harm only after acceptance                */
#define RKC_CHECK_L2 0x02u   /* write-admission denial followed by service        */
#define RKC_CHECK_L3 0x04u   /* refusal capacity proof and blocking attribution   */
#define RKC_CHECK_L45 0x08u  /* release (demote / expire) before loss, no harm    */
#define RKC_CHECK_L6 0x10u   /* materialization predicate consistency             */
#define RKC_CHECK_L7 0x20u   /* lifecycle legality / reconstruction = final state */
#define RKC_CHECK_I4 0x40u   /* contract lowering never harms an obligated claim  */
#define RKC_CHECK_LOST 0x80u /* the trace's event ring overflowed                 */
/* evidence int64[RKC_NEVIDENCE]: accepted, materialized, harmed, refusals
 * (incl. deferrals and insert refusals), attributed refusals, victims,
 * after-release victims, write-admission denials, failing traces */
#define RKC_NEVIDENCE 9
/* Check a compacted event stream (device pointers): events in (trace, step,
 * seq) order, offsets [num_traces+1] exclusive prefix, optional final claim
 * states [num_traces][claims_per_trace] (u8) and lowering bytes [num_traces]
 * (I4 is checked only when lowering is given).  verdict_out [num_traces] u32
 * and evidence_out int64[RKC_NEVIDENCE] are device pointers (evidence is
 * accumulated: zero it first).  Legal lifecycle per S:44 / S:66-68 (accepted
 * -> harmed included). */
RKC_API rkc_status rkc_conformance_check(const rkc_event* events, const uint32_t* offsets,
                                         uint32_t num_traces, const uint8_t* final_claim_states,
                                         uint32_t claims_per_trace, const uint8_t* lowering,
                                         uint32_t* verdict_out, int64_t* evidence_out, void* stream);
/* Check a pool's own event rings against its final claim table (device
 * outputs; a trace whose ring overflowed or was drained reports LOST /
 * skips the final-state comparison). */
RKC_API rkc_status rkc_pool_conformance(rkc_pool* pool, uint32_t* verdict_out, int64_t* evidence_out,
                                        void* stream);

/* Number of staged ops dropped because another op for the same trace was
 * already staged in this step (device-side staging conflicts). */
RKC_API rkc_status rkc_staging_conflicts(rkc_pool* pool, uint64_t* out);
/* Number of kernels this library has launched since it was loaded (all
 * pools, all streams): evidence for benchmark launch counts. */
RKC_API unsigned long long rkc_launch_count(void);
/* Test-only: set the pool step counter (e.g. after rkc_state_import). */
RKC_API rkc_status rkc_state_set_step(rkc_pool* pool, uint64_t step);

#ifdef __cplusplus
}
#endif
#endif /* RKC_H_ */
