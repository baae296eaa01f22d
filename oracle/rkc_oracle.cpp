/*
 * rkc_oracle.cpp -- plain, slow, single-threaded-per-trace CPU ORACLE of the
 * resident-KV-claim contract (arxiv/paper_2605_24259, "Resident KV Claims").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2605_24259_b200/, include/rkc.h, librkc.so) never
 * links, imports or calls it, and this file includes nothing from the
 * product path: every struct, enum value and layout below is written out
 * again here from DESIGN.md section "Semantics" (the reading of the paper).
 *
 * Style on purpose: array-of-structs state, std::vector, linear scans, a
 * full std::sort for victim choice, every derived quantity (leading prefix,
 * protected count P, active live A, blocking set) recomputed by brute force
 * from the block table each time it is needed.  No bitmaps, no intrinsics,
 * no incremental bookkeeping.
 *
 * Citations: "P:a-b" = /root/reference/PAPER.md lines a-b (section/table
 * named), "S:a-b" = SPEC.md lines, "Gn" = DESIGN.md ambiguity ledger entry.
 *
 * Parity pins: see DESIGN.md "Oracle pins" -- every function below is pinned
 * by tests/test_oracle_*.py against paper numbers, closed forms, brute force
 * or invariants.  The orderings the paper leaves open are the ledger's
 * readings, each pinned by a closed form or a property the paper states:
 * G1 tail-first stamps by P:615-616 "survived positions form leading ranges"
 * (invariant I11, asserted after every op in check mode) and the L-ORD
 * closed form; G6 soft bucket by the L-SOFT closed form and the exhaustive
 * victim search; G10 auto-demotion order and G18 event order by closed forms
 * (tests/test_oracle_readings.py); G24 block-to-position order by the
 * exhaustive victim search.  tools/oracle_mutants.py flips each of them.
 */
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <tuple>
#include <vector>

namespace {

/* ---------------- vocabulary (DESIGN.md "Semantics" tables) -------------- */
enum : uint8_t { B_FREE = 0, B_CACHED = 1, B_ACTIVE = 2 };
/* claim states, Table 2 "ResidentClaimState"; EMPTY = never submitted */
enum : uint8_t { C_EMPTY = 0, C_ACCEPTED = 1, C_MATERIALIZED = 2, C_DEMOTED = 3,
                 C_EXPIRED = 4, C_REFUSED = 5, C_HARMED = 6 };
/* protection modes, Table 3 */
enum : uint8_t { M_SOFT = 0, M_HARD = 1, M_DEMOTABLE = 2, M_OFFLOADABLE = 3,
                 M_EXPIRING = 4, M_BEST_EFFORT = 5 };
/* request status */
enum : uint8_t { R_EMPTY = 0, R_RUNNING = 1, R_DEFERRED = 2, R_REFUSED = 3, R_COMPLETED = 4 };
/* op kinds */
enum : uint8_t { OP_NOP = 0, OP_SUBMIT = 1, OP_ADMIT = 2, OP_ADVANCE = 3, OP_COMPLETE = 4,
                 OP_INSERT = 5, OP_DEMOTE = 6, OP_TOUCH = 7, OP_HIT_ADMIT = 8 };
/* event types (ClaimEvent; Table 4 required telemetry P:465-479) */
enum : uint8_t { E_CLAIM_ACCEPTED = 1, E_CLAIM_REJECTED = 2, E_CLAIM_MATERIALIZED = 3,
                 E_CLAIM_DEMOTED = 4, E_CLAIM_EXPIRED = 5, E_CLAIM_HARMED = 6,
                 E_ACTIVE_DEFERRED = 7, E_ACTIVE_REFUSED = 8, E_RESIDENT_INSERT_REFUSED = 9,
                 E_WRITE_ADMISSION_DENIED = 10, E_REQUEST_SERVED = 11, E_VICTIMS = 12,
                 E_REUSE_PROBE = 13, E_OP_ERROR = 14, E_PREFIX_HIT = 15 };
/* OP_ERROR codes */
enum : uint8_t { ERR_DUPLICATE_SLOT = 1, ERR_INVALID_ARG = 2, ERR_ILLEGAL_TRANSITION = 3,
                 ERR_UNKNOWN_CLAIM = 4, ERR_UNKNOWN_REQUEST = 5, ERR_NO_CHUNKS_REMAINING = 6,
                 ERR_OBJECT_IN_USE = 7, ERR_SEQ_EXHAUSTED = 8, ERR_UNKNOWN_OP = 9 };
/* claim rejection reasons (G3, G15, G26) */
enum : uint8_t { REJ_IDENTITY = 1, REJ_OBJECT_CLAIMED = 2, REJ_FOOTPRINT = 3, REJ_RESERVE = 4 };
/* refusal / deferral reasons (G7) */
enum : uint8_t { WHY_PROTECTED_RESIDENT = 1, WHY_ACTIVE_CAPACITY = 2, WHY_RESIDENT_RESERVE = 3 };
/* policy bytes */
enum : uint8_t { LOW_CONTRACT = 0, LOW_SOFT = 1, LOW_NATIVE = 2 };
enum : uint8_t { ADMIT_PEAK = 0, ADMIT_NONE = 1, ADMIT_RESERVE = 2 };
enum : uint8_t { ACCEPT_CAPACITY = 0, ACCEPT_RESERVE = 1 };
/* counters */
enum { K_OPS = 0, K_ACCEPTED, K_REJECTED, K_MATERIALIZED, K_DEMOTED_EXPLICIT, K_DEMOTED_AUTO,
       K_EXPIRED, K_HARMED_OBLIGATED, K_HARMED_UNOBLIGATED, K_ADMITTED, K_SERVED,
       K_DEFERRED_PROTECTED, K_DEFERRED_CAPACITY, K_REFUSED_PROTECTED, K_REFUSED_CAPACITY,
       K_INSERTED, K_INSERT_REFUSED, K_WRITE_DENIED, K_VICTIMS_ORDINARY, K_VICTIMS_AFTER_RELEASE,
       K_VICTIMS_CLAIMED, K_BLOCKS_ALLOCATED, K_BLOCKS_CACHED, K_REUSE_PROBES, K_REUSE_TOKENS,
       K_OP_ERRORS, K_STEPS, K_EVENTS, K_PREFIX_HITS, K_HIT_TOKENS, K_ALLOCATIONS,
       K_NCOUNTERS = 32 };

const uint32_t BLOCK_TOKENS = 16;              /* P:615 "16-token block size" */
const uint32_t NO_OBJ_CLAIM = 0xFF;            /* object has no claim binding */
const uint32_t SEQ_LIMIT = 0x3FFFFFFEu;        /* stamps must stay below */
const uint32_t MAX_TOKENS = 1u << 26;          /* prompt / decode / insert limits */

/* ------------------------------ records --------------------------------- */
#pragma pack(push, 1)
struct OpRec { uint8_t kind, a, b, c; uint32_t x, y, z; };                 /* 16 B */
struct TraceCfg { uint32_t U; uint8_t lowering, admit_check, defer_budget, auto_demote,
                  accept_rule, pad[3]; };                                    /* 12 B */
struct EventRec { uint32_t trace, step; uint8_t type, seq, slot, reason; uint32_t mask;
                  uint32_t f[4]; };                                          /* 32 B */
struct BlockView { uint8_t res, owner; uint16_t pad; uint32_t pos, seq; };  /* 12 B */
struct ClaimView { uint8_t state, mode, obj, pad; uint32_t F, R, D, decision_step,
                   protected_blocks; };                                      /* 24 B */
struct RequestView { uint8_t status, write_admit, target, defer_count;
                     uint32_t prompt, chunk, decode, done, live, hit, pad; };  /* 32 B */
struct ObjectView { uint8_t live, claim, pad[2]; uint32_t len, leading; };  /* 12 B */
struct HeaderView { uint32_t seq_ctr, free_blocks, alive, protected_total; }; /* 16 B */
#pragma pack(pop)
static_assert(sizeof(OpRec) == 16, "op");
static_assert(sizeof(TraceCfg) == 12, "cfg");
static_assert(sizeof(EventRec) == 32, "event");
static_assert(sizeof(BlockView) == 12, "bv");
static_assert(sizeof(ClaimView) == 24, "cv");
static_assert(sizeof(RequestView) == 32, "rv");
static_assert(sizeof(ObjectView) == 12, "ov");

struct Block { uint8_t res = B_FREE; uint8_t owner = 0; uint32_t pos = 0; uint32_t seq = 0; };
struct Object { bool live = false; uint32_t claim = NO_OBJ_CLAIM; uint32_t len = 0; };
struct Claim { uint8_t state = C_EMPTY, mode = 0, obj = 0; uint32_t F = 0, R = 0, D = 0,
               decision_step = 0; };
/* hit: leading blocks of the target object shared by a prefix hit (NEXT f3,
 * G28); live counts only the request's own (exclusive) blocks. */
struct Request { uint8_t status = R_EMPTY, write_admit = 0, target = 0, defer_count = 0;
                 uint32_t prompt = 0, chunk = 0, decode = 0, done = 0, live = 0, hit = 0; };

struct Dims { uint32_t N, C, Q, O; };

/* One independent allocator trace (one paged KV pool), "Instances are
 * independent".  All state lives here. */
struct Trace {
  uint32_t id = 0;
  TraceCfg cfg{};
  Dims dims{};
  std::vector<Block> blk;
  std::vector<Object> obj;
  std::vector<Claim> clm;
  std::vector<Request> req;
  uint32_t seq_ctr = 0;
  uint32_t ctr[K_NCOUNTERS] = {};
  std::vector<EventRec> events;
  uint32_t t = 0;          /* current step index */
  uint32_t ev_seq = 0;     /* emission index within (trace, step), G18 */
  bool check = false;      /* assert invariants I1-I11 after every op */
  bool injected = false;   /* state imported from views (I11 holds only for states it built) */
  int violation = 0;       /* first invariant violated (1..9), 0 = none */
  std::vector<uint32_t> lead_prev;  /* I8 bookkeeping (debug mode only) */

  void init(uint32_t trace_id, const TraceCfg& c, const Dims& d) {
    id = trace_id; cfg = c; dims = d;
    blk.assign(cfg.U, Block{});
    obj.assign(d.O, Object{});
    clm.assign(d.C, Claim{});
    req.assign(d.Q, Request{});
  }

  /* ---------------------------- telemetry -------------------------------- */
  void emit(uint8_t type, uint32_t slot, uint32_t reason, uint32_t mask,
            uint32_t f0 = 0, uint32_t f1 = 0, uint32_t f2 = 0, uint32_t f3 = 0) {
    EventRec e;
    std::memset(&e, 0, sizeof e);
    e.trace = id; e.step = t; e.type = type; e.seq = (uint8_t)ev_seq++;
    e.slot = (uint8_t)slot; e.reason = (uint8_t)reason; e.mask = mask;
    e.f[0] = f0; e.f[1] = f1; e.f[2] = f2; e.f[3] = f3;
    events.push_back(e);
    ctr[K_EVENTS]++;
  }
  void op_error(const OpRec& op, uint8_t code) {
    emit(E_OP_ERROR, op.a, code, 0, op.kind);
    ctr[K_OP_ERRORS]++;
  }

  /* -------------------- derived predicates (8c.3) ------------------------ */
  /* obligated(mode): Table 3 -- hard/demotable/offloadable/expiring carry a
   * preservation obligation; soft_priority "not a hard claim", best_effort
   * "telemetry only".  offloadable has no offload tier here and
   * is treated as obligated (G11). */
  static bool obligated(uint8_t mode) {
    return mode == M_HARD || mode == M_DEMOTABLE || mode == M_OFFLOADABLE || mode == M_EXPIRING;
  }
  /* A claim carries runtime responsibility only while accepted. */
  bool live_claim(uint32_t c) const {
    return c < clm.size() && (clm[c].state == C_ACCEPTED || clm[c].state == C_MATERIALIZED);
  }
  /* The claim bound to the owner object of cached block b, or NO_OBJ_CLAIM. */
  uint32_t claim_of_block(uint32_t b) const {
    if (blk[b].res != B_CACHED) return NO_OBJ_CLAIM;
    return obj[blk[b].owner].claim;
  }
  /* claimed(b): covered by a live claim's footprint (G12). */
  bool claimed(uint32_t b) const {
    uint32_t c = claim_of_block(b);
    return c != NO_OBJ_CLAIM && live_claim(c) && blk[b].pos < clm[c].F;
  }
  /* protected(b): hard resident victim exclusion (Table 5 "Resident victim
   * exclusion"; BlockPool touch probe P:953-959), only under the
   * contract lowering (G6). */
  bool is_protected(uint32_t b) const {
    if (cfg.lowering != LOW_CONTRACT || !claimed(b) || pinned(b)) return false;
    return obligated(clm[claim_of_block(b)].mode);
  }
  /* pin_prefix(o): the longest prefix of object o shared by a running
   * request's prefix hit (NEXT f3, "a leading-prefix hit", P:953
   * BlockPool.touch; G28): the refcount of block (o, p) is the number of
   * running requests with target o and hit > p. */
  uint32_t pin_prefix(uint32_t o) const {
    uint32_t m = 0;
    for (const Request& r : req)
      if (r.status == R_RUNNING && r.target == o && r.hit > m) m = r.hit;
    return m;
  }
  /* pinned(b): a cached block some running request executes on (refcount
   * > 0).  It is active live KV of that request, never a victim, and is
   * counted in A, not in P (G29). */
  bool pinned(uint32_t b) const {
    return blk[b].res == B_CACHED && blk[b].pos < pin_prefix(blk[b].owner);
  }
  /* Allocation class (G1, G2, G6): 0 free (key block id), 1 ordinary cached
   * (key LRU stamp), 2 soft-priority cached (evicted after all class 1,
   * S:181); -1 not a candidate (active or protected). */
  int alloc_class(uint32_t b) const {
    if (blk[b].res == B_FREE) return 0;
    if (blk[b].res == B_ACTIVE) return -1;
    if (pinned(b) || is_protected(b)) return -1;
    if (cfg.lowering != LOW_NATIVE && claimed(b)) {
      uint8_t m = clm[claim_of_block(b)].mode;
      if (m == M_SOFT || (cfg.lowering == LOW_SOFT && obligated(m))) return 2;
    }
    return 1;
  }
  /* leading(o): first missing position of the object's chain; "cached tokens
   * equal the first missing block times the 16-token block size",
   * "leading contiguous survival".  0 if the object never became
   * reusable; never exceeds len. */
  uint32_t leading(uint32_t o) const {
    if (!obj[o].live) return 0;
    /* one pass over the blocks marks the cached positions of o, then the
     * first unmarked position is the answer (same definition, O(N + len)) */
    std::vector<char> present(obj[o].len, 0);
    for (uint32_t b = 0; b < blk.size(); ++b)
      if (blk[b].res == B_CACHED && blk[b].owner == o && blk[b].pos < obj[o].len) present[blk[b].pos] = 1;
    for (uint32_t p = 0; p < obj[o].len; ++p)
      if (!present[p]) return p;
    return obj[o].len;
  }
  /* P = protected_resident_kv. */
  uint32_t protected_total() const {
    uint32_t n = 0;
    for (uint32_t b = 0; b < blk.size(); ++b) n += is_protected(b) ? 1u : 0u;
    return n;
  }
  uint32_t protected_of_claim(uint32_t c) const {
    uint32_t n = 0;
    for (uint32_t b = 0; b < blk.size(); ++b)
      if (is_protected(b) && claim_of_block(b) == c) ++n;
    return n;
  }
  /* Active live KV currently held: sum over running requests (G4),
   * plus every pinned cached block, counted once however many requests share
   * it (G29). */
  uint32_t alive() const {
    uint32_t n = 0;
    for (const Request& r : req) if (r.status == R_RUNNING) n += r.live;
    for (uint32_t b = 0; b < blk.size(); ++b) n += pinned(b) ? 1u : 0u;
    return n;
  }
  /* blocking_claim_ids: every claim with >= 1 protected block, ascending slot
   * = acceptance order (G7, G22). */
  uint32_t blocking_mask() const {
    uint32_t m = 0;
    for (uint32_t c = 0; c < clm.size(); ++c)
      if (protected_of_claim(c) > 0) m |= 1u << c;
    return m;
  }
  /* The resident reserve (NEXT f4): "Resident reserve -- Resident survives;
   * active work that cannot fit is refused.  Modeled reserve action" (Table 5,
   * P:573-574); "a static block count subtracted from usable headroom at
   * admission; default reserve equals the sum of accepted hard-protected
   * footprints".  Here: the footprints F of the live obligated claims when the
   * contract lowering protects them, 0 otherwise (G34). */
  uint64_t reserve_total() const {
    if (cfg.lowering != LOW_CONTRACT) return 0;
    uint64_t r = 0;
    for (uint32_t c = 0; c < clm.size(); ++c)
      if (live_claim(c) && obligated(clm[c].mode)) r += clm[c].F;
    return r;
  }
  /* the claims holding the reserve, ascending slot (the attribution of a
   * reserve refusal) */
  uint32_t reserve_mask() const {
    uint32_t m = 0;
    if (cfg.lowering != LOW_CONTRACT) return 0;
    for (uint32_t c = 0; c < clm.size(); ++c)
      if (live_claim(c) && obligated(clm[c].mode)) m |= 1u << c;
    return m;
  }
  uint32_t count_res(uint8_t res) const {
    uint32_t n = 0;
    for (const Block& b : blk) n += b.res == res ? 1u : 0u;
    return n;
  }

  /* release the active live blocks of request r to FREE (deferral / refusal /
   * no-admit completion, G9) */
  void release_request_blocks(uint32_t r) {
    for (Block& b : blk)
      if (b.res == B_ACTIVE && b.owner == r) { b.res = B_FREE; b.owner = 0; b.pos = 0; b.seq = 0; }
    req[r].live = 0;
    req[r].hit = 0;  /* its prefix-hit references are dropped too (G28) */
  }

  /* -------------------------- arbiter (8c.4) ------------------------------ */
  /* arbitrate(need): the feasibility boundary
   *     protected_resident_kv + active_live_kv <= usable_kv   (sec. 3.4)
   * with A = active live already held + need (G4).  On infeasibility: the
   * optional relax action (demote demotable claims before loss, P:423-424,
   * P:589-591, G10), else an explicit active-side action -- deferral or
   * refusal with blocking-claim attribution and the capacity proof
   * (P:477-479), or an insert refusal (G17).
   * requester: request slot, or -1 for INSERT of object `ins_obj`.
   * Returns true iff FEASIBLE. */
  bool arbitrate(uint32_t need, int requester, uint32_t ins_obj) {
    const uint32_t U = cfg.U;
    uint32_t P = protected_total();
    const uint64_t A = (uint64_t)alive() + need;
    if ((uint64_t)P + A <= U) return true;
    if (cfg.lowering == LOW_CONTRACT && cfg.auto_demote) {
      /* demotable live claims holding protected blocks, ascending slot */
      std::vector<uint32_t> dm; std::vector<uint32_t> g;
      for (uint32_t c = 0; c < clm.size(); ++c) {
        if (live_claim(c) && clm[c].mode == M_DEMOTABLE) {
          uint32_t pc = protected_of_claim(c);
          if (pc > 0) { dm.push_back(c); g.push_back(pc); }
        }
      }
      uint64_t rem = P; size_t j = 0; bool found = false;
      for (j = 0; j < dm.size(); ++j) {
        rem -= g[j];
        if (rem + A <= U) { found = true; break; }
      }
      if (found) {
        for (size_t i = 0; i <= j; ++i) {
          clm[dm[i]].state = C_DEMOTED;
          emit(E_CLAIM_DEMOTED, dm[i], 1 /*auto*/, 0, clm[dm[i]].obj, g[i]);
          ctr[K_DEMOTED_AUTO]++;
        }
        return true;
      }
    }
    const bool resident_cause = (A <= U) && P > 0;
    return infeasible(resident_cause ? WHY_PROTECTED_RESIDENT : WHY_ACTIVE_CAPACITY,
                      resident_cause ? blocking_mask() : 0u, P, A, requester, ins_obj);
  }

  /* admission under the resident reserve (admit_check = RESERVE, f4, G34):
   * the request's active live footprint estimate must fit the headroom the
   * reserve leaves, reserve + Alive + need <= U; otherwise the request is
   * deferred or refused with reason RESIDENT_RESERVE, the reserving claims as
   * the blocking set and the proof (reserve, A, U, reserve + A - U) -- or with
   * ACTIVE_CAPACITY and no claims when A > U alone (G7).  No auto-demotion:
   * the reserve is a static admission control. */
  bool admit_reserve(uint32_t need, int requester) {
    const uint64_t Rv = reserve_total();
    const uint64_t A = (uint64_t)alive() + need;
    if (Rv + A <= cfg.U) return true;
    const bool resident_cause = (A <= cfg.U) && Rv > 0;
    return infeasible(resident_cause ? WHY_RESIDENT_RESERVE : WHY_ACTIVE_CAPACITY,
                      resident_cause ? reserve_mask() : 0u, (uint32_t)Rv, A, requester, 0);
  }

  /* the explicit active-side action on an infeasible boundary: an insert
   * refusal (G17), or the request's deferral / refusal (G9) with the
   * capacity proof (P, A, U, shortfall = P + A - U) and attribution */
  bool infeasible(uint8_t why, uint32_t mask, uint32_t P, uint64_t A, int requester,
                  uint32_t ins_obj) {
    const uint32_t U = cfg.U;
    const uint32_t shortfall = (uint32_t)((uint64_t)P + A - U);
    const bool resident_cause = why != WHY_ACTIVE_CAPACITY;
    if (requester < 0) {
      emit(E_RESIDENT_INSERT_REFUSED, ins_obj, why, mask, P, (uint32_t)A, U, shortfall);
      ctr[K_INSERT_REFUSED]++;
      return false;
    }
    Request& r = req[requester];
    release_request_blocks(requester);
    r.done = 0;
    if (r.defer_count < cfg.defer_budget) {
      r.status = R_DEFERRED; r.defer_count++;
      emit(E_ACTIVE_DEFERRED, requester, why, mask, P, (uint32_t)A, U, shortfall);
      ctr[resident_cause ? K_DEFERRED_PROTECTED : K_DEFERRED_CAPACITY]++;
    } else {
      r.status = R_REFUSED;
      emit(E_ACTIVE_REFUSED, requester, why, mask, P, (uint32_t)A, U, shortfall);
      ctr[resident_cause ? K_REFUSED_PROTECTED : K_REFUSED_CAPACITY]++;
    }
    return false;
  }

  /* alloc(k): only after FEASIBLE, so all-or-nothing holds.  Takes
   * the first k candidates in (class, key) order: free blocks first by block
   * id (70 allocated with 20 free and 50 evicted), then ordinary
   * cached blocks oldest stamp first, then soft-priority ones (G1, G2, G6).
   * Protected and active blocks are never candidates.  Returns the
   * taken block ids sorted by block id (G24: the i-th taken block in block-id
   * order receives position base+i).  Emits one VICTIMS summary when cached
   * blocks were taken (G18). */
  std::vector<uint32_t> alloc(uint32_t k, uint32_t slot, uint32_t reason_kind) {
    std::vector<std::tuple<int, uint32_t, uint32_t>> cand;  /* (class, key, block) */
    for (uint32_t b = 0; b < blk.size(); ++b) {
      int cls = alloc_class(b);
      if (cls < 0) continue;
      uint32_t key = cls == 0 ? b : blk[b].seq;
      cand.emplace_back(cls, key, b);
    }
    std::sort(cand.begin(), cand.end());
    std::vector<uint32_t> taken;
    uint32_t ordinary = 0, after_release = 0, claimed_v = 0;
    for (uint32_t i = 0; i < k; ++i) {
      uint32_t b = std::get<2>(cand[i]);
      taken.push_back(b);
      if (blk[b].res == B_CACHED) {
        uint32_t c = obj[blk[b].owner].claim;
        /* victim attribution by the owner object's claim state at this moment
         * (Table 4; S:159 block_loss_after_release) */
        if (c == NO_OBJ_CLAIM || clm[c].state == C_HARMED || clm[c].state == C_REFUSED) ordinary++;
        else if (clm[c].state == C_DEMOTED || clm[c].state == C_EXPIRED) after_release++;
        else claimed_v++;
        if (check && is_protected(b)) violation = violation ? violation : 3; /* I3 */
      }
    }
    std::sort(taken.begin(), taken.end());
    ctr[K_VICTIMS_ORDINARY] += ordinary;
    ctr[K_VICTIMS_AFTER_RELEASE] += after_release;
    ctr[K_VICTIMS_CLAIMED] += claimed_v;
    ctr[K_BLOCKS_ALLOCATED] += k;
    ctr[K_ALLOCATIONS]++;  /* successful alloc calls (measurement: SURVEY 8(d) rows) */
    if (ordinary + after_release + claimed_v > 0)
      emit(E_VICTIMS, slot, reason_kind, 0, ordinary, after_release, claimed_v, k);
    return taken;
  }

  /* -------------------------- ops (8c.5) ---------------------------------- */
  /* SUBMIT: claim decision.  "A runtime is allowed to reject a resident
   * claim. The conformance obligation becomes binding only after the runtime
   * accepts the claim."; decision accepted/rejected with step and
   * reason (Table 2). */
  void op_submit(const OpRec& op) {
    const uint32_t c = op.a, o = op.b, mode = op.c & 0x7Fu;
    const bool id_mismatch = (op.c & 0x80u) != 0;
    const uint32_t F = op.x, R = op.y, D = op.z;
    if (c >= dims.C || o >= dims.O || mode > M_BEST_EFFORT) return op_error(op, ERR_INVALID_ARG);
    if (clm[c].state != C_EMPTY) return op_error(op, ERR_DUPLICATE_SLOT);
    if (F < 1 || R < 1 || R > F || (mode == M_EXPIRING && D == 0)) return op_error(op, ERR_INVALID_ARG);
    uint8_t rej = 0;
    if (id_mismatch) rej = REJ_IDENTITY;                                    /* G26 */
    else if (obj[o].claim != NO_OBJ_CLAIM && live_claim(obj[o].claim)) rej = REJ_OBJECT_CLAIMED; /* G15 */
    else if (F > cfg.U) rej = REJ_FOOTPRINT;
    else if (cfg.accept_rule == ACCEPT_RESERVE && obligated((uint8_t)mode)) {
      /* resident reserve (Table 5 "Resident reserve") */
      uint64_t sum = F;
      for (uint32_t j = 0; j < clm.size(); ++j)
        if (live_claim(j) && obligated(clm[j].mode)) sum += clm[j].F;
      if (sum > cfg.U) rej = REJ_RESERVE;
    }
    Claim& cl = clm[c];
    cl.mode = (uint8_t)mode; cl.obj = (uint8_t)o; cl.F = F; cl.R = R; cl.D = D; cl.decision_step = t;
    if (rej) {
      cl.state = C_REFUSED;
      emit(E_CLAIM_REJECTED, c, rej, 0, o, F, R, D);
      ctr[K_REJECTED]++;
    } else {
      cl.state = C_ACCEPTED;
      obj[o].claim = c;
      emit(E_CLAIM_ACCEPTED, c, 0, 0, o, F, R, D);
      ctr[K_ACCEPTED]++;
    }
  }

  /* peak(r): the request's active live footprint estimate:
   * full attention keeps every chunk live (Table 8). */
  static uint32_t peak_blocks(const Request& r) {
    return (uint32_t)(((uint64_t)r.prompt + r.decode + BLOCK_TOKENS - 1) / BLOCK_TOKENS);
  }

  void op_admit(const OpRec& op) {
    const uint32_t r = op.a, target = op.b, wa = op.c;
    if (r >= dims.Q || target >= dims.O || wa > 1) return op_error(op, ERR_INVALID_ARG);
    if (req[r].status == R_RUNNING || req[r].status == R_DEFERRED) return op_error(op, ERR_DUPLICATE_SLOT);
    if (op.x < 1 || op.y < 1 || op.x > MAX_TOKENS || op.z > MAX_TOKENS) return op_error(op, ERR_INVALID_ARG);
    Request& q = req[r];
    q.status = R_RUNNING; q.write_admit = (uint8_t)wa; q.target = (uint8_t)target; q.defer_count = 0;
    q.prompt = op.x; q.chunk = op.y; q.decode = op.z; q.done = 0; q.live = 0; q.hit = 0;
    ctr[K_ADMITTED]++;
    if (cfg.admit_check == ADMIT_PEAK) arbitrate(peak_blocks(q), (int)r, 0); /* G8 */
    else if (cfg.admit_check == ADMIT_RESERVE) admit_reserve(peak_blocks(q), (int)r);  /* f4 */
  }

  /* HIT_ADMIT (NEXT f3): admission of a request whose prompt begins with
   * object o's content.  The hit is the leading surviving prefix, the
   * materialization surface of P:303-304 and P:614-616 ("cached tokens equal
   * the first missing block times the 16-token block size"), capped so that
   * at least one prompt token is computed: h = min(leading(o),
   * floor((prompt-1)/16)) (G28).  The hit blocks are shared, not allocated:
   * the request starts at done = 16h, owns no block yet, and pins (o, 0..h-1)
   * while it runs.  Pinning moves blocks into A (G29), so the PEAK check
   * (G8) asks for the exclusive peak plus the newly pinned blocks that were
   * candidates before: need = (peak - h) + |[m, h)| - |protected in [m, h)|,
   * m = pin_prefix(o).  A hit refreshes the hit blocks' stamps tail-first,
   * like TOUCH (G23, G30).  Hit requests do not write back (write_admit 0). */
  void op_hit_admit(const OpRec& op) {
    const uint32_t r = op.a, o = op.b;
    if (r >= dims.Q || o >= dims.O || op.c != 0) return op_error(op, ERR_INVALID_ARG);
    if (req[r].status == R_RUNNING || req[r].status == R_DEFERRED) return op_error(op, ERR_DUPLICATE_SLOT);
    if (op.x < 1 || op.y < 1 || op.x > MAX_TOKENS || op.z > MAX_TOKENS) return op_error(op, ERR_INVALID_ARG);
    const uint32_t L = leading(o);
    const uint32_t h = std::min(L, (op.x - 1) / BLOCK_TOKENS);
    if ((uint64_t)seq_ctr + h > SEQ_LIMIT) return op_error(op, ERR_SEQ_EXHAUSTED);
    Request& q = req[r];
    q.status = R_RUNNING; q.write_admit = 0; q.target = (uint8_t)o; q.defer_count = 0;
    q.prompt = op.x; q.chunk = op.y; q.decode = op.z; q.done = 0; q.live = 0; q.hit = 0;
    ctr[K_ADMITTED]++;
    if (cfg.admit_check == ADMIT_PEAK) {
      const uint32_t m = pin_prefix(o);
      uint32_t newpin = 0, newprot = 0;
      for (uint32_t b = 0; b < blk.size(); ++b) {
        if (blk[b].res != B_CACHED || blk[b].owner != o || blk[b].pos < m || blk[b].pos >= h) continue;
        newpin++;
        if (is_protected(b)) newprot++;
      }
      if (!arbitrate(peak_blocks(q) - h + newpin - newprot, (int)r, 0)) return;
    } else if (cfg.admit_check == ADMIT_RESERVE) {
      /* f4: the exclusive part of the peak against the reserve (G34) */
      if (!admit_reserve(peak_blocks(q) - h, (int)r)) return;
    }
    const uint32_t base = seq_ctr;
    for (Block& b : blk)
      if (b.res == B_CACHED && b.owner == o && b.pos < h) b.seq = base + (h - 1 - b.pos);
    seq_ctr += h;
    q.hit = h;
    q.done = h * BLOCK_TOKENS;
    emit(E_PREFIX_HIT, r, 0, 0, o, h, h * BLOCK_TOKENS, L);
    ctr[K_PREFIX_HITS]++;
    ctr[K_HIT_TOKENS] += h * BLOCK_TOKENS;
  }

  /* ADVANCE: one prefill chunk or one decode token (G14).  Live
   * KV accumulates: live = ceil(done/16) (Table 8: 20/40/60/70). */
  void op_advance(const OpRec& op) {
    const uint32_t r = op.a;
    if (r >= dims.Q) return op_error(op, ERR_INVALID_ARG);
    Request& q = req[r];
    if (q.status != R_RUNNING && q.status != R_DEFERRED) return op_error(op, ERR_UNKNOWN_REQUEST);
    if (q.status == R_RUNNING && (uint64_t)q.done >= (uint64_t)q.prompt + q.decode)
      return op_error(op, ERR_NO_CHUNKS_REMAINING);
    if (q.status == R_DEFERRED) {
      /* retry of a deferred request: re-run the admission check (G9) */
      if (cfg.admit_check == ADMIT_PEAK && !arbitrate(peak_blocks(q), (int)r, 0)) return;
      if (cfg.admit_check == ADMIT_RESERVE && !admit_reserve(peak_blocks(q), (int)r)) return;
      q.status = R_RUNNING;
    }
    uint32_t n;
    if (q.done < q.prompt) n = std::min(q.chunk, q.prompt - q.done);
    else n = 1;
    const uint32_t need_total = (uint32_t)(((uint64_t)q.done + n + BLOCK_TOKENS - 1) / BLOCK_TOKENS);
    const uint32_t held = q.hit + q.live;  /* shared hit blocks + own blocks (G28) */
    const uint32_t need = need_total > held ? need_total - held : 0;
    if (need > 0) {
      if (!arbitrate(need, (int)r, 0)) return;
      std::vector<uint32_t> taken = alloc(need, r, 0);
      for (uint32_t i = 0; i < taken.size(); ++i) {
        Block& b = blk[taken[i]];
        b.res = B_ACTIVE; b.owner = (uint8_t)r; b.pos = q.live + i; b.seq = 0;
      }
      q.live += need;
    }
    q.done += n;
  }

  /* COMPLETE: future reusable admission is a separate decision from active
   * allocation (Table 7).  Only full blocks
   * become reusable (G16); stamps tail-first (G1). */
  void op_complete(const OpRec& op) {
    const uint32_t r = op.a;
    if (r >= dims.Q) return op_error(op, ERR_INVALID_ARG);
    Request& q = req[r];
    if (q.status != R_RUNNING) return op_error(op, ERR_UNKNOWN_REQUEST);
    const uint32_t full = q.done / BLOCK_TOKENS;
    const uint32_t o = q.target;
    const bool admitted = q.write_admit && !obj[o].live;
    if (admitted && (uint64_t)seq_ctr + full > SEQ_LIMIT) return op_error(op, ERR_SEQ_EXHAUSTED);
    const uint32_t held = q.live;
    if (admitted) {
      const uint32_t base = seq_ctr;
      for (Block& b : blk) {
        if (b.res != B_ACTIVE || b.owner != r) continue;
        if (b.pos < full) { b.res = B_CACHED; b.owner = (uint8_t)o; b.seq = base + (full - 1 - b.pos); }
        else { b.res = B_FREE; b.owner = 0; b.pos = 0; b.seq = 0; }
      }
      seq_ctr += full;
      obj[o].live = true; obj[o].len = full;
      ctr[K_BLOCKS_CACHED] += full;
    } else {
      release_request_blocks(r);
      emit(E_WRITE_ADMISSION_DENIED, r, q.write_admit ? 1u : 0u, 0, o, held);
      ctr[K_WRITE_DENIED]++;
    }
    emit(E_REQUEST_SERVED, r, admitted ? 1u : 0u, 0, q.done, admitted ? full : 0u, o);
    ctr[K_SERVED]++;
    q.status = R_COMPLETED; q.live = 0; q.hit = 0;
  }

  /* INSERT: resident insertion through the ordinary allocation path (G17). */
  void op_insert(const OpRec& op) {
    const uint32_t o = op.a, n = op.x;
    if (o >= dims.O) return op_error(op, ERR_INVALID_ARG);
    if (obj[o].live) return op_error(op, ERR_OBJECT_IN_USE);
    if (n < 1 || n > MAX_TOKENS) return op_error(op, ERR_INVALID_ARG);
    if ((uint64_t)seq_ctr + n > SEQ_LIMIT) return op_error(op, ERR_SEQ_EXHAUSTED);
    if (!arbitrate(n, -1, o)) return;
    std::vector<uint32_t> taken = alloc(n, o, 1);
    const uint32_t base = seq_ctr;
    for (uint32_t i = 0; i < taken.size(); ++i) {
      Block& b = blk[taken[i]];
      b.res = B_CACHED; b.owner = (uint8_t)o; b.pos = i; b.seq = base + (n - 1 - i);
    }
    seq_ctr += n;
    obj[o].live = true; obj[o].len = n;
    ctr[K_INSERTED]++;
    ctr[K_BLOCKS_CACHED] += n;
  }

  /* DEMOTE: "Accepted claim is demoted, then blocks are lost -- claim_demoted
   * before post-release block loss" (Table 4). */
  void op_demote(const OpRec& op) {
    const uint32_t c = op.a;
    if (c >= dims.C) return op_error(op, ERR_INVALID_ARG);
    if (clm[c].state == C_EMPTY) return op_error(op, ERR_UNKNOWN_CLAIM);
    if (!live_claim(c)) return op_error(op, ERR_ILLEGAL_TRANSITION);
    const uint32_t pc = protected_of_claim(c);
    clm[c].state = C_DEMOTED;
    emit(E_CLAIM_DEMOTED, c, 0 /*explicit*/, 0, clm[c].obj, pc);
    ctr[K_DEMOTED_EXPLICIT]++;
  }

  /* TOUCH: a reuse probe on the materialization surface (P:303-304,
   * P:614-616): hit length = leading prefix, cached tokens = 16 * leading;
   * refreshes the LRU stamps of the leading blocks tail-first (G23). */
  void op_touch(const OpRec& op) {
    const uint32_t o = op.a;
    if (o >= dims.O) return op_error(op, ERR_INVALID_ARG);
    const uint32_t L = leading(o);
    if ((uint64_t)seq_ctr + L > SEQ_LIMIT) return op_error(op, ERR_SEQ_EXHAUSTED);
    const uint32_t base = seq_ctr;
    for (Block& b : blk)
      if (b.res == B_CACHED && b.owner == o && b.pos < L) b.seq = base + (L - 1 - b.pos);
    seq_ctr += L;
    const uint32_t c = obj[o].claim;
    const bool has = c != NO_OBJ_CLAIM;
    const bool sat = has && live_claim(c) && L >= clm[c].R;
    emit(E_REUSE_PROBE, has ? c : 0xFFu, sat ? 1u : 0u, 0, o, L, L * BLOCK_TOKENS, has ? clm[c].R : 0u);
    ctr[K_REUSE_PROBES]++;
    ctr[K_REUSE_TOKENS] += L * BLOCK_TOKENS;
  }

  /* ------------------------- one step (8c.4) ------------------------------ */
  /* Phase order: expiry -> op -> post-op predicate pass (expiry
   * processes first so the release event precedes any loss). */
  void step(const OpRec& op) {
    ev_seq = 0;
    /* 1. expiry: "Runtime responsibility ends at expiry" (Table 3, P:427;
     *    Table 4); at the start of step t with decision+D <= t (G13) */
    for (uint32_t c = 0; c < clm.size(); ++c) {
      if (live_claim(c) && clm[c].D > 0 && (uint64_t)clm[c].decision_step + clm[c].D <= t) {
        const uint32_t pc = protected_of_claim(c);
        clm[c].state = C_EXPIRED;
        emit(E_CLAIM_EXPIRED, c, 0, 0, clm[c].obj, pc, clm[c].decision_step, clm[c].D);
        ctr[K_EXPIRED]++;
      }
    }
    /* 2. dispatch */
    if (op.kind != OP_NOP) ctr[K_OPS]++;
    switch (op.kind) {
      case OP_NOP: break;
      case OP_SUBMIT: op_submit(op); break;
      case OP_ADMIT: op_admit(op); break;
      case OP_ADVANCE: op_advance(op); break;
      case OP_COMPLETE: op_complete(op); break;
      case OP_INSERT: op_insert(op); break;
      case OP_DEMOTE: op_demote(op); break;
      case OP_TOUCH: op_touch(op); break;
      case OP_HIT_ADMIT: op_hit_admit(op); break;
      default: op_error(op, ERR_UNKNOWN_OP); break;
    }
    /* 3. post-op materialization predicate pass, ascending slot:
     *    accepted -> materialized when leading >= R;
     *    materialized -> harmed when the predicate breaks without a prior
     *    release: "claim_harmed with predicate and capacity context" (Table 4,
     *    P:474-476; harm definition; G5). */
    for (uint32_t c = 0; c < clm.size(); ++c) {
      if (!live_claim(c)) continue;
      const uint32_t o = clm[c].obj;
      const uint32_t L = leading(o);
      if (clm[c].state == C_ACCEPTED && obj[o].live && L >= clm[c].R) {
        clm[c].state = C_MATERIALIZED;
        emit(E_CLAIM_MATERIALIZED, c, 0, 0, L, clm[c].R, L * BLOCK_TOKENS, o);
        ctr[K_MATERIALIZED]++;
      } else if (clm[c].state == C_MATERIALIZED && L < clm[c].R) {
        const bool ob = obligated(clm[c].mode);
        clm[c].state = C_HARMED;
        emit(E_CLAIM_HARMED, c, ob ? 1u : 0u, 0, L, clm[c].R, protected_total(), alive());
        ctr[ob ? K_HARMED_OBLIGATED : K_HARMED_UNOBLIGATED]++;
      }
    }
    ctr[K_STEPS]++;
    if (check) check_invariants();
    ++t;
  }

  /* ----------------------- invariants (8c.7) ------------------------------ */
  void fail(int i) { if (!violation) violation = i; }
  void check_invariants() {
    /* I1 conservation */
    uint32_t nf = count_res(B_FREE), nc = count_res(B_CACHED), na = count_res(B_ACTIVE);
    if (nf + nc + na != cfg.U) fail(1);
    uint32_t held = 0;
    for (const Request& r : req) held += r.live;
    if (na != held) fail(1);
    uint32_t npin = 0;
    for (uint32_t b = 0; b < blk.size(); ++b) npin += pinned(b) ? 1u : 0u;
    if (na + npin != alive()) fail(1);
    /* I10 (f3): a pinned prefix is always fully present (never a victim) */
    for (uint32_t o = 0; o < obj.size(); ++o)
      if (pin_prefix(o) > leading(o)) fail(10);
    /* I2 (owner,pos) unique among non-free blocks; cached pos < len */
    std::vector<std::tuple<uint8_t, uint8_t, uint32_t>> ids;
    for (uint32_t i = 0; i < blk.size(); ++i) {
      if (blk[i].res == B_FREE) continue;
      if (blk[i].res == B_CACHED && (!obj[blk[i].owner].live || blk[i].pos >= obj[blk[i].owner].len)) fail(2);
      ids.emplace_back(blk[i].res, blk[i].owner, blk[i].pos);
    }
    std::sort(ids.begin(), ids.end());
    for (size_t i = 1; i < ids.size(); ++i) if (ids[i] == ids[i - 1]) fail(2);
    /* I8: leading never increases while the object stays live (chains only
     * shrink after insertion) */
    if (lead_prev.size() != obj.size()) lead_prev.assign(obj.size(), 0xFFFFFFFFu);
    for (uint32_t o = 0; o < obj.size(); ++o) {
      if (!obj[o].live) continue;
      uint32_t L = leading(o);
      if (lead_prev[o] != 0xFFFFFFFFu && L > lead_prev[o]) fail(8);
      lead_prev[o] = L;
    }
    /* I4: contract traces never harm an obligated claim (north star) */
    for (const EventRec& e : events)
      if (e.step == t && e.type == E_CLAIM_HARMED && e.reason == 1 && cfg.lowering == LOW_CONTRACT) fail(4);
    /* I11: "survived positions form leading ranges" (the paper's
     * ledger check on its vLLM traces): every live object's cached
     * positions are exactly [0, leading(o)).  This is what the tail-first
     * stamp order (G1) guarantees -- eviction eats each chain from its tail;
     * a head-first order would strand the tail.  (Injected states, e.g. L6's
     * position-0 hole, are exempt: they were not built by the runtime.) */
    if (!injected) {
      std::vector<uint32_t> cached(obj.size(), 0);
      for (const Block& b : blk) if (b.res == B_CACHED) cached[b.owner]++;
      for (uint32_t o = 0; o < obj.size(); ++o)
        if (obj[o].live && cached[o] != leading(o)) fail(11);
    }
    /* I9: running requests hold exactly ceil(done/16) blocks */
    for (const Request& r : req)
      if (r.status == R_RUNNING && r.hit + r.live != (r.done + BLOCK_TOKENS - 1) / BLOCK_TOKENS) fail(9);
  }
};

/* ------------------------------- batch ----------------------------------- */
struct Batch {
  Dims dims{};
  std::vector<Trace> traces;
};

}  // namespace

/* =========================== extern "C" surface ========================== */
extern "C" {

/* Create a batch of independent traces.  cfgs: num_traces 12-byte trace
 * configs {u32 U; u8 lowering, admit_check, defer_budget, auto_demote,
 * accept_rule, pad[3]}.  Returns NULL on invalid sizes. */
void* oracle_batch_create(const void* cfgs, uint32_t num_traces, uint32_t N, uint32_t C,
                          uint32_t Q, uint32_t O) {
  if (C < 1 || C > 32 || Q < 1 || Q > 32 || O < 1 || O > 128 || N < 1) return nullptr;
  Batch* b = new Batch();
  b->dims = Dims{N, C, Q, O};
  b->traces.resize(num_traces);
  const TraceCfg* tc = (const TraceCfg*)cfgs;
  for (uint32_t i = 0; i < num_traces; ++i) {
    if (tc[i].U < 1 || tc[i].U > N) { delete b; return nullptr; }
    b->traces[i].init(i, tc[i], b->dims);
  }
  return b;
}

void oracle_batch_free(void* h) { delete (Batch*)h; }

/* Run T lockstep steps.  ops: [T][op_stride] 16-byte records, trace i reads
 * column trace_offset + i.  Traces are independent, so a pool of
 * nthreads workers takes whole traces; each trace runs single-threaded.
 * check != 0 asserts invariants after every op.  Returns the number of
 * traces with an invariant violation. */
int oracle_batch_run(void* h, const void* ops, uint32_t T, uint64_t op_stride,
                     uint64_t trace_offset, int nthreads, int check) {
  Batch* b = (Batch*)h;
  const OpRec* rec = (const OpRec*)ops;
  const uint32_t n = (uint32_t)b->traces.size();
  std::atomic<uint32_t> next{0};
  auto worker = [&]() {
    for (;;) {
      uint32_t i = next.fetch_add(1);
      if (i >= n) return;
      Trace& tr = b->traces[i];
      tr.check = check != 0;
      for (uint32_t s = 0; s < T; ++s) tr.step(rec[(uint64_t)s * op_stride + trace_offset + i]);
    }
  };
  if (nthreads <= 1) worker();
  else {
    std::vector<std::thread> th;
    for (int k = 0; k < nthreads; ++k) th.emplace_back(worker);
    for (auto& x : th) x.join();
  }
  int bad = 0;
  for (auto& tr : b->traces) bad += tr.violation ? 1 : 0;
  return bad;
}

int oracle_trace_violation(void* h, uint32_t trace) { return ((Batch*)h)->traces[trace].violation; }

uint64_t oracle_batch_num_events(void* h) {
  uint64_t n = 0;
  for (auto& tr : ((Batch*)h)->traces) n += tr.events.size();
  return n;
}

/* Events in (trace, step, seq) order, 32 bytes each. */
uint64_t oracle_batch_events(void* h, void* out, uint64_t cap) {
  uint64_t k = 0;
  EventRec* o = (EventRec*)out;
  for (auto& tr : ((Batch*)h)->traces)
    for (auto& e : tr.events) { if (k < cap) o[k] = e; ++k; }
  return k;
}

/* counters: [num_traces][32] u32 */
void oracle_batch_counters(void* h, uint32_t* out) {
  Batch* b = (Batch*)h;
  for (size_t i = 0; i < b->traces.size(); ++i)
    std::memcpy(out + i * K_NCOUNTERS, b->traces[i].ctr, sizeof(uint32_t) * K_NCOUNTERS);
}

/* Neutral state views of one trace (layouts in DESIGN.md "State views").
 * blocks: [N] (entries >= U are zero), claims [C], requests [Q], objects [O]. */
void oracle_trace_export(void* h, uint32_t trace, void* hdr, void* blocks, void* claims,
                         void* requests, void* objects) {
  Batch* b = (Batch*)h;
  const Trace& tr = b->traces[trace];
  HeaderView* hv = (HeaderView*)hdr;
  hv->seq_ctr = tr.seq_ctr; hv->free_blocks = tr.count_res(B_FREE); hv->alive = tr.alive();
  hv->protected_total = tr.protected_total();
  BlockView* bv = (BlockView*)blocks;
  std::memset(bv, 0, sizeof(BlockView) * b->dims.N);
  for (uint32_t i = 0; i < tr.blk.size(); ++i) {
    bv[i].res = tr.blk[i].res;
    bv[i].owner = tr.blk[i].res == B_FREE ? 0 : tr.blk[i].owner;
    bv[i].pos = tr.blk[i].res == B_FREE ? 0 : tr.blk[i].pos;
    bv[i].seq = tr.blk[i].res == B_CACHED ? tr.blk[i].seq : 0;
  }
  ClaimView* cv = (ClaimView*)claims;
  for (uint32_t c = 0; c < b->dims.C; ++c) {
    std::memset(&cv[c], 0, sizeof(ClaimView));
    const Claim& k = tr.clm[c];
    cv[c].state = k.state; cv[c].mode = k.mode; cv[c].obj = k.obj;
    cv[c].F = k.F; cv[c].R = k.R; cv[c].D = k.D; cv[c].decision_step = k.decision_step;
    cv[c].protected_blocks = tr.protected_of_claim(c);
  }
  RequestView* rv = (RequestView*)requests;
  for (uint32_t r = 0; r < b->dims.Q; ++r) {
    std::memset(&rv[r], 0, sizeof(RequestView));
    const Request& q = tr.req[r];
    rv[r].status = q.status; rv[r].write_admit = q.write_admit; rv[r].target = q.target;
    rv[r].defer_count = q.defer_count; rv[r].prompt = q.prompt; rv[r].chunk = q.chunk;
    rv[r].decode = q.decode; rv[r].done = q.done; rv[r].live = q.live; rv[r].hit = q.hit;
  }
  ObjectView* ov = (ObjectView*)objects;
  for (uint32_t o = 0; o < b->dims.O; ++o) {
    std::memset(&ov[o], 0, sizeof(ObjectView));
    ov[o].live = tr.obj[o].live ? 1 : 0; ov[o].claim = (uint8_t)tr.obj[o].claim;
    ov[o].len = tr.obj[o].len; ov[o].leading = tr.leading(o);
  }
}

/* State injection (test-only, e.g. the L6 fixture P:1047-1050): overwrite a
 * trace's state from views; derived values are recomputed on demand anyway.
 * `step` sets the trace's step counter. */
void oracle_trace_import(void* h, uint32_t trace, uint32_t seq_ctr, uint32_t step,
                         const void* blocks, const void* claims, const void* requests,
                         const void* objects) {
  Batch* b = (Batch*)h;
  Trace& tr = b->traces[trace];
  tr.seq_ctr = seq_ctr; tr.t = step;
  tr.injected = true;
  const BlockView* bv = (const BlockView*)blocks;
  for (uint32_t i = 0; i < tr.blk.size(); ++i) {
    tr.blk[i].res = bv[i].res; tr.blk[i].owner = bv[i].owner; tr.blk[i].pos = bv[i].pos;
    tr.blk[i].seq = bv[i].seq;
  }
  const ClaimView* cv = (const ClaimView*)claims;
  for (uint32_t c = 0; c < b->dims.C; ++c) {
    Claim& k = tr.clm[c];
    k.state = cv[c].state; k.mode = cv[c].mode; k.obj = cv[c].obj; k.F = cv[c].F; k.R = cv[c].R;
    k.D = cv[c].D; k.decision_step = cv[c].decision_step;
  }
  const RequestView* rv = (const RequestView*)requests;
  for (uint32_t r = 0; r < b->dims.Q; ++r) {
    Request& q = tr.req[r];
    q.status = rv[r].status; q.write_admit = rv[r].write_admit; q.target = rv[r].target;
    q.defer_count = rv[r].defer_count; q.prompt = rv[r].prompt; q.chunk = rv[r].chunk;
    q.decode = rv[r].decode; q.done = rv[r].done; q.live = rv[r].live; q.hit = rv[r].hit;
  }
  const ObjectView* ov = (const ObjectView*)objects;
  for (uint32_t o = 0; o < b->dims.O; ++o) {
    tr.obj[o].live = ov[o].live != 0; tr.obj[o].claim = ov[o].claim; tr.obj[o].len = ov[o].len;
  }
}

/* The predicate alone on an explicit survivor set: leading =
 * first missing position among [0, len). Used by the Q1 / L6 fixtures. */
uint32_t oracle_leading_of_positions(const uint32_t* positions, uint32_t n, uint32_t len) {
  for (uint32_t p = 0; p < len; ++p) {
    bool present = false;
    for (uint32_t i = 0; i < n; ++i) if (positions[i] == p) { present = true; break; }
    if (!present) return p;
  }
  return len;
}

}  // extern "C"
