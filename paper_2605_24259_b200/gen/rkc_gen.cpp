/*
 * rkc_gen.cpp -- seeded synthetic allocator-trace generator (input only).
 *
 * Shared by the CUDA path, the oracle tests and bench.py.  It holds NONE of
 * the method's arithmetic: it never simulates allocation, feasibility,
 * eviction, materialization or lifecycle outcomes.  It only book-keeps what
 * it has itself issued (which request slots it admitted and not yet
 * completed, which claim/object slots it has handed out) so that ops target
 * plausible slots; ops that land on a slot the runtime has since refused or
 * retired produce deterministic OP_ERROR events on both sides.
 *
 * Randomness: counter-based per trace -- splitmix64(seed ^ trace_id * phi)
 * seeds a xoshiro256** stream -- so any trace range can be generated on any
 * rank/thread and the bytes are identical.
 *
 * The paper gives no workload distribution; the recipes below
 * are DESIGN.md "Input recipe".
 *
 * Record layouts:
 *   op        16 B {u8 kind, a, b, c; u32 x, y, z}
 *   trace cfg 12 B {u32 U; u8 lowering, admit_check, defer_budget,
 *                   auto_demote, accept_rule, pad[3]}
 */
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

#pragma pack(push, 1)
struct Op { uint8_t kind, a, b, c; uint32_t x, y, z; };
struct Cfg { uint32_t U; uint8_t lowering, admit_check, defer_budget, auto_demote, accept_rule, pad[3]; };
#pragma pack(pop)
static_assert(sizeof(Op) == 16, "op");
static_assert(sizeof(Cfg) == 12, "cfg");

enum : uint8_t { NOP = 0, SUBMIT = 1, ADMIT = 2, ADVANCE = 3, COMPLETE = 4, INSERT = 5, DEMOTE = 6, TOUCH = 7,
                 HIT_ADMIT = 8 };

inline uint64_t splitmix64(uint64_t& x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

struct Rng {
  uint64_t s[4];
  Rng(uint64_t seed, uint64_t trace) {
    uint64_t x = seed ^ (trace * 0x9E3779B97F4A7C15ull);
    for (int i = 0; i < 4; ++i) s[i] = splitmix64(x);
  }
  uint64_t next() {  /* xoshiro256** */
    const uint64_t r = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
    return r;
  }
  /* uniform integer in [lo, hi] */
  uint32_t uni(uint32_t lo, uint32_t hi) { return lo + (uint32_t)(next() % ((uint64_t)hi - lo + 1)); }
  double unit() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
  bool bern(double p) { return unit() < p; }
  template <int K> int pick(const double (&w)[K]) {
    double u = unit(), acc = 0;
    for (int i = 0; i < K; ++i) { acc += w[i]; if (u < acc) return i; }
    return K - 1;
  }
};

struct Recipe {
  uint32_t U;
  uint32_t C_lo, C_hi, Q, O;
  uint32_t insert_lo, insert_hi;
  uint32_t prompt_lo, prompt_hi;
  uint32_t chunks[3]; int n_chunks;
  uint32_t decode_hi;
  double op_w[8];          /* NOP SUBMIT ADMIT ADVANCE COMPLETE INSERT DEMOTE TOUCH */
  double mode_w[6];        /* soft hard demotable offloadable expiring best_effort */
  uint32_t exp_D_lo, exp_D_hi;  /* expiring duration */
  uint32_t D_lo, D_hi; double D_zero;  /* other modes */
};

/* c3: 100k traces, 1024-block pool, mixed chunked prefill/decode, 4-16 claims
 * (BASELINE.json configs[2]); c4: 65536-block pool, long shared prefixes with
 * demotion/expiry churn (configs[3]).  c5 = c3 recipe, 10^6 trace ids. */
Recipe recipe(int config, uint32_t N) {
  Recipe r{};
  if (config == 7) {
    /* c7 (parity only): slot stress -- every claim / request / object slot
     * the pool allows (C, Q, O from the caller, up to 32 / 32 / 128), small
     * objects and requests so that many coexist, hard-heavy claims so that
     * refusals carry blocking masks over high claim slots */
    r.U = N; r.C_lo = 32; r.C_hi = 32; r.Q = 32; r.O = 128;
    r.insert_lo = std::max<uint32_t>(1, N / 64); r.insert_hi = std::max<uint32_t>(4, N / 12);
    r.prompt_lo = 16; r.prompt_hi = std::max<uint32_t>(64, N * 4);
    r.chunks[0] = 16; r.chunks[1] = 64; r.chunks[2] = 128; r.n_chunks = 3;
    r.decode_hi = 32;
    const double w[8] = {0.05, 0.14, 0.16, 0.35, 0.06, 0.12, 0.04, 0.08};
    std::memcpy(r.op_w, w, sizeof w);
    const double m[6] = {0.10, 0.45, 0.15, 0.10, 0.10, 0.10};
    std::memcpy(r.mode_w, m, sizeof m);
    r.exp_D_lo = 8; r.exp_D_hi = 64; r.D_lo = 8; r.D_hi = 128; r.D_zero = 0.7;
  } else if (config == 4) {
    r.U = N; r.C_lo = 4; r.C_hi = 16; r.Q = 16; r.O = 128;
    r.insert_lo = 2048; r.insert_hi = 16384;
    r.prompt_lo = 8192; r.prompt_hi = 131072;
    r.chunks[0] = 8192; r.chunks[1] = 16384; r.chunks[2] = 32768; r.n_chunks = 3;
    r.decode_hi = 512;
    const double w[8] = {0.16, 0.06, 0.06, 0.40, 0.06, 0.06, 0.10, 0.10};
    std::memcpy(r.op_w, w, sizeof w);
    const double m[6] = {0.10, 0.15, 0.15, 0.05, 0.50, 0.05};
    std::memcpy(r.mode_w, m, sizeof m);
    r.exp_D_lo = 16; r.exp_D_hi = 128; r.D_lo = 16; r.D_hi = 256; r.D_zero = 0.7;
  } else {
    r.U = N; r.C_lo = 4; r.C_hi = 16; r.Q = 16; r.O = 64;
    r.insert_lo = 8; r.insert_hi = 192;
    r.prompt_lo = 16; r.prompt_hi = 4096;
    r.chunks[0] = 128; r.chunks[1] = 256; r.chunks[2] = 512; r.n_chunks = 3;  /* +1024 below */
    r.decode_hi = 128;
    const double w[8] = {0.17, 0.06, 0.08, 0.45, 0.07, 0.07, 0.03, 0.07};
    std::memcpy(r.op_w, w, sizeof w);
    const double m[6] = {0.15, 0.30, 0.15, 0.10, 0.15, 0.15};
    std::memcpy(r.mode_w, m, sizeof m);
    r.exp_D_lo = 8; r.exp_D_hi = 64; r.D_lo = 8; r.D_hi = 128; r.D_zero = 0.7;
  }
  return r;
}

struct ReqBook { bool active = false; uint32_t remaining = 0; };

void gen_trace(int config, uint64_t seed, uint64_t trace_id, uint32_t T, uint32_t N, uint32_t Cmax,
               uint32_t Qmax, uint32_t Omax, Cfg* cfg_out, Op* ops, uint64_t stride) {
  Rng g(seed, trace_id);
  Recipe rc = recipe(config, N);
  const uint32_t Q = std::min(rc.Q, Qmax), O = std::min(rc.O, Omax);
  Cfg cfg{};
  cfg.U = rc.U;
  { const double w[3] = {0.70, 0.15, 0.15}; cfg.lowering = (uint8_t)g.pick(w); }
  if (config == 8) {  /* c8 (NEXT f4): c3 with resident-reserve admission on 40 % of the traces */
    const double w[3] = {0.40, 0.20, 0.40};
    cfg.admit_check = (uint8_t)g.pick(w);
  } else {
    cfg.admit_check = g.bern(0.8) ? 0 : 1;
  }
  cfg.defer_budget = (uint8_t)g.uni(0, 2);
  cfg.auto_demote = g.bern(0.5) ? 1 : 0;
  cfg.accept_rule = g.bern(0.8) ? 0 : 1;
  *cfg_out = cfg;
  const uint32_t C = std::min(g.uni(rc.C_lo, rc.C_hi), Cmax);

  std::vector<ReqBook> rq(Q);
  std::vector<uint32_t> obj_len(O, 0);   /* generator's intended length, 0 = unused */
  std::vector<uint32_t> known_obj;       /* object slots handed out so far */
  std::vector<uint32_t> claims;          /* claim slots handed out so far */
  uint32_t next_claim = 0, next_obj = 0;

  auto take_obj = [&](uint32_t len) -> int {
    if (next_obj >= O) return -1;
    uint32_t o = next_obj++;
    obj_len[o] = len; known_obj.push_back(o);
    return (int)o;
  };

  for (uint32_t s = 0; s < T; ++s) {
    Op op{};
    int kind = g.pick(rc.op_w);
    /* retarget impossible kinds (a bounded chain, no outcome simulation) */
    for (int hop = 0; hop < 4; ++hop) {
      bool ok = true;
      std::vector<uint32_t> act;
      for (uint32_t r = 0; r < Q; ++r) if (rq[r].active) act.push_back(r);
      if (kind == ADVANCE || kind == COMPLETE) {
        if (act.empty()) { kind = ADMIT; ok = false; }
      } else if (kind == ADMIT) {
        if (act.size() == Q) { kind = ADVANCE; ok = false; }
      } else if (kind == INSERT) {
        if (next_obj >= O) { kind = TOUCH; ok = false; }
      } else if (kind == SUBMIT) {
        if (next_claim >= C) { kind = TOUCH; ok = false; }
      } else if (kind == TOUCH) {
        if (known_obj.empty()) { kind = INSERT; ok = false; }
      } else if (kind == DEMOTE) {
        if (claims.empty()) { kind = SUBMIT; ok = false; }
      }
      if (ok) break;
    }
    std::vector<uint32_t> act;
    for (uint32_t r = 0; r < Q; ++r) if (rq[r].active) act.push_back(r);
    switch (kind) {
      case ADVANCE: {
        if (act.empty()) break;
        uint32_t r = act[g.uni(0, (uint32_t)act.size() - 1)];
        if (rq[r].remaining == 0) {  /* generator believes it is finished */
          op.kind = COMPLETE; op.a = (uint8_t)r; rq[r].active = false;
        } else {
          op.kind = ADVANCE; op.a = (uint8_t)r; rq[r].remaining--;
        }
      } break;
      case COMPLETE: {
        if (act.empty()) break;
        std::vector<uint32_t> done;
        for (uint32_t r : act) if (rq[r].remaining == 0) done.push_back(r);
        uint32_t r = done.empty() ? act[g.uni(0, (uint32_t)act.size() - 1)]
                                  : done[g.uni(0, (uint32_t)done.size() - 1)];
        op.kind = COMPLETE; op.a = (uint8_t)r; rq[r].active = false;
      } break;
      case ADMIT: {
        uint32_t r = Q;
        for (uint32_t i = 0; i < Q; ++i) if (!rq[i].active) { r = i; break; }
        if (r == Q) break;
        uint32_t prompt = g.uni(rc.prompt_lo, rc.prompt_hi);
        uint32_t chunk;
        if (config == 4 || config == 7) chunk = rc.chunks[g.uni(0, 2)];
        else { const uint32_t ch[4] = {128, 256, 512, 1024}; chunk = ch[g.uni(0, 3)]; }
        uint32_t decode = g.uni(0, rc.decode_hi);
        if (config == 6 && !known_obj.empty() && g.bern(0.5)) {
          /* c6 (NEXT f3): a prompt that begins with a known object's content
           * -- a prefix hit on whatever of it survives -- plus new tokens */
          const uint32_t ho = known_obj[g.uni(0, (uint32_t)known_obj.size() - 1)];
          const uint32_t hp = 16 * g.uni(1, std::max<uint32_t>(1, obj_len[ho])) + g.uni(1, 2048);
          op.kind = HIT_ADMIT; op.a = (uint8_t)r; op.b = (uint8_t)ho; op.c = 0;
          op.x = hp; op.y = chunk; op.z = decode;
          rq[r].active = true;
          rq[r].remaining = (hp + chunk - 1) / chunk + decode;
          break;
        }
        uint8_t wa = g.bern(0.7) ? 1 : 0;
        int o = take_obj((prompt + decode) / 16);
        uint32_t target = o >= 0 ? (uint32_t)o : (known_obj.empty() ? 0 : known_obj[g.uni(0, (uint32_t)known_obj.size() - 1)]);
        op.kind = ADMIT; op.a = (uint8_t)r; op.b = (uint8_t)target; op.c = wa;
        op.x = prompt; op.y = chunk; op.z = decode;
        rq[r].active = true;
        rq[r].remaining = (prompt + chunk - 1) / chunk + decode;
      } break;
      case INSERT: {
        uint32_t n = g.uni(rc.insert_lo, rc.insert_hi);
        int o = take_obj(n);
        if (o < 0) break;
        op.kind = INSERT; op.a = (uint8_t)o; op.x = n;
      } break;
      case SUBMIT: {
        if (next_claim >= C) break;
        uint32_t c = next_claim++;
        uint32_t o;
        if (!known_obj.empty() && (g.bern(0.8) || next_obj >= O)) o = known_obj[g.uni(0, (uint32_t)known_obj.size() - 1)];
        else {
          int oo = take_obj(g.uni(rc.insert_lo, rc.insert_hi));
          o = oo >= 0 ? (uint32_t)oo : 0;
        }
        uint32_t len = std::max<uint32_t>(1, obj_len[o]);
        uint32_t F = g.bern(0.8) ? len : g.uni(1, len);
        uint32_t R = g.bern(0.7) ? F : g.uni(1, F);
        uint8_t mode = (uint8_t)g.pick(rc.mode_w);
        uint32_t D;
        if (mode == 4) D = g.uni(rc.exp_D_lo, rc.exp_D_hi);
        else D = g.bern(rc.D_zero) ? 0 : g.uni(rc.D_lo, rc.D_hi);
        uint8_t mismatch = g.bern(0.02) ? 0x80 : 0;
        op.kind = SUBMIT; op.a = (uint8_t)c; op.b = (uint8_t)o; op.c = (uint8_t)(mode | mismatch);
        op.x = F; op.y = R; op.z = D;
        claims.push_back(c);
      } break;
      case TOUCH: {
        if (known_obj.empty()) break;
        op.kind = TOUCH; op.a = (uint8_t)known_obj[g.uni(0, (uint32_t)known_obj.size() - 1)];
      } break;
      case DEMOTE: {
        if (claims.empty()) break;
        op.kind = DEMOTE; op.a = (uint8_t)claims[g.uni(0, (uint32_t)claims.size() - 1)];
      } break;
      default: break;
    }
    ops[(uint64_t)s * stride] = op;
  }
}

}  // namespace

extern "C" {

/* Generate n_traces random traces (trace ids trace_begin..trace_begin+n-1)
 * of T steps for recipe `config` (3 = c3/c5, 4 = c4, 6 = c6, 7 = slot stress, 8 = c3 with
 * resident-reserve admission) with pool size N and
 * slot limits C/Q/O.  cfg_out: [n] 12-byte configs; ops_out: [T][n] 16-byte
 * op records (step-major, the lockstep replay layout).  Returns 0. */
int rkc_gen_random(int config, uint64_t seed, uint64_t trace_begin, uint32_t n_traces, uint32_t T,
                   uint32_t N, uint32_t C, uint32_t Q, uint32_t O, void* cfg_out, void* ops_out,
                   int nthreads) {
  if (config != 3 && config != 4 && config != 6 && config != 7 && config != 8) return -1;
  Cfg* cfgs = (Cfg*)cfg_out;
  Op* ops = (Op*)ops_out;
  std::atomic<uint32_t> next{0};
  auto worker = [&]() {
    for (;;) {
      uint32_t i = next.fetch_add(1);
      if (i >= n_traces) return;
      gen_trace(config, seed, trace_begin + i, T, N, C, Q, O, &cfgs[i], ops + i, n_traces);
    }
  };
  if (nthreads <= 1) worker();
  else {
    std::vector<std::thread> th;
    for (int k = 0; k < nthreads; ++k) th.emplace_back(worker);
    for (auto& x : th) x.join();
  }
  return 0;
}

}  // extern "C"
