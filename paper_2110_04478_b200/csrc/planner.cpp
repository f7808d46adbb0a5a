// Host planner of libthemis: Themis Algorithm 1 + latency model + the
// deterministic intra-dimension pre-simulation, in exact integer arithmetic.
//
//   Splitter            ChunkSize = CS / CPC
//   Dim Load Tracker    reset to A_K, += n_K^i * B_K
//   Latency Model       A_K = steps * step_latency, n_K^i B_K
//   Threshold           RS/AG of chunk/16 on min-load dim
//   Scheduler           sort dims by load (RS asc / AG desc)
//   AR                  AG order = reverse(RS order)
//   Pre-simulation      per-dim op order enforced at run time
//
// Integer scaling (exact): with Lambda = lcm(bw_k) (MB/s) and W_k = Lambda/bw_k,
//   bytes  x byte_scale = P*C      (every per-stage chunk size is then integral),
//   time   x time_scale = Lambda*P*C per ns,
//   duration(op) = volume_scaled * W_k * 1000,  A_K = steps * lat_ns * time_scale.
// All comparisons are on 128-bit integers, so schedules and predicted times are
// bit-identical to the oracle's rational arithmetic.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>

#include "plan_internal.h"

namespace themis {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
themis_status_t fail(themis_status_t st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

namespace {

const u128 kLimit = ((u128)1) << 120;  // headroom for products below

u128 gcd128(u128 a, u128 b) {
  while (b) {
    u128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}

int num_steps(int kind, int p) {  // per phase; Table 1 + PAPER.md:477 (R7)
  switch (kind) {
    case THEMIS_DIM_RING: return p - 1;
    case THEMIS_DIM_DIRECT: return 1;
    default: {
      int s = 0;
      while ((1 << s) < p) ++s;
      return s;
    }
  }
}

themis_status_t validate(const themis_topology_t* t, const themis_plan_req_t* r) {
  if (!t || !r) return fail(THEMIS_ERR_INVALID_ARG, "null topology or request");
  if (t->ndims < 1 || t->ndims > THEMIS_MAX_DIMS) return fail(THEMIS_ERR_INVALID_ARG, "ndims must be 1..8");
  uint64_t P = 1;
  for (int k = 0; k < t->ndims; ++k) {
    if (t->size[k] < 2) return fail(THEMIS_ERR_INVALID_ARG, "dim" + std::to_string(k + 1) + ": size < 2");
    if (t->bw_mbps[k] == 0) return fail(THEMIS_ERR_INVALID_ARG, "dim" + std::to_string(k + 1) + ": bw == 0");
    if (t->kind[k] < 0 || t->kind[k] > 3) return fail(THEMIS_ERR_INVALID_ARG, "bad dim kind");
    if ((t->kind[k] == THEMIS_DIM_SWITCH || t->kind[k] == THEMIS_DIM_NVLS) && (t->size[k] & (t->size[k] - 1)))
      return fail(THEMIS_ERR_INVALID_ARG, "dim" + std::to_string(k + 1) + ": switch size not a power of two");
    P *= (uint64_t)t->size[k];
    if (P > (1u << 20)) return fail(THEMIS_ERR_INVALID_ARG, "more than 2^20 ranks");
  }
  if (r->coll < 0 || r->coll > 2) return fail(THEMIS_ERR_INVALID_ARG, "bad collective");
  if (r->policy < 0 || r->policy > 1) return fail(THEMIS_ERR_INVALID_ARG, "bad policy");
  if (r->intra < 0 || r->intra > 2) return fail(THEMIS_ERR_INVALID_ARG, "bad intra policy");
  if (r->n_chunks < 1 || r->n_chunks > THEMIS_MAX_CHUNKS) return fail(THEMIS_ERR_INVALID_ARG, "n_chunks must be 1..1024");
  if (r->bytes == 0) return fail(THEMIS_ERR_INVALID_ARG, "bytes must be > 0");
  if (r->threshold_div < 1) return fail(THEMIS_ERR_INVALID_ARG, "threshold_div must be >= 1");
  if (r->concurrency < 0 || r->concurrency > 64) return fail(THEMIS_ERR_INVALID_ARG, "concurrency must be 0..64");
  if (r->reserved != 0) return fail(THEMIS_ERR_INVALID_ARG, "reserved must be 0");
  if (r->chunk_release_ns > (1ull << 40)) return fail(THEMIS_ERR_INVALID_ARG, "chunk_release_ns must be <= 2^40");
  return THEMIS_OK;
}

uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const uint8_t* b = static_cast<const uint8_t*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 1099511628211ull;
  }
  return h;
}

struct Planner {
  themis_plan_t& pl;
  int D, C, P;
  u128 lambda, g_bytes = 1, W[THEMIS_MAX_DIMS], A_rs[THEMIS_MAX_DIMS], A_ag[THEMIS_MAX_DIMS],
      A_fused[THEMIS_MAX_DIMS];
  // DimLoadTracker.reset(CT): A_K of the collective on dim k
  u128 seed(int k) const {
    const int coll = pl.req.coll;
    if (coll == THEMIS_ALLREDUCE)
      return pl.topo.kind[k] == THEMIS_DIM_NVLS ? A_fused[k] : A_rs[k] + A_ag[k];  // R29
    return coll == THEMIS_REDUCE_SCATTER ? A_rs[k] : A_ag[k];
  }
  u128 chunk_scaled() const { return (u128)pl.req.bytes / g_bytes * P; }  // (S/C) * P*C/g

  explicit Planner(themis_plan_t& p) : pl(p), D(p.D), C(p.C), P(p.P) {}

  themis_status_t scales() {
    lambda = 1;
    for (int k = 0; k < D; ++k) {
      u128 b = pl.topo.bw_mbps[k];
      lambda = lambda / gcd128(lambda, b) * b;
      if (lambda > ((u128)1 << 62)) return fail(THEMIS_ERR_OVERFLOW, "lcm of bandwidths too large");
    }
    // smallest scale making every per-stage size S/(C*prod P_subset) integral
    const u128 pc = (u128)P * C;
    g_bytes = gcd128((u128)pl.req.bytes, pc);
    pl.byte_scale = pc / g_bytes;
    pl.time_scale = lambda * pl.byte_scale;
    for (int k = 0; k < D; ++k) {
      W[k] = lambda / pl.topo.bw_mbps[k] * 1000;
      u128 lat = (u128)pl.topo.step_latency_ns[k] * pl.time_scale;
      A_rs[k] = (u128)num_steps(pl.topo.kind[k], pl.topo.size[k]) * lat;
      A_ag[k] = A_rs[k];  // same step count per phase (R7)
      A_fused[k] = (u128)2 * lat;  // in-switch RS+AG pair: reduce + multicast traversals (R29)
    }
    u128 top = (u128)pl.req.bytes * P * 1000 * 16 * 1024;
    for (int k = 0; k < D; ++k)
      if (W[k] > kLimit / top) return fail(THEMIS_ERR_OVERFLOW, "planner arithmetic would overflow");
    return THEMIS_OK;
  }

  // RS volume of a stage holding b (scaled) on a dim of size p: (p-1)/p * b.
  static u128 rs_vol(u128 b, int p) { return b / p * (p - 1); }
  static u128 ag_vol(u128 b, int p) { return b * (p - 1); }

  // Walk a chunk through `order` (phase ph), adding n_K^i * W_K to inc.
  void walk(int ph, const uint8_t* order, u128 b, u128* inc, u128* b_out, int n = -1) const {
    for (int i = 0; i < (n < 0 ? D : n); ++i) {
      int d = order[i];
      int p = pl.topo.size[d];
      if (ph == 0) {
        inc[d] += rs_vol(b, p) * W[d];
        b /= p;
      } else {
        inc[d] += ag_vol(b, p) * W[d];
        b *= p;
      }
    }
    if (b_out) *b_out = b;
  }

  // R29: an All-Reduce chunk whose last RS dim is its first AG dim and an
  // NVLS dim runs that pair as one in-switch All-Reduce.
  bool fused(const uint8_t* rs, const uint8_t* ag) const {
    return pl.req.coll == THEMIS_ALLREDUCE && rs[D - 1] == ag[0] && pl.topo.kind[rs[D - 1]] == THEMIS_DIM_NVLS;
  }
  // n = (1 + 1/p) b of the fused pair (b = bytes held before it)
  static u128 fused_vol(u128 b, int p) { return b + b / p; }
  // AR tracker increments: RS walk + AG walk (R1), the fused pair as one op (R29)
  void ar_walk(const uint8_t* rs, const uint8_t* ag, u128 chunk, u128* inc) const {
    u128 b;
    if (fused(rs, ag)) {
      walk(0, rs, chunk, inc, &b, D - 1);
      const int k = rs[D - 1];
      inc[k] += fused_vol(b, pl.topo.size[k]) * W[k];
      walk(1, ag + 1, b, inc, nullptr, D - 1);
    } else {
      walk(0, rs, chunk, inc, &b);
      walk(1, ag, b, inc, nullptr);
    }
  }

  // SCHEDULER.SCHEDULE lines 18-27 (ct: 0 RS, 1 AG); returns true if greedy.
  bool schedule_one(int ct, const u128* L, u128 chunk, uint8_t* order) const {
    int m = 0;
    u128 mx = L[0], mn = L[0];
    for (int k = 1; k < D; ++k) {
      if (L[k] < L[m]) m = k;
      mx = std::max(mx, L[k]);
      mn = std::min(mn, L[k]);
    }
    // max-min < ((P_m-1)/P_m) * (chunk/div) * B_m, cross-multiplied (R2)
    int pm = pl.topo.size[m];
    u128 lhs = (mx - mn) * (u128)pm * (u128)pl.req.threshold_div;
    u128 rhs = chunk * (u128)(pm - 1) * W[m];
    int idx[THEMIS_MAX_DIMS];
    for (int k = 0; k < D; ++k) idx[k] = k;
    if (pl.req.policy == THEMIS_POLICY_BASELINE || lhs < rhs) {
      for (int k = 0; k < D; ++k) order[k] = (uint8_t)(ct == 0 ? k : D - 1 - k);
      return false;
    }
    std::stable_sort(idx, idx + D, [&](int a, int b) { return L[a] < L[b]; });  // ties: index (R3)
    for (int k = 0; k < D; ++k) order[k] = (uint8_t)(ct == 0 ? idx[k] : idx[D - 1 - k]);
    return true;
  }

  // SCHEDULE_COLLECTIVE (Algorithm 1 lines 1-14).
  void algorithm1() {
    const int coll = pl.req.coll;
    u128 L[THEMIS_MAX_DIMS];
    for (int k = 0; k < D; ++k) L[k] = seed(k);  // DimLoadTracker.reset(CT)
    const u128 chunk = chunk_scaled();  // CS/CPC x byte_scale
    pl.rs.assign((size_t)C * D, 0xFF);
    pl.ag.assign((size_t)C * D, 0xFF);
    pl.n_greedy = 0;
    for (int c = 0; c < C; ++c) {
      u128 inc[THEMIS_MAX_DIMS] = {0};
      uint8_t* rs = &pl.rs[(size_t)c * D];
      uint8_t* ag = &pl.ag[(size_t)c * D];
      if (coll == THEMIS_ALLREDUCE) {
        pl.n_greedy += schedule_one(0, L, chunk, rs);
        for (int k = 0; k < D; ++k) ag[k] = rs[D - 1 - k];  // line 8
        ar_walk(rs, ag, chunk, inc);  // RS + AG charged (R1), NVLS pair fused (R29)
      } else if (coll == THEMIS_REDUCE_SCATTER) {
        pl.n_greedy += schedule_one(0, L, chunk, rs);
        walk(0, rs, chunk, inc, nullptr);
      } else {
        pl.n_greedy += schedule_one(1, L, chunk, ag);
        walk(1, ag, chunk / P, inc, nullptr);  // first AG stage holds chunk/P (R4)
      }
      for (int k = 0; k < D; ++k) L[k] += inc[k];  // line 30
    }
    pl.load.assign(L, L + D);
  }

  // Caller-given per-chunk orders (any of the D! x D! per chunk):
  // the tracker is only walked (reported as final_load); n_greedy counts the
  // chunks whose order differs from the baseline.
  void custom_orders(const uint8_t* rs_in, const uint8_t* ag_in) {
    const int coll = pl.req.coll;
    u128 L[THEMIS_MAX_DIMS];
    for (int k = 0; k < D; ++k) L[k] = seed(k);
    const u128 chunk = chunk_scaled();
    pl.rs.assign((size_t)C * D, 0xFF);
    pl.ag.assign((size_t)C * D, 0xFF);
    pl.n_greedy = 0;
    for (int c = 0; c < C; ++c) {
      u128 inc[THEMIS_MAX_DIMS] = {0};
      uint8_t* rs = &pl.rs[(size_t)c * D];
      uint8_t* ag = &pl.ag[(size_t)c * D];
      bool differs = false;
      u128 b = coll == THEMIS_ALL_GATHER ? chunk / P : chunk;
      if (coll != THEMIS_ALL_GATHER)
        for (int k = 0; k < D; ++k) {
          rs[k] = rs_in[(size_t)c * D + k];
          differs |= rs[k] != k;
        }
      if (coll != THEMIS_REDUCE_SCATTER)
        for (int k = 0; k < D; ++k) {
          ag[k] = ag_in[(size_t)c * D + k];
          differs |= ag[k] != D - 1 - k;
        }
      if (coll == THEMIS_ALLREDUCE)
        ar_walk(rs, ag, b, inc);
      else if (coll == THEMIS_REDUCE_SCATTER)
        walk(0, rs, b, inc, nullptr);
      else
        walk(1, ag, b, inc, nullptr);
      pl.n_greedy += differs;
      for (int k = 0; k < D; ++k) L[k] += inc[k];
    }
    pl.load.assign(L, L + D);
  }

  void build_ops() {
    const int coll = pl.req.coll;
    pl.NS = coll == THEMIS_ALLREDUCE ? 2 * D : D;
    pl.ops.clear();
    for (int c = 0; c < C; ++c) {
      u128 b = chunk_scaled();
      uint32_t red = 0;
      if (coll == THEMIS_ALL_GATHER) {
        b /= P;
        red = (1u << D) - 1;
      }
      const bool fz = coll == THEMIS_ALLREDUCE && fused(&pl.rs[(size_t)c * D], &pl.ag[(size_t)c * D]);
      for (int s = 0; s < pl.NS; ++s) {
        Op op{};
        op.chunk = c;
        op.stage = s;
        bool is_rs = coll == THEMIS_REDUCE_SCATTER || (coll == THEMIS_ALLREDUCE && s < D);
        op.phase = is_rs ? 0 : 1;
        op.dim = is_rs ? pl.rs[(size_t)c * D + s] : pl.ag[(size_t)c * D + (coll == THEMIS_ALLREDUCE ? s - D : s)];
        int p = pl.topo.size[op.dim];
        op.reduced_before = red;
        op.bytes_before = b;
        op.volume = is_rs ? rs_vol(b, p) : ag_vol(b, p);
        if (fz && s == D - 1) op.volume = fused_vol(b, p);  // the in-switch pair (R29)
        if (fz && s == D) op.volume = 0;                    // its AG half: dependency only
        op.duration = op.volume * W[op.dim] * (u128)std::max(1, pl.req.concurrency);  // BW_K / servers
        if (pl.req.charge_latency && !(fz && s == D))
          op.duration += fz && s == D - 1 ? A_fused[op.dim] : is_rs ? A_rs[op.dim] : A_ag[op.dim];
        if (is_rs) {
          b /= p;
          red |= 1u << op.dim;
        } else {
          b *= p;
          red &= ~(1u << op.dim);
        }
        pl.ops.push_back(op);
      }
    }
  }

  // Deterministic pre-simulation.  One server per dim; all
  // chunks ready at t = 0; completions at t before starts at t (R11).
  void simulate() {
    const int NS = pl.NS;
    const int total = C * NS;
    struct Ready { int chunk, stage; u128 t; };
    std::vector<std::vector<Ready>> q(D);
    // chunk c's first stage is ready at 0, or at (c+1) * release with host streaming
    const u128 release = (u128)pl.req.chunk_release_ns * pl.time_scale;
    int released = 0;
    auto release_until = [&](u128 now) {
      for (; released < C && (release == 0 || (u128)(released + 1) * release <= now); ++released)
        q[pl.ops[(size_t)released * NS].dim].push_back({released, 0, release * (u128)(released + 1)});
    };
    // k parallel servers per dim (concurrency <= 1: one)
    const int SV = std::max(1, pl.req.concurrency);
    struct Run { bool on; int chunk, stage; u128 end; };
    std::vector<Run> run((size_t)D * SV, Run{false, 0, 0, 0});
    pl.dim_ops.assign(D, {});
    pl.start.assign(total, 0);
    pl.end.assign(total, 0);
    pl.server.assign(total, 0);
    pl.busy.assign(D, 0);
    pl.vol.assign(D, 0);
    std::vector<u128> finish(D, 0);
    auto less = [&](const Ready& a, const Ready& b) {
      const Op& oa = pl.ops[(size_t)a.chunk * NS + a.stage];
      const Op& ob = pl.ops[(size_t)b.chunk * NS + b.stage];
      switch (pl.req.intra) {
        case THEMIS_INTRA_FIFO:  // (ready, chunk) (R10)
          if (a.t != b.t) return a.t < b.t;
          return a.chunk < b.chunk;
        case THEMIS_INTRA_SCF_LITERAL:  // (bytes_before, chunk)
          if (oa.bytes_before != ob.bytes_before) return oa.bytes_before < ob.bytes_before;
          return a.chunk < b.chunk;
        default:  // SCF: (volume, ready, chunk) (R9)
          if (oa.volume != ob.volume) return oa.volume < ob.volume;
          if (a.t != b.t) return a.t < b.t;
          return a.chunk < b.chunk;
      }
    };
    u128 t = 0;
    int done = 0;
    while (done < total) {
      release_until(t);  // after the completions at t, before the starts at t (R11)
      for (int k = 0; k < D; ++k)
        for (int sv = 0; sv < SV; ++sv) {
          Run& rk = run[(size_t)k * SV + sv];
          if (rk.on || q[k].empty()) continue;
          size_t best = 0;
          for (size_t i = 1; i < q[k].size(); ++i)
            if (less(q[k][i], q[k][best])) best = i;
          Ready r = q[k][best];
          q[k].erase(q[k].begin() + best);
          const Op& op = pl.ops[(size_t)r.chunk * NS + r.stage];
          rk = Run{true, r.chunk, r.stage, t + op.duration};
          pl.start[(size_t)r.chunk * NS + r.stage] = t;
          pl.server[(size_t)r.chunk * NS + r.stage] = sv;
          pl.dim_ops[k].push_back(((uint32_t)r.chunk << 8) | (uint32_t)r.stage);
          pl.busy[k] += op.duration;  // x SV: rescaled below
          pl.vol[k] += op.volume;
        }
      u128 nt = 0;
      bool any = false;
      for (const Run& rk : run)
        if (rk.on && (!any || rk.end < nt)) {
          nt = rk.end;
          any = true;
        }
      if (released < C && (!any || (u128)(released + 1) * release < nt)) {  // next arrival first
        nt = (u128)(released + 1) * release;
        any = true;
      }
      t = nt;  // some op running or a chunk still to arrive: progress
      for (int k = 0; k < D; ++k)
        for (int sv = 0; sv < SV; ++sv) {
          Run& rk = run[(size_t)k * SV + sv];
          if (!rk.on || rk.end != t) continue;
          rk.on = false;
          int c = rk.chunk, s = rk.stage;
          pl.end[(size_t)c * NS + s] = t;
          finish[k] = t;
          ++done;
          if (s + 1 < NS) q[pl.ops[(size_t)c * NS + s + 1].dim].push_back({c, s + 1, t});
        }
    }
    // With SV servers busy_K = sum(durations) / SV; report every time in a
    // unit SV times finer so that all stay exact integers.
    if (SV > 1) {
      pl.time_scale *= SV;
      for (auto& x : pl.start) x *= SV;
      for (auto& x : pl.end) x *= SV;
      for (auto& x : finish) x *= SV;
      for (auto& x : pl.load) x *= SV;
    }
    pl.makespan = 0;
    pl.idle.assign(D, 0);
    for (int k = 0; k < D; ++k) {
      pl.makespan = std::max(pl.makespan, finish[k]);
      pl.idle[k] = finish[k] - pl.busy[k];
    }
  }

  void hash() {
    uint64_t h = 1469598103934665603ull;
    h = fnv(h, &pl.topo, sizeof(pl.topo));
    const themis_plan_req_t& r = pl.req;  // field by field: struct padding is not hashed
    const int64_t f[] = {r.coll, r.policy, r.intra, r.n_chunks, (int64_t)r.bytes, r.threshold_div,
                         r.charge_latency, r.concurrency, (int64_t)r.chunk_release_ns};
    h = fnv(h, f, sizeof(f));
    h = fnv(h, pl.rs.data(), pl.rs.size());
    h = fnv(h, pl.ag.data(), pl.ag.size());
    for (auto& v : pl.dim_ops) h = fnv(h, v.data(), v.size() * sizeof(uint32_t));
    pl.hash = h;
  }
};

bool fits64(u128 v) { return v <= (u128)UINT64_MAX; }

}  // namespace
}  // namespace themis

using namespace themis;

static themis_status_t build_plan(const themis_topology_t* topo, const themis_plan_req_t* req, const uint8_t* rs,
                                  const uint8_t* ag, bool custom, themis_plan_t** out) {
  if (!out) return fail(THEMIS_ERR_INVALID_ARG, "out is null");
  *out = nullptr;
  themis_status_t st = validate(topo, req);
  if (st != THEMIS_OK) return st;
  if (custom) {  // every given order must be a permutation of the dims
    const int D = topo->ndims, C = req->n_chunks;
    const bool need_rs = req->coll != THEMIS_ALL_GATHER, need_ag = req->coll != THEMIS_REDUCE_SCATTER;
    if ((need_rs && !rs) || (need_ag && !ag)) return fail(THEMIS_ERR_INVALID_ARG, "missing rs_order / ag_order");
    for (int c = 0; c < C; ++c)
      for (const uint8_t* o : {need_rs ? rs : nullptr, need_ag ? ag : nullptr}) {
        if (!o) continue;
        uint32_t seen = 0;
        for (int k = 0; k < D; ++k) {
          const uint8_t d = o[(size_t)c * D + k];
          if (d >= D || (seen >> d & 1u)) return fail(THEMIS_ERR_INVALID_ARG, "order is not a permutation of the dims");
          seen |= 1u << d;
        }
      }
  }
  try {
    auto* pl = new themis_plan_t();
    std::memset(&pl->topo, 0, sizeof(pl->topo));
    pl->topo.ndims = topo->ndims;
    for (int k = 0; k < topo->ndims; ++k) {
      pl->topo.size[k] = topo->size[k];
      pl->topo.bw_mbps[k] = topo->bw_mbps[k];
      pl->topo.step_latency_ns[k] = topo->step_latency_ns[k];
      pl->topo.kind[k] = topo->kind[k];
    }
    pl->req = *req;
    pl->D = topo->ndims;
    pl->C = req->n_chunks;
    pl->P = 1;
    for (int k = 0; k < pl->D; ++k) pl->P *= topo->size[k];
    Planner p(*pl);
    if ((st = p.scales()) != THEMIS_OK) {
      delete pl;
      return st;
    }
    if (custom)
      p.custom_orders(rs, ag);
    else
      p.algorithm1();
    p.build_ops();
    p.simulate();
    p.hash();
    bool ok = fits64(pl->makespan) && fits64(pl->time_scale);
    for (int k = 0; k < pl->D; ++k) ok = ok && fits64(pl->vol[k]) && fits64(pl->load[k]);
    if (!ok) {
      delete pl;
      return fail(THEMIS_ERR_OVERFLOW, "plan results exceed 64 bits");
    }
    *out = pl;
    return THEMIS_OK;
  } catch (const std::exception& e) {
    return fail(THEMIS_ERR_INVALID_ARG, std::string("planner: ") + e.what());
  }
}

// n_chunks = 0: pick the chunk count (extension of PAPER.md:374 CPC, NEXT-1).
// Candidates C = 1, 2, 4, ..., THEMIS_AUTO_MAX_CHUNKS whose 16-byte pieces tile
// the buffer (bytes % (P * C * 16) == 0); each is planned in full and the one
// with the smallest pre-simulated makespan wins (ties: the smaller C).  The
// makespan only charges per-op latency with charge_latency and step_latency_ns
// set; with A_K = 0 more chunks never lose in the model.
static themis_status_t plan_auto_chunks(const themis_topology_t* topo, const themis_plan_req_t* req,
                                        themis_plan_t** out) {
  themis_plan_req_t r = *req;
  r.n_chunks = 1;
  themis_status_t st = validate(topo, &r);
  if (st != THEMIS_OK) return st;
  uint64_t P = 1;
  for (int k = 0; k < topo->ndims; ++k) P *= (uint64_t)topo->size[k];
  themis_plan_t* best = nullptr;
  for (int C = 1; C <= THEMIS_AUTO_MAX_CHUNKS; C *= 2) {
    if (req->bytes % (P * (uint64_t)C * 16u)) continue;
    r.n_chunks = C;
    themis_plan_t* pl = nullptr;
    st = build_plan(topo, &r, nullptr, nullptr, false, &pl);
    if (st != THEMIS_OK) {
      delete best;
      return st;
    }
    // makespan / time_scale, compared exactly (both fit 64 bits)
    if (!best || (u128)pl->makespan * best->time_scale < (u128)best->makespan * pl->time_scale) {
      delete best;
      best = pl;
    } else {
      delete pl;
    }
  }
  if (!best) return fail(THEMIS_ERR_ALIGNMENT, "auto chunks: bytes is not a multiple of P * 16");
  *out = best;
  return THEMIS_OK;
}

extern "C" themis_status_t themis_plan(const themis_topology_t* topo, const themis_plan_req_t* req,
                                       themis_plan_t** out) {
  if (req && req->n_chunks == 0) {
    if (!out) return fail(THEMIS_ERR_INVALID_ARG, "out is null");
    *out = nullptr;
    return plan_auto_chunks(topo, req, out);
  }
  return build_plan(topo, req, nullptr, nullptr, false, out);
}

extern "C" themis_status_t themis_plan_custom(const themis_topology_t* topo, const themis_plan_req_t* req,
                                              const uint8_t* rs_order, const uint8_t* ag_order, themis_plan_t** out) {
  return build_plan(topo, req, rs_order, ag_order, true, out);
}

extern "C" themis_status_t themis_plan_info(const themis_plan_t* pl, themis_plan_info_t* info) {
  if (!pl || !info) return fail(THEMIS_ERR_INVALID_ARG, "null argument");
  std::memset(info, 0, sizeof(*info));
  info->ndims = pl->D;
  info->n_chunks = pl->C;
  info->n_ranks = pl->P;
  info->n_stages = pl->NS;
  info->n_greedy = pl->n_greedy;
  info->coll = pl->req.coll;
  info->policy = pl->req.policy;
  info->intra = pl->req.intra;
  info->time_scale = (uint64_t)pl->time_scale;
  info->byte_scale = (uint64_t)pl->byte_scale;
  info->makespan = (uint64_t)pl->makespan;
  for (int k = 0; k < pl->D; ++k) {
    info->busy[k] = (uint64_t)pl->busy[k];
    info->idle[k] = (uint64_t)pl->idle[k];
    info->dim_volume[k] = (uint64_t)pl->vol[k];
    info->final_load[k] = (uint64_t)pl->load[k];
  }
  info->hash = pl->hash;
  // R14 utilisation, exact: sum_K bw_K busy_K / (sum bw * makespan)
  u128 num = 0, sbw = 0;
  bool ovf = false;
  for (int k = 0; k < pl->D; ++k) {
    const u128 b = pl->topo.bw_mbps[k];
    sbw += b;
    if (pl->busy[k] && b > (((u128)-1) - num) / pl->busy[k]) ovf = true;
    else num += b * pl->busy[k];
  }
  u128 den = sbw * pl->makespan;
  if (pl->makespan && sbw > ((u128)-1) / pl->makespan) ovf = true;
  if (!ovf && den) {
    const u128 g = gcd128(num, den);
    num /= g;
    den /= g;
    info->util_exact = 1;
    while ((num >> 64) || (den >> 64)) {
      num >>= 1;
      den >>= 1;
      info->util_exact = 0;
    }
    info->util_num = (uint64_t)num;
    info->util_den = (uint64_t)den;
  }
  return THEMIS_OK;
}

extern "C" themis_status_t themis_default_ctas(const themis_topology_t* t, int32_t budget, int32_t* n) {
  if (!t || !n || t->ndims < 1 || t->ndims > THEMIS_MAX_DIMS)
    return fail(THEMIS_ERR_INVALID_ARG, "bad topology / output");
  const int D = t->ndims;
  if (budget < D) return fail(THEMIS_ERR_INVALID_ARG, "budget must be >= ndims (one CTA per dimension at least)");
  uint64_t sum = 0;
  for (int k = 0; k < D; ++k) {
    if (t->bw_mbps[k] == 0) return fail(THEMIS_ERR_INVALID_ARG, "bw == 0");
    sum += t->bw_mbps[k];
  }
  // x_k = budget * bw_k / sum;  n_k = max(1, floor(x_k));  r_k = (x_k - n_k) * sum
  // (negative for dims raised to the 1-CTA floor).  Largest r_k gains one CTA
  // while the caps sum below budget; the smallest r_k among n_k > 1 loses one
  // while they sum above (ties: lower dim index).  Exact integers.
  using i128 = __int128;
  i128 r[THEMIS_MAX_DIMS];
  int tot = 0;
  for (int k = 0; k < D; ++k) {
    const i128 x = (i128)budget * t->bw_mbps[k];
    n[k] = std::max<int32_t>(1, (int32_t)(x / (i128)sum));
    r[k] = x - (i128)n[k] * (i128)sum;
    tot += n[k];
  }
  while (tot < budget) {
    int best = 0;
    for (int k = 1; k < D; ++k)
      if (r[k] > r[best]) best = k;
    ++n[best];
    r[best] -= (i128)sum;
    ++tot;
  }
  while (tot > budget) {
    int best = -1;
    for (int k = 0; k < D; ++k)
      if (n[k] > 1 && (best < 0 || r[k] < r[best])) best = k;
    --n[best];
    r[best] += (i128)sum;
    --tot;
  }
  return THEMIS_OK;
}

extern "C" themis_status_t themis_plan_orders(const themis_plan_t* pl, uint8_t* rs, uint8_t* ag) {
  if (!pl) return fail(THEMIS_ERR_INVALID_ARG, "null plan");
  if (rs) std::memcpy(rs, pl->rs.data(), pl->rs.size());
  if (ag) std::memcpy(ag, pl->ag.data(), pl->ag.size());
  return THEMIS_OK;
}

extern "C" themis_status_t themis_plan_dim_ops(const themis_plan_t* pl, uint32_t* dim_ops, int32_t* n_dim_ops) {
  if (!pl || !dim_ops || !n_dim_ops) return fail(THEMIS_ERR_INVALID_ARG, "null argument");
  const size_t stride = (size_t)pl->C * pl->NS;
  for (int k = 0; k < pl->D; ++k) {
    n_dim_ops[k] = (int32_t)pl->dim_ops[k].size();
    std::memcpy(dim_ops + k * stride, pl->dim_ops[k].data(), pl->dim_ops[k].size() * sizeof(uint32_t));
  }
  return THEMIS_OK;
}

extern "C" themis_status_t themis_plan_servers(const themis_plan_t* pl, int32_t* server) {
  if (!pl || !server) return fail(THEMIS_ERR_INVALID_ARG, "null argument");
  std::memcpy(server, pl->server.data(), pl->server.size() * sizeof(int32_t));
  return THEMIS_OK;
}

extern "C" themis_status_t themis_plan_times(const themis_plan_t* pl, uint64_t* start, uint64_t* end) {
  if (!pl) return fail(THEMIS_ERR_INVALID_ARG, "null plan");
  for (size_t i = 0; i < pl->start.size(); ++i) {
    if (!fits64(pl->end[i])) return fail(THEMIS_ERR_OVERFLOW, "time exceeds 64 bits");
    if (start) start[i] = (uint64_t)pl->start[i];
    if (end) end[i] = (uint64_t)pl->end[i];
  }
  return THEMIS_OK;
}

extern "C" const char* themis_last_error(void) { return themis::g_last_error.c_str(); }
extern "C" const char* themis_version(void) { return "libthemis 0.1 (sm_100a)"; }
