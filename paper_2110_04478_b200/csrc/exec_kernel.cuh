// exec_kernel.cuh — device side of the Themis executor (included by comm.cu
// inside its anonymous namespace, after the shared constants).
//
// One cooperative launch per collective; CTAs are partitioned into D
// "dimension groups"; group k walks the plan's op list for dim k in the
// enforced order.  Each op (chunk c, stage s, dim k) is one
// stage of the hierarchical collective for every local logical rank and is
// executed with the basic algorithm Table 1 assigns to the dimension
// (PAPER.md:226-238):
//   direct (FullyConnected; also used for Switch dims):
//     RS: y = x_0 + x_1 + ... + x_{P_k-1} over the kept part (digit_k = c_k),
//         one pull of every member's copy, summed in coordinate order (R18);
//     AG: copy every member j's held part (digit_k = j).
//   ring (P_k >= 3): P_k - 1 neighbour steps (PAPER.md:214 figure
//     RingAllReduce, :477).  RS step i: part p = (c_k + P_k - 2 - i) mod P_k,
//     partial = left's partial (left's original at i = 0) + own value; after
//     the last step the rank holds its own part (digit_k = c_k) fully reduced.
//     AG step i: copy part (c_k - 1 - i) mod P_k from the left neighbour.
// A "unit" is one direct op or one ring step.

constexpr int kMaxCtas = 160;  // CTAs per dimension group (ring step flags)
enum UnitMode { U_DIRECT_RS = 0, U_DIRECT_AG = 1, U_RING_RS = 2, U_RING_AG = 3, U_DIRECT_AG_T = 4,
                U_NVLS = 5,   // fused NVLS All-Reduce of the own piece on a switch dim (RS op of an RS+AG pair)
                U_NONE = 6,   // its AG partner: no data (the NVLS broadcast delivered it), dependencies only
                U_PUSH_AG = 7,    // direct AG by writes: the own held part -> every dim peer (TMA bulk stores, R30)
                U_LL_RS = 8,      // small-collective RS: 8-byte {payload, epoch} packets pushed into the peers' inboxes (R31)
                U_LL_AG = 9 };    // small-collective AG, same packets

// Per-op descriptor uploaded at bind (a5).
struct OpDesc {
  int32_t chunk, stage, dim, phase;  // phase 0 RS, 1 AG
  uint32_t reduced;                  // dims reduce-scattered before the op
  int32_t next_dim;                  // dim of stage+1 (-1: last stage)
  int32_t ring;                      // 1: ring algorithm on this dim
  int32_t nvls;                      // 1: U_NVLS (fused RS+AG through the switch), 2: U_NONE (its AG partner)
  int32_t push;                      // 1: direct AG executed as pushes (U_PUSH_AG, R30)
  int32_t prev_push;                 // the chunk's previous stage was a push: wait for its k x k' plane (R30)
  int32_t prev_dim;                  // dim of stage - 1 (-1: first stage)
  int32_t ll;                        // 1: LL packets (R31): no peer flags, the data carries the epoch
  uint64_t ll_off;                   // byte offset of this op's region in every rank's LL inbox
  int32_t seq;                       // index of the op in its dim's enforced list
  int32_t width, offset;             // the op runs on CTAs [offset, offset+width) mod c_k of its group
  float pace_scale;                  // pacing: width / c_k for a lone narrow op (it gets the whole dim rate), else 1
  int32_t nfree;                     // dims whose block digit is free
  int32_t free_size[THEMIS_MAX_DIMS];
  int64_t free_stride[THEMIS_MAX_DIMS];
  int64_t nblk;                      // prod free sizes
};

struct KParams {
  int32_t D, P, V, W, my_gpu, C, NS;
  int32_t size[THEMIS_MAX_DIMS];
  int64_t stride[THEMIS_MAX_DIMS];
  int32_t grp_start[THEMIS_MAX_DIMS + 1];
  int32_t dim_ops_n[THEMIS_MAX_DIMS];
  const OpDesc* ops;        // [C*NS]
  const int32_t* dim_ops;   // [D][C*NS] op indices c*NS+s
  char* heap[THEMIS_MAX_GPUS];
  uint64_t data_rel;        // buf - heap[my_gpu]
  uint64_t vrank_stride, sig_bytes;
  uint64_t blk_elems;       // N / P
  uint64_t slice_elems;     // N / (P*C)
  int32_t elem_size;
  uint32_t* epoch_ctr;      // device: epoch of the last completed collective on this comm
  unsigned long long plan_hash;  // must be identical on every rank (checked at entry)
  uint32_t* opcnt;          // [kMaxOps] per-op CTA arrival counters
  uint32_t* done_cnt;
  uint32_t* abort_flag;     // device-local: someone timed out
  uint32_t* herr;           // host-mapped error word
  uint64_t timeout_ns;
  uint64_t* trace;          // [C*NS*2] or null
  uint64_t* tdetail;        // [C*NS*6] detailed per-op stamps (trace level 2) or null
  float pace_ns_per_byte[THEMIS_MAX_DIMS];  // per-CTA pacing of peer bytes, leaky bucket (0 = off)
  int32_t lookahead;        // runtime intra-dim order: ops of the enforced list a producer may pick from (<= 1: static)
  uint32_t dyn_mask;        // dims whose ops may be reordered at run time (no ring steps)
  int32_t push_ok;          // push AG allowed in this launch (off while host-buffer streaming)
  uint64_t ll_rel;          // LL inboxes: heap + ll_rel + (q % V) * ll_stride (R31)
  uint64_t ll_stride;
  int32_t stages;           // TMA ring depth in use: bytes in flight per CTA = stages x stage_bytes
  int32_t stage_bytes;      // bytes per ring stage (stages x stage_bytes <= kStages x kStageBytes)
  int32_t ag_rr;            // direct AG: 1 = one peer per ring stage (round robin), 0 = all peers per stage
  uint32_t host_seq;        // host-buffer streaming (themis_allreduce_host): value of this call's h2d / d2h flags; 0 = off
  uint32_t* d2h_flags;      // [THEMIS_MAX_CHUNKS] device: chunk c final on this GPU (read by a stream wait op)
  char* mc_heap;            // multicast (NVLS) mapping of this GPU's heap, same offsets; null = none
};

// ---------------------------------------------------------------- signal pads
// pad(q) = [entry u32 P][exit u32 P][ready u32 P x kMaxOps][ring u64 P x 8 x kMaxCtas]
__host__ __device__ __forceinline__ uint64_t ring_flags_offset(int P) { return 4ull * (2ull * P + (uint64_t)P * kMaxOps); }
__host__ __device__ __forceinline__ uint64_t hash_offset(int P) {
  return ring_flags_offset(P) + 8ull * P * THEMIS_MAX_DIMS * kMaxCtas;
}
__host__ __device__ __forceinline__ uint64_t h2d_offset(int P) { return hash_offset(P) + 8ull * P; }
// pad(q) continues: [hash u64 P][h2d u32 THEMIS_MAX_CHUNKS] (h2d used in local rank 0's pad only)
__host__ __device__ __forceinline__ uint64_t pad_bytes(int P) { return h2d_offset(P) + 4ull * THEMIS_MAX_CHUNKS; }
__device__ __forceinline__ uint32_t* sig_of(const KParams& p, int q) {
  return reinterpret_cast<uint32_t*>(p.heap[q / p.V] + (uint64_t)(q % p.V) * p.sig_bytes);
}
__device__ __forceinline__ uint32_t* entry_slot(const KParams& p, int q, int src) { return sig_of(p, q) + src; }
__device__ __forceinline__ uint32_t* exit_slot(const KParams& p, int q, int src) { return sig_of(p, q) + p.P + src; }
__device__ __forceinline__ uint32_t* ready_slot(const KParams& p, int q, int src, int op) {
  return sig_of(p, q) + 2 * p.P + (uint64_t)src * kMaxOps + op;
}
// ring step flag written by rank `src`'s CTA g of dim k's group into q's pad
__device__ __forceinline__ unsigned long long* ring_slot(const KParams& p, int q, int src, int k, int g) {
  return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(sig_of(p, q)) + ring_flags_offset(p.P)) +
         ((uint64_t)src * THEMIS_MAX_DIMS + k) * kMaxCtas + g;
}
// plan hash announced by rank `src` for the current call, in q's pad
__device__ __forceinline__ unsigned long long* hash_slot(const KParams& p, int q, int src) {
  return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(sig_of(p, q)) + hash_offset(p.P)) + src;
}
// host-buffer streaming: chunk c of GPU g's local ranks has arrived from the
// host (written by a stream memory op after the copies, value = host_seq)
__device__ __forceinline__ uint32_t* h2d_slot(const KParams& p, int g, int c) {
  return reinterpret_cast<uint32_t*>(p.heap[g] + h2d_offset(p.P)) + c;
}
__device__ __forceinline__ char* data_of(const KParams& p, int q) {
  return p.heap[q / p.V] + p.data_rel + (uint64_t)(q % p.V) * p.vrank_stride;
}
__device__ __forceinline__ char* inbox_of(const KParams& p, int q) {
  return p.heap[q / p.V] + p.ll_rel + (uint64_t)(q % p.V) * p.ll_stride;
}
// 32-bit arithmetic: a comm hosts <= 64 logical ranks (64-bit division is emulated)
__device__ __forceinline__ int coord(const KParams& p, int q, int k) {
  return (q / (int)p.stride[k]) % p.size[k];
}
// neighbour of q on dim k at coordinate offset delta (ring left = -1, right = +1)
__device__ __forceinline__ int ring_peer(const KParams& p, int q, int k, int delta) {
  const int pk = p.size[k], c = coord(p, q, k);
  return q + (((c + delta) % pk + pk) % pk - c) * (int)p.stride[k];
}

// This launch's epoch (a6), read once per CTA from the comm's device counter
// (so a collective captured in a CUDA graph gets a fresh epoch on every replay).
__shared__ uint32_t s_epoch;
__device__ __forceinline__ uint32_t cur_epoch() { return s_epoch; }

// Spin until *f >= e.  Returns false on timeout / abort (watchdog).
__device__ bool wait_geq(const KParams& p, const uint32_t* f, uint32_t e, uint32_t where) {
  if (dev::ld_acquire_sys(f) >= e) return true;
  const uint64_t t0 = dev::globaltimer();
  for (;;) {
#pragma unroll 1
    for (int i = 0; i < 256; ++i)
      if (dev::ld_acquire_sys(f) >= e) return true;
    if (*(volatile uint32_t*)p.abort_flag) return false;
    if (dev::globaltimer() - t0 > p.timeout_ns) {
      atomicExch(p.abort_flag, 1u);
      *(volatile uint32_t*)p.herr = (uint32_t)THEMIS_ERR_TIMEOUT | (where << 8);
      __threadfence_system();
      return false;
    }
  }
}
__device__ bool wait_geq64(const KParams& p, const unsigned long long* f, unsigned long long e, uint32_t where) {
  if (dev::ld_acquire_sys64(f) >= e) return true;
  const uint64_t t0 = dev::globaltimer();
  for (;;) {
#pragma unroll 1
    for (int i = 0; i < 256; ++i)
      if (dev::ld_acquire_sys64(f) >= e) return true;
    if (*(volatile uint32_t*)p.abort_flag) return false;
    if (dev::globaltimer() - t0 > p.timeout_ns) {
      atomicExch(p.abort_flag, 1u);
      *(volatile uint32_t*)p.herr = (uint32_t)THEMIS_ERR_TIMEOUT | (where << 8);
      __threadfence_system();
      return false;
    }
  }
}

// ---------------------------------------------------------------- work items
// An item is one contiguous slice (chunk c of block b, slice_bytes) of one
// local rank:  direct RS / ring RS / ring AG: (local rank v, free index f) ->
// V * nblk items;  direct AG: (v, source member j != c_k, f) -> V*(P_k-1)*nblk.
struct Item {
  int q;          // global logical rank the item belongs to
  int g0;         // rank of member 0 of q's dim-k group
  int j;          // direct AG: source member
  uint64_t off;   // byte offset of the slice inside a rank's data region
};

// Small ops run on a window of `width` CTAs so that several chunks' ops of the
// same dimension are in flight at once ("multiple chunks
// per dimension should be run in parallel" when one cannot saturate the BW).
// li = CTA index inside the window, wn = window width.
__device__ __forceinline__ bool op_member(const OpDesc& d, int gi, int gn, int& li, int& wn) {
  li = (gi - d.offset + gn) % gn;
  wn = d.width;
  return li < wn;
}

__device__ __forceinline__ int unit_mode(const OpDesc& d) {
  return d.ring ? (d.phase == 0 ? U_RING_RS : U_RING_AG) : (d.phase == 0 ? U_DIRECT_RS : U_DIRECT_AG);
}
// TMA path: a direct AG tile pulls the same offsets from all P_k - 1 peers at
// once (U_DIRECT_AG_T), so every CTA keeps requests in flight to every peer.
__device__ __forceinline__ bool is_push(const KParams& p, const OpDesc& d) { return d.push && p.push_ok; }
__device__ __forceinline__ int unit_mode_tma(const KParams& p, const OpDesc& d) {
  if (d.nvls) return d.nvls == 1 ? U_NVLS : U_NONE;
  if (d.ll) return d.phase == 0 ? U_LL_RS : U_LL_AG;
  if (is_push(p, d)) return U_PUSH_AG;
  const int m = unit_mode(d);
  return m == U_DIRECT_AG ? U_DIRECT_AG_T : m;
}
__device__ __forceinline__ uint64_t unit_items(const KParams& p, const OpDesc& d, int mode) {
  return (uint64_t)p.V * d.nblk * (mode == U_DIRECT_AG ? (uint64_t)(p.size[d.dim] - 1) : 1ull);
}
// byte distance between the same slice of two parts differing by 1 in digit_k
__device__ __forceinline__ uint64_t part_stride(const KParams& p, int k) {
  return (uint64_t)p.stride[k] * p.blk_elems * p.elem_size;
}
// the jj-th peer (jj = 0..P_k-2) of a rank with coordinate ck on its dim
__device__ __forceinline__ int peer_member(int jj, int ck) { return jj < ck ? jj : jj + 1; }

// 32-bit index arithmetic throughout: a unit has < 2^32 items (V * nblk *
// (P_k - 1) <= 64^3), and 64-bit div/mod (emulated, ~100 instructions each)
// made small ops latency-bound on this decode.
__device__ __forceinline__ Item decode_item(const KParams& p, const OpDesc& d, int mode, int step, uint64_t it64) {
  Item r;
  const int k = d.dim, pk = p.size[k];
  const uint32_t it = (uint32_t)it64, nblk = (uint32_t)d.nblk;
  uint32_t f;
  int digit;
  if (mode == U_DIRECT_AG) {
    const uint32_t per_v = (uint32_t)(pk - 1) * nblk;
    const uint32_t vq = it / per_v, rem = it - vq * per_v;
    r.q = p.my_gpu * p.V + (int)vq;
    const uint32_t jj = rem / nblk;
    const int ck = coord(p, r.q, k);
    r.j = (int)jj < ck ? (int)jj : (int)jj + 1;
    f = rem - jj * nblk;
    digit = r.j;
  } else {
    const uint32_t vq = it / nblk;
    r.q = p.my_gpu * p.V + (int)vq;
    f = it - vq * nblk;
    r.j = -1;
    const int ck = coord(p, r.q, k);
    digit = (mode == U_DIRECT_RS || mode == U_NVLS || mode == U_PUSH_AG || mode == U_LL_RS || mode == U_LL_AG) ? ck
          : mode == U_DIRECT_AG_T ? 0  // base: part j is at off + j * part_stride
          : mode == U_RING_RS     ? (ck + pk - 2 - step) % pk
                                  : ((ck - 1 - step) % pk + pk) % pk;
  }
  int b = digit * (int)p.stride[k];
  for (int dd = 0; dd < p.D; ++dd)  // other fixed digits: the rank's coords on the reduced dims
    if ((d.reduced >> dd & 1u) && dd != k) b += coord(p, r.q, dd) * (int)p.stride[dd];
  for (int i = 0; i < d.nfree; ++i) {
    const uint32_t fs = (uint32_t)d.free_size[i], fq = f / fs;
    b += (int)(f - fq * fs) * (int)d.free_stride[i];
    f = fq;
  }
  r.g0 = r.q - coord(p, r.q, k) * (int)p.stride[k];
  r.off = ((uint64_t)b * p.blk_elems + (uint64_t)d.chunk * p.slice_elems) * p.elem_size;
  return r;
}

// Visit this CTA's byte spans of a unit: fn(item index, a, e) with [a, e)
// inside the item.  Direct units split the unit's bytes evenly over the group;
// ring units give CTA g the same sub-range of every rank's part, so a ring
// step depends only on CTA g of the left neighbour.
template <class F>
__device__ __forceinline__ void for_each_span(const KParams& p, const OpDesc& d, int mode, int gi, int gn, F&& fn) {
  const uint64_t Lb = p.slice_elems * p.elem_size;
  if (mode == U_RING_RS || mode == U_RING_AG) {
    const uint64_t R16 = (uint64_t)d.nblk * (Lb / 16);
    const uint64_t r0 = R16 * gi / gn * 16, r1 = R16 * (gi + 1) / gn * 16;
    if (r0 >= r1) return;
    for (int v = 0; v < p.V; ++v)
      for (uint64_t f = r0 / Lb; f * Lb < r1; ++f) {
        const uint64_t a = r0 > f * Lb ? r0 - f * Lb : 0;
        const uint64_t e = r1 - f * Lb < Lb ? r1 - f * Lb : Lb;
        fn((uint64_t)v * d.nblk + f, a, e);
      }
    return;
  }
  const uint64_t tot16 = unit_items(p, d, mode) * (Lb / 16);
  const uint64_t u0 = tot16 * gi / gn * 16, u1 = tot16 * (gi + 1) / gn * 16;
  for (uint64_t it = u0 / Lb; it * Lb < u1; ++it) {
    const uint64_t a = u0 > it * Lb ? u0 - it * Lb : 0;
    const uint64_t e = u1 - it * Lb < Lb ? u1 - it * Lb : Lb;
    fn(it, a, e);
  }
}

__device__ __forceinline__ bool unit_has_work(const KParams& p, const OpDesc& d, int mode, int gi, int gn) {
  if (mode == U_NONE) return gi == 0;  // one CTA carries the dependency wait
  const uint64_t Lb16 = p.slice_elems * p.elem_size / 16;
  if (mode == U_RING_RS || mode == U_RING_AG) {
    const uint64_t R16 = (uint64_t)d.nblk * Lb16;
    return R16 * (gi + 1) / gn > R16 * gi / gn;
  }
  const uint64_t tot16 = unit_items(p, d, mode) * Lb16;
  return tot16 * (gi + 1) / gn > tot16 * gi / gn;
}

// sources of a unit's item, in summation order
__device__ __forceinline__ int unit_nsrc(const KParams& p, const OpDesc& d, int mode) {
  return mode == U_DIRECT_RS ? p.size[d.dim] : mode == U_DIRECT_AG_T ? p.size[d.dim] - 1 : mode == U_RING_RS ? 2 : 1;
}
__device__ __forceinline__ int unit_src_rank(const KParams& p, const OpDesc& d, int mode, const Item& m, int j) {
  const int k = d.dim;
  switch (mode) {
    case U_DIRECT_RS: return m.g0 + j * (int)p.stride[k];
    case U_DIRECT_AG: return m.g0 + m.j * (int)p.stride[k];
    case U_DIRECT_AG_T: return m.g0 + peer_member(j, coord(p, m.q, k)) * (int)p.stride[k];
    case U_RING_RS: return j == 0 ? ring_peer(p, m.q, k, -1) : m.q;  // left partial + own value
    case U_PUSH_AG: return m.q;                                      // the own held part
    default: return ring_peer(p, m.q, k, -1);
  }
}

// Address of dim-k member j's copy of the current piece (LDG path).
struct PeerSrc {
  const KParams* p;
  int q0, step;
  uint64_t off;
  __device__ __forceinline__ const uint4* operator()(int j) const {
    return reinterpret_cast<const uint4*>(data_of(*p, q0 + j * step) + off);
  }
};

// ------------------------------------------------------- path 1: LDG / STG
// Direct algorithm only: every thread issues NSRC*UNROLL 16-byte L1-bypassing
// loads before adding.  (Ring dims need the TMA engine.)
template <class Tag>
__device__ void run_op_ldg(const KParams& p, const OpDesc& d, int gi, int gn) {
  const int k = d.dim, pk = p.size[k];
  const int mode = unit_mode(d);
  for_each_span(p, d, mode, gi, gn, [&](uint64_t it, uint64_t a, uint64_t e) {
    const Item m = decode_item(p, d, mode, 0, it);
    uint4* dst = reinterpret_cast<uint4*>(data_of(p, m.q) + m.off);
    const PeerSrc src{&p, m.g0, (int)p.stride[k], m.off};
    if (mode == U_DIRECT_AG) {
      dev::copy_range<8>(dst, src(m.j), a / 16, e / 16);
      return;
    }
    switch (pk) {
      case 2: dev::reduce_range<Tag, 2, 4>(dst, src, a / 16, e / 16); break;
      case 3: dev::reduce_range<Tag, 3, 4>(dst, src, a / 16, e / 16); break;
      case 4: dev::reduce_range<Tag, 4, 2>(dst, src, a / 16, e / 16); break;
      case 8: dev::reduce_range<Tag, 8, 1>(dst, src, a / 16, e / 16); break;
      default: dev::reduce_range_generic<Tag>(dst, src, pk, a / 16, e / 16); break;
    }
  });
}

// ------------------------------------------------------- path 2: TMA bulk
// Warp-specialised CTA: warp 0 = producer (one lane streams each tile's
// sources into a kStages-deep shared-memory ring with cp.async.bulk, local HBM
// or a peer's HBM over NVLink), warps 1..8 = consumers (sum in order / pass
// through, 16-byte STG), warp 9 = completion (counts and publishes).
constexpr int kStages = 6;
constexpr int kStageBytes = 32 * 1024;
constexpr int kConsumerWarps = 8;
constexpr int kOpRing = 16;  // units the producer / consumers may run ahead of the completion warp
// ring [stages x stage bytes] | full, empty [kStages] | op_done, op_free, q_full [kOpRing] | unit queue int [kOpRing]
constexpr int kSmemBytes = kStages * kStageBytes + (2 * kStages + 3 * kOpRing) * 8 + kOpRing * 4;
constexpr int kMaxLookahead = 32;
static_assert(kThreads == 32 * (kConsumerWarps + 2), "producer + consumers + completion warp");

__device__ __forceinline__ uint32_t unit_tile(const KParams& p, int nsrc) { return ((uint32_t)p.stage_bytes / nsrc) & ~15u; }

// Producer (one lane): stream this CTA's tiles of one unit into the ring.
__device__ __forceinline__ bool empty_wait(const KParams& p, uint64_t* bar, uint32_t parity) {
  return dev::mbar_wait_or(bar, parity, p.abort_flag);
}

// Returns false if the kernel is aborting (watchdog): every wait for a free
// ring slot gives up on the abort flag, so a producer whose consumers stopped
// never spins forever (the CTA then reaches the exit barrier).
__device__ __forceinline__ bool produce_unit(const KParams& p, const OpDesc& d, int mode, int step, int gi, int gn,
                                             char* smem, uint64_t* full, uint64_t* empty, uint32_t& ctr,
                                             double& due) {
  if (mode == U_NVLS || mode == U_NONE || mode == U_LL_RS || mode == U_LL_AG) {
    // no TMA: a zero-byte token tells the consumers the deps hold
    const int s = ctr % p.stages;
    if (!empty_wait(p, &empty[s], ((ctr / p.stages) & 1) ^ 1)) return false;
    dev::mbar_arrive_token(&full[s]);
    ++ctr;
    return true;
  }
  bool ok = true;
  const int nsrc = unit_nsrc(p, d, mode);
  const uint32_t tile = unit_tile(p, nsrc);
  const float pace = p.pace_ns_per_byte[d.dim] * d.pace_scale;
  const int remote = (mode == U_DIRECT_RS || mode == U_DIRECT_AG_T || mode == U_PUSH_AG) ? p.size[d.dim] - 1
                                                                                          : 1;  // peer bytes / tile byte
  const uint64_t pstride = part_stride(p, d.dim);
  dev::fence_proxy_async_global();  // generic-proxy writes (ours and peers') -> async proxy (TMA)
  for_each_span(p, d, mode, gi, gn, [&](uint64_t it, uint64_t a, uint64_t e) {
    if (!ok) return;
    const Item m = decode_item(p, d, mode, step, it);
    const char* src[THEMIS_MAX_DIMS > 8 ? THEMIS_MAX_DIMS : 8];
    const int ns = nsrc <= 8 ? nsrc : 8;
    const int ck = coord(p, m.q, d.dim);
    for (int j = 0; j < ns; ++j)  // AG_T: peer j's own part sits at digit_k = member(j)
      src[j] = data_of(p, unit_src_rank(p, d, mode, m, j)) + m.off +
               (mode == U_DIRECT_AG_T ? (uint64_t)peer_member(j, ck) * pstride : 0);
    if (mode == U_DIRECT_AG_T && p.ag_rr) {
      // round-robin variant: each ring stage holds one whole stage_bytes tile
      // from one peer; consecutive stages cycle through the peers
      const uint32_t big = p.stage_bytes;
      for (uint64_t pos = a; pos < e; pos += big) {
        const uint32_t bytes = (uint32_t)(e - pos < big ? e - pos : big);
        for (int j = 0; j < nsrc; ++j, ++ctr) {
          if (pace > 0.f) {
            while ((double)dev::globaltimer() < due) {
            }
            due += (double)bytes * pace;
          }
          const int s = ctr % p.stages;
          if (!empty_wait(p, &empty[s], ((ctr / p.stages) & 1) ^ 1)) {
            ok = false;
            return;
          }
          dev::mbar_expect_tx(&full[s], bytes);
          const char* sj = j < 8 ? src[j]
                                 : data_of(p, unit_src_rank(p, d, mode, m, j)) + m.off +
                                       (uint64_t)peer_member(j, ck) * pstride;
          dev::bulk_g2s(smem + s * p.stage_bytes, sj + pos, bytes, &full[s]);
        }
      }
      return;
    }
    for (uint64_t pos = a; pos < e; pos += tile, ++ctr) {
      const uint32_t bytes = (uint32_t)(e - pos < tile ? e - pos : tile);
      if (pace > 0.f) {  // leaky bucket: this CTA's peer bytes at <= 1 / pace bytes/ns
        while ((double)dev::globaltimer() < due) {
        }
        due += (double)bytes * remote * pace;
      }
      const int s = ctr % p.stages;
      if (!empty_wait(p, &empty[s], ((ctr / p.stages) & 1) ^ 1)) {
        ok = false;
        return;
      }
      dev::mbar_expect_tx(&full[s], bytes * nsrc);
      char* dst = smem + s * p.stage_bytes;
      for (int j = 0; j < nsrc; ++j) {
        const char* sj = j < 8 ? src[j]
                               : data_of(p, unit_src_rank(p, d, mode, m, j)) + m.off +
                                     (mode == U_DIRECT_AG_T ? (uint64_t)peer_member(j, ck) * pstride : 0);
        dev::bulk_g2s(dst + j * tile, sj + pos, bytes, &full[s]);
      }
    }
  });
  return ok;
}

// R31: poll one LL packet group until it carries this launch's tag; the
// watchdog (timeout -> abort + THEMIS_ERR_TIMEOUT) as in wait_geq.
__device__ bool ll_wait(const KParams& p, const char* src, uint32_t tag, uint4& v) {
  if (dev::ld_ll_try(src, tag, v)) return true;
  const uint64_t t0 = dev::globaltimer();
  for (;;) {
#pragma unroll 1
    for (int i = 0; i < 256; ++i)
      if (dev::ld_ll_try(src, tag, v)) return true;
    if (*(volatile uint32_t*)p.abort_flag) return false;
    if (dev::globaltimer() - t0 > p.timeout_ns) {
      atomicExch(p.abort_flag, 1u);
      *(volatile uint32_t*)p.herr = (uint32_t)THEMIS_ERR_TIMEOUT | (0xFFFFFBu << 8);
      __threadfence_system();
      return false;
    }
  }
}

// Hand a ring slot back to the producer after this warp's reads of it: a
// release arrive (the reads happen-before the producer's acquire and its next
// TMA write into the slot; measured: no cost over a relaxed arrive).
__device__ __forceinline__ void slot_release(const KParams&, uint64_t* bar) { dev::mbar_arrive(bar); }

// R31 LL unit (consumer warps), kept out of line so the pull path's code is
// unchanged.  Returns false if the kernel is aborting (CTA-uniform).
template <class Tag>
__device__ __noinline__ bool consume_ll_unit(const KParams& p, const OpDesc& d, int mode, int step, int gi, int gn,
                                             uint64_t* full, uint64_t* empty, uint32_t& ctr) {
  const int ct = threadIdx.x - 32, lane = threadIdx.x & 31;
  constexpr int kCons = 32 * kConsumerWarps;
  bool ok = true;
    // R31: no flags between ranks -- every 8-byte packet {4 payload bytes,
    // epoch} is one single-copy-atomic store into the receiver's inbox and the
    // receiver polls the packets themselves.  Two passes over this CTA's
    // span: send the peers what they need from this rank, then poll what this
    // rank needs from them.
    if (!unit_has_work(p, d, mode, gi, gn)) return true;
    const int s = ctr % p.stages;
    // the consumer warps meet at a named barrier below: decide "go / abort"
    // for all of them at once (a warp that saw the abort flag while another
    // saw the token must not leave the others waiting at the barrier)
    if (!dev::named_bar_and(1, kCons, dev::mbar_wait_or(&full[s], (ctr / p.stages) & 1, p.abort_flag)))
      return false;
    const int k = d.dim, pk = p.size[k];
    const uint32_t tag = cur_epoch();
    const uint64_t ps = part_stride(p, k), Lb = p.slice_elems * p.elem_size, nblk = (uint64_t)d.nblk;
    // pass 1: send everything in this CTA's span (posted writes, never block)
    for_each_span(p, d, mode, gi, gn, [&](uint64_t it, uint64_t a, uint64_t e) {
      const Item m = decode_item(p, d, mode, step, it);
      const int ck = coord(p, m.q, k);
      const uint64_t f = it % nblk;  // the item's index among its rank's nblk slices
      for (uint64_t w = a / 16 + ct; w < e / 16; w += kCons) {
        const uint64_t pos = w * 16;
        // RS: peer j gets my copy of ITS part; AG: every peer gets my part
        for (int j = 0; j < pk; ++j) {
          if (j == ck) continue;
          const int qj = m.g0 + j * (int)p.stride[k];
          const uint64_t src_off = mode == U_LL_RS ? m.off + (int64_t)(j - ck) * (int64_t)ps : m.off;
          const uint4 v = dev::ld_cg(reinterpret_cast<const uint4*>(data_of(p, m.q) + src_off + pos));
          const int slot = ck < j ? ck : ck - 1;  // my slot among j's peers
          dev::st_ll(inbox_of(p, qj) + d.ll_off + (((uint64_t)slot * nblk + f) * Lb + pos) * 2, v, tag);
        }
      }
    });
    // every consumer thread of this CTA has sent before any waits: a CTA that
    // hosts several local ranks never waits on its own unsent packets, and
    // the receive pass mostly finds packets already landed
    dev::named_bar_sync(1, kCons);
    // pass 2: receive, reduce in coordinate order (R18) / copy
    for_each_span(p, d, mode, gi, gn, [&](uint64_t it, uint64_t a, uint64_t e) {
      if (!ok) return;
      const Item m = decode_item(p, d, mode, step, it);
      const int ck = coord(p, m.q, k);
      const uint64_t f = it % nblk;
      for (uint64_t w = a / 16 + ct; w < e / 16; w += kCons) {
        const uint64_t pos = w * 16;
        if (mode == U_LL_RS) {
          float acc[Tag::kAcc];
          for (int j = 0; j < pk; ++j) {
            uint4 v;
            if (j == ck) {
              v = dev::ld_cg(reinterpret_cast<const uint4*>(data_of(p, m.q) + m.off + pos));
            } else {
              const int slot = j < ck ? j : j - 1;
              if (!ll_wait(p, inbox_of(p, m.q) + d.ll_off + (((uint64_t)slot * nblk + f) * Lb + pos) * 2, tag, v)) {
                ok = false;
                return;
              }
            }
            if (j == 0) Tag::load(acc, v);
            else Tag::add(acc, v);
          }
          dev::st_v4(reinterpret_cast<uint4*>(data_of(p, m.q) + m.off + pos), Tag::store(acc));
        } else {
          for (int j = 0; j < pk; ++j) {
            if (j == ck) continue;
            const int slot = j < ck ? j : j - 1;
            uint4 v;
            if (!ll_wait(p, inbox_of(p, m.q) + d.ll_off + (((uint64_t)slot * nblk + f) * Lb + pos) * 2, tag, v)) {
              ok = false;
              return;
            }
            dev::st_v4(reinterpret_cast<uint4*>(data_of(p, m.q) + m.off + (int64_t)(j - ck) * (int64_t)ps + pos), v);
          }
        }
      }
    });
    // a thread with nothing left to poll must not run on while others gave up
    // (the next LL unit's barrier would wait for them): one answer per CTA
    ok = dev::named_bar_and(1, kCons, ok);
    if (lane == 0) slot_release(p, &empty[s]);
    ++ctr;
    return ok;
}

// Consumers: returns false if the kernel is aborting (watchdog).
template <class Tag>
__device__ __forceinline__ bool consume_unit(const KParams& p, const OpDesc& d, int mode, int step, int gi, int gn,
                                             const char* smem, uint64_t* full, uint64_t* empty, uint32_t& ctr) {
  const int ct = threadIdx.x - 32, lane = threadIdx.x & 31;
  constexpr int kCons = 32 * kConsumerWarps;
  const int nsrc = unit_nsrc(p, d, mode);
  const uint32_t tile = unit_tile(p, nsrc), tile16 = tile / 16;
  const bool reduce = mode == U_DIRECT_RS || mode == U_RING_RS;
  bool ok = true;
  if (mode == U_LL_RS || mode == U_LL_AG) return consume_ll_unit<Tag>(p, d, mode, step, gi, gn, full, empty, ctr);
  if (mode == U_NVLS || mode == U_NONE) {  // consumers reduce through the switch directly (no ring data)
    if (!unit_has_work(p, d, mode, gi, gn)) return true;
    const int s = ctr % p.stages;
    if (!dev::mbar_wait_or(&full[s], (ctr / p.stages) & 1, p.abort_flag)) return false;
    if (mode == U_NVLS)
      for_each_span(p, d, mode, gi, gn, [&](uint64_t it, uint64_t a, uint64_t e) {
        const Item m = decode_item(p, d, mode, step, it);
        char* mc = p.mc_heap + p.data_rel + (uint64_t)(m.q % p.V) * p.vrank_stride + m.off;
        // 4 independent in-switch reductions in flight per thread (the switch round trip is long)
        constexpr int U = 4;
        const uint64_t w0 = a / 16, w1 = e / 16;
        uint64_t w = w0 + ct;
        for (; w + (U - 1) * kCons < w1; w += U * kCons) {
          uint4 v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) v[u] = dev::mc_ld_reduce<Tag>(mc + 16 * (w + u * kCons));
#pragma unroll
          for (int u = 0; u < U; ++u) dev::mc_st(mc + 16 * (w + u * kCons), v[u]);
        }
        for (; w < w1; w += kCons) dev::mc_st(mc + 16 * w, dev::mc_ld_reduce<Tag>(mc + 16 * w));
      });
    __syncwarp();
    if (lane == 0) slot_release(p, &empty[s]);
    ++ctr;
    return true;
  }
  if (mode == U_PUSH_AG) {
    // R30: consumer thread 0 writes every landed tile of the own held part to
    // the P_k - 1 dim peers (TMA bulk stores, same offsets in their buffers),
    // one bulk group per tile, pipelined: a tile's slot is released (by warp
    // 1) once the NEXT tile's stores are issued and this tile's stores have
    // read it (wait_group.read 1); the other consumer warps release at once.
    // The unit ends only when every store's writes are complete (then
    // op_done -> the completion warp's release publish).
    const int pk = p.size[d.dim];
    int held = -1;  // warp 1: slot whose stores may still be reading it
    for_each_span(p, d, mode, gi, gn, [&](uint64_t it, uint64_t a, uint64_t e) {
      if (!ok) return;
      const Item m = decode_item(p, d, mode, step, it);
      const int ck = coord(p, m.q, d.dim);
      for (uint64_t pos = a; pos < e; pos += tile, ++ctr) {
        const uint32_t bytes = (uint32_t)(e - pos < tile ? e - pos : tile);
        const int s = ctr % p.stages;
        if (!dev::mbar_wait_or(&full[s], (ctr / p.stages) & 1, p.abort_flag)) {
          ok = false;
          return;
        }
        if (ct < 32) {
          if (ct == 0) {
            for (int j = 0; j < pk; ++j)
              if (j != ck)
                dev::bulk_s2g(data_of(p, m.g0 + j * (int)p.stride[d.dim]) + m.off + pos, smem + s * p.stage_bytes,
                              bytes);
            dev::bulk_commit();
            dev::bulk_wait_read1();
          }
          __syncwarp();
          if (held >= 0 && lane == 0) slot_release(p, &empty[held]);
          held = s;
        } else {
          __syncwarp();
          if (lane == 0) slot_release(p, &empty[s]);
        }
      }
    });
    if (ct < 32) {
      if (ct == 0) {
        dev::bulk_wait0();                 // writes performed ...
        dev::fence_proxy_async_global();   // ... and ordered before the generic-proxy release chain
      }
      __syncwarp();
      if (held >= 0 && lane == 0) slot_release(p, &empty[held]);
    }
    return ok;
  }
  for_each_span(p, d, mode, gi, gn, [&](uint64_t it, uint64_t a, uint64_t e) {
    if (!ok) return;
    const Item m = decode_item(p, d, mode, step, it);
    char* base = data_of(p, m.q) + m.off;
    if (mode == U_DIRECT_AG_T && p.ag_rr) {  // mirror of the producer's round-robin stages
      const uint32_t big = p.stage_bytes;
      const int ck = coord(p, m.q, d.dim);
      const uint64_t ps = part_stride(p, d.dim);
      for (uint64_t pos = a; pos < e; pos += big) {
        const uint32_t n16 = (uint32_t)((e - pos < big ? e - pos : big) / 16);
        for (int j = 0; j < nsrc; ++j, ++ctr) {
          const int s = ctr % p.stages;
          if (!dev::mbar_wait_or(&full[s], (ctr / p.stages) & 1, p.abort_flag)) {
            ok = false;
            return;
          }
          const uint4* sm = reinterpret_cast<const uint4*>(smem + s * p.stage_bytes);
          uint4* dj = reinterpret_cast<uint4*>(base + pos + (uint64_t)peer_member(j, ck) * ps);
          for (uint32_t w = ct; w < n16; w += kCons) dev::st_v4(dj + w, sm[w]);
          __syncwarp();
          if (lane == 0) slot_release(p, &empty[s]);
        }
      }
      return;
    }
    for (uint64_t pos = a; pos < e; pos += tile, ++ctr) {
      const uint32_t n16 = (uint32_t)((e - pos < tile ? e - pos : tile) / 16);
      const int s = ctr % p.stages;
      if (!dev::mbar_wait_or(&full[s], (ctr / p.stages) & 1, p.abort_flag)) {
        ok = false;
        return;
      }
      const uint4* sm = reinterpret_cast<const uint4*>(smem + s * p.stage_bytes);
      uint4* dst = reinterpret_cast<uint4*>(base + pos);
      if (reduce) {
        for (uint32_t w = ct; w < n16; w += kCons) {
          float acc[Tag::kAcc];
          Tag::load(acc, sm[w]);
          for (int j = 1; j < nsrc; ++j) Tag::add(acc, sm[j * tile16 + w]);
          dev::st_v4(dst + w, Tag::store(acc));
        }
      } else if (mode == U_DIRECT_AG_T) {  // slot j -> peer member(j)'s part
        const int ck = coord(p, m.q, d.dim);
        const uint64_t ps16 = part_stride(p, d.dim) / 16;
        for (int j = 0; j < nsrc; ++j) {
          uint4* dj = dst + (uint64_t)peer_member(j, ck) * ps16;
          for (uint32_t w = ct; w < n16; w += kCons) dev::st_v4(dj + w, sm[j * tile16 + w]);
        }
      } else {
        for (uint32_t w = ct; w < n16; w += kCons) dev::st_v4(dst + w, sm[w]);
      }
      __syncwarp();
      if (lane == 0) slot_release(p, &empty[s]);
    }
  });
  return ok;
}

// Sources whose (c, s-1) flag an op of local rank q waits for: q's dim-k
// group (P_k ranks) -- or, after a push stage on dim k' (R30), the whole
// k' x k plane through q (P_k' x P_k ranks: q's dim-k peers read data that
// their dim-k' peers wrote into them).
__device__ __forceinline__ int n_deps(const KParams& p, const OpDesc& d) {
  if (d.ll) return 1;  // R31: peers' data arrives tagged in the inbox; only the own (c, s-1) is a flag
  return p.size[d.dim] * ((d.prev_push && p.push_ok) ? p.size[d.prev_dim] : 1);
}
__device__ __forceinline__ int dep_src(const KParams& p, const OpDesc& d, int q, int t) {
  if (d.ll) return q;
  const int k = d.dim, pk = p.size[k];
  int src = q + (t % pk - coord(p, q, k)) * (int)p.stride[k];
  if (d.prev_push && p.push_ok) src += (t / pk - coord(p, q, d.prev_dim)) * (int)p.stride[d.prev_dim];
  return src;
}

// One warp: wait until the local ranks and their dim-k peers completed (c, s-1).
// Stage s > 0: every source finished (c, s-1).  Stage 0 in host-buffer mode:
// every source GPU's copy of chunk c has landed (h2d flag = host_seq).
__device__ __forceinline__ bool wait_deps_warp(const KParams& p, const OpDesc& d, int opi) {
  const int V = p.V, q0 = p.my_gpu * V, nd = n_deps(p, d);
  bool ok = true;
  for (int t = threadIdx.x & 31; t < V * nd; t += 32) {
    const int q = q0 + t / nd;
    const int src = dep_src(p, d, q, t % nd);
    if (d.stage > 0)
      ok &= wait_geq(p, ready_slot(p, q, src, opi - 1), cur_epoch(), (uint32_t)opi);
    else
      ok &= wait_geq(p, h2d_slot(p, src / V, d.chunk), p.host_seq, 0xFFFFFCu);
  }
  return __all_sync(0xFFFFFFFFu, ok);
}

// One warp, non-blocking: have the local ranks' and their dim-k peers' (c, s-1)
// (or the host copies of chunk c) completed?  One acquire load per flag.
__device__ __forceinline__ bool deps_ready_warp(const KParams& p, const OpDesc& d, int opi) {
  if (d.stage == 0 && !p.host_seq) return true;
  const int V = p.V, q0 = p.my_gpu * V, nd = n_deps(p, d);
  bool ok = true;
  for (int t = threadIdx.x & 31; t < V * nd; t += 32) {
    const int q = q0 + t / nd;
    const int src = dep_src(p, d, q, t % nd);
    ok &= d.stage > 0 ? dev::ld_acquire_sys(ready_slot(p, q, src, opi - 1)) >= cur_epoch()
                      : dev::ld_acquire_sys(h2d_slot(p, src / V, d.chunk)) >= p.host_seq;
  }
  return __all_sync(0xFFFFFFFFu, ok);
}

constexpr int kFewFlags = 16;  // flag stores a single lane issues after its one release fence

__device__ __forceinline__ unsigned long long ring_flag_value(uint32_t epoch, int seq, int steps_done) {
  return ((unsigned long long)epoch << 32) | ((unsigned long long)seq << 8) | (unsigned long long)steps_done;
}

// One warp: ring step `step` (>= 1) of CTA gi needs the left neighbours' CTA gi
// to have finished step - 1 of the same op.
__device__ __forceinline__ bool wait_ring_warp(const KParams& p, const OpDesc& d, int step, int gi) {
  const int V = p.V, q0 = p.my_gpu * V, k = d.dim;
  bool ok = true;
  for (int v = threadIdx.x & 31; v < V; v += 32) {
    const int q = q0 + v;
    ok &= wait_geq64(p, ring_slot(p, q, ring_peer(p, q, k, -1), k, gi), ring_flag_value(cur_epoch(), d.seq, step),
                     0xFFFFFCu);
  }
  return __all_sync(0xFFFFFFFFu, ok);
}

// One warp: this CTA finished ring step `step` -> tell the right neighbours.
__device__ __forceinline__ void publish_ring_warp(const KParams& p, const OpDesc& d, int step, int gi) {
  const int V = p.V, q0 = p.my_gpu * V, k = d.dim, lane = threadIdx.x & 31;
  bool local = true;
  for (int v = lane; v < V; v += 32) local &= ring_peer(p, q0 + v, k, +1) / V == p.my_gpu;
  local = __all_sync(0xFFFFFFFFu, local);
  // release pattern: a fence then relaxed flag stores in the same thread's
  // program order.  A fence on every lane of the warp costs ~10 % of NVLink
  // throughput (fence.acq_rel.sys is per thread), so few flags are stored by
  // lane 0 alone after its one fence.
  if (V <= kFewFlags) {
    if (lane == 0) {
      if (local)
        dev::fence_acq_rel_gpu();
      else
        dev::fence_acq_rel_sys();
      for (int v = 0; v < V; ++v)
        dev::st_relaxed_sys64(ring_slot(p, ring_peer(p, q0 + v, k, +1), q0 + v, k, gi),
                              ring_flag_value(cur_epoch(), d.seq, step + 1));
    }
  } else {
    if (local)
      dev::fence_acq_rel_gpu();
    else
      dev::fence_acq_rel_sys();
    for (int v = lane; v < V; v += 32) {
      const int q = q0 + v;
      dev::st_relaxed_sys64(ring_slot(p, ring_peer(p, q, k, +1), q, k, gi), ring_flag_value(cur_epoch(), d.seq, step + 1));
    }
  }
  __syncwarp();
}

// One warp: count this CTA's completion of op opi; the group's last CTA
// publishes the epoch to the consumers of (c, s): self and the next stage's
// dim peers.  Release chain: consumers' stores -> mbarrier arrive (release.cta)
// / bar.sync -> atom.acq_rel.gpu (all CTAs) -> fence.acq_rel.sys -> relaxed
// sys stores.
__device__ __forceinline__ void complete_op_warp(const KParams& p, const OpDesc& d, int opi, int gn) {
  const int lane = threadIdx.x & 31;
  uint32_t last = 0;
  if (lane == 0) {
    if (p.tdetail) p.tdetail[6 * opi + 2] = dev::globaltimer();  // (any CTA; last writer wins)
    // a one-CTA window (small op) is complete here: no counter round trip
    last = gn == 1 || dev::atom_add_acq_rel_gpu(&p.opcnt[opi], 1u) == (uint32_t)gn - 1;
    if (last && gn > 1) {
      if (p.tdetail) p.tdetail[6 * opi + 3] = dev::globaltimer();
      p.opcnt[opi] = 0;  // every CTA arrived; reset for the next call
    }
  }
  last = __shfl_sync(0xFFFFFFFFu, last, 0);
  if (!last) return;
  if (d.next_dim >= 0) {  // (the last stage has no consumer: the exit barrier orders it)
    const int V = p.V, q0 = p.my_gpu * V, kn = d.next_dim, pn = p.size[kn];
    // consumers of (c, s): self and the next stage's dim peers -- for a push
    // op (R30) the whole k x k_next plane (the next stage's peers read data
    // this op wrote into their dim-k peers)
    const bool push = is_push(p, d);
    const int pk = push ? p.size[d.dim] : 1;
    const int npe = d.ll ? 1 : pn * pk;  // R31: an LL op's only flag consumer is its own next stage
    const int nst = V * npe;
    auto dst_of = [&](int t, int& q) {
      q = q0 + t / npe;
      if (d.ll) return q;
      const int u = t % npe;
      int dst = q + (u % pn - coord(p, q, kn)) * (int)p.stride[kn];
      if (push) dst += (u / pn - coord(p, q, d.dim)) * (int)p.stride[d.dim];
      return dst;
    };
    // If every consumer (and, for a push, every rank it wrote to) is on this
    // GPU a gpu-scope release suffices; otherwise fence at sys scope.
    bool local = true;
    for (int t = lane; t < nst; t += 32) {
      int q;
      local &= dst_of(t, q) / V == p.my_gpu;
    }
    local = __all_sync(0xFFFFFFFFu, local);
    // release pattern (fence, then relaxed flag stores in the same thread's
    // program order); few flags: lane 0 alone, after one fence
    auto publish = [&](int t) {
      int q;
      const int dst = dst_of(t, q);
      if (local)
        dev::st_relaxed_gpu(ready_slot(p, dst, q, opi), cur_epoch());
      else
        dev::st_relaxed_sys(ready_slot(p, dst, q, opi), cur_epoch());
    };
    if (nst <= kFewFlags) {
      if (lane == 0) {
        if (local)
          dev::fence_acq_rel_gpu();
        else
          dev::fence_acq_rel_sys();
        if (p.tdetail) p.tdetail[6 * opi + 4] = dev::globaltimer();
        for (int t = 0; t < nst; ++t) publish(t);
      }
    } else {
      if (local)
        dev::fence_acq_rel_gpu();
      else
        dev::fence_acq_rel_sys();
      if (p.tdetail && lane == 0) p.tdetail[6 * opi + 4] = dev::globaltimer();
      for (int t = lane; t < nst; t += 32) publish(t);
    }
  }
  else if (p.host_seq && lane == 0) {  // last stage: chunk c is final here -> the D2H stream may copy it
    dev::fence_acq_rel_sys();
    dev::st_relaxed_sys(&p.d2h_flags[d.chunk], p.host_seq);
  }
  if (p.trace && lane == 0) p.trace[2 * opi + 1] = dev::globaltimer();
  __syncwarp();
}

template <class Tag, bool kTma>
__global__ void __launch_bounds__(kThreads, 1) themis_exec_kernel(const __grid_constant__ KParams p) {
  extern __shared__ __align__(128) char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* op_done = empty + kStages;
  uint64_t* op_free = op_done + kOpRing;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int g = 0;
  while (g + 1 < p.D && (int)blockIdx.x >= p.grp_start[g + 1]) ++g;
  const int gi = blockIdx.x - p.grp_start[g];
  const int gn = p.grp_start[g + 1] - p.grp_start[g];
  const int V = p.V, P = p.P;
  const int q0 = p.my_gpu * V;
  bool ok = true;
  // epoch = 1 + that of the previous collective on this comm (stream order:
  // the previous kernel stored it after every CTA had read its own).
  if (tid == 0) s_epoch = *(volatile uint32_t*)p.epoch_ctr + 1u;
  if (kTma && tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], kConsumerWarps);
    }
    for (int s = 0; s < kOpRing; ++s) {
      dev::mbar_init(&op_done[s], kConsumerWarps);
      dev::mbar_init(&op_free[s], 1);
      dev::mbar_init(&op_free[s] + kOpRing, 1);  // q_full[s]: the producer announced unit s
    }
    dev::fence_mbar_init();
  }
  __syncthreads();

  // a6: entry barrier — every local rank announces the epoch (and, ordered
  // before it by the release, its plan hash) to every rank.  Inter-dimension
  // schedule consistency: every CTA checks that all ranks
  // run the identical plan; a mismatch latches THEMIS_ERR_PLAN_MISMATCH.
  if (blockIdx.x == 0)
    for (int i = tid; i < V * P; i += blockDim.x) {
      dev::st_relaxed_sys64(hash_slot(p, i % P, q0 + i / P), p.plan_hash);
      dev::st_release_sys(entry_slot(p, i % P, q0 + i / P), cur_epoch());
    }
  for (int i = tid; i < V * P; i += blockDim.x) {
    ok &= wait_geq(p, entry_slot(p, q0 + i / P, i % P), cur_epoch(), 0xFFFFFFu);
    if (ok && *(volatile unsigned long long*)hash_slot(p, q0 + i / P, i % P) != p.plan_hash) {
      ok = false;
      atomicExch(p.abort_flag, 1u);
      *(volatile uint32_t*)p.herr = (uint32_t)THEMIS_ERR_PLAN_MISMATCH | ((uint32_t)(i % P) << 8);
      __threadfence_system();
    }
  }
  ok = __syncthreads_and(ok);

  // a9: walk this dimension's ops in the enforced order.
  const int* list = p.dim_ops + (uint64_t)g * p.C * p.NS;
  const int nops = ok ? p.dim_ops_n[g] : 0;
  if constexpr (kTma) {
    // Decoupled: the producer picks the next op, waits for its dependencies,
    // streams its tiles and moves on while the consumers finish; the
    // completion warp counts and publishes, so no sys fence ever stalls the
    // tile stream.  The producer announces every unit it takes (op, ring step)
    // in a shared-memory queue that the consumers and the completion warp
    // follow, so the order is the producer's alone:
    //   static (default; ring dims): the enforced order;
    //   runtime (lookahead L > 1, non-ring dims): the first op among the next L
    //   not-yet-taken ops of the enforced list whose dependencies already
    //   hold -- the pre-simulated order is the priority, readiness decides
    //   (SURVEY NEXT-3, R28).  Pull-based ops only read peers' finished
    //   (c, s-1) data, so ranks need not agree on the order (R28).
    uint32_t ctr = 0;  // tile ring position (identical sequence in producer and consumers)
    uint64_t* q_full = op_free + kOpRing;
    int* s_q = reinterpret_cast<int*>(q_full + kOpRing);
    // this CTA's units: sum of ring steps over the ops it is a member of
    int my_units = 0;
    if (warp > 0) {
      for (int i = lane; i < nops; i += 32) {
        const OpDesc& d = p.ops[list[i]];
        int li, wn;
        if (op_member(d, gi, gn, li, wn)) my_units += d.ring ? p.size[d.dim] - 1 : 1;
      }
      for (int o = 16; o; o >>= 1) my_units += __shfl_xor_sync(0xFFFFFFFFu, my_units, o);
    }
    if (warp == 0) {
      const bool dyn = p.lookahead > 1 && (p.dyn_mask >> g & 1u);
      const int LA = dyn ? (p.lookahead < kMaxLookahead ? p.lookahead : kMaxLookahead) : 1;
      int head = 0;           // first list position not yet taken
      uint32_t taken = 0;     // bit j: list[head + j] taken
      uint32_t nq = 0;        // units announced
      bool stop = false;
      uint64_t t_wait = 0;
      double pace_due = 0.0;  // lane 0: pacing bucket (ns)
      while (!stop) {
        while (head < nops) {  // drop taken / foreign ops at the head
          int li, wn;
          if (!(taken & 1u) && op_member(p.ops[list[head]], gi, gn, li, wn)) break;
          taken >>= 1;
          ++head;
        }
        if (head >= nops) break;
        int pick = 0;
        if (dyn) {
          pick = -1;
          for (int j = 0; j < LA && head + j < nops && pick < 0; ++j) {
            if (taken >> j & 1u) continue;
            const int opi = list[head + j];
            const OpDesc& d = p.ops[opi];
            int li, wn;
            if (!op_member(d, gi, gn, li, wn)) continue;
            if (!unit_has_work(p, d, unit_mode_tma(p, d), li, wn) || deps_ready_warp(p, d, opi)) pick = j;
          }
          if (pick < 0) {  // nothing ready yet: watchdog (decided on lane 0, warp-uniform), then scan again
            int give_up = 0;
            if (lane == 0) {
              const uint64_t now = dev::globaltimer();
              if (!t_wait) t_wait = now;
              if (*(volatile uint32_t*)p.abort_flag) {
                give_up = 1;
              } else if (now - t_wait > p.timeout_ns) {
                atomicExch(p.abort_flag, 1u);
                *(volatile uint32_t*)p.herr = (uint32_t)THEMIS_ERR_TIMEOUT | ((uint32_t)list[head] << 8);
                __threadfence_system();
                give_up = 1;
              }
            }
            if (__shfl_sync(0xFFFFFFFFu, give_up, 0)) break;
            continue;
          }
          t_wait = 0;
        }
        taken |= 1u << pick;
        const int opi = list[head + pick];
        const OpDesc& d = p.ops[opi];
        const int mode = unit_mode_tma(p, d);
        const int nu = d.ring ? p.size[d.dim] - 1 : 1;
        int li, wn;
        op_member(d, gi, gn, li, wn);
        const bool work = unit_has_work(p, d, mode, li, wn);
        for (int u = 0; u < nu && !stop; ++u, ++nq) {
          const int slot = nq % kOpRing;
          bool w = true;
          if (lane == 0) {  // announce the unit once the followers released the queue slot
            w = dev::mbar_wait_or(&op_free[slot], ((nq / kOpRing) & 1) ^ 1, p.abort_flag);
            if (w) {
              s_q[slot] = opi * 64 + u;
              dev::mbar_arrive(&q_full[slot]);
            }
          }
          if (!__shfl_sync(0xFFFFFFFFu, w, 0)) {
            stop = true;
            break;
          }
          if (!work) continue;  // nothing to wait for or move: the followers just count it
          // ring step flags are per absolute CTA index gi: each CTA's slot then
          // sees its ops in order (monotone), and CTA gi of the left neighbour
          // has the same window index li for this op (identical windows).
          if (u == 0 ? (!dyn && (d.stage > 0 || p.host_seq) && !wait_deps_warp(p, d, opi))
                     : !wait_ring_warp(p, d, u, gi)) {
            stop = true;
            break;
          }
          if (lane == 0) {
            if (u == 0) {
              if (p.trace) atomicMin(reinterpret_cast<unsigned long long*>(&p.trace[2 * opi]), dev::globaltimer());
              if (p.tdetail && li == 0) {  // stamp 5: after a proxy fence (its cost)
                dev::fence_proxy_async_global();
                p.tdetail[6 * opi + 5] = dev::globaltimer();
              }
            }
            // pacing (BW emulation): a per-CTA leaky bucket across all the
            // CTA's units -- no credit accrues while it waits for a unit's
            // dependencies, so a dim's c_k CTAs never exceed V * BW_k in total,
            // whatever order (or how many ops at once) they run
            const double now = (double)dev::globaltimer();
            if (pace_due < now) pace_due = now;
            if (!produce_unit(p, d, mode, u, li, wn, smem, full, empty, ctr, pace_due)) stop = true;
            if (p.tdetail && li == 0 && u + 1 == nu) p.tdetail[6 * opi + 0] = dev::globaltimer();
          }
          stop = __shfl_sync(0xFFFFFFFFu, stop, 0);
        }
      }
    } else if (warp <= kConsumerWarps) {
      // consumers: per announced unit, every consumer warp arrives on
      // op_done[slot] (mbarrier arrive = release.cta of its stores) after the
      // completion warp has freed that slot (ring of kOpRing units).
      for (int n = 0; n < my_units; ++n) {
        const int slot = n % kOpRing;
        if (!dev::mbar_wait_or(&q_full[slot], (n / kOpRing) & 1, p.abort_flag)) break;
        const int e = s_q[slot], opi = e >> 6, u = e & 63;
        const OpDesc& d = p.ops[opi];
        const int mode = unit_mode_tma(p, d);
        const int nu = d.ring ? p.size[d.dim] - 1 : 1;
        int li, wn;
        op_member(d, gi, gn, li, wn);
        // warp-uniform: a lane whose spans ended before an abort must stop with the others
        if (!__all_sync(0xFFFFFFFFu, consume_unit<Tag>(p, d, mode, u, li, wn, smem, full, empty, ctr))) break;
        __syncwarp();
        bool w = true;
        if (lane == 0) {
          if (p.tdetail && li == 0 && warp == 1 && u + 1 == nu) p.tdetail[6 * opi + 1] = dev::globaltimer();
          w = dev::mbar_wait_or(&op_free[slot], ((n / kOpRing) & 1) ^ 1, p.abort_flag);
          if (w) dev::mbar_arrive(&op_done[slot]);
        }
        if (!__shfl_sync(0xFFFFFFFFu, w, 0)) break;
      }
    } else {
      // completion warp: ring steps publish per-CTA step flags; the last unit
      // of an op counts group-wide and publishes the op's ready flags.
      for (int n = 0; n < my_units; ++n) {
        const int slot = n % kOpRing;
        bool w = true;
        if (lane == 0)
          w = dev::mbar_wait_or(&q_full[slot], (n / kOpRing) & 1, p.abort_flag) &&
              dev::mbar_wait_or(&op_done[slot], (n / kOpRing) & 1, p.abort_flag);
        if (!__shfl_sync(0xFFFFFFFFu, w, 0)) break;
        const int e = s_q[slot], opi = e >> 6, u = e & 63;
        const OpDesc& d = p.ops[opi];
        const int mode = unit_mode_tma(p, d);
        const int nu = d.ring ? p.size[d.dim] - 1 : 1;
        int li, wn;
        op_member(d, gi, gn, li, wn);
        if (u + 1 < nu) {
          if (unit_has_work(p, d, mode, li, wn)) publish_ring_warp(p, d, u, gi);
        } else {
          complete_op_warp(p, d, opi, wn);
        }
        __syncwarp();
        if (lane == 0) dev::mbar_arrive(&op_free[slot]);
      }
    }
  } else {
    for (int i = 0; ok && i < nops; ++i) {
      const int opi = list[i];
      const OpDesc& d = p.ops[opi];
      const int k = d.dim;
      int li, wn;
      if (!op_member(d, gi, gn, li, wn)) continue;
      if (d.stage > 0 || p.host_seq) {  // own and dim-k peers' previous stage (or host copy) of this chunk
        const int pk = p.size[k];
        for (int t = tid; t < V * pk; t += blockDim.x) {
          const int q = q0 + t / pk;
          const int src = q + (t % pk - coord(p, q, k)) * (int)p.stride[k];
          if (d.stage > 0)
            ok &= wait_geq(p, ready_slot(p, q, src, opi - 1), cur_epoch(), (uint32_t)opi);
          else
            ok &= wait_geq(p, h2d_slot(p, src / V, d.chunk), p.host_seq, 0xFFFFFCu);
        }
        ok = __syncthreads_and(ok);
        if (!ok) break;
      }
      if (p.trace && tid == 0) atomicMin(reinterpret_cast<unsigned long long*>(&p.trace[2 * opi]), dev::globaltimer());
      run_op_ldg<Tag>(p, d, li, wn);
      __syncthreads();
      if (warp == 0) complete_op_warp(p, d, opi, wn);
      __syncthreads();
    }
  }

  // exit: all CTAs done -> exit barrier so no peer still reads our buffers.
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    atomicAdd(p.done_cnt, 1u);
  }
  if (blockIdx.x != 0) return;
  if (tid == 0) {
    ok &= wait_geq(p, p.done_cnt, gridDim.x, 0xFFFFFEu);
    *p.done_cnt = 0;
    __threadfence_system();
  }
  __syncthreads();
  for (int i = tid; i < V * P; i += blockDim.x) dev::st_release_sys(exit_slot(p, i % P, q0 + i / P), cur_epoch());
  for (int i = tid; i < V * P; i += blockDim.x) wait_geq(p, exit_slot(p, q0 + i / P, i % P), cur_epoch(), 0xFFFFFDu);
  // host-buffer mode: every chunk's d2h flag is set by now; set them again so a
  // D2H stream waiting on them is released even when the kernel aborted
  // (the error is latched and reported by the next call)
  if (p.host_seq) {
    __threadfence_system();
    for (int i = tid; i < p.C; i += blockDim.x) dev::st_relaxed_sys(&p.d2h_flags[i], p.host_seq);
  }
  // every CTA has read the epoch (all counted in done_cnt): advance it for the next launch
  __syncthreads();
  if (tid == 0) *(volatile uint32_t*)p.epoch_ctr = cur_epoch();
}
