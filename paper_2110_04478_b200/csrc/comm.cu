// libthemis executor: symmetric heap, comm, plan binding and the persistent
// sm_100a kernel that runs a Themis plan.
//
// One cooperative launch per collective.  Its CTAs are partitioned into D
// "dimension groups"; group k walks the plan's op list for dim k in the
// enforced order, splitting every op over its c_k CTAs.  An op
// (chunk c, stage s, dim k) for local rank v waits until v and its dim-k peers
// completed (c, s-1), then:
//   RS: over v's held blocks with digit_k = c_k(v): y = sum_j x_{peer j} in
//       coordinate order, stored in place   (R16, R18)
//   AG: copies every peer j's held blocks (digit_k = j) into v's buffer.
// Capping c_k emulates per-dimension bandwidth (BASELINE.json north_star (d)).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "device.cuh"
#include "plan_internal.h"

using namespace themis;

namespace {

constexpr int kThreads = 320;  // TMA path: producer warp + 8 consumer warps + completion warp; LDG: all copy
constexpr int kMaxRanks = 64;                                       // logical ranks a comm may host
constexpr int kMaxOps = THEMIS_MAX_CHUNKS * 2 * THEMIS_MAX_DIMS;    // ops per plan
constexpr uint64_t kAlign = 1ull << 16;

uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
uint64_t signal_bytes(int P) { return round_up(4ull * (2ull * P + (uint64_t)P * kMaxOps), kAlign); }

themis_status_t cuda_fail(cudaError_t e, const char* what) {
  return fail(THEMIS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CUDA_TRY(call)                                 \
  do {                                                 \
    cudaError_t _e = (call);                           \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

// Per-op descriptor uploaded at bind (a5).
struct OpDesc {
  int32_t chunk, stage, dim, phase;  // phase 0 RS, 1 AG
  uint32_t reduced;                  // dims reduce-scattered before the op
  int32_t next_dim;                  // dim of stage+1 (-1: last stage)
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
  uint32_t epoch;
  uint32_t* opcnt;          // [kMaxOps] per-op CTA arrival counters
  unsigned long long* op_t0;  // [kMaxOps] group-wide pacing origin of each op (0 = unset)
  uint32_t* done_cnt;
  uint32_t* abort_flag;     // device-local: someone timed out
  uint32_t* herr;           // host-mapped error word
  uint64_t timeout_ns;
  uint64_t* trace;          // [C*NS*2] or null
  float pace_ns_per_byte[THEMIS_MAX_DIMS];  // per-CTA pacing of peer bytes (0 = off)
  int32_t stages;           // TMA ring depth in use (<= kStages): bytes in flight per CTA
};

__device__ __forceinline__ uint32_t* sig_of(const KParams& p, int q) {
  return reinterpret_cast<uint32_t*>(p.heap[q / p.V] + (uint64_t)(q % p.V) * p.sig_bytes);
}
__device__ __forceinline__ uint32_t* entry_slot(const KParams& p, int q, int src) { return sig_of(p, q) + src; }
__device__ __forceinline__ uint32_t* exit_slot(const KParams& p, int q, int src) { return sig_of(p, q) + p.P + src; }
__device__ __forceinline__ uint32_t* ready_slot(const KParams& p, int q, int src, int op) {
  return sig_of(p, q) + 2 * p.P + (uint64_t)src * kMaxOps + op;
}
__device__ __forceinline__ char* data_of(const KParams& p, int q) {
  return p.heap[q / p.V] + p.data_rel + (uint64_t)(q % p.V) * p.vrank_stride;
}
__device__ __forceinline__ int coord(const KParams& p, int q, int k) { return (int)((q / p.stride[k]) % p.size[k]); }

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

// ---------------------------------------------------------------- work items
// An op's work on this GPU is a list of "items", each one contiguous slice
// (chunk c of block b) of slice_bytes:
//   RS: item = (local rank v, free index f)          -> V * nblk items
//   AG: item = (local rank v, source member j != c_k, f) -> V * (P_k-1) * nblk
// The op's total bytes are split evenly (16-byte granules) over the group's
// CTAs; each CTA walks its contiguous range.
struct Item {
  int q;          // global logical rank this item belongs to
  int g0;         // rank of member 0 of q's dim-k group
  int j;          // AG: source member; RS: unused
  uint64_t off;   // byte offset of the slice inside a rank's data region
};

__device__ __forceinline__ Item decode_item(const KParams& p, const OpDesc& d, uint64_t it) {
  Item r;
  const int k = d.dim, pk = p.size[k];
  int64_t f;
  int64_t b = 0;
  if (d.phase == 0) {
    r.q = p.my_gpu * p.V + (int)(it / d.nblk);
    f = (int64_t)(it % d.nblk);
    r.j = -1;
    for (int dd = 0; dd < p.D; ++dd)  // fixed digits: my coords on reduced U {k}
      if ((d.reduced >> dd & 1u) || dd == k) b += (int64_t)coord(p, r.q, dd) * p.stride[dd];
  } else {
    const uint64_t per_v = (uint64_t)(pk - 1) * d.nblk;
    r.q = p.my_gpu * p.V + (int)(it / per_v);
    const uint64_t rem = it % per_v;
    const int jj = (int)(rem / d.nblk);
    const int ck = coord(p, r.q, k);
    r.j = jj < ck ? jj : jj + 1;
    f = (int64_t)(rem % d.nblk);
    b = (int64_t)r.j * p.stride[k];
    for (int dd = 0; dd < p.D; ++dd)  // fixed digits: my coords on reduced \ {k}, digit_k = j
      if ((d.reduced >> dd & 1u) && dd != k) b += (int64_t)coord(p, r.q, dd) * p.stride[dd];
  }
  for (int i = 0; i < d.nfree; ++i) {
    b += (f % d.free_size[i]) * d.free_stride[i];
    f /= d.free_size[i];
  }
  r.g0 = r.q - coord(p, r.q, k) * (int)p.stride[k];
  r.off = ((uint64_t)b * p.blk_elems + (uint64_t)d.chunk * p.slice_elems) * p.elem_size;
  return r;
}

__device__ __forceinline__ uint64_t op_items(const KParams& p, const OpDesc& d) {
  const int pk = p.size[d.dim];
  return (uint64_t)p.V * d.nblk * (d.phase == 0 ? 1 : (uint64_t)(pk - 1));
}

// Address of dim-k member j's copy of the current piece.
struct PeerSrc {
  const KParams* p;
  int q0, step;
  uint64_t off;
  __device__ __forceinline__ const uint4* operator()(int j) const {
    return reinterpret_cast<const uint4*>(data_of(*p, q0 + j * step) + off);
  }
};

// ------------------------------------------------------- path 1: LDG / STG
// Every thread issues NSRC*UNROLL 16-byte L1-bypassing loads before adding.
template <class Tag>
__device__ void run_op_ldg(const KParams& p, const OpDesc& d, int gi, int gn) {
  const int k = d.dim, pk = p.size[k];
  const uint64_t Lv = p.slice_elems * p.elem_size / 16;
  const uint64_t total = op_items(p, d) * Lv;
  const uint64_t u0 = total * gi / gn, u1 = total * (gi + 1) / gn;
  for (uint64_t it = u0 / Lv; it * Lv < u1; ++it) {
    const Item m = decode_item(p, d, it);
    const uint64_t a = (u0 > it * Lv ? u0 - it * Lv : 0);
    const uint64_t e = (u1 - it * Lv < Lv ? u1 - it * Lv : Lv);
    uint4* dst = reinterpret_cast<uint4*>(data_of(p, m.q) + m.off);
    const PeerSrc src{&p, m.g0, (int)p.stride[k], m.off};
    if (d.phase == 1) {
      dev::copy_range<8>(dst, src(m.j), a, e);
      continue;
    }
    switch (pk) {
      case 2: dev::reduce_range<Tag, 2, 4>(dst, src, a, e); break;
      case 3: dev::reduce_range<Tag, 3, 4>(dst, src, a, e); break;
      case 4: dev::reduce_range<Tag, 4, 2>(dst, src, a, e); break;
      case 8: dev::reduce_range<Tag, 8, 1>(dst, src, a, e); break;
      default: dev::reduce_range_generic<Tag>(dst, src, pk, a, e); break;
    }
  }
}

// ------------------------------------------------------- path 2: TMA bulk
// Warp 0 lane 0 streams each tile's P_k (RS) or 1 (AG) source ranges into a
// kStages-deep shared-memory ring with cp.async.bulk (mbarrier complete_tx);
// the kConsumerWarps consumer warps sum the P_k copies in coordinate order
// (RS) or pass the bytes through (AG) and store with 16-byte STG.
constexpr int kStages = 6;
constexpr int kStageBytes = 32 * 1024;
constexpr int kConsumerWarps = 8;
constexpr int kOpRing = 16;  // ops the consumers may run ahead of the completion warp
constexpr int kSmemBytes = kStages * kStageBytes + 2 * (kStages + kOpRing) * 8;
static_assert(kThreads == 32 * (kConsumerWarps + 2), "producer + consumers + completion warp");

// Geometry of op d for CTA gi of gn: byte range [u0, u1) of the op's items
// (16-byte granules), TMA tile size per source.
struct OpRange {
  uint64_t u0, u1, Lb;
  uint32_t tile;
  int nsrc, pk;
};
__device__ __forceinline__ OpRange op_range(const KParams& p, const OpDesc& d, int gi, int gn) {
  OpRange r;
  r.pk = p.size[d.dim];
  r.nsrc = d.phase == 0 ? r.pk : 1;
  r.Lb = p.slice_elems * p.elem_size;
  const uint64_t tot16 = op_items(p, d) * (r.Lb / 16);
  r.u0 = tot16 * gi / gn * 16;
  r.u1 = tot16 * (gi + 1) / gn * 16;
  r.tile = ((uint32_t)kStageBytes / r.nsrc) & ~15u;
  return r;
}

// Producer (one lane): stream the op's tiles into the shared-memory ring.
__device__ __forceinline__ void produce_op(const KParams& p, const OpDesc& d, int opi, const OpRange& r, char* smem,
                                           uint64_t* full, uint64_t* empty, uint32_t& ctr) {
  const int k = d.dim;
  dev::fence_proxy_async_global();  // generic-proxy writes (ours and peers') -> async proxy (TMA)
  // Bandwidth emulation by pacing: this CTA pulls peer bytes of this op no
  // faster than V * BW_k / c_k (the bound topology's bw, R6).  Due times are
  // absolute from the op start, so timer granularity does not accumulate.
  const float pace = p.pace_ns_per_byte[k];
  // The pacing origin is shared by the group's CTAs (first starter wins), so
  // a CTA that starts an op late catches up instead of stretching the op.
  uint64_t t_op = 0;
  if (pace > 0.f) {
    const unsigned long long now = dev::globaltimer();
    const unsigned long long prev = atomicCAS(&p.op_t0[opi], 0ull, now);
    t_op = prev ? prev : now;
  }
  double sent = 0.0;
  for (uint64_t it = r.u0 / r.Lb; it * r.Lb < r.u1; ++it) {
    const Item m = decode_item(p, d, it);
    const uint64_t a = (r.u0 > it * r.Lb ? r.u0 - it * r.Lb : 0);
    const uint64_t e = (r.u1 - it * r.Lb < r.Lb ? r.u1 - it * r.Lb : r.Lb);
    for (uint64_t pos = a; pos < e; pos += r.tile, ++ctr) {
      const uint32_t bytes = (uint32_t)(e - pos < r.tile ? e - pos : r.tile);
      if (pace > 0.f) {
        const uint64_t due = t_op + (uint64_t)(sent * pace);
        while (dev::globaltimer() < due) {
        }
        sent += (double)bytes * (d.phase == 0 ? r.pk - 1 : 1);
      }
      const int s = ctr % p.stages;
      dev::mbar_wait(&empty[s], ((ctr / p.stages) & 1) ^ 1);
      dev::mbar_expect_tx(&full[s], bytes * r.nsrc);
      char* dst = smem + s * kStageBytes;
      if (d.phase == 0) {
        for (int j = 0; j < r.pk; ++j)
          dev::bulk_g2s(dst + j * r.tile, data_of(p, m.g0 + j * (int)p.stride[k]) + m.off + pos, bytes, &full[s]);
      } else {
        dev::bulk_g2s(dst, data_of(p, m.g0 + m.j * (int)p.stride[k]) + m.off + pos, bytes, &full[s]);
      }
    }
  }
}

// Consumers (warps 1..kConsumerWarps): sum the P_k copies of each tile in
// coordinate order (RS) or pass the bytes through (AG), 16-byte STG.
// Returns false if the kernel is aborting (watchdog).
template <class Tag>
__device__ __forceinline__ bool consume_op(const KParams& p, const OpDesc& d, const OpRange& r, const char* smem,
                                           uint64_t* full, uint64_t* empty, uint32_t& ctr) {
  const int ct = threadIdx.x - 32, lane = threadIdx.x & 31;
  constexpr int kCons = 32 * kConsumerWarps;
  const uint32_t tile16 = r.tile / 16;
  for (uint64_t it = r.u0 / r.Lb; it * r.Lb < r.u1; ++it) {
    const Item m = decode_item(p, d, it);
    const uint64_t a = (r.u0 > it * r.Lb ? r.u0 - it * r.Lb : 0);
    const uint64_t e = (r.u1 - it * r.Lb < r.Lb ? r.u1 - it * r.Lb : r.Lb);
    char* base = data_of(p, m.q) + m.off;
    for (uint64_t pos = a; pos < e; pos += r.tile, ++ctr) {
      const uint32_t n16 = (uint32_t)((e - pos < r.tile ? e - pos : r.tile) / 16);
      const int s = ctr % p.stages;
      if (!dev::mbar_wait_or(&full[s], (ctr / p.stages) & 1, p.abort_flag)) return false;
      const uint4* sm = reinterpret_cast<const uint4*>(smem + s * kStageBytes);
      uint4* dst = reinterpret_cast<uint4*>(base + pos);
      if (d.phase == 0) {
        for (uint32_t w = ct; w < n16; w += kCons) {
          float acc[Tag::kAcc];
          Tag::load(acc, sm[w]);
          for (int j = 1; j < r.pk; ++j) Tag::add(acc, sm[j * tile16 + w]);
          dev::st_v4(dst + w, Tag::store(acc));
        }
      } else {
        for (uint32_t w = ct; w < n16; w += kCons) dev::st_v4(dst + w, sm[w]);
      }
      __syncwarp();
      if (lane == 0) dev::mbar_arrive(&empty[s]);
    }
  }
  return true;
}

// One warp: wait until the local ranks and their dim-k peers completed (c, s-1).
__device__ __forceinline__ bool wait_deps_warp(const KParams& p, const OpDesc& d, int opi) {
  const int V = p.V, q0 = p.my_gpu * V, k = d.dim, pk = p.size[k];
  bool ok = true;
  for (int t = threadIdx.x & 31; t < V * pk; t += 32) {
    const int q = q0 + t / pk;
    const int src = q + (t % pk - coord(p, q, k)) * (int)p.stride[k];
    ok &= wait_geq(p, ready_slot(p, q, src, opi - 1), p.epoch, (uint32_t)opi);
  }
  return __all_sync(0xFFFFFFFFu, ok);
}

// One warp: count this CTA's completion of op opi; the group's last CTA
// publishes the epoch to the consumers of (c, s): self and the next stage's
// dim peers.  Release chain: consumers' stores -> named barrier ->
// atom.acq_rel.gpu (all CTAs) -> fence.acq_rel.sys -> relaxed sys stores.
__device__ __forceinline__ void complete_op_warp(const KParams& p, const OpDesc& d, int opi, int gn) {
  const int lane = threadIdx.x & 31;
  uint32_t last = 0;
  if (lane == 0) {
    last = dev::atom_add_acq_rel_gpu(&p.opcnt[opi], 1u) == (uint32_t)gn - 1;
    if (last) {
      p.opcnt[opi] = 0;  // every CTA arrived; reset for the next call
      p.op_t0[opi] = 0;
      dev::fence_acq_rel_sys();
    }
  }
  last = __shfl_sync(0xFFFFFFFFu, last, 0);
  if (!last) return;
  if (d.next_dim >= 0) {
    const int V = p.V, q0 = p.my_gpu * V, kn = d.next_dim, pn = p.size[kn];
    for (int t = lane; t < V * pn; t += 32) {
      const int q = q0 + t / pn;
      const int dst = q + (t % pn - coord(p, q, kn)) * (int)p.stride[kn];
      dev::st_relaxed_sys(ready_slot(p, dst, q, opi), p.epoch);
    }
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
  if (kTma && tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], kConsumerWarps);
    }
    for (int s = 0; s < kOpRing; ++s) {
      dev::mbar_init(&op_done[s], kConsumerWarps);
      dev::mbar_init(&op_free[s], 1);
    }
    dev::fence_mbar_init();
  }

  // a6: entry barrier — every local rank announces the epoch to every rank.
  if (blockIdx.x == 0)
    for (int i = tid; i < V * P; i += blockDim.x) dev::st_release_sys(entry_slot(p, i % P, q0 + i / P), p.epoch);
  for (int i = tid; i < V * P; i += blockDim.x)
    ok &= wait_geq(p, entry_slot(p, q0 + i / P, i % P), p.epoch, 0xFFFFFFu);
  ok = __syncthreads_and(ok);

  // a9: walk this dimension's ops in the enforced order.
  const int* list = p.dim_ops + (uint64_t)g * p.C * p.NS;
  const int nops = ok ? p.dim_ops_n[g] : 0;
  if constexpr (kTma) {
    // Warp-specialised and decoupled: the producer warp waits for an op's
    // dependencies and streams its tiles, then moves on to the next op while
    // the consumer warps finish; the consumers count and publish completion.
    uint32_t ctr = 0;  // ring position (identical sequence in producer and consumers)
    if (warp == 0) {
      for (int i = 0; i < nops; ++i) {
        const int opi = list[i];
        const OpDesc& d = p.ops[opi];
        const OpRange r = op_range(p, d, gi, gn);
        if (r.u0 >= r.u1) continue;  // no bytes for this CTA: nothing to wait for
        if (d.stage > 0 && !wait_deps_warp(p, d, opi)) break;
        if (lane == 0) {
          if (p.trace && gi == 0) p.trace[2 * opi] = dev::globaltimer();
          produce_op(p, d, opi, r, smem, full, empty, ctr);
        }
        __syncwarp();
      }
    } else if (warp <= kConsumerWarps) {
      // consumers: per op, every consumer warp arrives on op_done[slot]
      // (mbarrier arrive = release.cta of its stores) once it is done, after
      // the completion warp has freed that slot (ring of kOpRing ops).
      for (int i = 0; i < nops; ++i) {
        const int opi = list[i];
        const OpDesc& d = p.ops[opi];
        const OpRange r = op_range(p, d, gi, gn);
        if (!consume_op<Tag>(p, d, r, smem, full, empty, ctr)) break;
        __syncwarp();
        bool w = true;
        if (lane == 0) {
          const int slot = i % kOpRing;
          w = dev::mbar_wait_or(&op_free[slot], ((i / kOpRing) & 1) ^ 1, p.abort_flag);
          if (w) dev::mbar_arrive(&op_done[slot]);
        }
        if (!__shfl_sync(0xFFFFFFFFu, w, 0)) break;
      }
    } else {
      // completion warp: counts ops done group-wide and publishes flags, so
      // the atomics / sys fences never stall the consumers' tile stream.
      for (int i = 0; i < nops; ++i) {
        const int opi = list[i];
        const int slot = i % kOpRing;
        bool w = true;
        if (lane == 0) w = dev::mbar_wait_or(&op_done[slot], (i / kOpRing) & 1, p.abort_flag);
        if (!__shfl_sync(0xFFFFFFFFu, w, 0)) break;
        complete_op_warp(p, p.ops[opi], opi, gn);
        if (lane == 0) dev::mbar_arrive(&op_free[slot]);
      }
    }
  } else {
    for (int i = 0; ok && i < nops; ++i) {
      const int opi = list[i];
      const OpDesc& d = p.ops[opi];
      const int k = d.dim;
      if (d.stage > 0) {  // own and dim-k peers' previous stage of this chunk
        const int pk = p.size[k];
        for (int t = tid; t < V * pk; t += blockDim.x) {
          const int q = q0 + t / pk;
          const int src = q + (t % pk - coord(p, q, k)) * (int)p.stride[k];
          ok &= wait_geq(p, ready_slot(p, q, src, opi - 1), p.epoch, (uint32_t)opi);
        }
        ok = __syncthreads_and(ok);
        if (!ok) break;
      }
      if (p.trace && gi == 0 && tid == 0) p.trace[2 * opi] = dev::globaltimer();
      run_op_ldg<Tag>(p, d, gi, gn);
      __syncthreads();
      if (warp == 0) complete_op_warp(p, d, opi, gn);
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
  for (int i = tid; i < V * P; i += blockDim.x) dev::st_release_sys(exit_slot(p, i % P, q0 + i / P), p.epoch);
  for (int i = tid; i < V * P; i += blockDim.x) wait_geq(p, exit_slot(p, q0 + i / P, i % P), p.epoch, 0xFFFFFDu);
}

}  // namespace

// ============================================================== host side
static const void* kernel_for(int dtype, int tma) {
  switch (dtype) {
    case THEMIS_F32: return tma ? (const void*)themis_exec_kernel<dev::F32Tag, true> : (const void*)themis_exec_kernel<dev::F32Tag, false>;
    case THEMIS_BF16: return tma ? (const void*)themis_exec_kernel<dev::BF16Tag, true> : (const void*)themis_exec_kernel<dev::BF16Tag, false>;
    case THEMIS_F16: return tma ? (const void*)themis_exec_kernel<dev::F16Tag, true> : (const void*)themis_exec_kernel<dev::F16Tag, false>;
    default: return tma ? (const void*)themis_exec_kernel<dev::I32Tag, true> : (const void*)themis_exec_kernel<dev::I32Tag, false>;
  }
}

static cudaError_t prepare_kernels() {
  for (int dt = 0; dt < 4; ++dt) {
    cudaError_t e = cudaFuncSetAttribute(kernel_for(dt, 1), cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}
struct themis_comm {
  int gpu_rank = 0, W = 1, P = 1, V = 1, device = 0, num_sms = 0;
  themis_topology_t topo{};
  char* heap[THEMIS_MAX_GPUS] = {};
  uint64_t heap_bytes = 0, vrank_stride = 0, sig_bytes = 0;
  uint32_t epoch = 0;
  uint32_t* opcnt = nullptr;
  unsigned long long* op_t0 = nullptr;
  uint32_t* done_cnt = nullptr;
  uint32_t* abort_flag = nullptr;
  uint32_t* herr_host = nullptr;
  uint32_t* herr_dev = nullptr;
  uint64_t* trace = nullptr;
  bool trace_on = false;
  bool pacing = false;  // emulate per-dim bandwidth by pacing (themis_comm_set_pacing)
  int stages = kStages;  // TMA ring depth (themis_comm_set_stages)
  uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;
  int max_blocks = 0;  // co-resident CTAs for the kernel
  int engine = 1;      // 1: TMA bulk-copy pipeline, 0: LDG/STG
};

namespace themis {
struct BindState {
  themis_comm* comm = nullptr;
  OpDesc* d_ops = nullptr;
  int32_t* d_dim_ops = nullptr;
  int32_t grp_start[THEMIS_MAX_DIMS + 1] = {};
  int32_t ctas[THEMIS_MAX_DIMS] = {};
  int32_t total_ctas = 0;
};
}  // namespace themis

extern "C" themis_status_t themis_heap_layout(int32_t n_ranks, int32_t n_gpus, uint64_t data_bytes,
                                              uint64_t* sig, uint64_t* stride, uint64_t* heap) {
  if (n_ranks < 1 || n_ranks > kMaxRanks || n_gpus < 1 || n_gpus > THEMIS_MAX_GPUS || n_ranks % n_gpus)
    return fail(THEMIS_ERR_INVALID_ARG, "need 1 <= n_gpus <= 8, n_ranks <= 64, n_ranks % n_gpus == 0");
  const int V = n_ranks / n_gpus;
  const uint64_t s = signal_bytes(n_ranks), st = round_up(std::max<uint64_t>(data_bytes, 1), kAlign);
  if (sig) *sig = s;
  if (stride) *stride = st;
  if (heap) *heap = (uint64_t)V * (s + st);
  return THEMIS_OK;
}

extern "C" themis_status_t themis_heap_alloc(uint64_t heap_bytes, void** heap) {
  if (!heap || heap_bytes == 0) return fail(THEMIS_ERR_INVALID_ARG, "bad heap args");
  CUDA_TRY(cudaMalloc(heap, heap_bytes));
  CUDA_TRY(cudaMemset(*heap, 0, heap_bytes));
  CUDA_TRY(cudaDeviceSynchronize());
  return THEMIS_OK;
}
extern "C" themis_status_t themis_heap_free(void* heap) {
  CUDA_TRY(cudaFree(heap));
  return THEMIS_OK;
}
extern "C" themis_status_t themis_heap_export(void* heap, uint8_t* handle) {
  if (!heap || !handle) return fail(THEMIS_ERR_INVALID_ARG, "null argument");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, heap));
  static_assert(sizeof(h) == THEMIS_IPC_HANDLE_BYTES, "ipc handle size");
  std::memcpy(handle, &h, sizeof(h));
  return THEMIS_OK;
}
extern "C" themis_status_t themis_heap_import(const uint8_t* handle, void** peer) {
  if (!handle || !peer) return fail(THEMIS_ERR_INVALID_ARG, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  CUDA_TRY(cudaIpcOpenMemHandle(peer, h, cudaIpcMemLazyEnablePeerAccess));
  return THEMIS_OK;
}
extern "C" themis_status_t themis_heap_close(void* peer) {
  CUDA_TRY(cudaIpcCloseMemHandle(peer));
  return THEMIS_OK;
}

extern "C" themis_status_t themis_comm_create(int32_t gpu_rank, int32_t n_gpus, const themis_topology_t* topo,
                                              void* const* heaps, uint64_t heap_bytes, uint64_t vrank_stride,
                                              themis_comm_t** out) {
  if (!out || !topo || !heaps) return fail(THEMIS_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  if (topo->ndims < 1 || topo->ndims > THEMIS_MAX_DIMS) return fail(THEMIS_ERR_INVALID_ARG, "bad ndims");
  int P = 1;
  for (int k = 0; k < topo->ndims; ++k) {
    if (topo->size[k] < 2) return fail(THEMIS_ERR_INVALID_ARG, "dim size < 2");
    P *= topo->size[k];
    if (P > kMaxRanks) return fail(THEMIS_ERR_INVALID_ARG, "a comm hosts at most 64 logical ranks");
  }
  if (n_gpus < 1 || n_gpus > THEMIS_MAX_GPUS || P % n_gpus || gpu_rank < 0 || gpu_rank >= n_gpus)
    return fail(THEMIS_ERR_INVALID_ARG, "bad gpu_rank / n_gpus for this topology");
  uint64_t sig, stride, hb;
  themis_heap_layout(P, n_gpus, vrank_stride, &sig, &stride, &hb);
  if (stride != vrank_stride || hb > heap_bytes)
    return fail(THEMIS_ERR_INVALID_ARG, "heap too small or vrank_stride not from themis_heap_layout");
  auto* c = new themis_comm();
  c->gpu_rank = gpu_rank;
  c->W = n_gpus;
  c->P = P;
  c->V = P / n_gpus;
  c->topo = *topo;
  for (int g = 0; g < n_gpus; ++g) c->heap[g] = static_cast<char*>(heaps[g]);
  c->heap_bytes = heap_bytes;
  c->vrank_stride = vrank_stride;
  c->sig_bytes = sig;
  cudaError_t e;
  if ((e = cudaGetDevice(&c->device)) != cudaSuccess ||
      (e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device)) != cudaSuccess ||
      (e = cudaMalloc(&c->opcnt, sizeof(uint32_t) * (kMaxOps + 8))) != cudaSuccess ||
      (e = cudaMalloc(&c->op_t0, sizeof(unsigned long long) * kMaxOps)) != cudaSuccess ||
      (e = cudaMemset(c->op_t0, 0, sizeof(unsigned long long) * kMaxOps)) != cudaSuccess ||
      (e = cudaMemset(c->opcnt, 0, sizeof(uint32_t) * (kMaxOps + 8))) != cudaSuccess ||
      (e = cudaMalloc(&c->trace, sizeof(uint64_t) * 2 * kMaxOps)) != cudaSuccess ||
      (e = cudaMemset(c->trace, 0, sizeof(uint64_t) * 2 * kMaxOps)) != cudaSuccess ||
      (e = cudaHostAlloc(&c->herr_host, sizeof(uint32_t), cudaHostAllocMapped)) != cudaSuccess ||
      (e = cudaHostGetDevicePointer(&c->herr_dev, c->herr_host, 0)) != cudaSuccess) {
    delete c;
    return cuda_fail(e, "themis_comm_create");
  }
  *c->herr_host = 0;
  c->done_cnt = c->opcnt + kMaxOps;
  c->abort_flag = c->opcnt + kMaxOps + 1;
  int nb = 0;
  if ((e = prepare_kernels()) != cudaSuccess ||
      (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, themis_exec_kernel<dev::F32Tag, true>, kThreads,
                                                         kSmemBytes)) != cudaSuccess) {
    delete c;
    return cuda_fail(e, "kernel attributes / occupancy query");
  }
  if (const char* env = getenv("THEMIS_COPY_ENGINE")) c->engine = std::string(env) == "ldg" ? 0 : 1;
  if (const char* env = getenv("THEMIS_STAGES")) c->stages = std::max(1, std::min(kStages, atoi(env)));
  c->max_blocks = nb * c->num_sms;
  *out = c;
  return THEMIS_OK;
}

extern "C" void themis_comm_free(themis_comm_t* c) {
  if (!c) return;
  cudaFree(c->opcnt);
  cudaFree(c->op_t0);
  cudaFree(c->trace);
  cudaFreeHost(c->herr_host);
  delete c;
}

extern "C" themis_status_t themis_comm_status(themis_comm_t* c) {
  if (!c) return fail(THEMIS_ERR_INVALID_ARG, "null comm");
  uint32_t v = *(volatile uint32_t*)c->herr_host;
  if (v) return fail((themis_status_t)(v & 0xFF), "device watchdog fired while waiting (code " + std::to_string(v >> 8) + ")");
  return THEMIS_OK;
}
extern "C" themis_status_t themis_comm_set_engine(themis_comm_t* c, int32_t engine) {
  if (!c || engine < 0 || engine > 1) return fail(THEMIS_ERR_INVALID_ARG, "engine must be 0 (LDG) or 1 (TMA)");
  c->engine = engine;
  return THEMIS_OK;
}
extern "C" themis_status_t themis_comm_set_stages(themis_comm_t* c, int32_t stages) {
  if (!c || stages < 1 || stages > kStages) return fail(THEMIS_ERR_INVALID_ARG, "stages must be 1..6");
  c->stages = stages;
  return THEMIS_OK;
}
extern "C" themis_status_t themis_comm_set_pacing(themis_comm_t* c, int32_t on) {
  if (!c) return fail(THEMIS_ERR_INVALID_ARG, "null comm");
  c->pacing = on != 0;
  return THEMIS_OK;
}
extern "C" themis_status_t themis_comm_set_timeout(themis_comm_t* c, uint64_t ns) {
  if (!c || ns == 0) return fail(THEMIS_ERR_INVALID_ARG, "bad timeout");
  c->timeout_ns = ns;
  return THEMIS_OK;
}
extern "C" themis_status_t themis_comm_enable_trace(themis_comm_t* c, int32_t on) {
  if (!c) return fail(THEMIS_ERR_INVALID_ARG, "null comm");
  c->trace_on = on != 0;
  return THEMIS_OK;
}
extern "C" themis_status_t themis_trace_fetch(themis_comm_t* c, uint64_t* out, size_t n) {
  if (!c || !out || n > 2ull * kMaxOps) return fail(THEMIS_ERR_INVALID_ARG, "bad trace args");
  CUDA_TRY(cudaMemcpy(out, c->trace, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return THEMIS_OK;
}

static void free_bind(themis_plan_t* pl) {
  if (!pl->bind) return;
  cudaFree(pl->bind->d_ops);
  cudaFree(pl->bind->d_dim_ops);
  delete pl->bind;
  pl->bind = nullptr;
}

extern "C" void themis_plan_free(themis_plan_t* pl) {
  if (!pl) return;
  free_bind(pl);
  delete pl;
}

extern "C" themis_status_t themis_plan_bind(themis_plan_t* pl, themis_comm_t* c, const int32_t* ctas) {
  if (!pl || !c) return fail(THEMIS_ERR_INVALID_ARG, "null argument");
  const int D = pl->D;
  if (c->topo.ndims != D) return fail(THEMIS_ERR_INVALID_ARG, "plan / comm topology mismatch");
  for (int k = 0; k < D; ++k)
    if (c->topo.size[k] != pl->topo.size[k]) return fail(THEMIS_ERR_INVALID_ARG, "plan / comm topology mismatch");
  if ((int64_t)pl->C * pl->NS > kMaxOps) return fail(THEMIS_ERR_INVALID_ARG, "too many ops");
  int32_t n[THEMIS_MAX_DIMS];
  int tot = 0;
  if (ctas) {
    for (int k = 0; k < D; ++k) {
      if (ctas[k] < 1) return fail(THEMIS_ERR_INVALID_ARG, "ctas_per_dim must be >= 1");
      n[k] = ctas[k];
      tot += n[k];
    }
  } else {  // proportional to bandwidth over all SMs, largest remainder, >= 1 each
    uint64_t sum = 0;
    for (int k = 0; k < D; ++k) sum += pl->topo.bw_mbps[k];
    const int budget = std::max(D, c->max_blocks);
    std::vector<std::pair<double, int>> rem;
    for (int k = 0; k < D; ++k) {
      double x = (double)budget * pl->topo.bw_mbps[k] / (double)sum;
      n[k] = std::max(1, (int)x);
      tot += n[k];
      rem.push_back({x - (int)x, k});
    }
    std::sort(rem.begin(), rem.end(), [](auto& a, auto& b) { return a.first > b.first || (a.first == b.first && a.second < b.second); });
    for (size_t i = 0; tot < budget && i < rem.size(); ++i, ++tot) ++n[rem[i].second];
    while (tot > budget) {  // the >= 1 floor overshot: trim the largest group
      int kmax = (int)(std::max_element(n, n + D) - n);
      --n[kmax];
      --tot;
    }
  }
  if (tot > c->max_blocks)
    return fail(THEMIS_ERR_INVALID_ARG, "sum of ctas_per_dim (" + std::to_string(tot) + ") exceeds co-resident CTAs (" +
                                            std::to_string(c->max_blocks) + ")");
  // descriptors
  std::vector<OpDesc> ops(pl->ops.size());
  for (size_t i = 0; i < pl->ops.size(); ++i) {
    const Op& o = pl->ops[i];
    OpDesc d{};
    d.chunk = o.chunk;
    d.stage = o.stage;
    d.dim = o.dim;
    d.phase = o.phase;
    d.reduced = o.reduced_before;
    d.next_dim = o.stage + 1 < pl->NS ? pl->ops[i + 1].dim : -1;
    const uint32_t fixed = o.phase == 0 ? (o.reduced_before | (1u << o.dim)) : o.reduced_before;
    d.nblk = 1;
    int64_t stride = 1;
    for (int k = 0; k < D; ++k) {
      if (!(fixed >> k & 1u)) {
        d.free_size[d.nfree] = pl->topo.size[k];
        d.free_stride[d.nfree] = stride;
        ++d.nfree;
        d.nblk *= pl->topo.size[k];
      }
      stride *= pl->topo.size[k];
    }
    ops[i] = d;
  }
  std::vector<int32_t> lists((size_t)D * pl->C * pl->NS, 0);
  for (int k = 0; k < D; ++k)
    for (size_t i = 0; i < pl->dim_ops[k].size(); ++i) {
      uint32_t e = pl->dim_ops[k][i];
      lists[(size_t)k * pl->C * pl->NS + i] = (int32_t)((e >> 8) * pl->NS + (e & 0xFF));
    }
  free_bind(pl);
  auto* b = new BindState();
  b->comm = c;
  cudaError_t e;
  if ((e = cudaMalloc(&b->d_ops, sizeof(OpDesc) * ops.size())) != cudaSuccess ||
      (e = cudaMemcpy(b->d_ops, ops.data(), sizeof(OpDesc) * ops.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMalloc(&b->d_dim_ops, sizeof(int32_t) * lists.size())) != cudaSuccess ||
      (e = cudaMemcpy(b->d_dim_ops, lists.data(), sizeof(int32_t) * lists.size(), cudaMemcpyHostToDevice)) != cudaSuccess) {
    pl->bind = b;
    free_bind(pl);
    return cuda_fail(e, "themis_plan_bind upload");
  }
  b->grp_start[0] = 0;
  for (int k = 0; k < D; ++k) {
    b->ctas[k] = n[k];
    b->grp_start[k + 1] = b->grp_start[k] + n[k];
  }
  b->total_ctas = tot;
  pl->bind = b;
  return THEMIS_OK;
}

extern "C" themis_status_t themis_plan_bound_ctas(const themis_plan_t* pl, int32_t* ctas) {
  if (!pl || !pl->bind || !ctas) return fail(THEMIS_ERR_PLAN_MISMATCH, "plan not bound");
  for (int k = 0; k < pl->D; ++k) ctas[k] = pl->bind->ctas[k];
  return THEMIS_OK;
}

static themis_status_t launch(int coll, void* buf, uint64_t count, int32_t dtype, const themis_plan_t* pl,
                              void* stream) {
  if (!pl || !pl->bind) return fail(THEMIS_ERR_PLAN_MISMATCH, "plan is not bound to a comm");
  if (pl->req.coll != coll) return fail(THEMIS_ERR_PLAN_MISMATCH, "plan was made for another collective");
  themis_comm* c = pl->bind->comm;
  themis_status_t st = themis_comm_status(c);
  if (st != THEMIS_OK) return st;
  int esz;
  switch (dtype) {
    case THEMIS_F32: case THEMIS_I32: esz = 4; break;
    case THEMIS_BF16: case THEMIS_F16: esz = 2; break;
    default: return fail(THEMIS_ERR_UNSUPPORTED_DTYPE, "unsupported dtype");
  }
  if (count * (uint64_t)esz != pl->req.bytes)
    return fail(THEMIS_ERR_INVALID_ARG, "count * elem_size != plan bytes");
  const uint64_t vec = 16 / esz;
  if (count % ((uint64_t)pl->P * pl->C * vec))
    return fail(THEMIS_ERR_ALIGNMENT, "count must be a multiple of P * n_chunks * (16 / elem_size)");
  char* mine = c->heap[c->gpu_rank];
  char* p = static_cast<char*>(buf);
  const uint64_t data0 = (uint64_t)c->V * c->sig_bytes;
  if (p < mine + data0 || (uint64_t)(p - mine - data0) >= c->vrank_stride ||
      (uint64_t)(p - mine - data0) + count * esz > c->vrank_stride)
    return fail(THEMIS_ERR_NOT_REGISTERED, "buf is not inside the comm's heap data region");
  if (reinterpret_cast<uintptr_t>(p) % 16) return fail(THEMIS_ERR_ALIGNMENT, "buf must be 16-byte aligned");

  KParams kp{};
  kp.D = pl->D;
  kp.P = c->P;
  kp.V = c->V;
  kp.W = c->W;
  kp.my_gpu = c->gpu_rank;
  kp.C = pl->C;
  kp.NS = pl->NS;
  int64_t s = 1;
  for (int k = 0; k < pl->D; ++k) {
    kp.size[k] = pl->topo.size[k];
    kp.stride[k] = s;
    s *= pl->topo.size[k];
    kp.dim_ops_n[k] = (int32_t)pl->dim_ops[k].size();
  }
  for (int k = 0; k <= pl->D; ++k) kp.grp_start[k] = pl->bind->grp_start[k];
  kp.ops = pl->bind->d_ops;
  kp.dim_ops = pl->bind->d_dim_ops;
  for (int g = 0; g < c->W; ++g) kp.heap[g] = c->heap[g];
  kp.data_rel = (uint64_t)(p - mine);
  kp.vrank_stride = c->vrank_stride;
  kp.sig_bytes = c->sig_bytes;
  kp.blk_elems = count / c->P;
  kp.slice_elems = count / ((uint64_t)c->P * pl->C);
  kp.elem_size = esz;
  kp.epoch = ++c->epoch;
  kp.opcnt = c->opcnt;
  kp.op_t0 = c->op_t0;
  kp.done_cnt = c->done_cnt;
  kp.abort_flag = c->abort_flag;
  kp.herr = c->herr_dev;
  kp.timeout_ns = c->timeout_ns;
  kp.trace = c->trace_on ? c->trace : nullptr;
  kp.stages = c->stages;
  for (int k = 0; k < pl->D; ++k)  // ns per byte per CTA = c_k / (V * bw_k[bytes/ns])
    kp.pace_ns_per_byte[k] =
        c->pacing ? (float)((double)pl->bind->ctas[k] * 1000.0 / ((double)c->V * pl->topo.bw_mbps[k])) : 0.f;

  void* args[] = {&kp};
  const void* fn = kernel_for(dtype, c->engine);
  cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(pl->bind->total_ctas), dim3(kThreads), args,
                                              c->engine ? kSmemBytes : 0,
                                              static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchCooperativeKernel");
  return THEMIS_OK;
}

extern "C" themis_status_t themis_allreduce(void* buf, uint64_t count, int32_t dtype, const themis_plan_t* pl, void* stream) {
  return launch(THEMIS_ALLREDUCE, buf, count, dtype, pl, stream);
}
extern "C" themis_status_t themis_reduce_scatter(void* buf, uint64_t count, int32_t dtype, const themis_plan_t* pl,
                                                 void* stream) {
  return launch(THEMIS_REDUCE_SCATTER, buf, count, dtype, pl, stream);
}
extern "C" themis_status_t themis_all_gather(void* buf, uint64_t count, int32_t dtype, const themis_plan_t* pl, void* stream) {
  return launch(THEMIS_ALL_GATHER, buf, count, dtype, pl, stream);
}

extern "C" themis_status_t themis_allreduce_host(const void* host_in, void* host_out, void* buf, uint64_t count,
                                                 int32_t dtype, const themis_plan_t* pl, void* stream) {
  if (!pl || !pl->bind) return fail(THEMIS_ERR_PLAN_MISMATCH, "plan is not bound to a comm");
  if (!host_in || !host_out) return fail(THEMIS_ERR_INVALID_ARG, "null host buffer");
  themis_comm* c = pl->bind->comm;
  const uint64_t bytes = pl->req.bytes;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int v = 0; v < c->V; ++v)
    CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(buf) + v * c->vrank_stride, static_cast<const char*>(host_in) + v * bytes,
                             bytes, cudaMemcpyHostToDevice, s));
  themis_status_t st = themis_allreduce(buf, count, dtype, pl, stream);
  if (st != THEMIS_OK) return st;
  for (int v = 0; v < c->V; ++v)
    CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(host_out) + v * bytes, static_cast<char*>(buf) + v * c->vrank_stride,
                             bytes, cudaMemcpyDeviceToHost, s));
  return THEMIS_OK;
}

extern "C" int32_t themis_launches_per_call(void) { return 1; }
