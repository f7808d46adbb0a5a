// Device-side building blocks of the Themis executor (sm_100a).
//
// Memory-ordering chain of the TMA executor (exec_kernel.cuh), per op:
//   consumer warps: 16-byte st.global of the op's output -> mbarrier.arrive
//     (release.cta) on the unit's op_done barrier;
//   completion warp: mbarrier wait (acquire.cta) -> atom.acq_rel.gpu on the
//     op's CTA counter; the group's last CTA then runs fence.acq_rel.gpu (every
//     consumer of the flag on this GPU) or fence.acq_rel.sys (some consumer on
//     a peer GPU) on every storing lane, and publishes the epoch with
//     st.relaxed.{gpu,sys} into the consumers' signal pads;
//   producer warp of a consumer: ld.acquire.sys polls of its own pad ->
//     fence.proxy.async.global -> cp.async.bulk (TMA) reads of the peer data;
//   ring slots: consumers' shared-memory reads -> mbarrier.arrive (release) on
//     empty[s] -> producer's acquire wait -> next TMA write into the slot.
// Ring-step flags follow the same fence-then-relaxed-store pattern; the entry
// and exit barriers use st.release.sys / ld.acquire.sys directly.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace themis {
namespace dev {

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// 16-byte vector moves.  .cg: cache in L2 only (no stale L1 lines for data
// other CTAs / GPUs wrote during this launch).
__device__ __forceinline__ uint4 ld_cg(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v4(uint4* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// ---- elementwise accumulate of one 16-byte vector, per dtype -------------
// Accumulator layout: 4 x f32 (f32), 8 x f32 (bf16/f16, one vector of 8
// elements), 4 x i32 (i32).  The sum is taken in coordinate order (R18).
struct F32Tag {
  static constexpr int kAcc = 4;
  __device__ static void load(float* a, const uint4& v) {
    a[0] = __uint_as_float(v.x); a[1] = __uint_as_float(v.y);
    a[2] = __uint_as_float(v.z); a[3] = __uint_as_float(v.w);
  }
  __device__ static void add(float* a, const uint4& v) {
    a[0] = __fadd_rn(a[0], __uint_as_float(v.x)); a[1] = __fadd_rn(a[1], __uint_as_float(v.y));
    a[2] = __fadd_rn(a[2], __uint_as_float(v.z)); a[3] = __fadd_rn(a[3], __uint_as_float(v.w));
  }
  __device__ static uint4 store(const float* a) {
    return make_uint4(__float_as_uint(a[0]), __float_as_uint(a[1]), __float_as_uint(a[2]), __float_as_uint(a[3]));
  }
};

struct BF16Tag {
  static constexpr int kAcc = 8;
  __device__ static float lo(uint32_t w) { return __uint_as_float(w << 16); }
  __device__ static float hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
  __device__ static void load(float* a, const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) { a[2 * i] = lo(w[i]); a[2 * i + 1] = hi(w[i]); }
  }
  __device__ static void add(float* a, const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[2 * i] = __fadd_rn(a[2 * i], lo(w[i]));
      a[2 * i + 1] = __fadd_rn(a[2 * i + 1], hi(w[i]));
    }
  }
  __device__ static uint32_t pack(float x, float y) {
    __nv_bfloat162 h = __floats2bfloat162_rn(x, y);  // round to nearest even
    return *reinterpret_cast<uint32_t*>(&h);
  }
  __device__ static uint4 store(const float* a) {
    return make_uint4(pack(a[0], a[1]), pack(a[2], a[3]), pack(a[4], a[5]), pack(a[6], a[7]));
  }
};

struct F16Tag {
  static constexpr int kAcc = 8;
  __device__ static void load(float* a, const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
      a[2 * i] = f.x; a[2 * i + 1] = f.y;
    }
  }
  __device__ static void add(float* a, const uint4& v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
      a[2 * i] = __fadd_rn(a[2 * i], f.x); a[2 * i + 1] = __fadd_rn(a[2 * i + 1], f.y);
    }
  }
  __device__ static uint4 store(const float* a) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = __floats2half2_rn(a[2 * i], a[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};

struct I32Tag {  // wraps mod 2^32 (R19); float slots hold raw bits
  static constexpr int kAcc = 4;
  __device__ static void load(float* a, const uint4& v) {
    a[0] = __uint_as_float(v.x); a[1] = __uint_as_float(v.y);
    a[2] = __uint_as_float(v.z); a[3] = __uint_as_float(v.w);
  }
  __device__ static void add(float* a, const uint4& v) {
    a[0] = __uint_as_float(__float_as_uint(a[0]) + v.x); a[1] = __uint_as_float(__float_as_uint(a[1]) + v.y);
    a[2] = __uint_as_float(__float_as_uint(a[2]) + v.z); a[3] = __uint_as_float(__float_as_uint(a[3]) + v.w);
  }
  __device__ static uint4 store(const float* a) {
    return make_uint4(__float_as_uint(a[0]), __float_as_uint(a[1]), __float_as_uint(a[2]), __float_as_uint(a[3]));
  }
};

// ---- the hot loops ---------------------------------------------------------
// RS piece: dst[u] = src[0][u] + src[1][u] + ... + src[n-1][u] for 16-byte
// vectors u in [a, e), all NSRC loads of UNROLL vectors issued before any add
// so that NSRC*UNROLL 16-byte requests are in flight per thread.
template <class Tag, int NSRC, int UNROLL, class Src>
__device__ __forceinline__ void reduce_range(uint4* __restrict__ dst, const Src& src, uint64_t a, uint64_t e) {
  const uint64_t step = (uint64_t)blockDim.x * UNROLL;
  const uint4* s[NSRC];
#pragma unroll
  for (int j = 0; j < NSRC; ++j) s[j] = src(j);
#pragma unroll 1
  for (uint64_t u = a + threadIdx.x; u < e; u += step) {
    uint4 x[NSRC][UNROLL];
#pragma unroll
    for (int r = 0; r < UNROLL; ++r) {
      const uint64_t uu = u + (uint64_t)r * blockDim.x;
      if (uu < e) {
#pragma unroll
        for (int j = 0; j < NSRC; ++j) x[j][r] = ld_cg(s[j] + uu);
      }
    }
#pragma unroll
    for (int r = 0; r < UNROLL; ++r) {
      const uint64_t uu = u + (uint64_t)r * blockDim.x;
      if (uu < e) {
        float acc[Tag::kAcc];
        Tag::load(acc, x[0][r]);
#pragma unroll
        for (int j = 1; j < NSRC; ++j) Tag::add(acc, x[j][r]);
        st_v4(dst + uu, Tag::store(acc));
      }
    }
  }
}

// Generic source count (P_k > 8): one source at a time, still in order.
template <class Tag, class Src>
__device__ __forceinline__ void reduce_range_generic(uint4* __restrict__ dst, const Src& src, int n, uint64_t a,
                                                     uint64_t e) {
#pragma unroll 1
  for (uint64_t u = a + threadIdx.x; u < e; u += blockDim.x) {
    float acc[Tag::kAcc];
    Tag::load(acc, ld_cg(src(0) + u));
    for (int j = 1; j < n; ++j) Tag::add(acc, ld_cg(src(j) + u));
    st_v4(dst + u, Tag::store(acc));
  }
}

// AG piece: bitwise copy of 16-byte vectors [a, e).
template <int UNROLL>
__device__ __forceinline__ void copy_range(uint4* __restrict__ dst, const uint4* __restrict__ src, uint64_t a,
                                           uint64_t e) {
  const uint64_t step = (uint64_t)blockDim.x * UNROLL;
#pragma unroll 1
  for (uint64_t u = a + threadIdx.x; u < e; u += step) {
    uint4 x[UNROLL];
#pragma unroll
    for (int r = 0; r < UNROLL; ++r) {
      const uint64_t uu = u + (uint64_t)r * blockDim.x;
      if (uu < e) x[r] = ld_cg(src + uu);
    }
#pragma unroll
    for (int r = 0; r < UNROLL; ++r) {
      const uint64_t uu = u + (uint64_t)r * blockDim.x;
      if (uu < e) st_v4(dst + uu, x[r]);
    }
  }
}

}  // namespace dev
}  // namespace themis

namespace themis {
namespace dev {
// ---- mbarrier + bulk async copy (TMA engine, no tensor map needed) --------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global (local HBM or a peer GPU over NVLink) -> shared, completes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// shared -> global (local HBM or a peer's HBM over NVLink): a TMA bulk store
// in the calling thread's bulk async-group
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the calling thread's bulk stores have finished READING shared memory
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// ... and their global writes are complete
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
}  // namespace dev
}  // namespace themis

namespace themis {
namespace dev {
// mbarrier wait that gives up when the kernel is aborting (watchdog fired).
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_wait_or(uint64_t* bar, uint32_t parity, const uint32_t* abort_flag) {
  for (;;) {
#pragma unroll 1
    for (int i = 0; i < 64; ++i)
      if (mbar_try_wait(bar, parity)) return true;
    if (*(volatile const uint32_t*)abort_flag) return false;
  }
}
// NVLS (NVSwitch in-switch reduction, PAPER.md:493-494 in-network offload):
// 16 bytes reduced over every GPU bound to the multicast address, then the
// result broadcast to all of them.  bf16 / f16 accumulate in fp32 in the
// switch and round once; int32 wraps; the switch's summation order is its own.
template <class Tag>
__device__ __forceinline__ uint4 mc_ld_reduce(const void* mc);
template <>
__device__ __forceinline__ uint4 mc_ld_reduce<F32Tag>(const void* mc) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
  return v;
}
template <>
__device__ __forceinline__ uint4 mc_ld_reduce<BF16Tag>(const void* mc) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
  return v;
}
template <>
__device__ __forceinline__ uint4 mc_ld_reduce<F16Tag>(const void* mc) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
  return v;
}
template <>
__device__ __forceinline__ uint4 mc_ld_reduce<I32Tag>(const void* mc) {
  const char* b = static_cast<const char*>(mc);
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(v.x) : "l"(b) : "memory");
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(v.y) : "l"(b + 4) : "memory");
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(v.z) : "l"(b + 8) : "memory");
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(v.w) : "l"(b + 12) : "memory");
  return v;
}
__device__ __forceinline__ void mc_st(void* mc, const uint4& v) {  // 16 bytes, bits as they are
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(mc), "f"(__uint_as_float(v.x)), "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)),
                  "f"(__uint_as_float(v.w)) : "memory");
}
// LL packets (R31): 16 payload bytes as four 8-byte {payload u32, tag u32}
// packets, each a single-copy-atomic 64-bit store (two 16-byte vector stores)
__device__ __forceinline__ void st_ll(void* dst, const uint4& v, uint32_t tag) {
  const unsigned long long a = (unsigned long long)v.x | ((unsigned long long)tag << 32);
  const unsigned long long b = (unsigned long long)v.y | ((unsigned long long)tag << 32);
  const unsigned long long c = (unsigned long long)v.z | ((unsigned long long)tag << 32);
  const unsigned long long d = (unsigned long long)v.w | ((unsigned long long)tag << 32);
  char* p = static_cast<char*>(dst);
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p + 16), "l"(c), "l"(d) : "memory");
}
// one poll of four packets: true (and the payload) if all carry `tag`
__device__ __forceinline__ bool ld_ll_try(const void* src, uint32_t tag, uint4& v) {
  const char* p = static_cast<const char*>(src);
  unsigned long long a, b, c, d;
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(c), "=l"(d) : "l"(p + 16) : "memory");
  if ((uint32_t)(a >> 32) != tag || (uint32_t)(b >> 32) != tag || (uint32_t)(c >> 32) != tag ||
      (uint32_t)(d >> 32) != tag)
    return false;
  v = make_uint4((uint32_t)a, (uint32_t)b, (uint32_t)c, (uint32_t)d);
  return true;
}
__device__ __forceinline__ void mbar_arrive_token(uint64_t* bar) {  // a zero-byte "go" for a ring slot
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// named barrier over nthreads threads that also ANDs a per-thread predicate:
// every participant gets the same answer (a CTA-uniform decision)
__device__ __forceinline__ bool named_bar_and(int id, int nthreads, bool v) {
  uint32_t r;
  asm volatile(
      "{\n"
      ".reg .pred p, q;\n"
      "setp.ne.u32 p, %1, 0;\n"
      "bar.red.and.pred q, %2, %3, p;\n"
      "selp.u32 %0, 1, 0, q;\n"
      "}\n"
      : "=r"(r)
      : "r"((uint32_t)v), "r"(id), "r"(nthreads)
      : "memory");
  return r != 0;
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
}  // namespace dev
}  // namespace themis

namespace themis {
namespace dev {
__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
}  // namespace dev
}  // namespace themis
