// NVLink transfer-engine probe (experiment for the executor's NVLink path,
// VERDICT r01 "Next round" item 3; not on the product path).
//
// One process drives every GPU of the box (peer access), all GPUs move data at
// the same time in a symmetric pattern, each GPU is timed with CUDA events on
// its own stream.  Modes (what one GPU g does, per peer p of its pattern):
//   pull   : TMA bulk copy p.src -> smem ring -> consumers st.global to g.dst
//            (the executor's engine today: remote reads)
//   push   : TMA bulk copy g.src -> smem ring -> TMA bulk store smem -> p.dst
//            (remote writes, no registers)
//   pushst : TMA bulk copy g.src -> smem ring -> consumers st.global to p.dst
//   memcpy : cudaMemcpyPeerAsync(g.dst <- p.src), one per peer
//   local  : TMA copy g.src -> smem -> g.dst (HBM reference)
// Patterns: pair1 (g^1), pair2 (g^2), all (every other GPU), mix (pair1 + pair2).
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o nvlink_probe nvlink_probe.cu
//   ./nvlink_probe <mode> <pattern> <ctas> <stages> <stage_kb> <mib_per_peer> [iters] [ngpus]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

constexpr int kThreads = 288;  // warp 0 producer, warps 1..8 consumers
constexpr int kMaxPeers = 8;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
          su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void g2s(void* s, const void* g, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(s)),
               "l"(g), "r"(n), "r"(su32(b))
               : "memory");
}
__device__ __forceinline__ void s2g(void* g, const void* s, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(su32(s)), "r"(n) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

struct Args {
  const char* src[kMaxPeers];  // per peer slot: where to read
  char* dst[kMaxPeers];        // per peer slot: where to write
  int npeers;
  uint64_t bytes;  // per peer
  int stages, stage_bytes, mode;  // mode 0 pull/local (consumers store), 1 push (TMA store)
};

__global__ void __launch_bounds__(kThreads, 1) xfer_kernel(const __grid_constant__ Args a) {
  extern __shared__ __align__(128) char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.stages * a.stage_bytes);
  uint64_t* empty = full + a.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], a.mode == 1 ? 1 : 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // CTA b serves peer b % npeers, sub-range (b / npeers) of that peer's bytes
  const int pe = blockIdx.x % a.npeers;
  const int per = gridDim.x / a.npeers + ((int)(blockIdx.x % a.npeers) < (int)(gridDim.x % a.npeers) ? 1 : 0);
  const int idx = blockIdx.x / a.npeers;
  const uint64_t n16 = a.bytes / 16;
  const uint64_t b0 = n16 * idx / per * 16, b1 = n16 * (idx + 1) / per * 16;
  const char* src = a.src[pe];
  char* dst = a.dst[pe];
  const uint32_t T = a.stage_bytes;
  const uint64_t ntiles = (b1 - b0 + T - 1) / T;
  if (warp == 0) {
    if (lane == 0) {
      for (uint64_t t = 0; t < ntiles; ++t) {
        const int s = t % a.stages;
        mbar_wait(&empty[s], ((t / a.stages) & 1) ^ 1);
        const uint64_t off = b0 + t * T;
        const uint32_t n = (uint32_t)(b1 - off < T ? b1 - off : T);
        mbar_expect_tx(&full[s], n);
        g2s(smem + s * T, src + off, n, &full[s]);
      }
    }
  } else if (a.mode == 1) {
    // push: one thread of warp 1 issues the bulk stores; frees a slot once its read is done
    if (warp == 1 && lane == 0) {
      for (uint64_t t = 0; t < ntiles; ++t) {
        const int s = t % a.stages;
        mbar_wait(&full[s], (t / a.stages) & 1);
        const uint64_t off = b0 + t * T;
        const uint32_t n = (uint32_t)(b1 - off < T ? b1 - off : T);
        s2g(dst + off, smem + s * T, n);
        commit();
        wait_read<0>();
        mbar_arrive(&empty[s]);
      }
      wait_all();
    }
  } else {
    const int ct = threadIdx.x - 32;
    for (uint64_t t = 0; t < ntiles; ++t) {
      const int s = t % a.stages;
      mbar_wait(&full[s], (t / a.stages) & 1);
      const uint64_t off = b0 + t * T;
      const uint32_t n = (uint32_t)(b1 - off < T ? b1 - off : T);
      const uint4* sm = reinterpret_cast<const uint4*>(smem + s * T);
      uint4* d = reinterpret_cast<uint4*>(dst + off);
      for (uint32_t w = ct; w < n / 16; w += 256) d[w] = sm[w];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
}

int main(int argc, char** argv) {
  if (argc < 7) {
    fprintf(stderr, "usage: %s mode pattern ctas stages stage_kb mib_per_peer [iters] [ngpus]\n", argv[0]);
    return 2;
  }
  const std::string mode = argv[1], pat = argv[2];
  const int ctas = atoi(argv[3]), stages = atoi(argv[4]), skb = atoi(argv[5]);
  const uint64_t bytes = (uint64_t)atoi(argv[6]) << 20;
  const int iters = argc > 7 ? atoi(argv[7]) : 5;
  int W = 0;
  CK(cudaGetDeviceCount(&W));
  if (argc > 8) W = std::min(W, atoi(argv[8]));
  std::vector<std::vector<int>> peers(W);
  for (int g = 0; g < W; ++g) {
    if (pat == "pair1") peers[g] = {g ^ 1};
    else if (pat == "pair2") peers[g] = {g ^ 2};
    else if (pat == "mix") peers[g] = {g ^ 1, g ^ 2};
    else if (pat == "all") { for (int p = 0; p < W; ++p) if (p != g) peers[g].push_back(p); }
    else if (pat == "self") peers[g] = {g};
    else { fprintf(stderr, "bad pattern\n"); return 2; }
    for (int p : peers[g]) if (p >= W) { fprintf(stderr, "pattern needs more GPUs\n"); return 2; }
  }
  const int maxp = W;  // dst regions: one per source GPU
  std::vector<char*> src(W), dst(W);
  std::vector<cudaStream_t> st(W);
  std::vector<cudaEvent_t> e0(W), e1(W);
  const int smem = stages * skb * 1024 + 2 * stages * 8;
  for (int g = 0; g < W; ++g) {
    CK(cudaSetDevice(g));
    for (int p = 0; p < W; ++p)
      if (p != g) {
        cudaError_t e = cudaDeviceEnablePeerAccess(p, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
        cudaGetLastError();
      }
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMalloc(&dst[g], bytes * maxp));
    CK(cudaMemset(src[g], g + 1, bytes));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
    CK(cudaFuncSetAttribute(xfer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  auto launch = [&](int g) {
    Args a{};
    a.npeers = (int)peers[g].size();
    a.bytes = bytes;
    a.stages = stages;
    a.stage_bytes = skb * 1024;
    for (int i = 0; i < a.npeers; ++i) {
      const int p = peers[g][i];
      if (mode == "pull" || mode == "local") {
        a.src[i] = src[mode == "local" ? g : p];
        a.dst[i] = dst[g] + (uint64_t)p * bytes;
        a.mode = 0;
      } else {  // push / pushst: own src -> region g of peer p's dst
        a.src[i] = src[g];
        a.dst[i] = dst[p] + (uint64_t)g * bytes;
        a.mode = mode == "push" ? 1 : 0;
      }
    }
    if (mode == "memcpy") {
      for (int i = 0; i < a.npeers; ++i) {
        const int p = peers[g][i];
        CK(cudaMemcpyPeerAsync(dst[g] + (uint64_t)p * bytes, g, src[p], p, bytes, st[g]));
      }
      return;
    }
    xfer_kernel<<<ctas, kThreads, smem, st[g]>>>(a);
    CK(cudaGetLastError());
  };
  std::vector<double> best(W, 1e30), sum(W, 0);
  for (int it = -2; it < iters; ++it) {
    for (int g = 0; g < W; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaDeviceSynchronize());
    }
    for (int g = 0; g < W; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaEventRecord(e0[g], st[g]));
      launch(g);
      CK(cudaEventRecord(e1[g], st[g]));
    }
    for (int g = 0; g < W; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaEventSynchronize(e1[g]));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
      if (it >= 0) {
        best[g] = std::min(best[g], (double)ms);
        sum[g] += ms;
      }
    }
  }
  double worst = 0, mean = 0;
  for (int g = 0; g < W; ++g) {
    worst = std::max(worst, sum[g] / iters);
    mean += sum[g] / iters / W;
  }
  const double per_gpu = (double)bytes * peers[0].size();
  printf("{\"mode\":\"%s\",\"pattern\":\"%s\",\"gpus\":%d,\"ctas\":%d,\"stages\":%d,\"stage_kb\":%d,\"mib_per_peer\":%d,"
         "\"peers\":%zu,\"gbs_per_gpu_worst\":%.1f,\"gbs_per_gpu_mean\":%.1f}\n",
         mode.c_str(), pat.c_str(), W, ctas, stages, skb, (int)(bytes >> 20), peers[0].size(),
         per_gpu / (worst * 1e-3) / 1e9, per_gpu / (mean * 1e-3) / 1e9);
  return 0;
}
