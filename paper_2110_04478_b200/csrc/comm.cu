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
#include <cuda.h>  // driver types for the stream memory ops (entry points fetched at run time, no -lcuda)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
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

themis_status_t cuda_fail(cudaError_t e, const char* what) {
  return fail(THEMIS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CUDA_TRY(call)                                 \
  do {                                                 \
    cudaError_t _e = (call);                           \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

#include "exec_kernel.cuh"

uint64_t signal_bytes(int P) { return round_up(pad_bytes(P), kAlign); }

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
  uint32_t* opcnt = nullptr;
  uint32_t* done_cnt = nullptr;
  uint32_t* abort_flag = nullptr;
  uint32_t* epoch_ctr = nullptr;  // device-resident collective epoch (graph-replay safe)
  uint32_t* herr_host = nullptr;
  uint32_t* herr_dev = nullptr;
  uint64_t* trace = nullptr;
  int trace_on = 0;  // 1: per-op start/end, 2: + detailed stamps
  bool pacing = false;  // emulate per-dim bandwidth by pacing (themis_comm_set_pacing)
  int stages = kStages;  // TMA ring depth (themis_comm_set_stages)
  int stage_bytes = kStageBytes;  // bytes per ring stage (themis_comm_set_stage_bytes)
  int ag_rr = 0;                  // direct-AG tile shape (env THEMIS_AG_RR, experiment)
  double min_cta_bytes = 0.0;  // op window sizing, 0 = full-width ops (themis_comm_set_min_cta_bytes)
  int window_rotate = 1;       // consecutive windows (1) or all from CTA 0 (0) (themis_comm_set_window_rotation)
  int lookahead = 1;           // runtime intra-dim order window (themis_comm_set_lookahead); 1 = static
  int push_ag = 0;             // direct AG ops as pushes (themis_comm_set_push, R30); applies at bind
  uint64_t ll_stride = 0;      // LL inbox bytes per local rank after the data regions (themis_comm_set_ll, R31)
  uint64_t ll_max_bytes = 0;   // plans of at most this many bytes run LL (0 = never)
  uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;
  int max_blocks = 0;  // co-resident CTAs for the kernel
  int engine = 1;      // 1: TMA bulk-copy pipeline, 0: LDG/STG
  // host-buffer streaming (themis_allreduce_host), created on first use
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  uint32_t* d2h_flags = nullptr;  // [THEMIS_MAX_CHUNKS] device
  uint32_t host_seq = 0;
  std::vector<themis_plan_t*> bound;  // plans bound to this comm (unbound when it is freed)
  char* mc_heap = nullptr;             // NVLS multicast mapping of the heap (themis_comm_set_multicast)
};

namespace themis {
struct BindState {
  themis_comm* comm = nullptr;
  OpDesc* d_ops = nullptr;
  int32_t* d_dim_ops = nullptr;
  int32_t grp_start[THEMIS_MAX_DIMS + 1] = {};
  int32_t ctas[THEMIS_MAX_DIMS] = {};
  int32_t total_ctas = 0;
  bool nvls = false;  // some op runs through the switch (TMA engine only)
  uint32_t dyn_mask = 0;  // dims whose ops may take the runtime order (no ring steps)
  int32_t nvls_pairs = 0;  // RS+AG pairs running in the switch
  bool ll = false;         // every op runs with LL packets (R31)
  uint64_t desc_hash = 0;  // of the uploaded op windows / algorithms (mixed into the launch's plan hash)
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
      (e = cudaMemset(c->opcnt, 0, sizeof(uint32_t) * (kMaxOps + 8))) != cudaSuccess ||
      (e = cudaMalloc(&c->trace, sizeof(uint64_t) * 8 * kMaxOps)) != cudaSuccess ||
      (e = cudaMemset(c->trace, 0, sizeof(uint64_t) * 8 * kMaxOps)) != cudaSuccess ||
      (e = cudaHostAlloc(&c->herr_host, sizeof(uint32_t), cudaHostAllocMapped)) != cudaSuccess ||
      (e = cudaHostGetDevicePointer(&c->herr_dev, c->herr_host, 0)) != cudaSuccess) {
    delete c;
    return cuda_fail(e, "themis_comm_create");
  }
  *c->herr_host = 0;
  c->done_cnt = c->opcnt + kMaxOps;
  c->abort_flag = c->opcnt + kMaxOps + 1;
  c->epoch_ctr = c->opcnt + kMaxOps + 2;
  int nb = 0;
  if ((e = prepare_kernels()) != cudaSuccess ||
      (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, themis_exec_kernel<dev::F32Tag, true>, kThreads,
                                                         kSmemBytes)) != cudaSuccess) {
    delete c;
    return cuda_fail(e, "kernel attributes / occupancy query");
  }
  if (const char* env = getenv("THEMIS_COPY_ENGINE")) c->engine = std::string(env) == "ldg" ? 0 : 1;
  if (const char* env = getenv("THEMIS_AG_RR")) c->ag_rr = atoi(env) != 0;
  if (const char* env = getenv("THEMIS_STAGE_KB"))
    c->stage_bytes = std::max(8, std::min(3 * kStageBytes / 1024, atoi(env))) * 1024;
  if (const char* env = getenv("THEMIS_STAGES"))
    c->stages = std::max(1, std::min(std::min(kStages, kStages * kStageBytes / c->stage_bytes), atoi(env)));
  if (const char* env = getenv("THEMIS_MIN_CTA_BYTES")) c->min_cta_bytes = std::max(0.0, atof(env));
  if (const char* env = getenv("THEMIS_WINDOW_ROTATE")) c->window_rotate = atoi(env) != 0;
  if (const char* env = getenv("THEMIS_PUSH")) c->push_ag = atoi(env) != 0;
  if (const char* env = getenv("THEMIS_LOOKAHEAD")) c->lookahead = std::max(1, std::min(kMaxLookahead, atoi(env)));
  c->max_blocks = nb * c->num_sms;
  *out = c;
  return THEMIS_OK;
}

static void free_bind(themis_plan_t* pl);

extern "C" void themis_comm_free(themis_comm_t* c) {
  if (!c) return;
  while (!c->bound.empty()) free_bind(c->bound.back());  // a plan may outlive its comm: unbind it
  if (c->h2d) {
    cudaStreamSynchronize(c->h2d);
    cudaStreamSynchronize(c->d2h);
    cudaStreamDestroy(c->h2d);
    cudaStreamDestroy(c->d2h);
    cudaEventDestroy(c->ev_in);
    cudaEventDestroy(c->ev_out);
    cudaFree(c->d2h_flags);
  }
  cudaFree(c->opcnt);
  cudaFree(c->trace);
  cudaFreeHost(c->herr_host);
  delete c;
}

extern "C" themis_status_t themis_comm_status(themis_comm_t* c) {
  if (!c) return fail(THEMIS_ERR_INVALID_ARG, "null comm");
  uint32_t v = *(volatile uint32_t*)c->herr_host;
  if ((v & 0xFF) == THEMIS_ERR_PLAN_MISMATCH)
    return fail(THEMIS_ERR_PLAN_MISMATCH, "rank " + std::to_string(v >> 8) +
                                              " launched a different plan / count / dtype / CTA caps (plan hash differs)");
  if (v) return fail((themis_status_t)(v & 0xFF), "device watchdog fired while waiting (code " + std::to_string(v >> 8) + ")");
  return THEMIS_OK;
}
extern "C" themis_status_t themis_comm_set_engine(themis_comm_t* c, int32_t engine) {
  if (!c || engine < 0 || engine > 1) return fail(THEMIS_ERR_INVALID_ARG, "engine must be 0 (LDG) or 1 (TMA)");
  c->engine = engine;
  return THEMIS_OK;
}
extern "C" themis_status_t themis_comm_set_multicast(themis_comm_t* c, void* mc_heap) {
  if (!c) return fail(THEMIS_ERR_INVALID_ARG, "null comm");
  c->mc_heap = static_cast<char*>(mc_heap);
  return THEMIS_OK;
}
extern "C" themis_status_t themis_comm_set_window_rotation(themis_comm_t* c, int32_t rotate) {
  if (!c || rotate < 0 || rotate > 1) return fail(THEMIS_ERR_INVALID_ARG, "rotate must be 0 or 1");
  c->window_rotate = rotate;
  return THEMIS_OK;
}
extern "C" themis_status_t themis_comm_set_ll(themis_comm_t* c, uint64_t inbox_bytes, uint64_t max_bytes) {
  if (!c) return fail(THEMIS_ERR_INVALID_ARG, "null comm");
  if (inbox_bytes % 16 ||
      (uint64_t)c->V * (c->sig_bytes + c->vrank_stride + inbox_bytes) > c->heap_bytes)
    return fail(THEMIS_ERR_INVALID_ARG, "LL inboxes (16-byte multiple, V per GPU after the data regions) do not fit the heap");
  c->ll_stride = inbox_bytes;
  c->ll_max_bytes = inbox_bytes ? max_bytes : 0;
  return THEMIS_OK;
}
extern "C" themis_status_t themis_comm_set_push(themis_comm_t* c, int32_t on) {
  if (!c || on < 0 || on > 1) return fail(THEMIS_ERR_INVALID_ARG, "push must be 0 or 1");
  c->push_ag = on;
  return THEMIS_OK;
}
extern "C" themis_status_t themis_comm_set_lookahead(themis_comm_t* c, int32_t lookahead) {
  if (!c || lookahead < 1 || lookahead > kMaxLookahead) return fail(THEMIS_ERR_INVALID_ARG, "lookahead must be 1..32");
  c->lookahead = lookahead;
  return THEMIS_OK;
}
extern "C" themis_status_t themis_comm_set_min_cta_bytes(themis_comm_t* c, uint64_t bytes) {
  if (!c) return fail(THEMIS_ERR_INVALID_ARG, "null comm");
  c->min_cta_bytes = (double)bytes;
  return THEMIS_OK;
}
extern "C" themis_status_t themis_comm_set_stages(themis_comm_t* c, int32_t stages) {
  if (!c || stages < 1 || stages > kStages || (int64_t)stages * c->stage_bytes > (int64_t)kStages * kStageBytes)
    return fail(THEMIS_ERR_INVALID_ARG, "stages must be 1..6 with stages * stage_bytes <= 192 KiB");
  c->stages = stages;
  return THEMIS_OK;
}
extern "C" themis_status_t themis_comm_set_stage_bytes(themis_comm_t* c, int32_t bytes) {
  if (!c || bytes < 8192 || bytes % 1024 || (int64_t)bytes * c->stages > (int64_t)kStages * kStageBytes)
    return fail(THEMIS_ERR_INVALID_ARG, "stage_bytes: multiple of 1 KiB, >= 8 KiB, stages * stage_bytes <= 192 KiB");
  c->stage_bytes = bytes;
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
  c->trace_on = on < 0 ? 0 : (on > 2 ? 2 : on);
  return THEMIS_OK;
}
extern "C" themis_status_t themis_trace_fetch(themis_comm_t* c, uint64_t* out, size_t n) {
  if (!c || !out || n > 2ull * kMaxOps) return fail(THEMIS_ERR_INVALID_ARG, "bad trace args");
  CUDA_TRY(cudaMemcpy(out, c->trace, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return THEMIS_OK;
}
extern "C" themis_status_t themis_trace_fetch_detail(themis_comm_t* c, uint64_t* out, size_t n) {
  if (!c || !out || n > 6ull * kMaxOps) return fail(THEMIS_ERR_INVALID_ARG, "bad trace args");
  CUDA_TRY(cudaMemcpy(out, c->trace + 2 * kMaxOps, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return THEMIS_OK;
}

static void free_bind(themis_plan_t* pl) {
  if (!pl->bind) return;
  auto& v = pl->bind->comm->bound;
  v.erase(std::remove(v.begin(), v.end(), pl), v.end());
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
  } else {  // proportional to bandwidth over every co-resident CTA (a9)
    themis_status_t st = themis_default_ctas(&pl->topo, std::max(D, c->max_blocks), n);
    if (st != THEMIS_OK) return st;
    for (int k = 0; k < D; ++k) tot += n[k];
  }
  if (tot > c->max_blocks)
    return fail(THEMIS_ERR_INVALID_ARG, "sum of ctas_per_dim (" + std::to_string(tot) + ") exceeds co-resident CTAs (" +
                                            std::to_string(c->max_blocks) + ")");
  // descriptors
  std::vector<OpDesc> ops(pl->ops.size());
  for (size_t i = 0; i < pl->ops.size(); ++i) {
    const Op& o = pl->ops[i];
    OpDesc d{};
    d.pace_scale = 1.0f;
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
    // Table 1: ring dims run the ring algorithm (P_k = 2 ring == direct)
    d.ring = pl->topo.kind[o.dim] == THEMIS_DIM_RING && pl->topo.size[o.dim] >= 3;
    ops[i] = d;
  }
  // NVLS (R27, R29): on an NVLS dim whose group is one rank per GPU at the
  // same local index (P_k == W, stride_k == V) and a comm with a multicast
  // mapping, an RS op immediately followed by the chunk's AG op on the same dim
  // (the pair the planner modelled as one in-switch All-Reduce) runs as one
  // in-switch All-Reduce of the own piece (multimem.ld_reduce + multimem.st);
  // the AG op then only carries the dependency.  Ineligible: direct RS + AG.
  bool any_nvls = false;
  int n_fused = 0;
  if (c->mc_heap) {
    int64_t stride = 1;
    bool elig[THEMIS_MAX_DIMS] = {};
    for (int k = 0; k < D; ++k) {
      elig[k] = pl->topo.kind[k] == THEMIS_DIM_NVLS && pl->topo.size[k] == c->W && stride == c->V && c->W > 1;
      stride *= pl->topo.size[k];
    }
    for (int ch = 0; ch < pl->C; ++ch)
      for (int st = 0; st + 1 < pl->NS; ++st) {
        const size_t i = (size_t)ch * pl->NS + st;
        const Op& a = pl->ops[i];
        const Op& b = pl->ops[i + 1];
        if (elig[a.dim] && a.phase == 0 && b.phase == 1 && b.dim == a.dim) {
          ops[i].nvls = 1;
          ops[i + 1].nvls = 2;
          any_nvls = true;
          ++n_fused;
        }
      }
  }
  // R30: direct (non-ring, non-NVLS) AG ops as pushes; the op after a push
  // waits for the push's k x k' plane
  for (size_t i = 0; i < ops.size(); ++i) {
    ops[i].prev_dim = ops[i].stage > 0 ? ops[i - 1].dim : -1;
    ops[i].push = c->push_ag && ops[i].phase == 1 && !ops[i].ring && !ops[i].nvls;
  }
  for (size_t i = 0; i < ops.size(); ++i) ops[i].prev_push = ops[i].stage > 0 && ops[i - 1].push;
  // R31: a small collective (bytes <= ll_max_bytes, no ring dims, no NVLS
  // pair) runs every op with LL packets; each op gets a region of every
  // rank's inbox: (P_k - 1) sources x the rank's part (nblk slices) x 2
  // (8-byte packets carry 4 payload bytes)
  bool ll = c->ll_max_bytes && pl->req.bytes <= c->ll_max_bytes && !any_nvls;
  for (const OpDesc& d : ops) ll = ll && !d.ring;
  if (ll) {
    const uint64_t slice = pl->req.bytes / ((uint64_t)pl->P * pl->C);
    uint64_t off = 0;
    for (OpDesc& d : ops) {
      d.ll = 1;
      d.push = 0;
      d.prev_push = 0;
      d.ll_off = off;
      off += (uint64_t)(pl->topo.size[d.dim] - 1) * (uint64_t)d.nblk * slice * 2;
    }
    if (off > c->ll_stride) ll = false;
    if (!ll)
      for (OpDesc& d : ops) d.ll = 0, d.ll_off = 0, d.push = c->push_ag && d.phase == 1 && !d.ring && !d.nvls;
    if (!ll)
      for (size_t i = 0; i < ops.size(); ++i) ops[i].prev_push = ops[i].stage > 0 && ops[i - 1].push;
  }
  std::vector<int32_t> lists((size_t)D * pl->C * pl->NS, 0);
  for (int k = 0; k < D; ++k)
    for (size_t i = 0; i < pl->dim_ops[k].size(); ++i) {
      uint32_t e = pl->dim_ops[k][i];
      const int opi = (int)((e >> 8) * pl->NS + (e & 0xFF));
      lists[(size_t)k * pl->C * pl->NS + i] = opi;
      ops[opi].seq = (int32_t)i;
    }
  for (int k = 0; k < D; ++k)
    if (n[k] > kMaxCtas) return fail(THEMIS_ERR_INVALID_ARG, "at most 160 CTAs per dimension group");
  // Op windows: an op that moves little gets only as many
  // CTAs as it can keep busy (>= min_cta_bytes each), and consecutive ops of a
  // dimension take consecutive CTA windows, so several small chunks' ops of a
  // dimension run concurrently.  Identical on every GPU (same plan, V, caps).
  const int SV = std::max(1, pl->req.concurrency);
  if (SV > 1) {
    // concurrency-aware plan: server s of dim k owns CTA slice [s*c_k/SV, (s+1)*c_k/SV)
    // and runs exactly the ops the pre-simulation gave it, in order
    for (int k = 0; k < D; ++k)
      if (n[k] < SV) return fail(THEMIS_ERR_INVALID_ARG, "concurrency exceeds the CTAs of a dimension group");
    for (size_t i = 0; i < ops.size(); ++i) {
      const int k = ops[i].dim, sv = pl->server[i];
      const int o0 = sv * n[k] / SV, o1 = (sv + 1) * n[k] / SV;
      ops[i].offset = o0;
      ops[i].width = o1 - o0;
    }
  } else {
    const double slice = (double)pl->req.bytes / ((double)pl->P * pl->C);
    const double min_b = c->min_cta_bytes;
    for (int k = 0; k < D; ++k) {
      int off = 0;
      for (size_t i = 0; i < pl->dim_ops[k].size(); ++i) {
        const uint32_t e = pl->dim_ops[k][i];
        OpDesc& d = ops[(e >> 8) * pl->NS + (e & 0xFF)];
        const double mult = (d.phase == 1 && !d.ring) ? (double)(pl->topo.size[k] - 1) : 1.0;
        const double work = (double)c->V * (double)d.nblk * slice * mult;
        int w = min_b > 0 ? (int)std::ceil(work / min_b) : n[k];
        w = std::max(1, std::min(n[k], w));
        d.width = w;
        d.offset = off;
        // a lone narrow op (no rotation: ops one at a time) carries the whole
        // dim rate on its w CTAs; rotating windows share it per CTA
        d.pace_scale = c->window_rotate ? 1.0f : (float)w / (float)n[k];
        off = c->window_rotate ? (off + w) % n[k] : 0;
      }
    }
  }
  // Everything a peer's CTAs assume about ours: ring step flags are indexed by
  // absolute CTA, so op windows (min_cta_bytes / window_rotate, settable per
  // process) and the NVLS rewrite (needs every GPU's multicast mapping) must
  // be identical on every rank -- hashed here, checked at kernel entry (R22).
  uint64_t dh = 1469598103934665603ull;
  auto mix = [&dh](int64_t v) { dh = (dh ^ (uint64_t)v) * 1099511628211ull; };
  for (const OpDesc& d : ops) {
    mix(d.width);
    mix(d.offset);
    mix(d.ring);
    mix(d.nvls);
    mix(d.seq);
    mix(d.push);
    mix(d.ll);
    mix((int64_t)d.ll_off);
    uint32_t ps;
    std::memcpy(&ps, &d.pace_scale, 4);
    mix(ps);
  }
  free_bind(pl);
  auto* b = new BindState();
  b->comm = c;
  b->desc_hash = dh;
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
  b->nvls = any_nvls;
  b->nvls_pairs = n_fused;
  b->dyn_mask = (1u << D) - 1;
  for (const OpDesc& d : ops)
    if (d.ring || d.ll) b->dyn_mask &= ~(1u << d.dim);  // ring steps / LL packets: the same op order on every rank
  b->ll = !ops.empty() && ops[0].ll;
  pl->bind = b;
  c->bound.push_back(pl);
  return THEMIS_OK;
}

// The plan hash covers the inputs, schedule and per-dim order; mix in the
// bound CTA caps, the op descriptors' windows and the byte count so every rank
// must launch identically (checked at kernel entry, R22).
static uint64_t launch_hash(const themis_plan_t* pl, uint64_t count, int32_t dtype) {
  uint64_t h = pl->hash ^ (count * 0x9E3779B97F4A7C15ull) ^ ((uint64_t)dtype << 56);
  for (int k = 0; k < pl->D; ++k) h = (h ^ (uint64_t)pl->bind->ctas[k]) * 1099511628211ull;
  return (h ^ pl->bind->desc_hash) * 1099511628211ull;  // op windows + NVLS rewrite (bind)
}

// Single-GPU profiling / fault injection: make GPU peer_gpu's logical ranks
// look as if they had entered, finished every op (and ring step) and exited
// for every epoch, with this plan's launch hash -- written into the signal pads
// of this GPU's local ranks.  The kernel on this GPU then never waits, while
// still pulling the peer's data over NVLink (ncu can replay it: no other GPU
// takes part).  Data results are meaningless.
extern "C" themis_status_t themis_debug_fake_peer_gpu(const themis_plan_t* pl, int32_t peer_gpu, uint64_t count,
                                                      int32_t dtype) {
  if (!pl || !pl->bind) return fail(THEMIS_ERR_PLAN_MISMATCH, "plan not bound");
  themis_comm* c = pl->bind->comm;
  if (peer_gpu < 0 || peer_gpu >= c->W || peer_gpu == c->gpu_rank) return fail(THEMIS_ERR_INVALID_ARG, "bad peer gpu");
  const int P = c->P, V = c->V;
  const uint64_t h = launch_hash(pl, count, dtype);
  std::vector<uint32_t> ones(kMaxOps, 0xFFFFFFFFu);
  std::vector<unsigned long long> ring(THEMIS_MAX_DIMS * kMaxCtas, ~0ull);
  for (int v = 0; v < V; ++v) {
    char* pad = c->heap[c->gpu_rank] + (uint64_t)v * c->sig_bytes;
    for (int src = peer_gpu * V; src < (peer_gpu + 1) * V; ++src) {
      const uint32_t m = 0xFFFFFFFFu;
      CUDA_TRY(cudaMemcpy(pad + 4ull * src, &m, 4, cudaMemcpyHostToDevice));                // entry
      CUDA_TRY(cudaMemcpy(pad + 4ull * (P + src), &m, 4, cudaMemcpyHostToDevice));          // exit
      CUDA_TRY(cudaMemcpy(pad + 4ull * (2ull * P + (uint64_t)src * kMaxOps), ones.data(), 4ull * kMaxOps,
                          cudaMemcpyHostToDevice));                                         // ready
      CUDA_TRY(cudaMemcpy(pad + ring_flags_offset(P) + 8ull * src * THEMIS_MAX_DIMS * kMaxCtas, ring.data(),
                          8ull * ring.size(), cudaMemcpyHostToDevice));                    // ring steps
      CUDA_TRY(cudaMemcpy(pad + hash_offset(P) + 8ull * src, &h, 8, cudaMemcpyHostToDevice));  // plan hash
    }
  }
  return THEMIS_OK;
}

extern "C" themis_status_t themis_plan_bound_ll(const themis_plan_t* pl, int32_t* ll) {
  if (!pl || !pl->bind || !ll) return fail(THEMIS_ERR_PLAN_MISMATCH, "plan not bound");
  *ll = pl->bind->ll;
  return THEMIS_OK;
}

extern "C" themis_status_t themis_plan_bound_nvls(const themis_plan_t* pl, int32_t* n_pairs) {
  if (!pl || !pl->bind || !n_pairs) return fail(THEMIS_ERR_PLAN_MISMATCH, "plan not bound");
  *n_pairs = pl->bind->nvls_pairs;
  return THEMIS_OK;
}

extern "C" themis_status_t themis_plan_bound_ctas(const themis_plan_t* pl, int32_t* ctas) {
  if (!pl || !pl->bind || !ctas) return fail(THEMIS_ERR_PLAN_MISMATCH, "plan not bound");
  for (int k = 0; k < pl->D; ++k) ctas[k] = pl->bind->ctas[k];
  return THEMIS_OK;
}

static themis_status_t check_call(int coll, void* buf, uint64_t count, int32_t dtype, const themis_plan_t* pl,
                                  int* esz_out) {
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
  *esz_out = esz;
  return THEMIS_OK;
}


extern "C" themis_status_t themis_plan_launch_hash(const themis_plan_t* pl, uint64_t count, int32_t dtype,
                                                   uint64_t* out) {
  if (!pl || !pl->bind || !out) return fail(THEMIS_ERR_PLAN_MISMATCH, "plan not bound / null output");
  *out = launch_hash(pl, count, dtype);
  return THEMIS_OK;
}

static themis_status_t launch(int coll, void* buf, uint64_t count, int32_t dtype, const themis_plan_t* pl,
                              void* stream, uint32_t host_seq = 0) {
  int esz = 0;
  themis_status_t st = check_call(coll, buf, count, dtype, pl, &esz);
  if (st != THEMIS_OK) return st;
  themis_comm* c = pl->bind->comm;
  char* mine = c->heap[c->gpu_rank];
  char* p = static_cast<char*>(buf);
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
  kp.epoch_ctr = c->epoch_ctr;
  kp.opcnt = c->opcnt;
  kp.done_cnt = c->done_cnt;
  kp.abort_flag = c->abort_flag;
  kp.herr = c->herr_dev;
  kp.timeout_ns = c->timeout_ns;
  kp.trace = c->trace_on ? c->trace : nullptr;
  kp.tdetail = c->trace_on >= 2 ? c->trace + 2 * kMaxOps : nullptr;
  kp.plan_hash = launch_hash(pl, count, dtype);
  kp.lookahead = c->lookahead;
  kp.push_ok = c->engine && !host_seq;
  kp.ll_rel = (uint64_t)c->V * (c->sig_bytes + c->vrank_stride);
  kp.ll_stride = c->ll_stride;  // host streaming publishes per-chunk d2h flags from the last stage: pull
  kp.dyn_mask = pl->bind->dyn_mask;
  kp.stages = c->stages;
  kp.stage_bytes = c->stage_bytes;
  kp.ag_rr = c->ag_rr;
  kp.host_seq = host_seq;
  kp.d2h_flags = c->d2h_flags;
  kp.mc_heap = c->mc_heap;
  for (int k = 0; k < pl->D; ++k)  // ns per byte per CTA = c_k / (V * bw_k[bytes/ns])
    kp.pace_ns_per_byte[k] =
        c->pacing ? (float)((double)pl->bind->ctas[k] * 1000.0 / ((double)c->V * pl->topo.bw_mbps[k])) : 0.f;

  void* args[] = {&kp};
  if (!c->engine)
    for (int k = 0; k < pl->D; ++k)
      if (pl->topo.kind[k] == THEMIS_DIM_RING && pl->topo.size[k] >= 3)
        return fail(THEMIS_ERR_INVALID_ARG, "ring dimensions need the TMA engine (themis_comm_set_engine(comm, 1))");
  if (!c->engine && pl->bind->nvls)
    return fail(THEMIS_ERR_INVALID_ARG, "NVLS ops need the TMA engine (themis_comm_set_engine(comm, 1))");
  if ((!c->engine || host_seq) && pl->bind->ll)
    return fail(THEMIS_ERR_INVALID_ARG, "LL plans need the TMA engine and device buffers (rebind with themis_comm_set_ll(comm, 0, 0))");
  const void* fn = kernel_for(dtype, c->engine);
  if (c->trace_on) {  // op start = earliest working CTA (atomicMin over an all-ones start)
    cudaError_t m = cudaMemsetAsync(c->trace, 0xFF, 2 * kMaxOps * sizeof(uint64_t), static_cast<cudaStream_t>(stream));
    if (m != cudaSuccess) return cuda_fail(m, "cudaMemsetAsync(trace)");
  }
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

// Stream memory ops (write / wait on a 32-bit device word) from the driver,
// fetched through the runtime so the library needs no -lcuda at link time.
typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static WriteValue32Fn g_write32 = nullptr;
static WaitValue32Fn g_wait32 = nullptr;

static themis_status_t host_stream_setup(themis_comm* c) {
  if (c->h2d) return THEMIS_OK;
  if (!g_write32 || !g_wait32) {
    cudaDriverEntryPointQueryResult q1, q2;
    void *w = nullptr, *t = nullptr;
    CUDA_TRY(cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1));
    CUDA_TRY(cudaGetDriverEntryPoint("cuStreamWaitValue32", &t, cudaEnableDefault, &q2));
    if (q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !w || !t)
      return fail(THEMIS_ERR_CUDA, "driver stream memory ops unavailable");
    g_write32 = reinterpret_cast<WriteValue32Fn>(w);
    g_wait32 = reinterpret_cast<WaitValue32Fn>(t);
  }
  CUDA_TRY(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
  CUDA_TRY(cudaMalloc(&c->d2h_flags, sizeof(uint32_t) * THEMIS_MAX_CHUNKS));
  CUDA_TRY(cudaMemset(c->d2h_flags, 0, sizeof(uint32_t) * THEMIS_MAX_CHUNKS));
  CUDA_TRY(cudaDeviceSynchronize());
  return THEMIS_OK;
}

// Host buffers in and out, streamed chunk by chunk so PCIe overlaps the
// collective: an H2D stream copies chunk c of every local rank (one 2-D copy
// per rank: P slices of slice bytes, block pitch) and then writes the chunk's
// h2d flag (= this call's sequence number) into local rank 0's signal pad; the
// kernel's stage-0 op of chunk c waits for the flags of every source GPU; the
// last stage of chunk c publishes a d2h flag that a D2H stream waits on
// before copying the chunk back.  Chunks are fed in the order of their
// pre-simulated stage-0 start and drained in the order of their final-stage
// end.  The user stream waits for the D2H stream at the end, so stream order
// semantics are those of a single call.
extern "C" themis_status_t themis_allreduce_host(const void* host_in, void* host_out, void* buf, uint64_t count,
                                                 int32_t dtype, const themis_plan_t* pl, void* stream) {
  if (!pl || !pl->bind) return fail(THEMIS_ERR_PLAN_MISMATCH, "plan is not bound to a comm");
  if (!host_in || !host_out) return fail(THEMIS_ERR_INVALID_ARG, "null host buffer");
  if (pl->req.coll != THEMIS_ALLREDUCE) return fail(THEMIS_ERR_PLAN_MISMATCH, "plan was made for another collective");
  int esz = 0;
  themis_status_t st = check_call(THEMIS_ALLREDUCE, buf, count, dtype, pl, &esz);  // before any copy lands
  if (st != THEMIS_OK) return st;
  themis_comm* c = pl->bind->comm;
  if ((st = host_stream_setup(c)) != THEMIS_OK) return st;
  const uint64_t bytes = pl->req.bytes;
  const int P = c->P, C = pl->C, NS = pl->NS;
  const uint64_t blk = bytes / P, slice = blk / C;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t seq = ++c->host_seq;
  // the copy streams start after the user stream's prior work (incl. the
  // previous collective on this comm, hence every peer's reads of our buffer)
  CUDA_TRY(cudaEventRecord(c->ev_in, s));
  CUDA_TRY(cudaStreamWaitEvent(c->h2d, c->ev_in, 0));
  CUDA_TRY(cudaStreamWaitEvent(c->d2h, c->ev_in, 0));
  std::vector<int> in_order(C), out_order(C);
  for (int i = 0; i < C; ++i) in_order[i] = out_order[i] = i;
  std::stable_sort(in_order.begin(), in_order.end(),
                   [&](int a, int b) { return pl->start[(size_t)a * NS] < pl->start[(size_t)b * NS]; });
  std::stable_sort(out_order.begin(), out_order.end(), [&](int a, int b) {
    return pl->end[(size_t)a * NS + NS - 1] < pl->end[(size_t)b * NS + NS - 1];
  });
  char* pad0 = c->heap[c->gpu_rank];  // local rank 0's signal pad
  for (int ch : in_order) {
    for (int v = 0; v < c->V; ++v)
      CUDA_TRY(cudaMemcpy2DAsync(static_cast<char*>(buf) + v * c->vrank_stride + ch * slice, blk,
                                 static_cast<const char*>(host_in) + v * bytes + ch * slice, blk, slice, P,
                                 cudaMemcpyHostToDevice, c->h2d));
    const CUdeviceptr flag = reinterpret_cast<CUdeviceptr>(pad0 + h2d_offset(P) + 4ull * ch);
    if (g_write32(reinterpret_cast<CUstream>(c->h2d), flag, seq, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
      return fail(THEMIS_ERR_CUDA, "cuStreamWriteValue32 (h2d flag)");
  }
  st = launch(THEMIS_ALLREDUCE, buf, count, dtype, pl, stream, seq);
  if (st != THEMIS_OK) return st;
  for (int ch : out_order) {
    const CUdeviceptr flag = reinterpret_cast<CUdeviceptr>(c->d2h_flags + ch);
    if (g_wait32(reinterpret_cast<CUstream>(c->d2h), flag, seq, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return fail(THEMIS_ERR_CUDA, "cuStreamWaitValue32 (d2h flag)");
    for (int v = 0; v < c->V; ++v)
      CUDA_TRY(cudaMemcpy2DAsync(static_cast<char*>(host_out) + v * bytes + ch * slice, blk,
                                 static_cast<char*>(buf) + v * c->vrank_stride + ch * slice, blk, slice, P,
                                 cudaMemcpyDeviceToHost, c->d2h));
  }
  CUDA_TRY(cudaEventRecord(c->ev_out, c->d2h));
  CUDA_TRY(cudaStreamWaitEvent(s, c->ev_out, 0));
  return THEMIS_OK;
}

extern "C" int32_t themis_launches_per_call(void) { return 1; }
