/*
 * themis.h — C ABI of libthemis: the B200-native hot path of Themis
 * (arXiv 2110.04478): a chunked hierarchical All-Reduce (and its
 * Reduce-Scatter / All-Gather halves) over a logical P_1 x ... x P_D topology,
 * each chunk traversing the dimensions in the order Themis's greedy policy
 * (Algorithm 1) picks, executed by hand-written sm_100a kernels that pull peer
 * data over NVLink / NVSwitch.
 *
 * Citations are to /root/reference/PAPER.md lines; "R<n>" are the readings
 * listed in DESIGN.md where the paper is silent or ambiguous.
 *
 * Conventions (all entry points):
 *   - Every call returns themis_status_t; THEMIS_OK == 0.  No C++ exception
 *     crosses the ABI.  themis_last_error() returns a thread-local message for
 *     the last failing call on the calling thread.
 *   - Pointers marked [host] are host memory, [device] are device memory (or
 *     UVA pointers to a peer GPU's memory), [out] are written by the call.
 *   - Collectives are enqueue-only and asynchronous on the given CUDA stream.
 *     Device-side failures (watchdog timeout) are latched in the comm and
 *     reported by the next collective call or themis_comm_status().
 *   - Objects are owned by the caller: every *_create / plan has a matching
 *     *_free.  The library never frees memory it did not allocate.
 *
 * Units: bandwidth in MB/s (10^6 bytes/s, integer), latency in ns, sizes in
 * bytes.  Planner arithmetic is exact (integers, 128-bit intermediates); time
 * is reported in integer units of 1/time_scale ns and per-dimension volumes in
 * units of 1/byte_scale bytes (themis_plan_info_t), so schedules and
 * predicted times are bit-exact against the oracle's rational arithmetic.
 */
#ifndef THEMIS_H_
#define THEMIS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define THEMIS_MAX_DIMS 8      /* D <= 8 (the paper uses D <= 4, Table 2) */
#define THEMIS_MAX_CHUNKS 1024 /* CPC <= 1024 (paper: 4..512) */
#define THEMIS_AUTO_MAX_CHUNKS 256 /* largest candidate of n_chunks = 0 (auto) */
#define THEMIS_MAX_GPUS 8      /* GPUs of one NVSwitch box */
#define THEMIS_IPC_HANDLE_BYTES 64

typedef enum {
  THEMIS_OK = 0,
  THEMIS_ERR_INVALID_ARG = 1,     /* malformed topology / request / argument */
  THEMIS_ERR_ALIGNMENT = 2,       /* count not a multiple of P*C*vec, or misaligned buf */
  THEMIS_ERR_UNSUPPORTED_DTYPE = 3,
  THEMIS_ERR_OVERFLOW = 4,        /* exact planner arithmetic would overflow */
  THEMIS_ERR_NOT_REGISTERED = 5,  /* buf outside the comm's registered heap */
  THEMIS_ERR_PLAN_MISMATCH = 6,   /* plan not bound / bound to another comm / wrong coll */
  THEMIS_ERR_CUDA = 7,            /* a CUDA runtime call failed (message has details) */
  THEMIS_ERR_TIMEOUT = 8          /* device watchdog fired (peer never signalled) */
} themis_status_t;

typedef enum { THEMIS_F32 = 0, THEMIS_BF16 = 1, THEMIS_F16 = 2, THEMIS_I32 = 3 } themis_dtype_t;
typedef enum { THEMIS_ALLREDUCE = 0, THEMIS_REDUCE_SCATTER = 1, THEMIS_ALL_GATHER = 2 } themis_coll_t;
/* Table 3: Baseline = fixed dim1->dimD order;
 * Themis = Algorithm 1. */
typedef enum { THEMIS_POLICY_BASELINE = 0, THEMIS_POLICY_THEMIS = 1 } themis_policy_t;
/* Intra-dimension order: SCF keyed on the op's transfer volume
 * (R9), FIFO (R10), or SCF keyed on bytes-before (SPEC.md:330 literal). */
typedef enum { THEMIS_INTRA_SCF = 0, THEMIS_INTRA_FIFO = 1, THEMIS_INTRA_SCF_LITERAL = 2 } themis_intra_t;
/* Table 1: per-dimension topology -> basic algorithm.
 * THEMIS_DIM_NVLS (extension, PAPER.md:493-494 in-network offload; DESIGN R29):
 * a Switch dim whose switch reduces.  The latency model runs an All-Reduce
 * chunk's last RS stage + first AG stage on it (the same dim, Algorithm 1 line
 * 8) as ONE op of n = (1 + 1/P_k) x bytes-held (each member's copy into the
 * switch + the multicast of the reduced piece) and 2 steps of latency; the AG
 * half becomes a zero-volume op.  Bound to a comm with a multicast heap whose
 * dim group is one rank per GPU (P_k == W, stride_k == V), the executor runs
 * the pair in the switch (multimem.ld_reduce + multimem.st); otherwise as
 * direct RS + AG (same result, themis_plan_bound_nvls reports 0). */
typedef enum { THEMIS_DIM_RING = 0, THEMIS_DIM_DIRECT = 1, THEMIS_DIM_SWITCH = 2, THEMIS_DIM_NVLS = 3 } themis_dim_kind_t;

/* Logical topology P_1 x ... x P_D.  Rank r has coordinates
 * c_k = floor(r / prod_{i<k} P_i) mod P_k (dim1 fastest, R15).
 * bw[k]: aggregate uni-directional per-NPU bandwidth of dim k in MB/s
 * (PAPER.md:505, :136); with zero latencies only the ratios matter.
 * Validation: 1 <= ndims <= 8, size >= 2, bw > 0,
 * SWITCH / NVLS => size is a power of two. */
typedef struct {
  int32_t ndims;
  int32_t size[THEMIS_MAX_DIMS];
  uint32_t bw_mbps[THEMIS_MAX_DIMS];
  uint32_t step_latency_ns[THEMIS_MAX_DIMS];
  int32_t kind[THEMIS_MAX_DIMS]; /* themis_dim_kind_t */
} themis_topology_t;

/* One collective to plan (Algorithm 1 inputs CT, CS, CPC). */
typedef struct {
  int32_t coll;            /* themis_coll_t (CT) */
  int32_t policy;          /* themis_policy_t */
  int32_t intra;           /* themis_intra_t */
  int32_t n_chunks;        /* CPC, 1..THEMIS_MAX_CHUNKS (paper default 64);
                              0 (themis_plan only) = auto: the power of two C <=
                              THEMIS_AUTO_MAX_CHUNKS with bytes % (P*C*16) == 0 whose
                              pre-simulated makespan is smallest (ties: smaller C);
                              ALIGNMENT if bytes % (P*16) != 0.  Meaningful with
                              step_latency_ns + charge_latency (measured A_K); the
                              choice is themis_plan_info().n_chunks. */
  uint64_t bytes;          /* CS: bytes of the full buffer on each rank (> 0) */
  int32_t threshold_div;   /* Threshold = time of an RS/AG of chunk/threshold_div on
                              the min-load dim (paper uses 16) */
  int32_t charge_latency;  /* 0 (default, F5): the pre-simulation charges A_K only via
                              the tracker seed; 1: also per op */
  int32_t concurrency;     /* ops in flight per dimension, 0/1 = one (the paper's model);
                              k > 1: the pre-simulation runs k parallel servers of BW_K/k per
                              dim and assigns each op a server; bound plans
                              run server s's ops on the s-th slice of the dim's CTAs */
  int32_t reserved;        /* must be 0 */
  uint64_t chunk_release_ns; /* 0 (the paper's model): every chunk is ready at t = 0.
                              r > 0: chunk c's first stage becomes ready at (c+1)*r ns in
                              the pre-simulation — chunks streamed in from the host at
                              one per r ns (themis_allreduce_host), so the enforced
                              per-dim order drains early chunks while later ones arrive */
} themis_plan_req_t;

/* Summary of a plan.  Times in units of 1/time_scale ns, volumes in units of
 * 1/byte_scale bytes (exact; see the header comment). */
typedef struct {
  int32_t ndims, n_chunks, n_ranks;
  int32_t n_stages;        /* stages per chunk: 2D for AR, D for RS / AG */
  int32_t n_greedy;        /* chunks whose order came from the sort (not the threshold fallback) */
  int32_t coll, policy, intra;
  uint64_t time_scale;     /* integer time units per ns */
  uint64_t byte_scale;     /* integer volume units per byte (= P * C) */
  uint64_t makespan;       /* predicted makespan of the pre-simulation */
  uint64_t busy[THEMIS_MAX_DIMS];       /* N_K*B_K (+A_K if charged) */
  uint64_t idle[THEMIS_MAX_DIMS];       /* idle_K: idle before dim K's last op ends */
  uint64_t dim_volume[THEMIS_MAX_DIMS]; /* N_K = sum_i n_K^i, x byte_scale */
  uint64_t final_load[THEMIS_MAX_DIMS]; /* Dim Load Tracker after the last chunk */
  uint64_t hash;           /* FNV-1a of inputs + schedule + per-dim order; equal on all ranks */
  /* The paper's average BW utilisation of the pre-simulated run (PAPER.md:292,
   * R14): sum_K BW_K busy_K / (sum_K BW_K * makespan) = util_num / util_den,
   * reduced by their gcd.  util_exact = 1 when the reduced fraction fits in 64
   * bits (always for the BASELINE configs); 0 = both were shifted right until
   * they fit (relative error < 2^-60). */
  uint64_t util_num, util_den;
  int32_t util_exact;
  int32_t reserved_info;
} themis_plan_info_t;

typedef struct themis_plan themis_plan_t;
typedef struct themis_comm themis_comm_t;

/* ---------------------------------------------------------------- planner
 * themis_plan: host-only, pure, thread-safe.  Runs the Splitter, the Dim Load
 * Tracker seeded with A_K, Algorithm 1 with the Threshold
 * or the baseline order, then the deterministic
 * pre-simulation that fixes every dimension's op order.
 * Errors: INVALID_ARG (validation), OVERFLOW.  *out is owned by the caller
 * (themis_plan_free). */
themis_status_t themis_plan(const themis_topology_t* topo /*[host]*/, const themis_plan_req_t* req /*[host]*/,
                            themis_plan_t** out /*[out]*/);
/* themis_plan_custom: a plan whose per-chunk dim orders are given by the
 * caller instead of Algorithm 1 — any RS order x any AG order per chunk
 * (Observations 1-2; e.g. a brute-force optimum, or a
 * projection of a larger topology's schedule).  rs_order / ag_order: [host]
 * C*D 0-based dims, row-major (rs_order may be NULL for AG, ag_order NULL
 * for RS).  The intra-dimension order is pre-simulated as in themis_plan;
 * req->policy is ignored.  Errors: INVALID_ARG (not a permutation, missing
 * order), OVERFLOW. */
themis_status_t themis_plan_custom(const themis_topology_t* topo /*[host]*/, const themis_plan_req_t* req /*[host]*/,
                                   const uint8_t* rs_order, const uint8_t* ag_order, themis_plan_t** out /*[out]*/);
themis_status_t themis_plan_info(const themis_plan_t* plan, themis_plan_info_t* info /*[host, out]*/);
/* Per-chunk dim orders, 0-based dims, row-major [C][D]; ag_order for AR is
 * reverse(rs_order) (Algorithm 1 line 8).  RS plans leave ag_order rows 0xFF,
 * AG plans leave rs_order rows 0xFF.  Either pointer may be NULL. */
themis_status_t themis_plan_orders(const themis_plan_t* plan, uint8_t* rs_order /*[host,out] C*D*/,
                                   uint8_t* ag_order /*[host,out] C*D*/);
/* Per-dimension enforced op order: dim_ops[k*(C*n_stages) + i] = (chunk << 8) | stage,
 * n_dim_ops[k] entries valid per dim (row stride C*n_stages).  Every rank
 * executes exactly this order on each dimension. */
themis_status_t themis_plan_dim_ops(const themis_plan_t* plan, uint32_t* dim_ops /*[host,out] D*C*n_stages*/,
                                    int32_t* n_dim_ops /*[host,out] D*/);
/* Server (0..concurrency-1) of every op, [C][n_stages] (all 0 for concurrency <= 1). */
themis_status_t themis_plan_servers(const themis_plan_t* plan, int32_t* server /*[host,out] C*n_stages*/);
/* Pre-simulated start / end time of every op, [C][n_stages], time units. */
themis_status_t themis_plan_times(const themis_plan_t* plan, uint64_t* start /*[host,out]*/,
                                  uint64_t* end /*[host,out]*/);
void themis_plan_free(themis_plan_t* plan);

/* ---------------------------------------------------------------- memory
 * A comm spans W GPUs (one process each) hosting P = prod P_k logical ranks,
 * V = P / W consecutive ranks per GPU (V > 1 emulates several ranks on one
 * GPU: W = 1 runs the whole topology inside one GPU's HBM).  Each GPU owns
 * one "heap": [V signal pads of themis_signal_bytes(P) each][V data regions
 * of vrank_stride bytes].  Peers' heaps are mapped with CUDA IPC.
 * themis_heap_layout: signal bytes per pad and total heap bytes for
 * V ranks with data_bytes per rank (data_bytes rounded up to 4 KiB). */
themis_status_t themis_heap_layout(int32_t n_ranks, int32_t n_gpus, uint64_t data_bytes,
                                   uint64_t* signal_bytes /*[out]*/, uint64_t* vrank_stride /*[out]*/,
                                   uint64_t* heap_bytes /*[out]*/);
/* cudaMalloc on the current device, signal pads zeroed.  Caller frees. */
themis_status_t themis_heap_alloc(uint64_t heap_bytes, void** heap /*[out, device]*/);
themis_status_t themis_heap_free(void* heap /*[device]*/);
/* CUDA IPC handle of a heap (64 bytes) to send to the other processes. */
themis_status_t themis_heap_export(void* heap /*[device]*/, uint8_t* handle /*[host,out] 64 B*/);
/* Map a peer's heap into this process; returns its UVA base pointer. */
themis_status_t themis_heap_import(const uint8_t* handle /*[host] 64 B*/, void** peer_heap /*[out]*/);
themis_status_t themis_heap_close(void* peer_heap /*[device]*/);

/* ---------------------------------------------------------------- comm
 * gpu_rank / n_gpus: this process's index among the W GPUs.  heaps[g]: UVA
 * base of GPU g's heap as mapped in this process (own heap at heaps[gpu_rank]).
 * Allocates small device-local state (op counters, error word, trace).
 * Errors: INVALID_ARG, CUDA. */
themis_status_t themis_comm_create(int32_t gpu_rank, int32_t n_gpus, const themis_topology_t* topo /*[host]*/,
                                   void* const* heaps /*[host] n_gpus UVA pointers*/, uint64_t heap_bytes,
                                   uint64_t vrank_stride, themis_comm_t** out /*[out]*/);
/* Frees the comm's device state (waits for its host-stream copies).  Plans
 * still bound to it are unbound (themis_plan_bind them again to reuse them);
 * the heaps stay the caller's (themis_heap_free / themis_heap_close). */
void themis_comm_free(themis_comm_t* comm);
/* Latched asynchronous device errors (THEMIS_ERR_TIMEOUT) or THEMIS_OK.
 * Non-blocking: reads a host-mapped error word the kernel writes. */
themis_status_t themis_comm_status(themis_comm_t* comm);
/* Copy engine of the kernel: 1 (default) = TMA bulk copies (cp.async.bulk)
 * into a shared-memory ring + warp-specialised reduction; 0 = per-thread
 * 16-byte LDG/STG.  Env THEMIS_COPY_ENGINE=ldg|tma sets the default. */
themis_status_t themis_comm_set_engine(themis_comm_t* comm, int32_t engine);
/* Bandwidth emulation by pacing (TMA engine): when on, every CTA of dim k's
 * group pulls peer bytes no faster than V * bw_mbps[k] / ctas[k] (a per-CTA
 * leaky bucket over all its units: no credit accrues while it waits for
 * dependencies), so dim k's per-rank rate is capped
 * at the bound plan topology's absolute bw_mbps[k] (B_K =
 * 1/BW_K); a lone narrow op (op windows without rotation) on w CTAs paces at
 * V * bw_mbps[k] / w per CTA.  Off (default): only the CTA caps limit it. */
themis_status_t themis_comm_set_pacing(themis_comm_t* comm, int32_t on);
/* TMA ring per CTA: `stages` slots of `stage_bytes` (bytes in flight per CTA
 * = stages x stage_bytes <= 192 KiB); defaults 6 x 32 KiB, env THEMIS_STAGES /
 * THEMIS_STAGE_KB.  A tile moves stage_bytes / n_sources bytes per source.
 * Errors: INVALID_ARG (product too large, stage_bytes < 8 KiB or not KiB-aligned). */
themis_status_t themis_comm_set_stages(themis_comm_t* comm, int32_t stages);
themis_status_t themis_comm_set_stage_bytes(themis_comm_t* comm, int32_t stage_bytes);
/* Op windows (PAPER.md:461, :491 — several chunks per dimension in flight when
 * one chunk cannot saturate it): at bind, an op whose bytes on this GPU are
 * below c_k * min_cta_bytes runs on ceil(bytes / min_cta_bytes) CTAs of its
 * dimension group, consecutive ops taking consecutive windows.  0 (default,
 * env THEMIS_MIN_CTA_BYTES) = every op on all c_k CTAs, one op at a time per
 * dimension as in the pre-simulation.  Takes effect at the next
 * themis_plan_bind.  Errors: INVALID_ARG. */
themis_status_t themis_comm_set_min_cta_bytes(themis_comm_t* comm, uint64_t bytes);
/* Window placement for min_cta_bytes > 0: rotate = 1 (default, env
 * THEMIS_WINDOW_ROTATE) consecutive ops of a dimension take consecutive CTA
 * windows (several small ops in flight); rotate = 0: every narrow op starts at
 * the group's first CTA, so ops stay one at a time in the enforced order but a
 * small op occupies (and synchronises) only the CTAs it needs.  Takes effect at
 * the next themis_plan_bind.  Errors: INVALID_ARG. */
themis_status_t themis_comm_set_window_rotation(themis_comm_t* comm, int32_t rotate);
/* LL small collectives (DESIGN R31).  inbox_bytes > 0: every local rank has
 * an inbox of inbox_bytes right after the heap's data regions (the caller
 * allocated heap_bytes >= V * (signal_bytes + vrank_stride + inbox_bytes);
 * 16-byte multiple).  At the next themis_plan_bind, a plan of at most
 * max_bytes with no ring dim and no NVLS pair whose ops' inbox regions fit
 * (sum over ops of (P_k - 1) x part x 2) runs EVERY op with LL packets: the
 * sender stores 8-byte {4 payload bytes, epoch} packets straight into the
 * receivers' inboxes and the receivers poll the packets -- no flag, fence or
 * read round trip between ranks (each op waits only for its own previous
 * stage); the per-dim orders stay the enforced ones (the exchange is
 * pairwise, like the paper's collective ops).  Same summation order as the
 * pull path: results bit-identical.  themis_plan_bound_ll reports whether a
 * bound plan runs LL.  Host-buffer streaming and the LDG engine refuse LL
 * plans.  All ranks must use the same setting (launch hash).
 * Errors: INVALID_ARG (does not fit the heap). */
themis_status_t themis_comm_set_ll(themis_comm_t* comm, uint64_t inbox_bytes, uint64_t max_bytes);
/* Push-mode All-Gather (DESIGN R30): on = 1 (env THEMIS_PUSH), at the next
 * themis_plan_bind every direct-algorithm AG op (not ring, not NVLS) runs by
 * WRITES: each rank streams its own held part through shared memory and TMA
 * bulk-stores it into its P_k - 1 dim peers' buffers (NVLink carries data in
 * write requests instead of read responses + read requests), and the chunk's
 * next stage waits for the whole k x k' plane of ranks that wrote into its
 * sources.  Same results bit for bit (AG copies).  All ranks must bind with
 * the same setting (part of the launch hash).  Host-buffer streaming
 * (themis_allreduce_host) and the LDG engine run AG ops as pulls.
 * Errors: INVALID_ARG. */
themis_status_t themis_comm_set_push(themis_comm_t* comm, int32_t on);
/* Runtime intra-dimension order (DESIGN R28).  lookahead = 1
 * (default, env THEMIS_LOOKAHEAD): every dimension group runs its ops in the
 * pre-simulated enforced order.  L in 2..32: on every dim
 * without ring steps (direct, switch and NVLS dims), each CTA's producer
 * takes, among the next L not-yet-taken ops of the enforced list, the first
 * whose dependencies already hold (the enforced order stays the priority;
 * readiness decides), so a late op no longer blocks ready ones behind it.
 * Ranks may then run a dimension's ops in different orders, which the
 * pull-based executor tolerates (every op reads only its peers' finished
 * (c, s-1) data; R28).  Takes effect at the next collective.
 * Errors: INVALID_ARG. */
themis_status_t themis_comm_set_lookahead(themis_comm_t* comm, int32_t lookahead);
/* NVLS (in-switch reduction): mc_heap [device] = the
 * multicast (NVSwitch) mapping of this GPU's heap, at the same offsets, bound
 * on all W GPUs (e.g. torch symmetric memory's multicast pointer); NULL = off.
 * At the next themis_plan_bind, on every THEMIS_DIM_SWITCH dim whose group is
 * one rank per GPU at the same local index (P_k == W, stride_k == V), an RS op
 * directly followed by the chunk's AG op on that dim runs as one in-switch
 * All-Reduce of the rank's piece (multimem.ld_reduce + multimem.st; the switch
 * sums in its own order, bf16/f16 accumulate in fp32 and round once; R27).
 * TMA engine only.  Errors: INVALID_ARG. */
themis_status_t themis_comm_set_multicast(themis_comm_t* comm, void* mc_heap);
/* Watchdog: spin-waits give up after timeout_ns (default 20 s) and latch TIMEOUT. */
themis_status_t themis_comm_set_timeout(themis_comm_t* comm, uint64_t timeout_ns);
/* Trace: when enabled, each dim group records %globaltimer start/end of every
 * op it runs (PAPER.md:640/:658 activity).  Fetch after the stream is synced:
 * out[(chunk*n_stages + stage)*2 + {0,1}] in ns, n = C*n_stages*2 entries;
 * start = the earliest CTA of the group that begins the op (its dependencies
 * met), end = the op's completion published by its last CTA.  With tracing on
 * each collective also enqueues a memset of the trace buffer before the kernel. */
themis_status_t themis_comm_enable_trace(themis_comm_t* comm, int32_t enable);
themis_status_t themis_trace_fetch(themis_comm_t* comm, uint64_t* out /*[host,out]*/, size_t n);
/* Trace level 2 (themis_comm_enable_trace(comm, 2)): 6 extra %globaltimer
 * stamps per op, out[op*6 + j]: 0 producer issued its last tile (window CTA 0),
 * 1 consumers done (window CTA 0), 2 a CTA's completion warp reached the op
 * counter, 3 last CTA's atomic returned, 4 after its fence.acq_rel.sys, 5 unused. */
themis_status_t themis_trace_fetch_detail(themis_comm_t* comm, uint64_t* out /*[host,out]*/, size_t n);

/* CTA caps proportional to bandwidth (BW emulation by CTA caps, SURVEY a9,
 * north_star (d)): splits `budget` CTAs over the dims of `topo` as
 * c_k = max(1, floor(budget * bw_k / sum bw)), then one more CTA to the dims
 * with the largest remainders budget * bw_k / sum bw - c_k (ties: lower dim
 * index) while the caps sum below `budget`, or one fewer from the dims with
 * the smallest remainders among c_k > 1 while they sum above (largest
 * remainder with a floor of one CTA).  Whenever the roundings
 * max(1, round(budget * bw_k / sum bw)) sum to `budget` (and no share is a
 * half-integer), this equals SURVEY a9's c_k = max(1, round(c_tot BW_k / sum BW)).
 * Exact integer arithmetic.  Errors: INVALID_ARG (budget < ndims, bad topology). */
themis_status_t themis_default_ctas(const themis_topology_t* topo /*[host]*/, int32_t budget,
                                    int32_t* ctas_per_dim /*[host,out] ndims*/);
/* Attach a plan to a comm with per-dimension CTA counts.  ctas_per_dim[k] =
 * CTAs (SMs) of dimension k's group; NULL = themis_default_ctas over every
 * co-resident CTA of the device.  Capping CTAs per dim emulates heterogeneous per-dimension bandwidth
 * on the uniform NVSwitch fabric.  Uploads the per-dim op lists (the plan is
 * immutable afterwards).  Errors: INVALID_ARG (topology differs from the
 * comm's, too many CTAs for co-residency), CUDA. */
themis_status_t themis_plan_bind(themis_plan_t* plan, themis_comm_t* comm, const int32_t* ctas_per_dim /*[host] D or NULL*/);
/* The 64-bit hash a collective launched with this bound plan, count and dtype
 * announces at its entry barrier (plan hash + count + dtype + CTA caps + op
 * windows / NVLS rewrite); ranks whose hashes differ latch PLAN_MISMATCH
 * (R22).  For diagnosing mismatches and for fault-injection tests.
 * Errors: PLAN_MISMATCH if the plan is not bound. */
themis_status_t themis_plan_launch_hash(const themis_plan_t* plan, uint64_t count, int32_t dtype,
                                        uint64_t* hash /*[host,out]*/);
/* Debug (single-GPU profiling, fault injection): write into this GPU's local
 * ranks' signal pads that every logical rank of GPU peer_gpu entered, finished
 * every op / ring step and exited for all epochs, announcing the launch hash of
 * (plan, count, dtype).  This GPU's collectives then run alone -- pulling the
 * peer's heap over NVLink without waiting for it -- so one GPU's kernel can be
 * profiled (ncu replays it) with real NVLink traffic.  Results are garbage.
 * Errors: PLAN_MISMATCH (not bound), INVALID_ARG, CUDA. */
themis_status_t themis_debug_fake_peer_gpu(const themis_plan_t* plan, int32_t peer_gpu, uint64_t count, int32_t dtype);
/* 1 if a bound plan runs with LL packets (R31), else 0.
 * Errors: PLAN_MISMATCH if the plan is not bound. */
themis_status_t themis_plan_bound_ll(const themis_plan_t* plan, int32_t* ll /*[host,out]*/);
/* Number of a bound plan's chunk RS+AG pairs that run as in-switch
 * All-Reduces (NVLS dims on a multicast-capable comm, R29); 0 otherwise.
 * Errors: PLAN_MISMATCH if the plan is not bound. */
themis_status_t themis_plan_bound_nvls(const themis_plan_t* plan, int32_t* n_pairs /*[host,out]*/);
/* CTAs per dimension group a bound plan launches with ([host, out] D entries).
 * Errors: PLAN_MISMATCH if the plan is not bound. */
themis_status_t themis_plan_bound_ctas(const themis_plan_t* plan, int32_t* ctas_per_dim /*[host,out]*/);

/* ---------------------------------------------------------------- collectives
 * buf: [device] local rank 0's data region inside this GPU's heap (local rank
 * v's data is at buf + v*vrank_stride), the same offset on every GPU.
 * count: elements of the FULL buffer on each rank (all three calls).
 *   AR: every rank ends with sum_r x_r.
 *   RS: rank r ends with block r of the sum at buf + r*count/P (in place).
 *   AG: rank r's input block r is at buf + r*count/P; output is the full buffer.
 * Requirements: count * elem_size == plan bytes; count % (P * C * (16/elem_size)) == 0
 * (ALIGNMENT); the plan's coll matches the call (PLAN_MISMATCH); all ranks
 * call the same collectives, with identical plans, in the same order.
 * Float sums: fp32 accumulate in coordinate order within each stage, one
 * round-to-nearest-even per RS stage for bf16/f16 (R18); int32 wraps (R19).
 * Each call is one cooperative kernel launch on `stream` and may be captured
 * into a CUDA graph: the collective epoch is kept on the device, so every
 * replay is a new collective (all ranks must replay the same sequence). */
themis_status_t themis_allreduce(void* buf, uint64_t count, int32_t dtype, const themis_plan_t* plan, void* stream);
themis_status_t themis_reduce_scatter(void* buf, uint64_t count, int32_t dtype, const themis_plan_t* plan, void* stream);
themis_status_t themis_all_gather(void* buf, uint64_t count, int32_t dtype, const themis_plan_t* plan, void* stream);
/* End-to-end All-Reduce with HOST buffers: copies host_in (V local ranks,
 * contiguous, count elements each; pinned memory recommended) into the heap,
 * runs themis_allreduce, copies the result to host_out; all on `stream`. */
themis_status_t themis_allreduce_host(const void* host_in /*[host]*/, void* host_out /*[host,out]*/, void* buf,
                                      uint64_t count, int32_t dtype, const themis_plan_t* plan, void* stream);

/* Number of kernel launches the last collective call made (1 per call). */
int32_t themis_launches_per_call(void);
const char* themis_last_error(void);
const char* themis_version(void);

#ifdef __cplusplus
}
#endif
#endif /* THEMIS_H_ */
