/* libcoconet_cuda — C-ABI of the B200-native CoCoNet fused compute/communication
 * backend (sm_100a). Plain pointers and sizes only; never throws.
 *
 * The reference (ccopt, /root/reference/proj) executes every op inside the
 * simulated Engine::exec_data (runtime.hpp:367-524) on per-rank host vectors.
 * This library is what that dispatch lowers to: each entry point below is one
 * `exec_data` case (or one fused schedule the paper evaluates) re-designed for
 * B200 and replaces the cited reference routine. GpuEngine
 * (include/coconet/gpu_engine.hpp) is the drop-in host that walks a ccopt
 * Program and calls these; see INTEGRATION.md for the bindings.
 *
 * Execution model
 *  - One context per process. Two modes:
 *      VIRTUAL     : all `world` ranks live on one device in this process
 *                    (the reference's in-process rank model, state.hpp:17-20);
 *                    one call executes every rank, with the same cross-rank
 *                    flag protocol, co-resident CTAs standing in for peer GPUs.
 *      DISTRIBUTED : one process per GPU (rank = this process); peer heaps are
 *                    mapped over NVLink/NVSwitch with CUDA IPC.
 *  - Every rank owns a symmetric heap of the same size; symmetric buffers have
 *    the same OFFSET on every rank. Pointers passed to collective entry points
 *    must point into the caller's heap (VIRTUAL: rank 0's heap); the same
 *    offset is used on every rank of the group.
 *  - Calls are asynchronous on the caller's stream and collective: all ranks of
 *    a group issue the same calls in the same order (runtime.hpp:101-138 walks
 *    one plan for all ranks).
 *  - Cross-rank synchronisation is device-side (epoch flags with release /
 *    acquire at system scope); spin-waits are bounded by a watchdog that
 *    records COCONET_ERR_TIMEOUT instead of hanging (see coconet_check).
 */
#ifndef COCONET_CUDA_H
#define COCONET_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COCONET_MAX_RANKS 8

/* Status codes. 1..20 mirror ccopt::ErrCode (types.hpp:102-124) as
 * (ErrCode index + 1), so GpuEngine can re-throw ccopt::Error(code - 1). */
enum coconet_status {
  COCONET_OK = 0,
  COCONET_ERR_LAYOUT_MISMATCH = 1,
  COCONET_ERR_SHAPE_MISMATCH = 2,
  COCONET_ERR_INVALID_INPUT = 3,
  COCONET_ERR_NO_SUCH_RANK = 14,
  COCONET_ERR_OPERAND_LAYOUT_MISMATCH = 15,
  COCONET_ERR_DIVISIBILITY = 16,
  COCONET_ERR_REPLICATION_VIOLATION = 17,
  COCONET_ERR_UNKNOWN_ID = 19,
  COCONET_ERR_CUDA = 100,    /* a CUDA runtime/driver call failed */
  COCONET_ERR_TIMEOUT = 101, /* device watchdog: a peer never arrived */
  COCONET_ERR_UNSUPPORTED = 102,
  COCONET_ERR_OOM = 103      /* symmetric heap exhausted */
};

enum coconet_mode { COCONET_MODE_VIRTUAL = 0, COCONET_MODE_DISTRIBUTED = 1 };

/* Element types. ccopt::Elem has F16/F32 (types.hpp:12); BF16 is added for
 * B200 activations. Values are widened to fp32 for arithmetic. */
enum coconet_elem { COCONET_F32 = 0, COCONET_F16 = 1, COCONET_BF16 = 2 };

/* ccopt::Reducer (types.hpp:58) */
enum coconet_reducer { COCONET_SUM = 0, COCONET_MAX = 1, COCONET_MIN = 2 };

/* Arithmetic of the element-wise expression (SURVEY §5 "fp64-exact vs
 * fp32-fast"): EXACT evaluates in IEEE double with no contraction, exactly as
 * eval_expr does (expr.hpp:186-222), so results are bit-identical to the
 * reference Engine; FAST evaluates in fp32 with FMA. Both use the reference's
 * fp32 ring-order reduction (runtime.hpp:302-327). */
enum coconet_math { COCONET_MATH_EXACT = 0, COCONET_MATH_FAST = 1 };

/* Collective algorithm (paper §6.1 crossover):
 * TWO_SHOT = reduce-scatter pull + all-gather push (sliced state),
 * ONE_SHOT = every rank pulls all peers (replicated state), AUTO = by size. */
enum coconet_algo { COCONET_ALGO_AUTO = 0, COCONET_ALGO_TWO_SHOT = 1, COCONET_ALGO_ONE_SHOT = 2,
                    /* NVLS: two-shot through the NVSwitch multicast view of the heaps (multimem.ld_reduce
                     * for the reduce-scatter, multimem.st for the all-gather); explicit only, needs
                     * coconet_nvls_setup. The switch sums in its own order: results are within fp32
                     * rounding of TWO_SHOT, not bitwise. */
                    COCONET_ALGO_NVLS = 3 };

/* Symmetric-heap backing (coconet_init_ex). CUDAMALLOC: one cudaMalloc per rank,
 * peers through CUDA IPC. CUMEM: cuMemCreate + cuMemMap, peers import a POSIX
 * descriptor (fetched over a Unix socket). CUMEM_NVLS: a CUMEM heap sized to the
 * multicast granularity, ready for coconet_nvls_setup. DEFAULT reads the
 * environment variable COCONET_HEAP (cudamalloc | cumem | nvls; unset = cudamalloc). */
enum coconet_heap_kind { COCONET_HEAP_DEFAULT = 0, COCONET_HEAP_CUDAMALLOC = 1, COCONET_HEAP_CUMEM = 2,
                         COCONET_HEAP_CUMEM_NVLS = 3 };

typedef struct coconet_ctx* coconet_ctx_t;
typedef struct coconet_tlist* coconet_tlist_t;

/* ---- errors -------------------------------------------------------------- */
const char* coconet_last_error(void); /* thread-local message of the last failure */
const char* coconet_status_name(int status);

/* ---- lifecycle (replaces the in-process rank model, state.hpp:17-20) ------ */
/* VIRTUAL: rank is ignored, `world` ranks are created on `device`.
 * DISTRIBUTED: this process is `rank`; call coconet_exchange_handles next. */
int coconet_init(coconet_ctx_t* out, int mode, int rank, int world, int device,
                 size_t heap_bytes_per_rank);
/* coconet_init with an explicit heap kind (enum coconet_heap_kind). */
int coconet_init_ex(coconet_ctx_t* out, int mode, int rank, int world, int device,
                    size_t heap_bytes_per_rank, int heap_kind);
int coconet_heap_kind(coconet_ctx_t ctx); /* the resolved kind, -1 for a null ctx */
int coconet_finalize(coconet_ctx_t ctx);
int coconet_world(coconet_ctx_t ctx, int* world, int* rank, int* mode);
/* DISTRIBUTED bootstrap: export this rank's heap handle (`*len` bytes), then
 * pass the allgathered blob (world * len bytes, rank order) to open peers. */
int coconet_heap_handle(coconet_ctx_t ctx, void* handle_out, size_t* len);
int coconet_open_peers(coconet_ctx_t ctx, const void* all_handles, size_t len_per_rank);
/* NVLS (NVSwitch multicast). coconet_nvls_supported: 1 if `device` can join a
 * `world`-device multicast object, else 0 with the reason in `why`.
 * coconet_nvls_setup: collective, stages 0, 1, 2 in order after
 * coconet_open_peers with a process barrier after each (0: rank 0 creates the
 * multicast object; 1: the others import it, every rank adds its device; 2:
 * every rank binds its heap and maps the multicast range). Then
 * coconet_nvls_mapped is 1 and COCONET_ALGO_NVLS runs on the world group.
 * Replaces the AllReduce data path runtime.hpp:384-395 with in-switch sums. */
int coconet_nvls_supported(int device, int world, char* why, size_t why_len);
int coconet_nvls_setup(coconet_ctx_t ctx, int stage);
int coconet_nvls_mapped(coconet_ctx_t ctx);
/* Symmetric allocation: same offset on every rank; 256-byte aligned. */
/* Deterministic first-fit over a free list (256-byte granules, neighbours
 * coalesced on free): alloc/free are collective - every rank issues the same
 * sequence and gets the same offsets. */
int coconet_symm_alloc(coconet_ctx_t ctx, size_t bytes, size_t* offset);
int coconet_symm_free(coconet_ctx_t ctx, size_t offset); /* INVALID_INPUT if not live */
int coconet_symm_reset(coconet_ctx_t ctx); /* frees every symmetric allocation */
size_t coconet_symm_high_water(coconet_ctx_t ctx); /* highest offset ever allocated */
size_t coconet_heap_bytes(coconet_ctx_t ctx); /* per-rank heap size incl. reserved pad */
/* Device pointer of `offset` in `rank`'s heap (VIRTUAL: any rank;
 * DISTRIBUTED: own rank, or a mapped peer pointer). */
void* coconet_symm_ptr(coconet_ctx_t ctx, int rank, size_t offset);
/* ProcessGroup (types.hpp:42-50): contiguous rank interval. Group 0 is the
 * world group, created by init. */
int coconet_group_create(coconet_ctx_t ctx, int first_rank, int size, int* group);
/* Waits for `stream` and reports the first device-side failure (watchdog). */
int coconet_check(coconet_ctx_t ctx, void* stream);
/* Device watchdog bound for every spin-wait, in milliseconds (default 20000). */
int coconet_set_timeout_ms(coconet_ctx_t ctx, uint32_t ms);
/* Number of kernels this context launched so far (bench evidence). */
uint64_t coconet_launch_count(coconet_ctx_t ctx);

/* ---- synthetic inputs: gen_decl_values (state.hpp:55-74) on device -------- */
/* Writes rank-local storage of a decl into dst (elem type out_elem):
 * value(gi) = float(0.1 + 0.8 * counter_uniform(seed, key', gi)) where
 * key' = fnv1a(name) ^ (rank+1)*phi for LOCAL decls. Sliced decls
 * (sliced_dim >= 0) store only rank's slice (view.hpp:62-70 index map). */
int coconet_gen_values(coconet_ctx_t ctx, void* dst, int out_elem, uint64_t seed,
                       uint64_t name_key, int is_local, int rank, int ndim,
                       const int64_t* global_shape, int sliced_dim, int group_size,
                       void* stream);

/* ---- tensor lists: BucketTable (runtime.hpp:575-614) on device ----------- */
/* Buckets of <= bucket_cap elements per tensor, round-robin across tensors
 * (build_bucket_table). The flat bucket-order space is split into `group`'s
 * contiguous flat chunks total*c/W (runtime.hpp:63-66, uneven allowed): chunk
 * c is owned by group rank c. Built once, reused every step (paper §5.4). */
int coconet_tlist_create(coconet_ctx_t ctx, int group, int n_tensors, const int64_t* counts,
                         int64_t bucket_cap, coconet_tlist_t* out);
/* Host-only plan of the same tables for a group of `world` ranks (no device,
 * no context): for inspection and CPU tests; cannot be passed to kernels. */
int coconet_tlist_plan(int world, int n_tensors, const int64_t* counts, int64_t bucket_cap,
                       coconet_tlist_t* out);
int coconet_tlist_destroy(coconet_tlist_t tl);
/* Elements of shard storage each rank needs for sliced state (m, v): the
 * owned flat chunk plus alignment padding (so shard quads align with tensor
 * quads). Identical on every rank. */
int64_t coconet_tlist_shard_elems(coconet_tlist_t tl);
int64_t coconet_tlist_total(coconet_tlist_t tl);
/* ONE_SHOT replicated-state storage (padded full bucket-order space). */
int64_t coconet_tlist_state_elems(coconet_tlist_t tl);
int64_t coconet_tlist_buckets(coconet_tlist_t tl);
int64_t coconet_tlist_metadata_bytes(coconet_tlist_t tl); /* device bucket table bytes */
/* Flat chunk [lo, hi) owned by group rank r. */
int coconet_tlist_chunk(coconet_tlist_t tl, int r, int64_t* lo, int64_t* hi);
/* Segment table of group rank r (TWO_SHOT), or r = -1 for the ONE_SHOT table:
 * (tensor, element offset, length, state index) per segment; returns the count
 * (or -count if cap is too small). */
int64_t coconet_tlist_segments(coconet_tlist_t tl, int r, int64_t* tensor, int64_t* toff,
                               int64_t* len, int64_t* sidx, int64_t cap);
/* ONCHIP-LAMB plan of the last ONCHIP launch on this list: elements whose u
 * is not held on chip (beyond a CTA's hold, or a per-window cover item; their
 * pass 2 re-reads m', v'), or -1 if none was built.
 * Pass-level bytes at fp16 g: 30 per element + 8 per spilled element. */
int64_t coconet_tlist_onchip_spilled(coconet_tlist_t tl);
/* Shard index of flat position `pos` inside its owner's shard storage. */
int64_t coconet_tlist_shard_index(coconet_tlist_t tl, int64_t pos);
/* STREAMED-LAMB work list of rank r for a pass-1 -> pass-2 lag of `lag`
 * elements (see coconet_lamb_sched): items in execution order with their pass
 * (0/1). Host-only (works on a plan-only list). Returns the item count,
 * -count if cap is too small, -(2^62) on error. */
int64_t coconet_tlist_stream_items(coconet_tlist_t tl, int64_t lag, int r, int64_t* tensor,
                                   int64_t* toff, int64_t* len, int64_t* pass, int64_t cap);

/* ---- fused data-parallel optimizer: FusedAllReduce (runtime.hpp:471-516) -- */
/* Adam step of goldens/adam.json under schedules/adam_fused.json:
 *   m' = m*beta1 + c_m*g ; v' = v*beta2 + c_v*g*g ; m1 = m'/bc1 ; v1 = v'/bc2
 *   p' = p - lr*m1/(sqrt(v1) + eps)
 * with g = the ring-order reduce-scatter of the ranks' gradients. The golden
 * uses c_m = c_v = 1 - beta1 (its verbatim (1-beta1) typo) and eps = 0.
 * Scalars are the f32 decl values; the host forms the double constants
 * exactly as eval_expr would (pow on the host, expr.hpp:199-200). */
typedef struct {
  float lr, beta1, beta2, t;
  float eps;     /* 0 reproduces the golden (no epsilon) */
  int cv_beta1;  /* 1: c_v = 1-beta1 (golden), 0: c_v = 1-beta2 (textbook Adam) */
  int math;      /* coconet_math */
  int algo;      /* coconet_algo */
} coconet_adam_params;

/* g[i]: grads (elem g_elem) and p[i]: fp32 params of tensor i, symmetric.
 * TWO_SHOT: m_shard/v_shard hold coconet_tlist_shard_elems fp32 each (sliced
 * state, as_slice transform.hpp:515-558); p is all-gathered in place
 * (gather_decl "p", runtime.hpp:506-510).
 * ONE_SHOT: m_shard/v_shard hold the full flat bucket-order state
 * (coconet_tlist_state_elems elements; replicated m, v). */
int coconet_fused_rs_adam_ag(coconet_ctx_t ctx, coconet_tlist_t tl, const void* const* g,
                             int g_elem, float* const* p, float* m_shard, float* v_shard,
                             const coconet_adam_params* hp, void* stream);

/* LAMB step, per-tensor trust ratio (the paper's LAMB, PAPER.md:884-939;
 * golden authored in the reference JSON format, tests/golden/lamb_*):
 *   m' = m*beta1 + (1-beta1)*g ; v' = v*beta2 + (1-beta2)*g*g
 *   u  = m'/(1-beta1^t) / (sqrt(v'/(1-beta2^t)) + eps) + wd*p
 *   p' = p - lr*sqrt(sum(p*p))/sqrt(sum(u*u))*u        (sums per tensor)
 * The per-tensor sums are partial per rank, exchanged over the open
 * symmetric buffers and combined in rank order (state.hpp:139-174), inside
 * the same kernel (K12). */
typedef struct {
  float lr, beta1, beta2, t, eps, wd;
  int math;  /* FAST: fp32 element math, m'/v' stored in pass 1 (38 B/element at fp16 g).
                EXACT: the reference's double element math (expr.hpp:186-222) with a
                read-only pass 1 and m', v', u recomputed in pass 2 from the same old
                values, as eval_pointwise does (state.hpp:139-190); only the norm
                summation order differs from the Engine. `sched` is ignored. */
  int sched; /* coconet_lamb_sched; both give bit-identical results */
  int64_t lag_elems; /* STREAMED: pass-1 -> pass-2 distance in elements (0 = default) */
  int trust_guard;   /* 0: the golden's raw lr*sqrt(P)/sqrt(U) (reference parity);
                        1: ratio = lr when either norm is 0 (apex/NVLAMB; FusedLAMB) */
  int pad_;
} coconet_lamb_params;

/* LAMB schedules (bit-identical results). GRID: pass 1 over the whole shard,
 * grid-wide sync, norms, pass 2 over the whole shard (m, v, p read twice
 * from HBM: 38 B/element at fp16 g). STREAMED: the shard's segments in tensor
 * order, one small CTA per segment; a tensor's pass 2 is scheduled lag_elems
 * of pass-1 work after its pass 1 and waits only on that tensor's norms
 * (per-tensor completion counters, cross-rank ready flags), so part of its
 * m, v, p re-reads hit L2. TMA: GRID's two passes with the local m, v, p
 * (and g at group size 1) fed by bulk copies; across ranks g is pulled and p
 * pushed by the consumer threads. AUTO = TMA with buckets of >= 4096
 * elements, GRID otherwise. m and v are bit-identical across
 * schedules; TMA sums the norms in another fixed order. */
enum coconet_lamb_sched {
  COCONET_LAMB_AUTO = 0,
  COCONET_LAMB_GRID = 1,
  COCONET_LAMB_STREAMED = 2,
  COCONET_LAMB_TMA = 3, /* GRID's two passes fed by TMA bulk copies into a shared-memory ring
                          (norms summed in a different fixed order) */
  COCONET_LAMB_WINDOWED = 4, /* group size 1: the TMA ring over windows of consecutive tensors
                               (lag_elems = window size), pass 2 of a window one window after
                               its pass 1 so its m, v, p re-reads hit L2; per-window arrival
                               counters instead of grid-wide syncs. m, v bit-identical to TMA */
  COCONET_LAMB_ONCHIP = 5, /* group size 1: pass 1 keeps u = m'/(sqrt(v')+eps) + wd*p on chip
                             (TMEM + shared memory of one CTA per SM) for windows of whole
                             tensors, so pass 2 reads only p (30 B/element at fp16 g against
                             38); items beyond a CTA's on-chip capacity take TMA's pass 2.
                             m, v bit-identical to TMA */
  COCONET_LAMB_NVLS = 6 /* GRID's two passes with the RS pull as one multimem.ld_reduce and the AG
                           push as one multimem.st through the NVSwitch multicast view
                           (coconet_nvls_setup; world group only; never chosen by AUTO) */
};

int coconet_fused_rs_lamb_ag(coconet_ctx_t ctx, coconet_tlist_t tl, const void* const* g,
                             int g_elem, float* const* p, float* m_shard, float* v_shard,
                             const coconet_lamb_params* hp, void* stream);

/* The unfused GPU baseline the north star measures against ("NCCL plus
 * separate kernels"; the paper's LAMB comparison is DDP AllReduce + apex
 * FusedLAMB): the same LAMB step as FOUR separate multi-tensor
 * kernels - stage 1 (m', v', u into u_scratch), per-segment L2-norm partials
 * of p and u, per-tensor combine, stage 2 (p -= ratio*u) - over a list whose
 * group has ONE rank (after an all-reduce every rank updates every element,
 * replicated state). m, v, u_scratch: coconet_tlist_shard_elems fp32 each;
 * norms_scratch: 2 * n_tensors doubles. 46 B/element at fp16 g against the
 * fused kernel's 38. Same element math as FAST. */
int coconet_unfused_lamb(coconet_ctx_t ctx, coconet_tlist_t tl, const void* const* g, int g_elem,
                         float* const* p, float* m, float* v, float* u_scratch, double* norms_scratch,
                         const coconet_lamb_params* hp, void* stream);

/* ---- collectives (runtime.hpp:306-414, exec_gather_decl :529-557) --------- */
/* Flat-chunk AllReduce over a tensor list (AR: x -> out, in place allowed),
 * fp32 ring-order reduction; elem = storage type of x and out. This is also
 * scattered_collective (runtime.hpp:624-675) without the flatten copy. */
int coconet_allreduce(coconet_ctx_t ctx, coconet_tlist_t tl, const void* const* x,
                      void* const* out, int elem, int reducer, int algo, void* stream);

/* Axis-sliced ReduceScatter / AllGather of one tensor (ChunkSpec axis_chunks,
 * runtime.hpp:78-85; DistView::to_global view.hpp:62-70). Shapes are global.
 * RS: x (Local, full) -> out (rank's slice). AG: x (rank's slice) -> out (full).
 * AG with x == NULL gathers `out` in place from each rank's owned region
 * (the gather_decl form, exec_gather_decl). */
int coconet_reduce_scatter(coconet_ctx_t ctx, int group, const void* x, void* out, int elem,
                           int reducer, int ndim, const int64_t* shape, int axis, void* stream);
int coconet_all_gather(coconet_ctx_t ctx, int group, const void* x, void* out, int elem, int ndim,
                       const int64_t* shape, int axis, void* stream);

/* Rooted collectives (runtime.hpp:415-436). Reduce: the root's out = fold of
 * every rank's x (n elements) in RANK order 0..G-1 in fp32 (the Engine's
 * order), other ranks' out = 0 (Local layout: meaningful on the root only,
 * program.hpp:315-321); x may alias out. Broadcast: every rank's out = the
 * root's x. `root` is a group rank. */
int coconet_reduce(coconet_ctx_t ctx, int group, const void* x, void* out, int elem, int reducer, int64_t n,
                   int root, void* stream);
int coconet_broadcast(coconet_ctx_t ctx, int group, const void* x, void* out, int elem, int64_t n, int root,
                      void* stream);

/* Send / Recv (runtime.hpp:439-470): group rank r of src_group stores its n
 * local elements of x into out on group rank r of dst_group (same sizes,
 * "peer group sizes differ" otherwise). Every rank of the interval covering
 * both groups calls; the destination sees the data after the call. */
int coconet_send(coconet_ctx_t ctx, int src_group, int dst_group, const void* x, void* out, int elem,
                 int64_t n, void* stream);

/* Element-type conversion of a plain device array of n elements (16-bit
 * staging of fp32-stored decls for the tcgen05 MatMul). Not collective. */
int coconet_convert(coconet_ctx_t ctx, const void* src, int src_elem, void* dst, int dst_elem, int64_t n,
                    void* stream);

/* ---- fused MP / PP epilogues (goldens/model_parallel.json, pipeline.json) - */
/* out = dropout(x + b, rate, key) + r, element-wise, dropout index = global
 * flat index (expr.hpp:15-27, state.hpp:178-181); b broadcast over leading
 * axes (BroadcastView view.hpp:75-98). */
typedef struct {
  double rate; /* the parsed double literal (json_io.hpp:205) */
  uint64_t seed, key;
  int math;
} coconet_bdr_params;

/* FusedAllReduce with the MP expression: RS of x (Local [rows, H], axis =
 * last dim, chunk c = column block c) -> bias+dropout+residual on the slice
 * -> AG into out (Replicated [rows, H]). */
int coconet_fused_rs_bdr_ag(coconet_ctx_t ctx, int group, const void* x, const void* b,
                            const void* r, void* out, int elem, int64_t rows, int64_t cols,
                            const coconet_bdr_params* hp, void* stream);

/* PP stage boundary, pipeline_overlap.json: RS in group src (x Local [n]) ->
 * bias+dropout+residual on the rank's slice -> remote store into the peer
 * rank of group dst (same group-relative index; runtime.hpp:439-470) -> AG in
 * group dst into out. intergroup bytes per sender = n/W * bw. */
int coconet_rs_fused_send_ag(coconet_ctx_t ctx, int src_group, int dst_group, const void* x,
                             const void* b, const void* r, void* out, int elem, int64_t n,
                             const coconet_bdr_params* hp, void* stream);

/* ---- MatMul (state.hpp:94-121) ------------------------------------------ */
/* Row-major C[M,N] = A[M,K] * B[K,N] per rank; BF16/F16 inputs on tcgen05
 * (TMEM accumulators, TMA-fed), fp32 accumulation; out_elem F32 or BF16.
 * EXACT with F32 inputs: fp64 accumulation in k order (bit-exact with
 * eval_matmul). */
int coconet_matmul(coconet_ctx_t ctx, int group, const void* a, const void* b, void* c,
                   int in_elem, int out_elem, int64_t m, int64_t n, int64_t k, int math,
                   void* stream);

/* OverlapGroup{MatMul, FusedAllReduce(bias+dropout+residual)} (mp_overlap.json,
 * runtime.hpp:517-522). Three schedules:
 *  - AUTO (aggemm): ONE all-gather -> GEMM kernel when cols/W is a multiple
 *    of 128 (run as 384-, 256- or 128-column sub-blocks), rows % 256 == 0 and
 *    k_local % 64 == 0. The owner of column block c
 *    streams every rank's A_r and B_r[:, c] through one K loop (TMA from the
 *    peers' memory), accumulates in fp32 TMEM, applies bias + dropout (masks
 *    bit-exact) + residual and pushes the finished tile into every rank's
 *    `out`. The partial products are never formed, so `partial` is not
 *    written; results are within 1e-2 of the two-kernel schedule (fp32 sum
 *    over the whole K instead of 16-bit partials folded in ring order).
 *  - sequential: coconet_matmul into `partial`, then coconet_fused_rs_bdr_ag.
 *  - fused: one cooperative kernel, the GEMM publishing a flag per output
 *    tile (row tile outermost) and comm warps running RS->epilogue->AG per
 *    (row tile, column block) unit; bitwise equal to sequential.
 * COCONET_MP_OVERLAP=aggemm|sequential|fused forces one; other shapes run
 * sequential. */
int coconet_mm_overlap_fused_ar(coconet_ctx_t ctx, int group, const void* a, const void* w,
                                const void* b, const void* r, void* partial, void* out,
                                int in_elem, int64_t rows, int64_t cols, int64_t k_local,
                                const coconet_bdr_params* hp, void* stream);

/* ---- generic element-wise expressions (eval_pointwise, state.hpp:126-193) --
 * Any ccopt ExprDag (expr.hpp:29-173) lowered to a node list in evaluation
 * order (children before parents, only nodes reachable from the root without
 * entering ReduceTensor children). Evaluated in IEEE double without
 * contraction like eval_expr (expr.hpp:186-222); element-uniform subtrees
 * (scalar-only, e.g. 1 - pow(beta1, t)) arrive pre-folded by the host as
 * CONST, per rank. Used by GpuEngine for Pointwise nodes and for fused
 * expressions no specialised kernel matches. */
enum coconet_expr_op {
  COCONET_OP_CONST = 0, COCONET_OP_INPUT = 1, COCONET_OP_ADD = 2, COCONET_OP_SUB = 3,
  COCONET_OP_MUL = 4, COCONET_OP_DIV = 5, COCONET_OP_SQRT = 6, COCONET_OP_POW = 7,
  COCONET_OP_DROPOUT = 8, COCONET_OP_REDUCED = 9, COCONET_OP_UPDATE = 10
};

#define COCONET_EXPR_MAX_NODES 160
#define COCONET_EXPR_MAX_OPERANDS 12
#define COCONET_EXPR_MAX_DIMS 6

typedef struct {
  int32_t op;       /* coconet_expr_op */
  int32_t a, b;     /* operand node positions in this list */
  int32_t slot;     /* INPUT: operand slot; UPDATE: target slot; REDUCED: reduce index;
                       CONST: per-rank constant index (-1 = use `value`) */
  double value;     /* CONST */
  double rate;      /* DROPOUT */
  uint64_t key;     /* DROPOUT */
} coconet_expr_node;

/* A tensor as the element loop sees it: its heap offset, its GLOBAL shape
 * right-aligned to the output rank (BroadcastView, view.hpp:75-98), and its
 * storage layout (sliced_dim >= 0: only the rank's slice is stored,
 * DistView::to_local view.hpp:49-60). */
typedef struct {
  int64_t off;
  int32_t elem;                          /* coconet_elem */
  int32_t ndim;
  int64_t shape[COCONET_EXPR_MAX_DIMS];  /* global shape, ndim entries */
  int32_t sliced_dim;                    /* in this operand's own dims, -1 if not sliced */
  int32_t pad_;
} coconet_operand;

typedef struct {
  int32_t n_nodes, n_inputs, n_targets, n_reduce;
  int32_t root;
  int32_t out_sliced_dim;      /* iteration space: the output's layout */
  int32_t out_ndim;
  int32_t n_rank_consts;       /* per-rank constants (folded uniform subtrees) */
  int64_t out_shape[COCONET_EXPR_MAX_DIMS];
  uint64_t seed;
  coconet_operand out;
  coconet_operand inputs[COCONET_EXPR_MAX_OPERANDS];
  coconet_operand targets[4];
  coconet_expr_node nodes[COCONET_EXPR_MAX_NODES];
} coconet_expr_program;

/* Per-element pass: out[r] and Update targets for every local rank.
 * rank_consts[r * n_rank_consts + i], reduced[r * n_reduce + j] (may be NULL). */
int coconet_pointwise(coconet_ctx_t ctx, int group, const coconet_expr_program* prog,
                      const double* rank_consts, const double* reduced, void* stream);
/* ReduceTensor pre-pass: for reduce node `node` (sum/max/min = red) evaluates
 * its subtree (no Update stores) over each rank's local iteration space and
 * writes one partial per local rank into host memory partial[r] (synchronous).
 * Deterministic (fixed-order two-level reduction). */
int coconet_pointwise_reduce(coconet_ctx_t ctx, int group, const coconet_expr_program* prog, int node,
                             int red, const double* rank_consts, double* partial, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* COCONET_CUDA_H */
