/*
 * marrow.h — C-ABI of libmarrow.so, the B200-native hot path of the Marrow
 * skeleton framework (Soldado, Alexandre, Paulino, arXiv:1510.06585).
 *
 * "P:n" cites /root/reference/PAPER.md line n; "S:n" cites SPEC.md line n.
 * The entry points mirror the paper's constructors and run request (Table 1,
 * P:181-214): build a skeleton computation tree (SCT) bottom-up from built-in
 * kernels, set the workload-distribution vector, run it (asynchronously,
 * returning a future), monitor per-partition times and rebalance.
 *
 * Execution model (§3.1 "locality-aware domain decomposition"):
 * the input domain is split into P = nranks * parts_per_rank contiguous
 * partitions ("parallel executions" j of P:355-372), one process per GPU
 * (rank) owning parts_per_rank consecutive partitions; every partition runs
 * the WHOLE tree on its slice and intermediates stay in device memory.
 * Inter-partition exchange (hysteresis halos, MapReduce merge, N-body COPY
 * re-replication, loop-condition reduction) uses device copies inside a rank
 * and NCCL over NVLink between ranks.
 *
 * Conventions for every function:
 *  - returns MW_OK (0) or an error code; on error, out-params are untouched
 *    and mw_last_error() holds a message naming the violated rule;
 *  - no C++ exception crosses this boundary;
 *  - pointers are borrowed (the caller owns every buffer it passes; device
 *    buffers must stay valid until the run's future completes);
 *  - one host thread drives a given mw_ctx.  Node builders touch no
 *    device and are thread-safe.
 *  - "collective": every rank must call it, in the same order.
 */
#ifndef MARROW_H
#define MARROW_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MW_ABI_VERSION 1

/* ------------------------------------------------------------------ status */
typedef int32_t mw_status;
enum {
    MW_OK = 0,
    MW_E_INVALID_SPEC = 1,          /* ill-formed tree, params or distribution */
    MW_E_EPU_NU = 2,                /* epu mod nu != 0            */
    MW_E_INFEASIBLE_PARTITION = 3,  /* strict divisibility impossible        */
    MW_E_SHAPE_MISMATCH = 4,        /* args do not match the root's interface*/
    MW_E_MISSING_ITERATION_COUNT = 5, /* execution order needs a while count  */
    MW_E_NOT_CONVERGED = 6,         /* while-loop hit max_iters (result still valid) */
    MW_E_CUDA = 7,
    MW_E_NCCL = 8,
    MW_E_STATE = 9,                 /* wrong call order / released handle            */
    MW_E_OOM = 10,
    MW_E_UNSUPPORTED = 11,          /* valid SCT outside the built hot path (NEXT-4)  */
};

typedef struct mw_ctx mw_ctx;
typedef struct mw_node mw_node;
typedef struct mw_future mw_future;

const char* mw_status_string(mw_status s);
/* Last error message of the calling thread (ctx may be NULL). Never NULL.    */
const char* mw_last_error(const mw_ctx* ctx);
int32_t mw_abi_version(void);

/* ------------------------------------------------------------------ context */
/* Device memory callbacks (PyTorch's caching allocator in the Python
 * binding).  alloc returns a device pointer (256-B aligned) or NULL; stream
 * is the cudaStream_t the memory will be used on.  NULL => cudaMalloc/Free. */
typedef struct mw_alloc_fns {
    void* (*alloc)(size_t bytes, void* stream, void* user);
    void (*free)(void* ptr, void* user);
    void* user;
} mw_alloc_fns;

/* NCCL unique id for mw_ctx_create (call on one rank, broadcast the 128 bytes
 * with torch.distributed).                                                   */
mw_status mw_nccl_unique_id(uint8_t out[128]);

/* Transport of the cross-rank exchanges (halo rows, merges, COPY
 * re-replication, loop condition, timings; P:224, P:376, P:705-707,
 * P:736-737).                                                                */
enum {
    MW_TRANSPORT_AUTO = 0,     /* NCCL when nranks > 1, none for one rank      */
    MW_TRANSPORT_NCCL = 1,     /* NCCL even for one rank (1-rank communicator) */
    /* TEST-ONLY: the ranks are threads of ONE process sharing a device; every
     * exchange is device copies between their buffers ordered by CUDA events
     * and host barriers, with NCCL's completion semantics.  It runs the
     * cross-rank code paths of the executor on a one-GPU machine.  The id is
     * any 128 bytes shared by the group (e.g. mw_nccl_unique_id's).        */
    MW_TRANSPORT_LOOPBACK = 2
};
/* Create a context on CUDA device `device` for rank `rank` of `nranks`
 * processes (or loopback threads), each owning `parts_per_rank` (>= 1)
 * consecutive partitions.
 * nccl_id: the group id, required when nranks > 1 or transport != AUTO (then
 * a communicator is created — collective: blocks until every rank joined),
 * ignored otherwise.
 * The initial distribution is uniform over the P partitions (identical
 * B200s have equal relative performance).  Errors: MW_E_INVALID_SPEC (bad
 * rank / transport / missing id), MW_E_NCCL, MW_E_CUDA.                     */
mw_status mw_ctx_create(int32_t device, int32_t rank, int32_t nranks, int32_t parts_per_rank,
                        const uint8_t* nccl_id, int32_t transport, const mw_alloc_fns* alloc,
                        mw_ctx** out);
/* Collective when the ctx owns an NCCL communicator.  Frees all scratch; when
 * futures or graphs of the ctx are still alive the teardown happens at the
 * release of the last of them (the ctx is unusable from this call on).     */
mw_status mw_ctx_destroy(mw_ctx* ctx);
/* Number of partitions P (= nranks * parts_per_rank) and this rank's first. */
mw_status mw_ctx_info(const mw_ctx* ctx, int32_t* n_parts, int32_t* first_part,
                      int32_t* parts_per_rank, int32_t* rank, int32_t* nranks);

/* ------------------------------------------------------------------ kernels
 * Built-in kernel leaves (P:168-178 Kernel objects; the paper's OpenCL
 * sources become fixed sm_100a kernels).  Each leaf carries its argument
 * interface (value kind, epu, nu, PARTITION/COPY, Size/Offset traits) and its
 * scalar parameters.  Definitions: DESIGN.md §Readings (R1-R12).            */
mw_status mw_kernel_saxpy(float a, mw_node** out);
/* Gaussian noise (R1): n_c = (popcount((h>>10c)&0x3FF) - 5) * scale,
 * h = lowbias32(idx ^ lowbias32(seed ^ 0x9E3779B9)), idx = global y*W + x.
 * scale in [0, 255].                                                         */
mw_status mw_kernel_gauss_noise(uint32_t seed, int32_t scale, mw_node** out);
mw_status mw_kernel_solarize(int32_t threshold, mw_node** out);          /* P:725, R2 */
mw_status mw_kernel_mirror(mw_node** out);
/* 3-class threshold {0,128,255}, 0 <= lo <= hi <= 256 (R6); also the
 * hysteresis threshold2d stage.                                              */
mw_status mw_kernel_segment(int32_t lo, int32_t hi, mw_node** out);
mw_status mw_kernel_hysteresis_step(mw_node** out);      /* 8-neighbour Jacobi, R11 */
mw_status mw_kernel_hysteresis_finalize(mw_node** out);  /* 128 -> 0, R11           */
mw_status mw_kernel_nbody_step(float dt, float eps2, mw_node** out);
mw_status mw_kernel_nbody_accel(float eps2, mw_node** out);  /* test leaf: a_i only */
mw_status mw_kernel_map_identity(mw_node** out);         /* MapReduce map stage: x   */
mw_status mw_kernel_map_product(mw_node** out);          /* MapReduce map stage: x*y */
/* Reduction-stage leaf (NEXT-4; Table 1 P:191 "map_reduce(SCT map_stage, SCT
 * reduction_stage)", "It is thus up to the programmer to decide where
 * the reduction takes place" — here: on the device).  It reduces the terms
 * of a map stage (x or x*y, each exact in fp64) with an associative,
 * commutative operator; the partitions' partial results are merged with the
 * same operator, so the result is the reduction over the whole domain
 * (reading R28): SUM = the canonical fp64 sum (as MW_MERGE_ADD), MAX / MIN =
 * IEEE maxNum / minNum (a NaN term is ignored; exact, bit-identical for every
 * distribution).  Empty domain: 0, -inf, +inf.  Only usable as the second
 * argument of mw_map_reduce_sct; op outside 0..2: MW_E_INVALID_SPEC.        */
enum { MW_REDUCE_SUM = 0, MW_REDUCE_MAX = 1, MW_REDUCE_MIN = 2 };
mw_status mw_kernel_reduce(int32_t op, mw_node** out);
/* Test leaf: writes each element's partition (SIZE, OFFSET) trait
 * values.  epu/nu feed the constraint system;
 * strict != 0 forbids the L mod granule tail.                                */
mw_status mw_kernel_debug_traits(int64_t epu, int64_t nu, int32_t strict, mw_node** out);
/* FFT leaf (NEXT-3; "a set of Fast-Fourier Transformations ...
 * pipelined with its inversion ... The elementary partitioning unit is the
 * size of each FFT which is 512 KBytes"; readings R23-R25): every row of a
 * complex64 batch f32[B][N][2] (interleaved re, im; N = 2^log2n, log2n in
 * 13..16, default benchmark 16 = 512 KiB) is transformed; inverse != 0 gives
 * the inverse transform including the 1/N factor.  Consecutive FFT leaves of
 * a Pipeline fuse (a forward followed by an inverse is one launch: each FFT
 * crosses HBM once).  Partitioned by whole transforms.  log2n outside 13..16
 * or inverse not 0/1: MW_E_INVALID_SPEC.                                    */
mw_status mw_kernel_fft(int32_t log2n, int32_t inverse, mw_node** out);

/* ------------------------------------------------------------------ skeletons
 * Table 1.  Composites retain their children; trees are
 * immutable and may be shared across runs and contexts.           */
mw_status mw_pipeline(mw_node* const* stages, int32_t n, mw_node** out);  /* n >= 2 */
mw_status mw_map(mw_node* tree, mw_node** out);
/* Merging functions ("a set of predefined functions (addition,
 * subtraction, multiplication and division) and also ... user-defined
 * functions"; NEXT-4, reading R26).  ADD returns the canonical sum of all
 * terms (chunk partials combined in global order: bit-identical for every
 * distribution).  SUB / MUL / DIV / USER combine the per-partition partial
 * results r_p (each partition's own reduction, partitions with work in
 * global order): acc = r_first; acc = op(acc, r_p) — on the host, when the
 * future completes; the result depends on the distribution by definition.
 * MapReduce roots with SUB..USER cannot be captured in a graph.              */
enum { MW_MERGE_ADD = 0, MW_MERGE_SUB = 1, MW_MERGE_MUL = 2, MW_MERGE_DIV = 3, MW_MERGE_USER = 4 };
typedef double (*mw_merge_fn)(double acc, double partial, void* user);
mw_status mw_map_reduce(mw_node* map_stage, int32_t merge_op, mw_node** out);   /* ADD..DIV */
/* User-defined merging function (called on the host thread that waits on the
 * future; fn must not call back into libmarrow).                           */
mw_status mw_map_reduce_user(mw_node* map_stage, mw_merge_fn fn, void* user, mw_node** out);
/* MapReduce with a device reduction stage (an mw_kernel_reduce leaf, or the
 * reduction-stage SCT below; NEXT-4): the map stage's terms are
 * reduced on the device, partition partials merged with the same operator
 * across ranks (NCCL all-reduce).  Result as for mw_map_reduce
 * (mw_future_result out[0] fp64, out[1] fp32).  A reduction stage that is
 * not such a tree, or a map_stage not producing terms: MW_E_INVALID_SPEC.  */
mw_status mw_map_reduce_sct(mw_node* map_stage, mw_node* reduction_stage, mw_node** out);
/* Reduction-stage SCT leaves (NEXT-4, P:191 map_reduce(SCT, SCT) with the
 * reduction placed on the device).  The reduction stage of
 * mw_map_reduce_sct may be pipeline(term maps..., mw_kernel_reduce(op),
 * scalar maps...): a term map applies to every fp64 term before the fold
 * (ABS: |t|, SQUARE: t*t in fp64, exact for identity terms), a scalar map to
 * the reduced fp64 value after the merge (SQRT, SCALE by c).  E.g. the L2
 * norm = map_reduce_sct(map_identity, pipeline(term_map(SQUARE),
 * reduce(SUM), scalar_map(SQRT))).  Fused into the reduction kernels (term
 * maps) and its combine (scalar maps).  Unknown kind: MW_E_INVALID_SPEC.   */
enum { MW_TERM_ABS = 0, MW_TERM_SQUARE = 1 };
enum { MW_SCALAR_SQRT = 0, MW_SCALAR_SCALE = 1 };
mw_status mw_kernel_term_map(int32_t kind, mw_node** out);
mw_status mw_kernel_scalar_map(int32_t kind, double c, mw_node** out);
mw_status mw_loop_for(mw_node* body, int64_t n, mw_node** out);           /* n >= 0 */
/* while(changed && executions < max_iters) body.
 * The stop condition is evaluated on the device and reduced across ranks
 * every `check_every` (>= 1) executions; extra executions past the fixed
 * point are no-ops and the reported execution count E is exact.            */
mw_status mw_loop_while_changed(mw_node* body, int64_t max_iters, int32_t check_every,
                                mw_node** out);
/* Loop with a host-side condition / state update ("1 - evaluation
 * of the condition, on the host; 2 - execution of the body (the SCT), on the
 * device(s); and 3 - the update of the loop's state ... (also performed on
 * the host)"; NEXT-4, reading R27).  Before iteration i (0-based, i <
 * max_iters) the library synchronizes the run's stream and calls
 * cond(i, user) on the calling thread; 0 ends the loop.  The callback may
 * read or write host state (stage 3).  Iteration i reads the previous
 * iteration's output (ping-pong; src -> dst for i = 0), so a body of k
 * iterations equals loop_for(body, k).  Executions are reported like
 * LoopWhileChanged's.  The root, or one stage of a root pipeline (the stages
 * before it run into an intermediate buffer, the ones after it from its
 * output; deeper nesting: MW_E_UNSUPPORTED); not capturable.
 * mw_run returns after the last condition evaluation.                        */
typedef int32_t (*mw_loop_cond_fn)(int64_t iteration, void* user);
mw_status mw_loop_host(mw_node* body, int64_t max_iters, mw_loop_cond_fn cond, void* user,
                       mw_node** out);
void mw_node_retain(mw_node* n);
void mw_node_release(mw_node* n);
/* Deterministic content hash (SHA-256 of a canonical serialization): equal
 * for structurally equal trees, different when any kernel parameter differs
 * (profile item (a) P:447).                                       */
mw_status mw_node_id(const mw_node* n, uint8_t out[32]);
/* Value kinds flowing in/out of a tree (MW_VK_*), see mw_run for the args.  */
enum {
    MW_VK_SAXPY = 1, MW_VK_RGBA = 2, MW_VK_U8 = 3, MW_VK_U8_2D = 4, MW_VK_NBODY = 5,
    MW_VK_VEC1 = 6, MW_VK_VEC2 = 7, MW_VK_TERMS = 8, MW_VK_ACCEL = 9, MW_VK_TRAITS = 10,
    MW_VK_SCALAR = 11, MW_VK_CPLX = 12,
};
mw_status mw_node_signature(const mw_node* n, int32_t* in_kind, int32_t* out_kind);
/* Sequential single-device kernel order (depth-first): leaves are
 * numbered 0.. in pre-order; LoopFor bodies repeat n times; each
 * LoopWhileChanged node (pre-order) consumes one count from while_counts.
 * *inout_len: capacity in, length out (MW_E_INVALID_SPEC if too small, with
 * *inout_len set to the needed length).                                      */
mw_status mw_kernel_execution_order(const mw_node* root, const int64_t* while_counts,
                                    int32_t n_counts, int32_t* out_ids, int64_t* inout_len);

/* ------------------------------------------------------------------ partition
 * Granule g (in units of the partitioned outermost dimension) of a tree:
 * lcm of every leaf's epu/nu and the alignment unit of its value kind
 * (R5/R14).                                            */
mw_status mw_granule(const mw_node* root, int64_t* out);
/* Pure: largest-remainder apportionment of L units over k fractions with
 * granule g (R13).  offsets/lengths: k entries each.              */
mw_status mw_partition_plan(int64_t L, int64_t g, const double* fractions, int32_t k,
                            int32_t strict, int64_t* offsets, int64_t* lengths);
/* fractions: P entries, each >= 0, at least one > 0, sum 1 +- 1e-9.         */
mw_status mw_set_distribution(mw_ctx* ctx, const double* fractions, int32_t n);
mw_status mw_get_distribution(const mw_ctx* ctx, double* out, int32_t n);
/* All P partitions of a domain of L outer units for `root` under the ctx's
 * current distribution — identical on every rank.                           */
mw_status mw_partition(const mw_ctx* ctx, const mw_node* root, int64_t L, int64_t* offsets,
                       int64_t* lengths);

/* ------------------------------------------------------------------ run
 * Buffer argument.  shape is the GLOBAL shape, outermost (partitioned)
 * dimension first.  A PARTITION buffer on this rank holds global outer rows
 * [local_offset, local_offset + local_rows) at ptr; it must cover this
 * rank's partitions (else MW_E_SHAPE_MISMATCH), so both "exactly my slice"
 * and "the whole array" work.  A COPY buffer holds the whole
 * array on every rank.  location MW_LOC_HOST: ptr is host memory (pinned for
 * overlap) — the library stages this rank's slice through device memory with
 * chunked, multi-stream H2D / compute / D2H overlap (the paper's GPU
 * "overlap").
 *
 * Interfaces by the root's input value kind (mut = written by the run):
 *   SAXPY        x f32[L], y f32[L] (mut, in place)
 *   RGBA         src u8[H][W][4], dst u8[H][W][4] (mut)          partition rows
 *   U8 / U8_2D   src u8[L][...], dst u8 same shape (mut)         outermost dim
 *   NBODY->NBODY pos f32[N][4] COPY (mut), vel f32[N][4] COPY (mut)  (x,y,z,m)
 *   NBODY->ACCEL pos f32[N][4] COPY, acc f32[N][4] (mut)
 *   VEC1 / VEC2  x f32[L] (, y f32[L]); the MapReduce result is in the future
 *   TRAITS       out i64[L][2] (mut): (SIZE, OFFSET) of each element's partition
 *   CPLX         src f32[B][N][2], dst f32[B][N][2] (mut); N = 2^log2n of
 *                every FFT leaf (else MW_E_SHAPE_MISMATCH); partition B
 */
enum { MW_DT_U8 = 1, MW_DT_F32 = 2, MW_DT_F64 = 3, MW_DT_I64 = 4 };
enum { MW_PARTITION = 0, MW_COPY = 1 };
enum { MW_LOC_DEVICE = 0, MW_LOC_HOST = 1 };
typedef struct mw_arg {
    void* ptr;
    int32_t dtype;
    int32_t ndim;          /* 1..4 */
    int64_t shape[4];
    int32_t mode;          /* MW_PARTITION / MW_COPY */
    int32_t location;      /* MW_LOC_DEVICE / MW_LOC_HOST */
    int64_t local_offset;  /* PARTITION only */
    int64_t local_rows;    /* PARTITION only */
} mw_arg;

/* Enqueue one execution of `root` on the CUDA stream `stream` (cudaStream_t;
 * NULL = legacy default stream) and return a future.
 * Runs of one ctx are FIFO (first-come-first-served), also when
 * issued on different streams: each run (and graph replay) first waits on
 * the device for the end of the ctx's previous one.  Trees with
 * a while-loop synchronise the host every check_every executions; all others
 * return without host synchronisation (device args).  Collective when the
 * tree exchanges data between ranks (MapReduce, hysteresis, N-body).         */
mw_status mw_run(mw_ctx* ctx, const mw_node* root, const mw_arg* args, int32_t nargs,
                 void* stream, mw_future** out);
mw_status mw_future_wait(mw_future* f);                 /* async CUDA/NCCL errors here */
mw_status mw_future_query(mw_future* f, int32_t* done);
/* After wait: out[0] = MapReduce result (fp64), out[1] = its fp32 rounding,
 * out[2] = while-loop executions E (total over all while loops), out[3] = 1
 * if every while loop converged else 0.  n <= 4 values are written.         */
mw_status mw_future_result(mw_future* f, double* out, int32_t n);
/* Releases the handle without blocking: a run still in flight is retired and
 * its resources are reclaimed once it completes (by a later mw_run on the
 * same ctx, or at mw_ctx_destroy, which waits for retired runs).  The buffers
 * the run reads and writes must stay valid until it completes.             */
void mw_future_release(mw_future* f);

/* ------------------------------------------------------------------ graphs
 * A built SCT receives many execution requests over time.
 * mw_graph_capture records one run of `root` on `args` into a CUDA graph
 * (the partition under the current distribution is frozen into it); each
 * mw_graph_launch replays exactly that run on the same buffers with no host
 * work (for launch-bound trees and small partitions).  `stream` must not be
 * the legacy default stream.  MW_E_UNSUPPORTED for host-resident args and
 * for while-loops whose condition needs the host (multi-partition byte
 * stencil); the one-partition hysteresis loop runs on the device and is
 * capturable.  Timing events are not recorded inside graphs.               */
typedef struct mw_graph mw_graph;
mw_status mw_graph_capture(mw_ctx* ctx, const mw_node* root, const mw_arg* args, int32_t nargs,
                           void* stream, mw_graph** out);
/* Same, capturing `nsets` back-to-back runs of `root`, run k on
 * args[k*nargs .. k*nargs+nargs) (e.g. rotating buffer sets); one
 * mw_graph_launch then replays all of them in order.                       */
mw_status mw_graph_capture_many(mw_ctx* ctx, const mw_node* root, const mw_arg* args,
                                int32_t nargs, int32_t nsets, void* stream, mw_graph** out);
mw_status mw_graph_launch(mw_graph* g, void* stream);
/* Results of the most recent replay (same layout as mw_future_result); call
 * after the launch stream has synchronised.                                */
mw_status mw_graph_result(mw_graph* g, double* out, int32_t n);
mw_status mw_graph_kernels(const mw_graph* g, int64_t* kernels_per_replay);
mw_status mw_graph_destroy(mw_graph* g);

/* Host-staged runs (MW_LOC_HOST arguments, NEXT-1): by default a run's
 * uploads start after the work enqueued on its stream before the call (a
 * pinned host input may be produced by an asynchronous D2H on that stream).
 * on != 0 promises that every host input is complete when mw_run is called;
 * the uploads of a run then overlap the previous run's downloads (no start
 * barrier).  Default off.                                                    */
mw_status mw_ctx_set_staging_overlap(mw_ctx* ctx, int32_t on);
/* Run pipelining.  on != 0 promises that between runs of this ctx on a
 * stream no other work writes what a run reads (the runs' only data
 * dependencies are through their arguments).  A fused Map/Pipeline chain run
 * whose source the previous run did not write then issues its first loads
 * before the programmatic-dependent-launch wait, overlapping the previous
 * run's drain (consecutive runs over rotating buffers, e.g. a rank's small
 * share); its stores still follow the wait, so the stream order of every
 * write is kept.  Default off.                                              */
mw_status mw_ctx_set_run_pipelining(mw_ctx* ctx, int32_t on);
/* Monitoring (per-device execution times feed the load balancer)
 * is on by default: every run records CUDA events around each partition's
 * kernels (mw_last_timings, mw_kernel_stats, mw_rebalance).  Off: no events,
 * so back-to-back runs carry no timing work between them (mw_last_timings
 * and mw_rebalance then return MW_E_STATE).                                 */
mw_status mw_ctx_set_monitoring(mw_ctx* ctx, int32_t on);
/* ------------------------------------------------------------------ monitor / balance
 * Per-partition compute times of the last completed run (events placed
 * around each partition's kernels, before any collective wait),
 * for all P partitions (collective when nranks > 1: an all-gather), and the
 * run's wall time on this rank.  per_part_ms: n >= P floats.                */
mw_status mw_last_timings(mw_ctx* ctx, float* per_part_ms, int32_t n, float* wall_ms);
/* Partition lengths (outer units) of the last run, n >= P.                  */
mw_status mw_last_lengths(const mw_ctx* ctx, int64_t* per_part_len, int32_t n);

/* Kernel statistics.  While enabled (mw_stats_enable(ctx, 1) synchronises
 * the device and clears them), every partition's kernels of each class are
 * bracketed by CUDA events on the launching stream and kept; mw_kernel_stats
 * synchronises and returns the summed event-measured duration (ms) and the
 * number of kernel launches of that class since enabling.                   */
enum {
    MW_KC_SAXPY = 0, MW_KC_RGBA = 1, MW_KC_U8 = 2, MW_KC_STENCIL = 3, MW_KC_NBODY = 4,
    MW_KC_REDUCE = 5, MW_KC_TRAITS = 6, MW_KC_FFT = 7, MW_KC_COUNT = 8
};
mw_status mw_stats_enable(mw_ctx* ctx, int32_t on);
mw_status mw_kernel_stats(mw_ctx* ctx, int32_t kernel_class, double* total_ms, int64_t* launches);

enum { MW_BALANCE_PROPORTIONAL = 0, MW_BALANCE_ABS = 1 };
typedef struct mw_balance_params {
    double weight;    /* lbt history weight, default 2/3              */
    double max_dev;   /* balanced iff dev / c_factor >= max_dev, default 0.85 */
    double c_factor;  /* correction factor, default 1                 */
    double trigger;   /* lbt >= trigger starts balancing, default 0.95*/
    int32_t mode;     /* MW_BALANCE_PROPORTIONAL or MW_BALANCE_ABS (2 parts)  */
} mw_balance_params;
typedef struct mw_balance_state {
    double lbt;
    int32_t active;
    int32_t abs_last_dir;
    double abs_t;
    int32_t abs_count;
    int32_t pad;
    int64_t runs;
} mw_balance_state;
void mw_balance_defaults(mw_balance_params* p);
/* Pure host function: one monitoring step (P:613-638 lbt; P:649-667 ABS;
 * proportional = P:388's relative-performance rule with measured rates).
 * Algorithm: DESIGN.md R15-R17.  next: n fractions.                         */
mw_status mw_balance_step(const mw_balance_params* p, mw_balance_state* inout,
                          const float* per_part_ms, const int64_t* per_part_len,
                          const double* cur, int32_t n, double* next, int32_t* triggered);
/* Convenience (collective): last timings -> mw_balance_step -> set the new
 * distribution.  The ctx keeps the mw_balance_state.                        */
mw_status mw_rebalance(mw_ctx* ctx, const mw_balance_params* p, int32_t* triggered);
mw_status mw_get_balance_state(const mw_ctx* ctx, mw_balance_state* out);

/* Slowdown injector (the analogue of the paper's CPU-load generator,
 * P:1110-1113): partition `part` computes as on a device `factor` (>= 1;
 * 1 = off) times slower.  Idempotent work (the N-body step, RGBA chains
 * src -> dst) is repeated round(factor) times (time exactly proportional);
 * the other kernels launch on 1/factor of their usual grid (grid-stride
 * loops).  Results never change.                                           */
mw_status mw_ctx_set_slowdown(mw_ctx* ctx, int32_t part, float factor);

/* Tuning knobs: the B200 platform configuration of a profile (P:446-456
 * item (d)) — block/element shapes the profile builder (mw_autotune)
 * searches.  Every value gives bit-identical results (MW_TUNE_FFT_4STEP:
 * two FFT algorithms, both within the oracle's bound).  Defaults are the
 * measured best on B200 (MW_* environment variables override them).       */
enum {
    MW_TUNE_RGBA_TMA = 0,     /* fused RGBA chain: 0 LSU path, 1 = 16 KiB TMA ring, 2 stages
                                 for launches of >= 8 waves of chunks else 3 (default),
                                 2 = 8 KiB x 4, 3 = 8 KiB x 3, 4 = 4 KiB x 4, 5 = 32 KiB x 3,
                                 6 = 16 KiB x 6, 9 = 16 KiB x 2; warp-granular rings:
                                 7 = 4 KiB x 3 x 8 warps, 8 = 8 KiB x 2 x 6 warps         */
    MW_TUNE_RGBA_UNROLL = 1,  /* LSU path: 16-byte vectors per thread (2, 4, 8)            */
    MW_TUNE_HYST_PLANES = 2,  /* 1: one-partition hysteresis on bit planes; 0: byte stencil */
    MW_TUNE_HYST_T = 3,       /* executions per pass of the plane loop (4, 6, 8, 12)        */
    MW_TUNE_HYST_ROWS = 4,    /* register rows per plane tile (32, 40)                      */
    MW_TUNE_NBODY_SPLIT = 5,  /* 1: split packed/scalar FP32 across the FMA pipes           */
    MW_TUNE_U8_TMA = 6,       /* 1: TMA bulk-copy ring for contiguous u8 chains (volumes)   */
    MW_TUNE_HYST_FUSED = 7,   /* 1: several partitions of one rank run the whole plane loop in
                                 ONE cooperative kernel (in-kernel halo exchange, device loop
                                 condition); 0: one launch per partition and pass            */
    MW_TUNE_GRAPH_LANES = 8,  /* mw_graph_capture_many: runs of a scratch-free fused chain whose
                                 argument sets are pairwise independent (no write overlaps
                                 another set's buffers) are captured on up to this many
                                 parallel lanes (1, 2, 4); 1 = strictly serialized replays   */
    MW_TUNE_FFT_4STEP = 9,    /* pipeline(fft, ifft) at N = 65536 as a four-step FFT,
                                 16 x 4096 (column DFT-16s in registers, one 4096-point
                                 row per CTA) as 1 = ONE persistent dataflow launch (work
                                 items from an atomic ticket, the passes of a transform
                                 ordered by device readiness counters, the intermediate
                                 consumed from L2; default) or 4 = three launches;
                                 256 x 256 as 2 (dataflow launch) or 3 (three launches);
                                 0 = one thread-block cluster per transform (distributed
                                 shared memory).  1 and 4 are bit-identical, so are 2 and 3 */
    MW_TUNE_COUNT = 10
};
mw_status mw_ctx_set_tuning(mw_ctx* ctx, int32_t knob, int32_t value);
mw_status mw_ctx_get_tuning(const mw_ctx* ctx, int32_t knob, int32_t* value);

/* ------------------------------------------------------------------ profiles / Knowledge Base
 * NEXT-2 of SURVEY §8(f): the paper's Knowledge Base stores, per
 * (SCT id, workload), the best configuration found (profile items (a)-(f),
 * P:446-456): the tree's content hash, the global shape, the distribution
 * vector, the tuning knobs, the best time and the provenance.  Lookup
 * derives a configuration for an unseen workload by narrowing the scope
 * SCT -> workload -> dimensionality, nearest neighbour in
 * log2-size space (R22).  The file is plain text, one record per
 * line, rewritten by mw_kb_save / mw_kb_close.                             */
typedef struct mw_kb mw_kb;
enum { MW_PROV_BUILT = 0, MW_PROV_DERIVED = 1, MW_PROV_BALANCED = 2 };
enum { MW_KB_NONE = 0, MW_KB_EXACT = 1, MW_KB_SCT = 2, MW_KB_WORKLOAD = 3,
       MW_KB_DIMENSIONALITY = 4 };
mw_status mw_kb_open(const char* path /* NULL or "" = in memory */, mw_kb** out);
mw_status mw_kb_save(const mw_kb* kb);
mw_status mw_kb_close(mw_kb* kb);                      /* saves, then frees */
mw_status mw_kb_count(const mw_kb* kb, int32_t* n);
/* Keeps the better of an existing (SCT, workload) record and this one
 * (progressive refinement); derived records are always replaced. */
mw_status mw_kb_store(mw_kb* kb, const mw_node* root, const int64_t* dims, int32_t ndims,
                      const int32_t* tune /* MW_TUNE_COUNT */, const double* fractions,
                      int32_t nparts, double best_ms, int32_t provenance);
/* *scope = MW_KB_NONE when nothing applies (outputs untouched), else the
 * narrowing level that matched; fractions_out (nparts) gets the record's
 * distribution when its partition count matches, else uniform.             */
mw_status mw_kb_lookup(const mw_kb* kb, const mw_node* root, const int64_t* dims, int32_t ndims,
                       int32_t* tune_out, double* fractions_out, int32_t nparts, int32_t* scope);
/* Profile building (Alg. 1, over the B200 knobs): runs `root` on
 * `args` (collective like mw_run) warm-up + `reps` times per candidate
 * setting of the knobs that apply to its plan, keeps the fastest in the ctx,
 * stores it in `kb` (if not NULL, provenance BUILT) and returns it.
 * In-place arguments (Saxpy y, N-body state) are restored afterwards.        */
mw_status mw_autotune(mw_ctx* ctx, const mw_node* root, const mw_arg* args, int32_t nargs,
                      void* stream, int32_t reps, mw_kb* kb, int32_t* tune_out, double* best_ms);

/* The exact (SCT, workload) record: *found = 0/1, its provenance and time.  */
mw_status mw_kb_find(const mw_kb* kb, const mw_node* root, const int64_t* dims, int32_t ndims,
                     int32_t* found, int32_t* provenance, double* best_ms);

/* Heterogeneous devices (NEXT-4): partition `part` runs on a
 * device of class `cls` (>= 0) whose relative performance is rel_perf (> 0).
 * The distribution becomes proportional to the partitions' relative
 * performances (P:388's static rule).  Classes are the device types of the
 * profile builder's workload-distribution generator (Alg. 1).
 * On one B200 a class is realised with the slowdown injector (or MIG).     */
mw_status mw_ctx_set_device_class(mw_ctx* ctx, int32_t part, int32_t cls, double rel_perf);

/* Profile building, Alg. 1 over the B200 configuration space:
 * the knob dimensions that apply to the plan are iterated in nested loops,
 * most likely values first, and a value that does not improve on the
 * previous one discards the rest of its dimension; innermost, the
 * workload-distribution generator binary-searches the share of
 * device class A (partition 0's class) against the other classes, binding
 * half of the transferable share to the faster type per iteration
 * (transferableSize(n) = 1/2^n); every proposal runs warm-up + `executions`
 * times (mean, step 13; with several partitions per rank — virtual devices —
 * the time is the makespan, the longest partition's compute time of the last
 * execution, i.e. what concurrent devices would take); a result better than
 * the stored best is stored, and
 * an improvement below precision_ms ends the search direction (steps 14-17).
 * The best configuration is left in the ctx (tuning + distribution), stored
 * in kb (provenance BUILT) when kb != NULL and returned.  Collective like
 * mw_run; in-place arguments are restored afterwards.                      */
typedef struct mw_profile_params {
    int32_t executions;      /* runs per proposal (quality factor), default 3 */
    double precision_ms;     /* step 17 stop, default 0                        */
    int32_t max_dist_iters;  /* generator iterations (two device types), 10    */
} mw_profile_params;
void mw_profile_defaults(mw_profile_params* p);
mw_status mw_profile_build(mw_ctx* ctx, const mw_node* root, const mw_arg* args, int32_t nargs,
                           void* stream, const mw_profile_params* params, mw_kb* kb,
                           int32_t* tune_out /* MW_TUNE_COUNT or NULL */,
                           double* fractions_out /* n_parts or NULL */, int32_t nfrac,
                           double* best_ms, int32_t* runs);

/* Managed execution, the Fig. 5 decision process around mw_run:
 * a new (SCT, workload) — different from the previous managed run's — gets
 * its configuration (tuning + distribution) from the KB: the exact record or
 * one derived by scope narrowing; a recurrent one first persists
 * the previous run's attained time with the process that produced it
 * (provenance DERIVED / BALANCED / BUILT), then runs the monitor
 * (mw_rebalance with params->balance): when it triggers, the distribution is
 * adjusted, or — with build_profiles set and no BUILT record yet — the
 * profile is built from scratch (mw_profile_build, once per pair).
 * *action says which branch ran.  Needs monitoring on; collective.          */
enum {
    MW_MANAGED_NO_KNOWLEDGE = 0, /* new pair, KB empty for it: current configuration */
    MW_MANAGED_FROM_KB = 1,      /* new pair, exact KB record                         */
    MW_MANAGED_DERIVED = 2,      /* new pair, configuration derived by scope narrowing */
    MW_MANAGED_RECURRENT = 3,    /* recurrent pair, balanced: nothing changed          */
    MW_MANAGED_ADJUSTED = 4,     /* recurrent, unbalanced: distribution adjusted        */
    MW_MANAGED_BUILT = 5         /* recurrent, unbalanced: profile built from scratch   */
};
typedef struct mw_managed_params {
    mw_balance_params balance;
    int32_t build_profiles;      /* 0 (default): never build, only adjust */
    mw_profile_params profile;
} mw_managed_params;
void mw_managed_defaults(mw_managed_params* p);
mw_status mw_run_managed(mw_ctx* ctx, mw_kb* kb, const mw_managed_params* params,
                         const mw_node* root, const mw_arg* args, int32_t nargs, void* stream,
                         mw_future** out, int32_t* action);
/* Persist the last managed run's result now (otherwise done by the next
 * managed run).  Call after its future completed.                          */
mw_status mw_managed_flush(mw_ctx* ctx);

/* Number of kernels this library launched on the ctx since creation.        */
mw_status mw_ctx_launch_count(const mw_ctx* ctx, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* MARROW_H */
