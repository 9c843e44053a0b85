/* scratchpipe.h — C ABI of the B200-native ScratchPipe hot path.
 *
 * ScratchPipe (Kwon & Rhu, ISCA'22, arXiv 2205.04702; PAPER.md = the LaTeX
 * source, cited as P:<line>) keeps the full embedding tables in host memory
 * and, because the sparse IDs of upcoming mini-batches are known ahead of
 * time, plans a GPU scratchpad so that the Train stage always hits
 * (P:159-163).  This library is that scratchpad on one B200:
 *
 *   sp_plan     [Plan]  (Alg. 1): index ingest, dedup,
 *               Hit-Map probe, hit/miss, window-safe LRU victim selection
 *               (past window P:840-861, future window P:864-884, superset
 *               P:887-896), Hit-Map/Storage bookkeeping.
 *               [Collect]+[Exchange]+[Insert] run in the
 *               library's transfer engine: CPU threads gather the missed
 *               rows into a contiguous pinned slot, one bounded-grid kernel
 *               per batch moves them into the freed slots and writes the
 *               victims contiguously into pinned staging (zero-copy, TMA
 *               bulk copies), CPU threads scatter the staged victims into
 *               their host rows (no CUDA call on those threads).
 *   sp_forward  [Training] part 1: EmbeddingBag gather-reduce.
 *   sp_train    [Training] part 2: gradient duplication + coalescing
 *                and the SGD update in place in the scratchpad
 *               (P:713-715).
 *   sp_flush    end-of-run write-back of every (dirty) resident row.
 *
 * Everything on the path runs in this library's sm_100a kernels; the
 * caller supplies device memory for pooled outputs / gradients and a stream.
 *
 * Conventions
 * - All calls return sp_status; no exceptions, no exit(), no host aborts.
 * - Batch indices are laid out [T][N][L] (table, sample, lookup position),
 *   int64 by default (SP_FLAG_INDEX_I32 for int32), host memory by default
 *   (SP_FLAG_INDEX_DEVICE for a device pointer).
 * - pooled / pooled_grad are DEVICE pointers, fp32, layout [T][N][D],
 *   ordered on desc.stream like any CUDA library argument.
 * - Host tables: caller-owned, row-major fp32 [rows[t]][dim], pinned
 *   (cudaHostAlloc) or, with SP_FLAG_REGISTER_HOST, registered by the
 *   library for the context's lifetime.  They are NOT coherent between
 *   sp_create and sp_flush: resident rows are newer in HBM.
 * - Errors found on the device (SP_ERR_INDEX_RANGE, SP_ERR_CAPACITY) are
 *   latched in device memory and returned by the next call that observes
 *   them (at the latest sp_flush); sp_last_error_batch() then gives the
 *   (batch, table) where it happened.  After CAPACITY, INDEX_RANGE, CUDA
 *   errors the context is poisoned: only sp_error_string, sp_last_error_batch,
 *   sp_get_stats and sp_destroy remain valid.
 * - One context per GPU; a context is not thread-safe.
 *
 * Environment (read at sp_create; tuning experiments and diagnostics only,
 * the defaults are the measured best on B200):
 *   SP_CPU_GATHER=0|1     0: the transfer kernel pulls the missed rows from
 *                         their random host rows itself; 1: CPU threads gather
 *                         them into a contiguous pinned slot first (default:
 *                         all gathered when T*N*L*dim*4 <= 32 MB, i.e. few rows
 *                         per batch; above, the hybrid split with f = 0.5)
 *   SP_WRITEBACK=gpu|cpu  victims' write-back: gpu = the transfer kernel stores
 *                         each victim row straight into its host row (TMA bulk
 *                         store); cpu = staged contiguously, CPU threads scatter
 *   SP_GATHER_FRAC=f      hybrid: the CPU gathers the share f in (0,1) of each
 *                         batch's missed rows, the transfer kernel pulls the rest
 *                         at the same time (1: all gathered, 0: all pulled)
 *   SP_GATHER_DMA=1       with the CPU gather, copy the gathered slot to HBM by
 *                         copy-engine DMA before the transfer kernel (default 0)
 *   SP_PULL_CTAS=n        transfer-kernel grid (one-warp CTAs, default 16)
 *   SP_XFER_STREAMS=1     one transfer stream instead of two alternating ones
 *   SP_XFER_PRIO=1        transfer streams at the highest priority
 *   SP_PLAN_PRIO=0        plan stream / plan graphs at the default priority
 *   SP_CARVEOUT=pct       shared-memory carveout hint for every kernel
 *   SP_DIAG_SERIAL=1      every GPU stage on the caller's stream (no overlap)
 *   SP_DIAG=mask          1: the transfer kernel moves nothing, 2: the Train
 *                         kernels do nothing, 4: victims are not staged, 8 / 16:
 *                         k_bwd skips hot segments / chunk records --
 *                         RESULTS ARE WRONG (timing only)
 *   SP_NO_GRAPHS=1        sp_run_steps without CUDA-graph replay
 *   SP_PDL=0              no programmatic dependent launch of k_surrogate / k_bwd
 */
#ifndef SCRATCHPIPE_H
#define SCRATCHPIPE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_ABI_VERSION 4

typedef struct sp_ctx sp_ctx;

typedef enum {
    SP_OK = 0,
    SP_ERR_INVALID_ARG = 1,  /* bad descriptor / pointer / size                 */
    SP_ERR_CAPACITY = 2,     /* no evictable slot: the window working set does  */
                             /* not fit in Storage                */
    SP_ERR_INDEX_RANGE = 3,  /* a sparse ID < 0 or >= rows[t]                   */
    SP_ERR_STATE = 4,        /* call-order violation (see sp_forward/sp_train)  */
    SP_ERR_CUDA = 5,         /* CUDA runtime error                              */
    SP_ERR_NCCL = 6,         /* NCCL library missing or an NCCL call failed     */
    SP_ERR_OOM = 7           /* device or pinned allocation failed              */
} sp_status;

/* desc.flags */
#define SP_FLAG_REGISTER_HOST (1u << 0) /* cudaHostRegister the host tables      */
#define SP_FLAG_INDEX_I32     (1u << 1) /* batch indices are int32              */
#define SP_FLAG_INDEX_DEVICE  (1u << 2) /* batch indices are a device pointer   */
#define SP_FLAG_PROFILE       (1u << 3) /* CUDA events around every kernel ->   */
                                        /* per-kernel times in sp_get_stats     */
#define SP_FLAG_PADDING       (1u << 4) /* ragged bags: an ID of -1 is "no      */
                                        /* lookup" (a bag with none pools to    */
                                        /* zeros; reading R27); sp_plan_csr     */
#define SP_FLAG_BF16          (1u << 5) /* bf16 Storage (reading */
                                        /* R28): the scratchpad holds each row  */
                                        /* rounded to bf16 (nearest even) on    */
                                        /* fill and after every update; pooled, */
                                        /* gradients and host tables stay fp32  */
                                        /* (a write-back widens exactly).       */
                                        /* Requires dim % 8 == 0.               */

/* sp_create(tables, dim, slots, window) of the problem statement. */
typedef struct {
    int32_t num_tables;          /* T tables on THIS device (>= 1)                 */
    const int64_t *rows;         /* [T] rows per table, 1 <= rows[t] < 2^32 - 1    */
    float *const *host_tables;   /* [T] host pointers, rows[t] x dim fp32 each      */
    int32_t dim;                 /* D, multiple of 4, 4 <= D <= 1024                */
    const int64_t *slots;        /* [T] scratchpad rows per table (per-table        */
                                 /* pools: one cache manager per table)     */
    int32_t window;              /* w: past hold P = w, future hold F = w - 1;      */
                                 /* w = 3 is the paper's 3 past + current + 2       */
                                 /* future = six batches     */
    int32_t past, future;        /* >= 0 overrides P / F (requires F <= P + 1);     */
                                 /* -1 = derive from window                         */
    int32_t batch_size, pooling; /* N bags per table, L lookups per bag (fixed)     */
    int32_t device;              /* CUDA device ordinal                             */
    void *stream;                /* cudaStream_t for sp_forward / sp_train /        */
                                 /* sp_surrogate_grad (NULL = legacy default)       */
    uint32_t flags;              /* SP_FLAG_*                                       */
    int32_t log_factor;          /* LRU-log ring capacity per table =               */
                                 /* log_factor * slots[t] + 4*N*L (0 -> 32)         */
    int32_t host_threads;        /* CPU row-copy helpers per transfer-engine pool   */
                                 /* (gather, scatter); 0 -> from the node's cores:  */
                                 /* (ncpu - pools) / pools, pools = 2 * max(1,      */
                                 /* world) contexts' pools, clamped to [1, 6]       */
    int32_t policy;              /* replacement policy among the window-safe        */
                                 /* candidates: SP_POLICY_*           */
    uint32_t reserved;           /* must be 0                                       */
    uint64_t policy_seed;        /* SP_POLICY_RANDOM: seed of the victim draws      */
    /* Table-wise sharding over G GPUs (one cache manager per
     * table, "no further inter-GPU RAW hazards"), one context per GPU.  With
     * world > 1 the context owns num_tables of the num_tables_all global
     * tables and the library exchanges pooled rows / gradients with NCCL
     * (send/recv over NVLink, on desc.stream): sp_forward then writes the
     * batch-sharded [num_tables_all][N/G][D] layout a data-parallel MLP
     * consumes (rank r holds samples r*N/G .. (r+1)*N/G-1 of every table)
     * and sp_train takes its gradient in that layout.  world == 1: none of
     * these fields is read. */
    int32_t world;               /* G ranks (0 or 1: single GPU)                    */
    int32_t rank;                /* this context's rank                             */
    const void *nccl_id;         /* 128-byte ncclUniqueId from sp_nccl_unique_id on */
                                 /* one rank, the same bytes on every rank          */
    int32_t num_tables_all;      /* T_all                                           */
    int32_t reserved2;           /* must be 0                                       */
    const int32_t *table_owner;  /* [T_all] rank owning each global table           */
    const int32_t *table_ids;    /* [num_tables] global id of each local table,     */
                                 /* ascending; rows/slots/host_tables follow it     */
} sp_desc;

/* desc.policy (readings R8, R23-R25).  Every policy evicts only
 * candidates: slots whose row is outside the window B(b-P..b+F) and not pinned.
 *   LRU     ascending (last Plan that used the slot, resident ID)  [default]
 *   RANDOM  vacant slots lowest first, then draws s_i = H(seed, t, b, i) mod O
 *           over the O occupied slots, a candidate taken when first drawn
 *           (H: splitmix64 chain of seed ^ "RAND", t, b, i)
 *   LFU     ascending (use count saturating at 8, last use, resident ID); the
 *           use count is 1 at fill and +1 per Plan that hits the slot */
#define SP_POLICY_LRU    0
#define SP_POLICY_RANDOM 1
#define SP_POLICY_LFU    2

typedef enum {
    SP_K_PLAN = 0,      /* dedup + future probe + Plan (one launch per sp_plan)  */
    SP_K_TRANSFER = 1,  /* k_pullfill: victims staged to host, freed slots filled */
    SP_K_FORWARD = 2,   /* EmbeddingBag gather-reduce                             */
    SP_K_BACKWARD = 3,  /* duplicate-coalescing segmented reduce + fused SGD      */
    SP_K_SURROGATE = 4, /* harness MLP stand-in g = fmaf(gamma, pooled, delta)    */
    SP_K_FLUSH = 5,     /* write-back of all resident rows                        */
    SP_K_H2D = 6,       /* (unused: the transfer kernel pulls rows itself)        */
    SP_K_D2H = 7,       /* (unused: the transfer kernel stages victims itself)    */
    SP_K_COUNT = 8
} sp_kernel_kind;

typedef struct {
    int64_t pushed, planned, transferred, forwarded, trained;
    /* cumulative over planned batches, summed over tables (device counters,  */
    /* read with a plan-stream synchronisation)                               */
    int64_t uniques, hits, misses, evictions;
    int64_t h2d_index_bytes;        /* batch indices uploaded                  */
    int64_t h2d_row_bytes;          /* missed rows pulled from host tables     */
    int64_t d2h_row_bytes;          /* victim rows written back                */
    int64_t kernel_launches[SP_K_COUNT];
    double kernel_ms[SP_K_COUNT];   /* SP_FLAG_PROFILE only: summed CUDA-event */
                                    /* durations of completed launches         */
    int64_t kernel_timed[SP_K_COUNT];
    double host_gather_ms;          /* transfer engine: CPU time gathering missed */
    double host_scatter_ms;         /* rows / scattering victims (wall, summed)   */
    int64_t host_rows_gathered, host_rows_scattered;
    double wait_xfer_ms;            /* caller thread waiting for the transfer     */
    double wait_list_ms;            /* engine (forward / host-list ring reuse)    */
    int64_t graph_steps;            /* sp_run_steps steps replayed as CUDA graphs */
    double graph_step_host_ms;      /* caller-thread wall time spent issuing them */
    int32_t transfer_mode;          /* how missed rows reach HBM: SP_XFER_*        */
    int32_t engine_threads;         /* CPU threads of the transfer engine (workers */
                                    /* + row-copy helpers)                          */
    int32_t gpu_writeback;          /* 1: k_pullfill writes victims straight into  */
                                    /* their host rows (SP_WRITEBACK=gpu)           */
    int32_t backward_kernels;       /* kernels per backward launch (kernel_launches */
                                    /* counts launches of the stage): 2 = k_bwd_tile */
                                    /* + k_bwd_rows (two-phase), else 1             */
    double gather_share;            /* share of the missed rows the CPU gathers    */
} sp_stats;

/* sp_stats.transfer_mode (missed rows in); victims out: CPU scatter from
 * pinned staging, or with sp_stats.gpu_writeback TMA bulk stores from the
 * transfer kernel straight into the host rows */
#define SP_XFER_GPU_PULL   0  /* k_pullfill reads each missed row from its host row */
#define SP_XFER_CPU_GATHER 1  /* CPU threads gather into a contiguous pinned slot   */
#define SP_XFER_GATHER_DMA 2  /* CPU gather, then copy-engine DMA of the slot       */
#define SP_XFER_HYBRID     3  /* CPU gathers a share (gather_share) into the slot,  */
                              /* k_pullfill pulls the rest concurrently            */

int32_t sp_abi_version(void);

/* A fresh NCCL unique id (128 bytes into out) for sp_desc.nccl_id: created on
 * one rank and broadcast to the others by the caller.  SP_ERR_NCCL if the
 * NCCL library cannot be loaded. */
sp_status sp_nccl_unique_id(void *out);

/* Host-only layout of the sharded exchange (no GPU): for rank `rank` of
 * `world`, the sends of sp_forward's exchange as (peer, local table,
 * global table) triples in the order they are posted, and the receives as
 * (peer, global table) pairs; each message is one table's N/G contiguous
 * rows.  send[3*k..3*k+2], recv[2*k..2*k+1]; *nsend = T_local * world,
 * *nrecv = T_all.  sp_train's exchange is the mirror image. */
sp_status sp_shard_plan(int32_t world, int32_t rank, int32_t num_tables_all, const int32_t *table_owner,
                        int32_t *send, int64_t *nsend, int32_t *recv, int64_t *nrecv);

/* Host-table allocator: `bytes` of anonymous host memory backed by 2 MB
 * transparent huge pages where the OS allows (the CPU side of the transfer
 * engine gathers / scatters random rows), registered with CUDA as mapped +
 * portable.  Pass the pointer in desc.host_tables WITHOUT
 * SP_FLAG_REGISTER_HOST.  Free with sp_host_free.  Returns SP_ERR_OOM when
 * the pages cannot be mapped or pinned. */
sp_status sp_host_alloc(size_t bytes, void **out);

/* The same, with the pages placed on the host NUMA node closest to CUDA
 * device `device` (cudaDevAttrHostNumaId; mbind MPOL_PREFERRED before the
 * pages are first touched), so each GPU's tables sit behind its own memory
 * controllers on a multi-socket node ("pinned host rows, placed
 * NUMA-local to that GPU").  On a single-node host, or when the device
 * reports no NUMA id, it is sp_host_alloc.  *numa_node_out (nullable) gets
 * the node used, -1 for none. */
sp_status sp_host_alloc_near(size_t bytes, int32_t device, void **out, int32_t *numa_node_out);
sp_status sp_host_free(void *ptr, size_t bytes);

/* Create a context: validates the descriptor, allocates Storage
 * (sum slots x dim fp32), the Hit-Map, per-slot metadata, the LRU log and a
 * ring of per-batch buffers in HBM of desc.device; creates the plan and
 * transfer streams.  *out is NULL on failure. */
sp_status sp_create(const sp_desc *desc, sp_ctx **out);

/* Push the next mini-batch B(j) into the look-forward window.
 * batch_indices: [T][N][L] (int64 | int32; host | device per flags).  Host
 * indices are copied before return.  Device indices must stay unmodified
 * until sp_forward of that batch has returned; they are read on the plan
 * stream after all work previously enqueued on desc.stream.
 * One kernel launch dedups B(j) and, beside it, runs Plan(j - F - 1), whose
 * future window B(j - 1) was deduped by the previous call (when j > F).  Asynchronous: never waits for the GPU except
 * to recycle a pinned staging buffer.  Returns SP_ERR_STATE if the caller is
 * more than 16 batches ahead of sp_train. */
sp_status sp_plan(sp_ctx *c, const void *batch_indices);

/* Ragged mini-batch B(j) in CSR form (the EmbeddingBag "offsets" layout;
 * PAPER.md Fig. 2 P:257-263 has bags of 2 and 3 lookups): values int64 [nnz],
 * offsets int64 [T*N + 1], bag k = t*N + s holds values[offsets[k] ..
 * offsets[k+1]); offsets[0] == 0; every bag has at most desc.pooling lookups
 * (so tables may differ in pooling: per-table pooling is bags of different
 * sizes).  Host pointers, copied before return.  Requires SP_FLAG_PADDING:
 * the library expands the bags on the GPU (k_csr_pad) into the padded
 * [T][N][L] layout, -1 in the unused positions, and plans that.
 * SP_ERR_INVALID_ARG for malformed offsets or a bag longer than pooling. */
sp_status sp_plan_csr(sp_ctx *c, const int64_t *values, const int64_t *offsets);

/* Static partition (the paper's static top-N cache design
 * point P:472-495, reading R26): before the first sp_plan, load rows
 * ids[0..count) of table t (distinct, in range) into the table's LAST `count`
 * slots, in order, and map them in the Hit-Map.  Pinned rows always hit and
 * are never victims; the remaining slots are the scratchpad as usual.
 * SP_ERR_STATE after the first sp_plan or a second call for the table;
 * SP_ERR_INVALID_ARG for bad IDs or count > slots[t].  Synchronous. */
sp_status sp_pin_rows(sp_ctx *c, int32_t t, const int64_t *ids, int64_t count);

/* Same as sp_plan with SP_FLAG_INDEX_DEVICE for this one call: dev_indices
 * is a device pointer ([T][N][L], index width per SP_FLAG_INDEX_I32), read
 * on the plan stream after all work previously enqueued on desc.stream; it
 * must stay unmodified until sp_forward of that batch has returned. */
sp_status sp_plan_device(sp_ctx *c, const void *dev_indices);

/* No more batches: the future window truncates at the last batch (reading
 * R9); enqueues the Plans of the last F batches. */
sp_status sp_end_of_data(sp_ctx *c);

/* Forward of the oldest untrained batch b into pooled [T][N][D] (device).
 * Requires B(b + F + 1) to have been pushed, or sp_end_of_data.  sp_forward and
 * sp_train strictly alternate. */
sp_status sp_forward(sp_ctx *c, float *pooled);

/* Backward + SGD of the batch last passed to sp_forward: pooled_grad is
 * [T][N][D] on the device (one gradient per reduced embedding);
 * w <- fmaf(-lr, g_row, w) for every unique row, in place in Storage. */
sp_status sp_train(sp_ctx *c, const float *pooled_grad, float lr);

/* Harness utility (the MLP stand-in, not part of the method):
 * grad[i] = fmaf(gamma, pooled[i], delta) for i < count (count = 0 means
 * T*N*D; count must be a multiple of 4; device pointers, 16-byte aligned),
 * on desc.stream. */
sp_status sp_surrogate_grad(sp_ctx *c, const float *pooled, float *grad, int64_t count,
                            float gamma, float delta);

/* Enqueue (on desc.stream, after the work already enqueued there) an
 * asynchronous copy of batch b's Plan counters into host_out[T][4]
 * (U, hits, misses, evictions per table; host_out should be pinned).  Valid
 * while batch b's ring entry is live (until batch b + 16 is pushed). */
sp_status sp_copy_batch_stats(sp_ctx *c, int64_t b, uint32_t *host_out);

/* Turn per-kernel CUDA-event timing (SP_FLAG_PROFILE) on or off.  Turning it
 * on records a reference event on desc.stream and clears the timeline. */
sp_status sp_set_profiling(sp_ctx *c, int32_t on);

/* Timeline of profiled kernel launches since profiling was last turned on:
 * kind (sp_kernel_kind), batch index, start / end in ms relative to the
 * reference event (CUDA events, all streams).  Synchronises the device;
 * writes min(cap, *n) records. */
sp_status sp_get_timeline(sp_ctx *c, int32_t *kind, int64_t *batch, double *start_ms,
                          double *end_ms, int64_t cap, int64_t *n);

/* Harness driver loop (benchmarks, tests): runs `steps` training iterations
 * without returning to the caller, each exactly
 *   sp_plan_device(indices + j*stride) while the look-ahead is short (sp_end_of_data
 *   once the trace is exhausted and the next batch cannot be planned otherwise),
 *   sp_forward(pooled), sp_surrogate_grad(pooled, grad, 0, gamma, delta),
 *   sp_train(grad, lr)
 * The first call pushes F+P+1 batches ahead.  `indices` is a DEVICE array, or
 * a PINNED HOST array (cudaHostAlloc / registered; the plan kernel then reads
 * each batch over the host link, so its H2D is part of the step), of
 * `num_batches` batches [T][N][L] (index width per SP_FLAG_INDEX_I32) with
 * `stride` bytes between batches; batch j of the trace is pushed at most once
 * (the loop continues from the context's counters).  pooled / grad: device
 * [T][N][D].  When stats_out (pinned host, [steps][T][4]) is non-NULL, every
 * step's Plan counters are copied back (sp_copy_batch_stats).  Returns the
 * first error. */
sp_status sp_run_steps(sp_ctx *c, const void *indices, int64_t num_batches, int64_t stride,
                       int64_t steps, float *pooled, float *grad, float gamma, float delta,
                       float lr, uint32_t *stats_out);

/* Drain and write every resident row back to its host table; on return the
 * host tables are coherent.  Requires every pushed batch to be trained (call
 * sp_end_of_data first).  Synchronises the device. */
sp_status sp_flush(sp_ctx *c);

/* All-resident warm start, the paper's GPU-only design point (Table 1;
 * SURVEY §8(f) f3): with slots[t] == rows[t] for every table, copy every host
 * row into Storage (slot_base[t] + id) and map it in the Hit-Map before the
 * first sp_plan, so no batch ever misses.  SP_ERR_INVALID_ARG unless every
 * table is fully resident, SP_ERR_STATE after the first sp_plan.  Synchronous. */
sp_status sp_prefill(sp_ctx *c);

/* Free everything (unregisters host tables registered by the library). */
sp_status sp_destroy(sp_ctx *c);

/* Human-readable description of the last error (never NULL). */
const char *sp_error_string(const sp_ctx *c);
/* Batch / table of the latched device error (-1 if none or not device). */
sp_status sp_last_error_batch(const sp_ctx *c, int64_t *batch, int32_t *table);

/* Statistics (synchronises the plan stream to read device counters, and the
 * streams whose profiled kernel events are pending). */
sp_status sp_get_stats(sp_ctx *c, sp_stats *out);

/* ---- introspection for parity tests (synchronise the plan stream) ---- */
/* Plan record of batch b, table t, in the same format as the oracle's Part B:
 * counts[4] = U, hits, misses, evictions; for k < U (arrays of capacity N*L):
 * uniq[k] = k-th smallest unique ID, slot[k] = table-local Storage slot after
 * the Plan, hit[k] = 1/0, evicted[k] = ID previously in the victim slot of a
 * miss (-1 if vacant or a hit).  Valid while batch b's ring entry is live
 * (until batch b + 16 is pushed). */
sp_status sp_debug_plan(sp_ctx *c, int64_t b, int32_t t, int64_t *counts, int64_t *uniq,
                        int64_t *slot, int64_t *hit, int64_t *evicted);
/* Sorted resident IDs of table t as planned so far (Hit-Map view). */
sp_status sp_debug_resident(sp_ctx *c, int32_t t, int64_t *ids, int64_t cap, int64_t *n);
/* Per-slot view of table t: resident ID (-1 vacant), last_use (INT64_MIN if
 * never used).  Arrays of slots[t] entries. */
sp_status sp_debug_slots(sp_ctx *c, int32_t t, int64_t *resident, int64_t *last_use);
/* Copy Storage rows [first, first+count) of table t to host (synchronises). */
/* Stage timing on/off (default off): when on, the steady-state step graphs are
 * (re)captured with CUDA event records around k_push, k_fwd, k_surrogate and
 * k_bwd, and every transfer launch is bracketed by events (read with
 * sp_stage_times).  Off keeps the event nodes out of the graphs. */
sp_status sp_set_stage_timing(sp_ctx *c, int32_t on);

/* Stage durations of the LAST RING (16) steps, from CUDA events recorded on
 * the stages' own streams inside the steady-state step graphs (sp_run_steps)
 * and around every transfer launch: out_ms[5] = mean ms of {plan (k_push),
 * transfer (k_pullfill), forward, surrogate, backward}, n_out[5] = steps
 * averaged (0: stage never timed).  Synchronises the device. */
sp_status sp_stage_times(sp_ctx *c, double *out_ms, int32_t *n_out);

/* Raw stage-event timestamps of the same last RING steps: out_ms[16][8] = ms
 * of event k of ring residue r relative to the earliest plan-start event of
 * the window (k: 0/1 plan start/end, 2 forward start, 3 forward end =
 * surrogate start, 4 surrogate end, 5 backward end, 6/7 transfer start/end),
 * NaN where not recorded.  Lets the caller take the union of each stream's
 * busy intervals instead of summing spans.  Synchronises the device. */
sp_status sp_stage_events(sp_ctx *c, double *out_ms);

/* Span timing of the steady state as it runs (diagnostic).  on != 0: every
 * CTA of the five stage kernels (k_push Plan, the transfer kernel, k_fwd,
 * k_surrogate, k_bwd) stamps %globaltimer when it starts its work and when it
 * is done; the step graphs are recaptured with the stamp buffer (no event
 * nodes).  Turning it on clears the stamps.  sp_span_times then returns, per
 * kind k (0 plan, 1 transfer, 2 forward, 3 surrogate, 4 backward) and ring
 * slot r (batch % 16), out_ms[(k*16 + r)*2 + {0,1}] = the earliest CTA start
 * and latest CTA end of the last launch for that slot, in ms from the
 * earliest recorded start (NaN: not recorded).  Synchronises the device. */
sp_status sp_set_span_timing(sp_ctx *c, int32_t on);
sp_status sp_span_times(sp_ctx *c, double *out_ms);

/* k_push per-CTA wall time while profiling is on (sp_set_profiling / SP_FLAG_PROFILE),
 * from %globaltimer at CTA entry and exit.  out[18T+2+4096] (caller-owned host array):
 * out[t] = summed ns of the Plan CTA of table t, out[T+t] = summed ns of the
 * dedup CTA of table t, out[2T] / out[2T+1] = CTAs timed per role (summed
 * over tables), out[2T+2 + (role*T + t)*8 + k] = summed ns of phase k of that
 * CTA (role 0 Plan: P1..P6; role 1 dedup: D1, D2 sort, D2 unique, D3a, D3b);
 * then per launch q = j mod 1024 of the current profiling window: [q] first
 * CTA start, [1024+q] last CTA end (ns), [2048+q] slowest Plan CTA,
 * [3072+q] slowest dedup CTA (ns).
 * Synchronises the plan stream.  Diagnostics only. */
sp_status sp_debug_plan_profile(sp_ctx *c, uint64_t *out);

/* Storage rows [first, first+count) of table t's slots into out (fp32; with
 * SP_FLAG_BF16 the bf16 rows widened exactly).  Synchronises the device.
 * Diagnostics only. */
sp_status sp_debug_storage(sp_ctx *c, int32_t t, int64_t first, int64_t count, float *out);

#ifdef __cplusplus
}
#endif
#endif /* SCRATCHPIPE_H */
