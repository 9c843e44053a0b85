// sp_internal.cuh — device-side layout and kernel launch declarations of the
// B200-native ScratchPipe hot path.  Internal to libscratchpipe.so.
//
// Data layout in HBM (one context = the tables of one GPU):
//   hitmap   [sum_t R_t]      u32   Hit-Map as a direct-indexed
//                                   array: row_off[t]+id -> global slot or EMPTY
//   resident [S]              u32   table-local ID held by each slot (or EMPTY)
//   last_use [S]              i32   last Plan index that hit/filled the slot
//                                   (VACANT for never used): the LRU key and the
//                                   past-window hold
//   next_need[S]              i32   latest future batch that probed the slot
//                                   (RAW-4 future-window hold)
//   storage  [S][D]           f32   the Storage array
//   log_slot/log_stamp [C]    u32/i32  per-table LRU log ring (append-only,
//                                   lazily invalidated: valid iff
//                                   last_use[slot] == stamp)
//   ring of 16 per-batch buffers, per table region of n = N*L entries.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sp {

constexpr int RING = 16;                    // batches in flight (>= P+F+2)
constexpr uint32_t EMPTY = 0xFFFFFFFFu;     // empty Hit-Map entry / vacant slot
constexpr int32_t VACANT = INT32_MIN;       // last_use of a never-used slot
constexpr int32_t NEVER = INT32_MIN;        // next_need of a slot with no future use
constexpr int CH = 16;                      // occurrences per backward chunk
// hot-row segment record packing: occurrences of the segment (<= hs <= HOT_SEG_MAX)
// in the low HOT_LEN_BITS of .z, the row's segment count above them (< 2^22)
constexpr int HOT_LEN_BITS = 10;
constexpr uint32_t HOT_LEN_MASK = (1u << HOT_LEN_BITS) - 1u;
constexpr int HOT_SEG_MAX = 512;
constexpr long long HOT_NSEG_MAX = (1ll << (32 - HOT_LEN_BITS)) - 1;
#ifndef SP_PUSH_THREADS
#define SP_PUSH_THREADS 1024
#endif
constexpr int PUSH_THREADS = SP_PUSH_THREADS;  // one CTA per table and role (k_push)
#ifndef SP_PUSH_MIN_BLOCKS
#define SP_PUSH_MIN_BLOCKS (SP_PUSH_THREADS >= 1024 ? 1 : 2)  // resident k_push CTAs per SM
#endif
constexpr int SMEM_SORT_MAX = 8192;         // n handled by the shared-memory radix sort
constexpr unsigned long long NO_ERR = ~0ull;

// device error word: min over (batch << 24 | table << 8 | kind)
enum DevErr : unsigned { DERR_INDEX = 3, DERR_CAPACITY = 2 };
__host__ __device__ inline unsigned long long err_key(long long b, int t, unsigned kind) {
    return ((unsigned long long)b << 24) | ((unsigned long long)(t & 0xFFFF) << 8) | kind;
}

// Per-batch ring buffers, all with a per-table region.  Strides:
//   n  = N*L         (sorted_occ, sorted_uid, uniq_id, slot_u, hit, slot_of_occ,
//                     fill_*)
//   n1 = n + 1       (seg_off)
//   nc = n + n/CH + 1 (chunk_rec)
//   nh = n/hs + n/(CH+1) + 1 (hot_rec: a hot row has > CH occurrences and
//                     ceil(len/hs) <= len/hs + 1 segments)
// chunk_rec[c]: one unique row with <= CH occurrences, their bag indices inline
// (ascending occurrence order), so the backward pass needs one record load
// before the gradient rows.
// hot_rec[h] = {u -> slot, first sorted occurrence, occurrences | nseg << 10, k}:
// segment k of nseg of a row with more than CH occurrences (Zipf head), at most
// hs occurrences each.  One CTA of k_bwd folds a segment from sorted_occ; a
// row's segments meet through fp64 partials and hot_cnt (last arriver folds).
struct ChunkRec {
    uint32_t slot;      // unique index at dedup, Storage slot after Plan
    uint32_t meta;      // occurrences (1..CH)
    uint32_t bag[CH];   // table-local bag (sample) index of each occurrence
    uint32_t pad[2];
};
static_assert(sizeof(ChunkRec) == 80, "ChunkRec is 5 x 16 bytes");

struct BatchBufs {
    uint32_t *sorted_occ, *sorted_uid, *uniq_id, *seg_off, *U;
    ChunkRec *chunk_rec;
    uint32_t *nchunks;
    uint4 *hot_rec;
    uint32_t *nhot;
    uint32_t *hot_cnt;  // [T][nh] arrivals per hot row (at its segment-0 index)
    uint32_t *slot_u, *slot_of_occ;
    uint32_t *sorted_slot;  // [T][n] Storage slot of each sorted occurrence (k_bwd_tile)
    uint8_t *hit;
    uint32_t *fill_slot, *fill_row, *evict_row, *m;
    uint32_t *stats;  // [T][4] U, hits, misses, evictions
    uint32_t *work;   // [ceil(T/64)] k_bwd dynamic work counters (zeroed at dedup)
};

struct Geometry {
    int T, N, L, D;
    int n, n1, nc, nh;    // strides
    int hs;               // occurrences per hot-row segment (k_bwd: one CTA round)
    int pad;              // SP_FLAG_PADDING: slot_of_occ may hold EMPTY (no lookup)
    int bf16;             // SP_FLAG_BF16: Storage rows are bf16 (reading R28)
};

// A Storage row seen four columns at a time: fp32 rows hold a float4, bf16
// rows (SP_FLAG_BF16, reading R28) a uint2 of four bf16 (column 4c+0 in the
// low half of .x).  wid widens exactly; nar rounds to nearest even
// (cvt.rn.bf16x2.f32), the rounding the oracle's orc_bf16_round writes out.
template <bool BF>
struct SRow {
    using V = float4;
    static constexpr uint32_t bytes = 16;
    __device__ __forceinline__ static float4 wid(const V &v) { return v; }
    __device__ __forceinline__ static V nar(const float4 &x) { return x; }
};
template <>
struct SRow<true> {
    using V = uint2;
    static constexpr uint32_t bytes = 8;
    __device__ __forceinline__ static float4 wid(const V &v) {
        return make_float4(__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u),
                           __uint_as_float(v.y << 16), __uint_as_float(v.y & 0xffff0000u));
    }
    __device__ __forceinline__ static V nar(const float4 &x) {
        const __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.y), hi = __floats2bfloat162_rn(x.z, x.w);
        return make_uint2(*reinterpret_cast<const uint32_t *>(&lo), *reinterpret_cast<const uint32_t *>(&hi));
    }
};

// Missed-row lists of one Plan, mirrored into pinned host memory by the plan
// kernel for the CPU gather of the transfer engine (per ring slot, per table).
struct HostList {
    unsigned long long *ready;  // [T] = b + 1 once table t's list of batch b is complete
    uint32_t *m;                // [T] fills of table t
    uint32_t *row;              // [T][n] missed row of each fill
};

// replacement policies (R23-R25)
enum Policy : int { POL_LRU = 0, POL_RANDOM = 1, POL_LFU = 2 };
constexpr int LFU_FMAX = 8;                 // LFU use counts saturate here (R24)
constexpr int LOG_CLASSES_MAX = LFU_FMAX + 1;

struct PushArgs {
    Geometry g;
    int P, F;
    // policy: LRU walks one log per table; LFU one log per use-count class
    // (log ids t*log_classes + c); RANDOM keeps no log (log_classes = 0) and
    // draws from the occupied dynamic slots [slot_base, slot_base + nfill)
    int policy, log_classes;
    unsigned long long seed;            // RANDOM draw seed
    const uint32_t *pin_base;           // [T] first pinned (static) slot of table t
    const uint8_t *log_skip;            // [T] 1: dynamic slots >= rows (never evicts): no log appends
    uint32_t *nfill;                    // [T] RANDOM: dynamic slots filled so far
    unsigned long long *claim;          // [S] RANDOM: per-slot draw claims
    uint8_t *freq;                      // [S] LFU: use count (saturating)
    int pad;                            // SP_FLAG_PADDING: -1 is "no lookup"
    int bwd_recs;                       // build the record-based k_bwd's work lists (SP_BWD=rec)
    const unsigned long long *row_off;  // [T+1]
    const long long *rows;              // [T]
    const uint32_t *slot_base;          // [T+1]
    uint32_t *hitmap, *resident;
    int32_t *last_use, *next_need;
    uint32_t *log_slot;
    int32_t *log_stamp;
    const unsigned long long *log_base, *log_cap;
    unsigned long long *log_head, *log_tail;
    unsigned long long *err;
    unsigned long long *err_host;  // pinned mapped flag: set on any device error
    unsigned long long *cum;  // [4] cumulative U, hits, misses, evictions
    uint32_t *miss_u, *victims;  // plan scratch [T*n]
    uint32_t *sort_tmp;          // [4][T*n] scratch for the large-n radix path
    // CTAs [T, 2T): dedup of the new batch B(j)
    int has_new;
    long long j;
    const void *idx;
    int idx_i32;
    BatchBufs nb;
    // CTAs [0, T): Plan(b), whose future window ends at B(b+F) (already deduped)
    int do_plan;
    long long b;
    BatchBufs pb;
    int has_future;
    BatchBufs fb;
    HostList hl;                 // pinned mirror of Plan(b)'s missed rows (CPU gather)
    // graph replay: j is read from ctl[ctl_r] (b = j - F - 1, idx = idx + j*stride)
    // and ctl[(ctl_r + 1) % RING] = j + 1 is written for the next step
    long long *ctl;
    int ctl_r;
    long long idx_stride;
    // profiling (nullable): [0,T) plan-CTA ns, [T,2T) dedup-CTA ns summed over
    // launches, [2T] plan launches, [2T+1] dedup launches
    unsigned long long *prof;
    unsigned long long *span;  // span timing (nullable): Plan(b) at slot b % RING
};

constexpr int TCTR_GROUPS = 8;
constexpr int TCTR_STRIDE = (TCTR_GROUPS + 1) * 32;
struct TrainArgs {
    Geometry g;
    BatchBufs bb;
    float *storage;
    const float *grad;   // bwd
    float *pooled;       // fwd
    float lr;
    double *partial;     // [T][nh][D] fp64 partial sums of hot-row segments
    const unsigned long long *err;
    int diag;            // timing diagnostic (k_bwd): 8 = skip hot segments, 16 = skip chunk records
    // k_bwd_tile: the table's sorted occurrence list cut into tiles of `tr`
    // rows (ntiles per table); a row spanning tiles meets through fp64 pieces
    double *tpart;       // [T][ntiles][2][D] pieces (slot 0: the tile's first segment, 1: its last)
    uint32_t *seg_cnt;   // [T][n] arrivals per multi-tile row (self-resetting)
    uint32_t *grp_cnt;   // [T][ntiles][2] arrivals per group of 8 pieces (self-resetting)
    int tr, ntiles;
    // k_bwd_tile dynamic tiles (nullable: static round robin): [RING][2]
    // {claims, exits} per batch slot; a CTA's first two tiles are static
    // (blockIdx.x, + gridDim.x), later ones claimed, so a CTA that becomes
    // resident late (its SM shared with the transfer / plan kernels) takes
    // fewer tiles; the last CTA to exit resets the pair
    uint32_t *tctr;      // [RING][TCTR_STRIDE]: TCTR_GROUPS claim counters + the exit counter, 128 B apart
    uint32_t *fctr;      // k_fwd dynamic bag chunks (nullable: static grid stride), same layout
    // two-phase backward (default; SP_BWD_2P=0: one phase with last-arriver
    // counters): k_bwd_tile only writes the fp64 pieces of rows spanning
    // tiles, k_bwd_rows then folds each such row's pieces and applies SGD
    int tp2;
    int bwd2_small;      // k_bwd_rows: rows of up to this many pieces are folded by one warp (0: default)
    int bwd_tma;         // k_bwd_tile stages rows by TMA bulk copies (default) or LDGSTS (SP_BWD_TMA=0)
    int g4;              // (set by the launcher) TMA tile::gather4, 4 rows per request, via tensor maps
    long long srows;     // Storage rows (tensor map of Storage)
    unsigned long long *span;  // span timing (nullable), slot = batch % RING
    long long span_b;
};

struct XferArgs {
    Geometry g;
    BatchBufs bb;
    float *storage;
    float *const *host;       // [T] device-visible (mapped) host table pointers
    float *wb_stage;          // [sum m][D] victims: pinned host staging (device alias)
    unsigned long long *wb_dst;  // [sum m] host address of each staged victim's row (0: none)
    unsigned long long *staged_cnt;  // pinned: sum m of this batch (written before `staged`)
    int diag_nowb;                // timing diagnostic: skip the victims' staging stores
    int wb_direct;                // victims go straight to their host rows (no staging)
    uint32_t wb_q16;              // k_xfer_warp: share of the valid victims written back by the
                                  // kernel itself (65536 = all), the rest staged for the CPU
    const float *in_dev;          // device copy of the first in_dev_rows rows of in_stage
    uint32_t in_dev_rows;         //   (copy-engine DMA), or nullptr / 0
    uint32_t gfrac_q16;           // share of the fills gathered by the CPU (65536 = all)
    const unsigned long long *gwait;  // hybrid split: pinned "batches gathered" counter the
                                      // CTAs reading gathered rows wait on (else nullptr)
    const float *in_stage;        // [sum m][D] missed rows gathered by the CPU into pinned
                                  // host memory (contiguous, flattened over tables), or
                                  // nullptr: pull each row from its host table
    uint32_t *done_ctr;       // CTA arrivals (the last CTA resets it)
    unsigned long long *staged;  // pinned host flag: = b + 1 once every victim is staged
    long long b;
    const unsigned long long *err;
    unsigned long long *span;  // span timing (nullable)
};


struct FlushArgs {
    Geometry g;             // (g.bf16: Storage rows widened to fp32 on the way out)
    int S_total;
    const uint32_t *slot_base;
    const uint32_t *resident;
    const float *storage;
    float *const *host;
};

// fp32 rows -> bf16 Storage rows (SP_FLAG_BF16: sp_prefill, sp_pin_rows);
// src may be a mapped host pointer; count rows of D columns
cudaError_t launch_rows_to_bf16(const float *src, void *dst, long long count, int D, cudaStream_t s);

// Exclusive prefix of per-table counts[t0 .. t0+tcount) into s_pref[0..tcount]
// (tcount <= 64).  Loads are issued in parallel (one per thread) and scanned
// by warp 0: a serial loop of dependent-latency global loads would cost
// ~0.5 us per table.  Contains __syncthreads.
__device__ __forceinline__ void table_prefix(const uint32_t *counts, int t0, int tcount,
                                             uint32_t *s_pref) {
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        uint32_t a = lane < tcount ? counts[t0 + lane] : 0u;
        uint32_t b = lane + 32 < tcount ? counts[t0 + lane + 32] : 0u;
        uint32_t x = a, y = b;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t xa = __shfl_up_sync(0xffffffffu, x, o);
            uint32_t yb = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) { x += xa; y += yb; }
        }
        const uint32_t tot_a = __shfl_sync(0xffffffffu, x, 31);
        s_pref[lane] = x - a;
        s_pref[lane + 32] = tot_a + y - b;
        if (lane == 31) s_pref[64] = tot_a + y;
    }
    __syncthreads();
}

// Two prefixes at once (warp 0: counts_a -> pa, warp 1: counts_b -> pb), so
// their global loads are in flight together.  Contains __syncthreads.
__device__ __forceinline__ void table_prefix2(const uint32_t *counts_a, const uint32_t *counts_b, int t0,
                                              int tcount, uint32_t *pa, uint32_t *pb) {
    __syncthreads();
    if (threadIdx.x < 64) {
        const int lane = threadIdx.x & 31;
        const uint32_t *counts = threadIdx.x < 32 ? counts_a : counts_b;
        uint32_t *s_pref = threadIdx.x < 32 ? pa : pb;
        uint32_t a = lane < tcount ? counts[t0 + lane] : 0u;
        uint32_t b = lane + 32 < tcount ? counts[t0 + lane + 32] : 0u;
        uint32_t x = a, y = b;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t xa = __shfl_up_sync(0xffffffffu, x, o);
            uint32_t yb = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) { x += xa; y += yb; }
        }
        const uint32_t tot_a = __shfl_sync(0xffffffffu, x, 31);
        s_pref[lane] = x - a;
        s_pref[lane + 32] = tot_a + y - b;
        if (lane == 31) s_pref[64] = tot_a + y;
    }
    __syncthreads();
}

// Table of a flattened work item: the tl with s_pref[tl] <= item < s_pref[tl+1]
// (binary search; empty tables have equal prefixes and are skipped).
__device__ __forceinline__ int find_table(const uint32_t *s_pref, int tcount, uint32_t item) {
    int lo = 0, hi = tcount;  // invariant: s_pref[lo] <= item < s_pref[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_pref[mid] <= item) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Span timing (sp_set_span_timing): every CTA of the five stage kernels
// stamps %globaltimer when it starts its work and when it is done, into
// span[kind][ring slot][cta][start, end]; the host takes min / max per
// (kind, slot).  No atomics, no events in the graphs: the steady state is
// timed as it runs (bench.py's per-stage durations and overlap).
enum SpanKind : int { SPK_PLAN = 0, SPK_XFER = 1, SPK_FWD = 2, SPK_SURR = 3, SPK_BWD = 4, SPAN_KINDS = 5 };
constexpr int SPAN_MAXCTA = 8192;
constexpr int SPAN_BWD2_OFF = 7168;  // k_bwd_rows (the backward's second phase) stamps CTAs from here
__device__ __forceinline__ unsigned long long *span_base(unsigned long long *span, int kind, long long b) {
    return span ? span + (((size_t)kind * RING + (size_t)(b % RING)) * SPAN_MAXCTA) * 2 : nullptr;
}
__device__ __forceinline__ void span_mark(unsigned long long *base, int which, unsigned off = 0) {
    if (base && threadIdx.x == 0 && off + blockIdx.x < (unsigned)SPAN_MAXCTA) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        base[(size_t)(off + blockIdx.x) * 2 + which] = t;
    }
}

// launchers (return cudaGetLastError())
cudaError_t launch_push(const PushArgs &a, cudaStream_t s);
cudaError_t launch_forward(const TrainArgs &a, cudaStream_t s);
cudaError_t launch_backward(const TrainArgs &a, cudaStream_t s);
int backward_hot_segment(int D);
int backward_tile_rows(int D);   // k_bwd_tile rows per tile
bool backward_tiled();           // k_bwd_tile (default) vs the record-based k_bwd (SP_BWD=rec)
cudaError_t launch_surrogate(const float *pooled, float *grad, long long count, float gamma,
                             float delta, cudaStream_t s, unsigned long long *span = nullptr, long long span_b = 0);
cudaError_t launch_pullfill(const XferArgs &a, int ctas, cudaStream_t s);
cudaError_t launch_xfer_warp(const XferArgs &a, int ctas, cudaStream_t s);
cudaError_t launch_flush(const FlushArgs &a, cudaStream_t s);
cudaError_t launch_prefill_map(const uint32_t *slot_base, const unsigned long long *row_off, int T,
                               long long S_total, uint32_t *resident, uint32_t *hitmap, cudaStream_t s);
cudaError_t launch_log_init(const uint32_t *slot_base, const unsigned long long *log_base0, int T, long long S_total,
                            uint32_t *log_slot, int32_t *log_stamp, cudaStream_t s);
cudaError_t launch_csr_pad(const long long *values, const long long *offsets, long long nbags, int L, void *out,
                           int out_i32, cudaStream_t s);
size_t push_smem_bytes(int n);
// shared-memory carveout (percent) requested for every kernel of the library,
// -1 = driver default; set once at sp_create (SP_CARVEOUT) so consecutive
// kernels on an SM do not force an L1/shared reconfiguration
extern int g_carveout;
// Programmatic dependent launch for k_surrogate and k_bwd (SP_PDL, default on):
// each may be launched while its predecessor on the stream drains, runs the
// prologue that reads no predecessor output, then griddepcontrol.wait
extern int g_pdl;
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <typename K>
inline void apply_carveout(K kernel) {
    if (g_carveout >= 0) cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, g_carveout);
}
cudaError_t configure_push_kernel();
cudaError_t configure_xfer_kernels();
cudaError_t configure_train_kernels();
int device_sms();  // SM count of the current device (cached per device)

}  // namespace sp
