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
#include <cuda_runtime.h>
#include <stdint.h>

namespace sp {

constexpr int RING = 16;                    // batches in flight (>= P+F+2)
constexpr uint32_t EMPTY = 0xFFFFFFFFu;     // empty Hit-Map entry / vacant slot
constexpr int32_t VACANT = INT32_MIN;       // last_use of a never-used slot
constexpr int32_t NEVER = INT32_MIN;        // next_need of a slot with no future use
constexpr int CH = 32;                      // occurrences per backward chunk
constexpr int PUSH_THREADS = 512;
constexpr int SMEM_SORT_MAX = 16384;        // n_pad handled by the smem bitonic path
constexpr unsigned long long NO_ERR = ~0ull;

// device error word: min over (batch << 24 | table << 8 | kind)
enum DevErr : unsigned { DERR_INDEX = 3, DERR_CAPACITY = 2 };
__host__ __device__ inline unsigned long long err_key(long long b, int t, unsigned kind) {
    return ((unsigned long long)b << 24) | ((unsigned long long)(t & 0xFFFF) << 8) | kind;
}

// Per-batch ring buffers, all with a per-table region.  Strides:
//   n  = N*L         (sorted_occ, sorted_uid, uniq_id, slot_u, hit, slot_of_occ,
//                     fill_*, chunk_first)
//   n1 = n + 1       (seg_off)
//   nc = n + n/CH + 1 (chunk_u)
struct BatchBufs {
    uint32_t *sorted_occ, *sorted_uid, *uniq_id, *seg_off, *U;
    uint32_t *chunk_u, *chunk_first, *nchunks;
    uint32_t *slot_u, *slot_of_occ;
    uint8_t *hit;
    uint32_t *fill_slot, *fill_row, *evict_row, *m;
    uint32_t *stats;  // [T][4] U, hits, misses, evictions
};

struct Geometry {
    int T, N, L, D;
    int n, n1, nc;        // strides
};

struct PushArgs {
    Geometry g;
    int n_pad, P, F;
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
    unsigned long long *cum;  // [4] cumulative U, hits, misses, evictions
    uint32_t *miss_u, *victims;  // plan scratch [T*n]
    uint64_t *sort_tmp;          // [T*n] x2 scratch for the large-n radix path
    // new batch j (dedup + future probe)
    int has_new;
    long long j;
    const void *idx;
    int idx_i32;
    BatchBufs nb;
    // Plan(b)
    int do_plan;
    long long b;
    BatchBufs pb;
};

struct TrainArgs {
    Geometry g;
    BatchBufs bb;
    float *storage;
    const float *grad;   // bwd
    float *pooled;       // fwd
    float lr;
    double *partial;     // [T][nc][D]
    uint32_t *cnt;       // [T][n]
    const unsigned long long *err;
};

struct XferArgs {
    Geometry g;
    BatchBufs bb;
    float *storage;
    float *const *host;  // [T] device-visible host table pointers
    const unsigned long long *err;
};

struct FlushArgs {
    Geometry g;
    int S_total;
    const uint32_t *slot_base;
    const uint32_t *resident;
    const float *storage;
    float *const *host;
};

// launchers (return cudaGetLastError())
cudaError_t launch_push(const PushArgs &a, cudaStream_t s);
cudaError_t launch_forward(const TrainArgs &a, cudaStream_t s);
cudaError_t launch_backward(const TrainArgs &a, cudaStream_t s);
cudaError_t launch_surrogate(const float *pooled, float *grad, long long count, float gamma,
                             float delta, cudaStream_t s);
cudaError_t launch_transfer(const XferArgs &a, int max_ctas, cudaStream_t s);
cudaError_t launch_flush(const FlushArgs &a, cudaStream_t s);
size_t push_smem_bytes(int n_pad);
cudaError_t configure_push_kernel();

}  // namespace sp
