// runtime.cu — host runtime behind include/scratchpipe.h.
//
// Pipeline schedule: PAPER.md Fig. 8 re-expressed with CUDA
// streams, events and a native transfer-engine thread instead of lock-step
// cycles:
//
//   plan stream     push(j): [H2D of B(j)] -> k_push: dedup B(j) beside
//                   Plan(b = j-F-1) -> record ev_plan[b]
//   transfer streams (two, alternating batches) Transfer(b) once
//                   Train(b-P-1) is enqueued (past window): waits
//                   ev_plan[b], ev_train[b-P-1] and, on the GPU, for the
//                   pinned counter "scattered >= b-F" (RAW-4: the
//                   CPU write-back of batch b-F-1 has landed) -> k_pullfill
//                   ([Collect] + [Exchange]: missed rows pulled into the freed
//                   slots, victims written to pinned staging with their host
//                   addresses; the last CTA raises h_staged[b]) -> ev_xfer[b]
//   transfer engine (scatter thread + row-copy helpers, no CUDA calls): for
//                   b in order, once h_staged[b] is up, CPU scatter of the
//                   staged victims into the host tables ([Insert]), then
//                   scattered = b+1
//   compute stream  forward(b) waits ev_xfer[b]; train(b) -> record ev_train[b]
//
// No host synchronisation on the caller's thread in the steady state.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <immintrin.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/scratchpipe.h"
#include "sp_internal.cuh"

using namespace sp;

namespace {

struct ProfEv {
    int kind;
    long long batch;
    cudaEvent_t a, b;
};

struct TimelineRec {
    int kind;
    long long batch;
    double start_ms, end_ms;  // relative to the profiling reference event
};

// Fork-join pool of spinning threads copying rows between host tables and
// pinned staging (the CPU side of Collect / Insert).
struct RowPool {
    std::vector<std::thread> th;
    std::atomic<uint64_t> gen{0};
    std::atomic<long> next{0};
    std::atomic<int> done{0};
    std::atomic<bool> stop{false};
    const float *const *src = nullptr;
    float *const *dst = nullptr;
    long n = 0;
    size_t bytes = 0;

    static constexpr long CHUNK = 16;

    void run_chunks() {
        for (;;) {
            const long i0 = next.fetch_add(CHUNK, std::memory_order_relaxed);
            if (i0 >= n) break;
            const long i1 = std::min(n, i0 + CHUNK);
            // all source lines of the chunk in flight first (random host rows:
            // memory-level parallelism, not bandwidth, bounds a core here)
            for (long i = i0; i < i1; i++) {
                const char *p = reinterpret_cast<const char *>(src[i]);
                for (size_t o = 0; o < bytes; o += 64) __builtin_prefetch(p + o, 0, 2);
                __builtin_prefetch(dst[i], 1, 2);  // the destination's translation, walked early
            }
            // non-temporal stores: a random destination row costs no
            // read-for-ownership, and staging never pollutes the caches
            for (long i = i0; i < i1; i++) {
                const uintptr_t a = reinterpret_cast<uintptr_t>(src[i]) | reinterpret_cast<uintptr_t>(dst[i]);
                if ((a & 15) == 0 && (bytes & 15) == 0) {
                    const __m128i *sp = reinterpret_cast<const __m128i *>(src[i]);
                    __m128i *dp = reinterpret_cast<__m128i *>(dst[i]);
                    for (size_t q = 0; q < bytes / 16; q++) _mm_stream_si128(dp + q, _mm_load_si128(sp + q));
                } else {
                    std::memcpy(dst[i], src[i], bytes);
                }
            }
            _mm_sfence();
        }
    }

    void helper() {
        uint64_t seen = 0;
        int idle = 0;
        while (!stop.load(std::memory_order_relaxed)) {
            const uint64_t g = gen.load(std::memory_order_acquire);
            if (g == seen) {
                if (++idle > 4096) std::this_thread::yield();
                else _mm_pause();
                continue;
            }
            idle = 0;
            seen = g;
            run_chunks();
            done.fetch_add(1, std::memory_order_acq_rel);
        }
    }

    void start(int nthreads) {
        for (int i = 0; i < nthreads; i++) th.emplace_back([this] { helper(); });
    }

    std::mutex job_mu;  // one copy job at a time (a pool shared by the gather and scatter threads)

    void copy(const float *const *s, float *const *d, long count, size_t row_bytes) {
        if (count <= 0) return;
        std::lock_guard<std::mutex> lk(job_mu);
        src = s;
        dst = d;
        n = count;
        bytes = row_bytes;
        next.store(0, std::memory_order_relaxed);
        done.store(0, std::memory_order_relaxed);
        gen.fetch_add(1, std::memory_order_acq_rel);
        run_chunks();
        while (done.load(std::memory_order_acquire) < (int)th.size()) _mm_pause();
    }

    void shutdown() {
        stop = true;
        for (auto &t : th) t.join();
        th.clear();
    }
};


// ---- NCCL, loaded at run time (libnccl.so.2: the copy torch already loaded
// if any, so a comm created here and torch's share one library)
struct NcclApi {
    typedef int (*init_rank_t)(void **, int, std::array<char, 128>, int);
    typedef int (*uid_t)(std::array<char, 128> *);
    typedef int (*p2p_t)(const void *, size_t, int, int, void *, cudaStream_t);
    typedef int (*recv_t)(void *, size_t, int, int, void *, cudaStream_t);
    typedef int (*void_t)();
    typedef int (*destroy_t)(void *);
    typedef const char *(*err_t)(int);
    init_rank_t init_rank = nullptr;
    uid_t unique_id = nullptr;
    p2p_t send = nullptr;
    recv_t recv = nullptr;
    void_t group_start = nullptr, group_end = nullptr;
    destroy_t destroy = nullptr;
    err_t err = nullptr;
    bool ok = false;
};

NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        api.init_rank = reinterpret_cast<NcclApi::init_rank_t>(dlsym(h, "ncclCommInitRank"));
        api.unique_id = reinterpret_cast<NcclApi::uid_t>(dlsym(h, "ncclGetUniqueId"));
        api.send = reinterpret_cast<NcclApi::p2p_t>(dlsym(h, "ncclSend"));
        api.recv = reinterpret_cast<NcclApi::recv_t>(dlsym(h, "ncclRecv"));
        api.group_start = reinterpret_cast<NcclApi::void_t>(dlsym(h, "ncclGroupStart"));
        api.group_end = reinterpret_cast<NcclApi::void_t>(dlsym(h, "ncclGroupEnd"));
        api.destroy = reinterpret_cast<NcclApi::destroy_t>(dlsym(h, "ncclCommDestroy"));
        api.err = reinterpret_cast<NcclApi::err_t>(dlsym(h, "ncclGetErrorString"));
        api.ok = api.init_rank && api.unique_id && api.send && api.recv && api.group_start && api.group_end &&
                 api.destroy && api.err;
    });
    return api;
}
constexpr int NCCL_FLOAT32 = 7;

// The sharded exchange's message list (host logic, sp_shard_plan): sends in
// (peer, local table) order, receives in (peer, global table) order, one
// message = one table's N/G rows.
void shard_plan(int world, int rank, int T_all, const int32_t *owner, std::vector<std::array<int, 3>> &send,
                std::vector<std::array<int, 2>> &recv) {
    send.clear();
    recv.clear();
    std::vector<int> local;
    for (int t = 0; t < T_all; t++)
        if (owner[t] == rank) local.push_back(t);
    for (int g = 0; g < world; g++) {
        for (int k = 0; k < (int)local.size(); k++) send.push_back({g, k, local[k]});
        for (int t = 0; t < T_all; t++)
            if (owner[t] == g) recv.push_back({g, t});
    }
}

}  // namespace

struct sp_ctx {
    // configuration
    int T = 0, D = 0, N = 0, L = 0, n = 0, P = 0, F = 0;
    int device = 0;
    uint32_t flags = 0;
    std::vector<long long> rows, slots;
    std::vector<float *> host;
    std::vector<unsigned long long> row_off;  // [T+1]
    std::vector<uint32_t> slot_base;          // [T+1]
    long long S_total = 0;
    unsigned long long hit_total = 0;
    bool registered = false;
    Geometry g{};
    cudaStream_t compute = nullptr, plan_s = nullptr, xfer_s = nullptr;
    // Transfer(b) runs on xfer_s if b is even, xfer_s2 if odd: consecutive
    // transfers touch disjoint slots and host rows (a victim of Plan(b+1) has
    // last_use <= b-P, a row evicted at Plan(b) is not in B(b+1..b+F)), and
    // every real dependency is an explicit wait (Plan, Train(b-P-1), scatter)
    cudaStream_t xfer_s2 = nullptr;
    cudaStream_t own_plan_s = nullptr, own_xfer_s = nullptr, own_xfer_s2 = nullptr;  // created here
    // device memory
    std::vector<void *> allocs;
    unsigned long long *d_row_off = nullptr;
    long long *d_rows = nullptr;
    uint32_t *d_slot_base = nullptr;
    uint32_t *d_hitmap = nullptr, *d_resident = nullptr;
    int32_t *d_last_use = nullptr, *d_next_need = nullptr;
    float *d_storage = nullptr;
    uint32_t *d_log_slot = nullptr;
    int32_t *d_log_stamp = nullptr;
    unsigned long long *d_log_base = nullptr, *d_log_cap = nullptr, *d_log_head = nullptr,
                       *d_log_tail = nullptr;  // [T * log_classes]
    // replacement policy (sp_desc.policy) and its per-slot / per-table state
    int policy = 0, log_classes = 1;
    unsigned long long policy_seed = 0;
    uint32_t *d_pin_base = nullptr;           // [T] first pinned slot (slot_base[t+1]: none)
    uint8_t *d_log_skip = nullptr;            // [T] dynamic slots >= unpinned rows: no log appends
    std::vector<uint8_t> log_skip;
    std::vector<uint32_t> pin_base;
    std::vector<bool> pinned_t;
    uint32_t *d_nfill = nullptr;              // [T] RANDOM: dynamic slots filled so far
    unsigned long long *d_claim = nullptr;    // [S] RANDOM: draw claims
    uint8_t *d_freq = nullptr;                // [S] LFU: use counts
    // ragged bags in CSR form (sp_plan_csr): pinned host staging + device copies per ring slot
    int64_t *h_csr = nullptr;                 // pinned [RING][T*n + T*N + 1]
    int64_t *d_csr = nullptr;                 // device [RING][T*n + T*N + 1]
    unsigned long long *d_err = nullptr, *d_cum = nullptr;
    unsigned long long *d_pprof = nullptr;  // k_push per-CTA timing [2T+2] (profiling only)
    uint32_t *d_miss_u = nullptr, *d_victims = nullptr;
    uint32_t *d_sort_tmp = nullptr;
    double *d_partial = nullptr;  // [T][nh][D] hot-row segment partials (k_bwd)
    // k_bwd_tile: pieces of rows spanning tiles, self-resetting arrival counters
    double *d_tpart = nullptr;    // [T][ntiles][2][D]
    uint32_t *d_seg_cnt = nullptr, *d_grp_cnt = nullptr;  // [T][n], [T][ntiles][2]
    int bwd_tr = 0, bwd_ntiles = 0;
    uint32_t *d_tctr = nullptr;   // [RING][TCTR_STRIDE] k_bwd_tile tile claims / exits per batch slot
    bool bwd_dyn = true;
    bool bwd_2p = true;
    int bwd2_small = 0;           // SP_BWD2_SMALL: k_bwd_rows one-warp threshold (A/B)
    uint32_t *d_fctr = nullptr;   // [RING][TCTR_STRIDE] k_fwd bag-chunk claims / exits per batch slot
    bool fwd_dyn = true;          // k_fwd claims bag chunks dynamically (SP_FWD_DYN=0: static grid stride)           // two-phase backward (SP_BWD_2P=0: last-arriver counters in k_bwd_tile)          // k_bwd_tile claims tiles dynamically (SP_BWD_DYN=0: static round robin)
    int bwd_tma = 1;  // k_bwd_tile stages rows with TMA bulk copies; SP_BWD_TMA=0: LDGSTS (A/B, slower)
    float **d_host = nullptr;
    std::vector<float *> host_dev;  // [T] device-visible (mapped) host table pointers
    void *d_idx[RING] = {};
    BatchBufs ring[RING];
    // victim staging: XSR slots of sum(m) rows (<= T*n) in pinned host memory,
    // written by k_pullfill (contiguous rows over the host link); the kernel's
    // last CTA sets h_staged[b % RING] = b + 1 for the scatter thread
    int XSR = 4;
    float *h_wb = nullptr;                     // pinned mapped [XSR][T*n][D]
    float *hd_wb = nullptr;                    // its device alias
    unsigned long long *h_staged = nullptr;    // pinned mapped [RING]
    unsigned long long *hd_staged = nullptr;   // device alias
    unsigned long long *h_wbdst = nullptr;     // pinned mapped [XSR][T*n]: host row of each staged victim
    unsigned long long *hd_wbdst = nullptr;    // device alias
    unsigned long long *h_scnt = nullptr;      // pinned mapped [RING]: staged items of the batch
    unsigned long long *hd_scnt = nullptr;     // device alias
    uint32_t *d_xdone = nullptr;               // [RING] k_pullfill CTA arrival counters
    // GPU write-back (SP_WRITEBACK=gpu): k_pullfill stores each victim row
    // straight into its host row (TMA bulk store over the link); no staging,
    // no scatter thread; RAW-4 is then an event wait on Transfer(b-F-1)
    bool gpu_wb = false;
    unsigned long long *h_scat = nullptr;      // pinned mapped: batches scattered
    unsigned long long *d_scat = nullptr;      // its device alias (stream wait-value)
    int pull_ctas = 16;  // k_pullfill grid (one warp per CTA); SP_PULL_CTAS overrides
    // transfer kernel: k_pullfill (TMA bulk copies from 16 one-warp CTAs,
    // default) or k_xfer_warp (plain loads from ~1,200 warps, SP_XFER=warp:
    // measured slower in the pipeline, its sysmem loads slow the Train
    // kernels 1.3-1.8x; profiles/r02_xs1_sweep.txt)
    bool xfer_warp = false;
    int xfer_ctas = 0;          // k_xfer_warp grid (0: 2 x SMs); SP_XFER_CTAS overrides
    uint32_t wb_q16 = 0;        // k_xfer_warp: victims written back by the GPU (SP_WB_GPU_FRAC)
    // timing diagnostics (SP_DIAG bit mask; results are then WRONG): 1 = the
    // transfer kernel moves nothing, 2 = the Train kernels do nothing, 4 = the
    // transfer kernel pulls but does not stage the victims; k_bwd_tile: 32 =
    // every row through the fp64 fold, 64 = no fold, 128 = no staging
    int diag = 0;
    long long xfer_enq = 0;                    // transfers enqueued (caller's thread)
    // pinned index staging
    void *h_stage = nullptr;
    unsigned long long *h_err = nullptr;      // exact device error key (sync copies)
    unsigned long long *h_errflag = nullptr;  // pinned mapped: kernels set it on error
    unsigned long long *d_errflag = nullptr;  // device alias of h_errflag
    size_t idx_bytes = 0;
    // events
    cudaEvent_t ev_plan[RING] = {}, ev_xfer[RING] = {}, ev_train[RING] = {},
                ev_h2d[RING] = {};
    cudaEvent_t ev_user = nullptr;
    // timing events of the steady state (sp_stage_times): recorded by the step
    // graphs of residue r around k_push / k_fwd / k_surrogate / k_bwd
    // ([0..1] plan, [2..5] forward start, forward end, surrogate end, backward
    // end) and around every transfer ([6..7]); the last RING steps are timed
    cudaEvent_t sev[RING][8] = {};
    bool sev_used[RING][2] = {};
    bool stage_timing = false;  // sp_set_stage_timing: record sev in new graphs
    bool span_on = false;       // sp_set_span_timing: kernels stamp their CTA spans
    unsigned long long *d_span = nullptr;  // [SPAN_KINDS][RING][SPAN_MAXCTA][2] %globaltimer ns
    bool h2d_used[RING] = {};
    // schedule state (caller's thread)
    long long pushed = 0, planned = 0, forwarded = 0, trained = 0;
    bool eod = false, fwd_pending = false;
    // published to the transfer engine
    std::atomic<long long> trained_pub{0};
    std::atomic<long long> x_enqueued{0}, x_scattered{0};
    std::atomic<int> x_error{0};
    std::atomic<long long> x_gather_ns{0}, x_scatter_ns{0}, x_rows_g{0}, x_rows_s{0};
    std::string x_errmsg;
    std::thread scatter_worker;
    std::atomic<bool> stop{false};
    RowPool spool;  // scatter helpers
    int host_threads = 6;
    int scatter_helpers = 0, gather_helpers = 0;  // per pool (0: host_threads); SP_SCATTER_THREADS / SP_GATHER_THREADS
    // CPU gather of the missed rows (default; SP_CPU_GATHER=0 lets the transfer
    // kernel pull random host rows itself): Plan mirrors its
    // missed-row lists to pinned memory, the gather thread copies the rows
    // into a contiguous pinned slot, the transfer kernel reads that slot
    // (sequential pages) instead of random host rows
    bool cpu_gather = false;
    uint32_t gather_q16 = 65536;  // CPU-gathered share of each batch's fills (hybrid < 65536)
    std::thread gather_worker;
    RowPool gpool;  // gather helpers
    bool shared_pool = false;  // SP_SHARED_POOL=1: gather and scatter jobs take turns on one pool of both sizes
    unsigned long long *hl_ready = nullptr;    // pinned mapped [RING][T]
    uint32_t *hl_m = nullptr;                  // pinned mapped [RING][T]
    uint32_t *hl_row = nullptr;                // pinned mapped [RING][T][n]
    HostList hl_dev[RING];                     // device aliases
    float *h_in = nullptr, *hd_in = nullptr;   // pinned mapped [XSR][T*n][D] gathered rows
    unsigned long long *h_gathered = nullptr;  // pinned mapped: batches gathered
    unsigned long long *d_gathered = nullptr;  // device alias (stream wait-value)
    std::atomic<long long> x_gathered{0};
    // copy-engine H2D of the gathered slot (SP_GATHER_DMA=1; off by default:
    // measured 4% slower on Kaggle, the DMA's HBM writes slow k_fwd/k_bwd more
    // than it saves the surrogate): the first rows of the slot go to d_in by
    // DMA on the transfer stream; k_pullfill reads them from HBM and any rows
    // beyond from the pinned slot (zero-copy).
    bool gather_dma = false;
    float *d_in = nullptr;                     // device [XSR][T*n][D]
    std::atomic<long long> x_max_m{0};         // largest of the last 16 gathered batches (rows)
    // table-wise sharding (world > 1): NCCL comm, local pooled / gradient
    // buffers [T][N][D], the message lists of the exchange
    int world = 1, rank = 0, T_all = 0;
    void *comm = nullptr;
    float *d_pooled_local = nullptr, *d_grad_local = nullptr;
    std::vector<std::array<int, 3>> x_send;  // (peer, local table, global table)
    std::vector<std::array<int, 2>> x_recv;  // (peer, global table)
    // errors
    sp_status poisoned = SP_OK;
    std::string err = "no error";
    long long err_batch = -1;
    int err_table = -1;
    // stats (guarded by prof_mu where shared with the worker)
    std::mutex prof_mu;
    long long h2d_index_bytes = 0;
    long long launches[SP_K_COUNT] = {};
    double kms[SP_K_COUNT] = {};
    long long ktimed[SP_K_COUNT] = {};
    std::vector<ProfEv> prof_pending;
    std::vector<cudaEvent_t> ev_pool;
    cudaEvent_t prof_ref = nullptr;
    std::vector<TimelineRec> timeline;
    std::atomic<bool> profiling{false};
    // CUDA-graph replay of the steady-state step (sp_run_steps): per ring
    // residue r, one plan-stream graph and one compute-stream graph
    long long *d_ctl = nullptr;                 // [RING] device batch-index chain
    cudaGraphExec_t gplan[RING] = {}, gcomp[RING] = {};
    cudaStream_t cap_s = nullptr;
    // plan graphs are captured on a high-priority stream: a captured kernel
    // node keeps the priority of its capture stream, and k_push must stay
    // ahead of the wide Train grids in graph mode as in eager mode
    cudaStream_t cap_hi = nullptr;
    struct GraphKey {
        const void *trace = nullptr;
        long long stride = 0;
        float *pooled = nullptr, *grad = nullptr;
        float gamma = 0, delta = 0, lr = 0;
        bool operator==(const GraphKey &o) const {
            return trace == o.trace && stride == o.stride && pooled == o.pooled && grad == o.grad &&
                   gamma == o.gamma && delta == o.delta && lr == o.lr;
        }
    } gkey;
    long long g_next_j = -1;                    // j the device chain expects next
    long long graph_steps = 0;
    long long graph_step_ns = 0;  // caller-thread time issuing graph steps
    long long wait_xfer_ns = 0, wait_list_ns = 0;  // caller-thread waits on the engine
};

namespace {

sp_status fail(sp_ctx *c, sp_status s, const std::string &msg) {
    if (c) c->err = msg;
    return s;
}

sp_status cuda_fail(sp_ctx *c, cudaError_t e, const char *where) {
    if (c) {
        c->poisoned = SP_ERR_CUDA;
        c->err = std::string(where) + ": " + cudaGetErrorString(e);
    }
    return SP_ERR_CUDA;
}

#define CK(call)                                                   \
    do {                                                           \
        cudaError_t e_ = (call);                                   \
        if (e_ != cudaSuccess) return cuda_fail(c, e_, #call);     \
    } while (0)

template <typename T>
cudaError_t dalloc(sp_ctx *c, T **p, size_t count) {
    void *q = nullptr;
    cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
    if (e == cudaSuccess) {
        c->allocs.push_back(q);
        *p = static_cast<T *>(q);
    }
    return e;
}

cudaEvent_t pool_event(sp_ctx *c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// caller holds prof_mu
void harvest_profile(sp_ctx *c, bool blocking) {
    std::vector<ProfEv> keep;
    for (auto &p : c->prof_pending) {
        if (blocking) cudaEventSynchronize(p.b);
        if (cudaEventQuery(p.b) == cudaSuccess) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, p.a, p.b);
            c->kms[p.kind] += ms;
            c->ktimed[p.kind] += 1;
            if (c->prof_ref && c->timeline.size() < (1u << 20)) {
                float t0 = 0.f, t1 = 0.f;
                cudaEventElapsedTime(&t0, c->prof_ref, p.a);
                cudaEventElapsedTime(&t1, c->prof_ref, p.b);
                c->timeline.push_back({p.kind, p.batch, (double)t0, (double)t1});
            }
            c->ev_pool.push_back(p.a);
            c->ev_pool.push_back(p.b);
        } else {
            keep.push_back(p);
        }
    }
    (void)cudaGetLastError();  // clear cudaErrorNotReady
    c->prof_pending.swap(keep);
}

// wraps one kernel launch / DMA: counts it, optionally brackets it with events
template <typename Fn>
cudaError_t launch(sp_ctx *c, int kind, long long batch, cudaStream_t s, Fn &&fn) {
    const bool prof = c->profiling.load(std::memory_order_relaxed);
    ProfEv pe{kind, batch, nullptr, nullptr};
    if (prof) {
        std::lock_guard<std::mutex> lk(c->prof_mu);
        if (c->prof_pending.size() > 4096) harvest_profile(c, false);
        pe.a = pool_event(c);
        pe.b = pool_event(c);
        cudaEventRecord(pe.a, s);
    }
    cudaError_t e = fn();
    std::lock_guard<std::mutex> lk(c->prof_mu);
    c->launches[kind] += 1;
    if (prof) {
        cudaEventRecord(pe.b, s);
        c->prof_pending.push_back(pe);
    }
    return e;
}

BatchBufs carve(sp_ctx *c, cudaError_t *st) {
    BatchBufs b{};
    const size_t Tn = (size_t)c->T * c->n;
    cudaError_t e = cudaSuccess;
    auto A = [&](auto **p, size_t cnt) {
        if (e == cudaSuccess) e = dalloc(c, p, cnt);
    };
    A(&b.sorted_occ, Tn);
    A(&b.sorted_uid, Tn);
    A(&b.uniq_id, Tn);
    A(&b.seg_off, (size_t)c->T * c->g.n1);
    A(&b.U, (size_t)c->T);
    A(&b.chunk_rec, (size_t)c->T * c->g.nc);  // ChunkRec (80 B)
    A(&b.nchunks, (size_t)c->T);
    A(&b.hot_rec, (size_t)c->T * c->g.nh);
    A(&b.nhot, (size_t)c->T);
    A(&b.hot_cnt, (size_t)c->T * c->g.nh);
    A(&b.slot_u, Tn);
    A(&b.slot_of_occ, Tn);
    A(&b.sorted_slot, Tn);
    A(&b.hit, Tn);
    A(&b.fill_slot, Tn);
    A(&b.fill_row, Tn);
    A(&b.evict_row, Tn);
    A(&b.m, (size_t)c->T);
    A(&b.stats, (size_t)c->T * 4);
    A(&b.work, (size_t)(c->T + 63) / 64);
    *st = e;
    return b;
}

sp_status check_async_error(sp_ctx *c) {
    if (c->poisoned != SP_OK) return c->poisoned;
    if (*(volatile unsigned long long *)c->h_errflag && *(volatile unsigned long long *)c->h_err == NO_ERR) {
        // a kernel latched an error: read the exact (earliest) key
        cudaStreamSynchronize(c->plan_s);
        cudaMemcpy(c->h_err, c->d_err, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    }
    unsigned long long e = *(volatile unsigned long long *)c->h_err;
    if (e != NO_ERR && e != 0ull) {
        unsigned kind = (unsigned)(e & 0xFF);
        c->err_table = (int)((e >> 8) & 0xFFFF);
        c->err_batch = (long long)(e >> 24);
        c->poisoned = kind == DERR_CAPACITY ? SP_ERR_CAPACITY : SP_ERR_INDEX_RANGE;
        char buf[256];
        snprintf(buf, sizeof buf,
                 kind == DERR_CAPACITY
                     ? "SP_ERR_CAPACITY: no evictable Storage slot at batch %lld table %d "
                       "(window working set exceeds slots, PAPER.md P:1030-1035)"
                     : "SP_ERR_INDEX_RANGE: sparse ID out of range at batch %lld table %d",
                 c->err_batch, c->err_table);
        c->err = buf;
        return c->poisoned;
    }
    if (c->x_error.load(std::memory_order_acquire)) {
        c->poisoned = SP_ERR_CUDA;
        c->err = "transfer engine: " + c->x_errmsg;
        return c->poisoned;
    }
    return SP_OK;
}

// synchronous error read (device -> pinned word)
sp_status sync_error(sp_ctx *c) {
    if (c->poisoned != SP_OK) return c->poisoned;
    cudaError_t e = cudaMemcpyAsync(c->h_err, c->d_err, sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, c->plan_s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->plan_s);
    if (e != cudaSuccess) return cuda_fail(c, e, "sync_error");
    return check_async_error(c);
}

// spin until pred() (the transfer engine made progress) or an error shows up
template <typename Pred>
sp_status wait_engine(sp_ctx *c, Pred pred) {
    int idle = 0;
    while (!pred()) {
        if (sp_status s = check_async_error(c)) return s;
        if (++idle > 1024) std::this_thread::yield();
        else _mm_pause();
    }
    return SP_OK;
}

PushArgs push_args(sp_ctx *c) {
    PushArgs a{};
    a.span = c->span_on ? c->d_span : nullptr;
    a.g = c->g;
    a.P = c->P;
    a.F = c->F;
    a.row_off = c->d_row_off;
    a.rows = c->d_rows;
    a.slot_base = c->d_slot_base;
    a.hitmap = c->d_hitmap;
    a.resident = c->d_resident;
    a.last_use = c->d_last_use;
    a.next_need = c->d_next_need;
    a.log_slot = c->d_log_slot;
    a.log_stamp = c->d_log_stamp;
    a.log_base = c->d_log_base;
    a.log_cap = c->d_log_cap;
    a.log_head = c->d_log_head;
    a.log_tail = c->d_log_tail;
    a.err = c->d_err;
    a.err_host = c->d_errflag;
    a.cum = c->d_cum;
    a.miss_u = c->d_miss_u;
    a.victims = c->d_victims;
    a.sort_tmp = c->d_sort_tmp;
    a.idx_i32 = (c->flags & SP_FLAG_INDEX_I32) ? 1 : 0;
    a.prof = c->profiling.load() ? c->d_pprof : nullptr;
    a.policy = c->policy;
    a.log_classes = c->log_classes;
    a.seed = c->policy_seed;
    a.pin_base = c->d_pin_base;
    a.log_skip = c->d_log_skip;
    a.nfill = c->d_nfill;
    a.claim = c->d_claim;
    a.freq = c->d_freq;
    a.pad = (c->flags & SP_FLAG_PADDING) ? 1 : 0;
    a.bwd_recs = c->d_tpart ? 0 : 1;
    return a;
}

sp_status wait_gather_slot(sp_ctx *c, long long b);

sp_status enqueue_plan_only(sp_ctx *c, long long b) {
    if (sp_status s = wait_gather_slot(c, b)) return s;
    PushArgs a = push_args(c);
    a.has_new = 0;
    a.do_plan = 1;
    a.b = b;
    a.pb = c->ring[b % RING];
    if (c->cpu_gather) a.hl = c->hl_dev[b % RING];
    a.has_future = (b + c->F < c->pushed) ? 1 : 0;  // future window truncates at the end
    a.fb = c->ring[(b + c->F) % RING];
    CK(launch(c, SP_K_PLAN, b, c->plan_s, [&] { return launch_push(a, c->plan_s); }));
    CK(cudaEventRecord(c->ev_plan[b % RING], c->plan_s));
    c->planned = b + 1;
    return SP_OK;
}

TrainArgs train_args(sp_ctx *c, long long b) {
    TrainArgs a{};
    a.g = c->g;
    a.bb = c->ring[b % RING];
    a.storage = c->d_storage;
    a.partial = c->d_partial;
    a.tpart = c->d_tpart;  // null: the record-based k_bwd (SP_BWD=rec)
    a.seg_cnt = c->d_seg_cnt;
    a.grp_cnt = c->d_grp_cnt;
    a.tr = c->bwd_tr;
    a.ntiles = c->bwd_ntiles;
    a.tctr = c->bwd_dyn ? c->d_tctr : nullptr;
    a.tp2 = c->bwd_2p ? 1 : 0;
    a.bwd2_small = c->bwd2_small;
    a.fctr = c->fwd_dyn ? c->d_fctr : nullptr;
    a.bwd_tma = c->bwd_tma;
    a.srows = c->S_total;
    a.span = c->span_on ? c->d_span : nullptr;
    a.span_b = b;
    a.err = c->d_err;
    if (c->diag & 2) a.g.T = 0;  // diagnostic: Train kernels launched, no work
    a.diag = c->diag;
    return a;
}

// --------------------------------------------------------------- transfer engine

// On a device error or at teardown the engine threads stop; the GPU stream
// waits on their progress counters are released so that queued transfers run
// (and return at once on the latched error) instead of blocking forever.
void release_engine_waits(sp_ctx *c) {
    const unsigned long long all = 1ull << 62;
    if (c->h_scat) *(volatile unsigned long long *)c->h_scat = all;
    if (c->h_gathered) *(volatile unsigned long long *)c->h_gathered = all;
    std::atomic_thread_fence(std::memory_order_seq_cst);
}

// [Insert] CPU scatter of batch s's victims into the host tables once
// Transfer(s) has staged them in pinned host memory (k_pullfill's last CTA
// sets h_staged), in batch order, on its own thread.  No CUDA API call: the
// thread only polls pinned memory, so it never contends for the driver with
// the caller's thread.  Rows evicted at s are not in B(s+1..s+F), so the
// scatter overlaps the next transfers; Transfer(s+F+1) waits for it on the
// GPU (RAW-4, h_scat).
void scatter_main(sp_ctx *c) {
    const size_t rowb = (size_t)c->D * sizeof(float);
    const size_t slab = (size_t)c->T * c->n * c->D;
    std::vector<const float *> src;
    std::vector<float *> dst;
    std::vector<uint32_t> pref(c->T + 1);
    long long s = 0;  // next batch to scatter
    int idle = 0;
    auto ready = [&](long long b) {
        if (((volatile unsigned long long *)c->h_staged)[b % RING] != (unsigned long long)(b + 1)) return false;
        std::atomic_thread_fence(std::memory_order_acquire);
        return true;
    };
    while (!c->stop.load(std::memory_order_relaxed)) {
        if (*(volatile unsigned long long *)c->h_errflag) {
            release_engine_waits(c);
            break;
        }
        if (s < c->x_enqueued.load(std::memory_order_acquire) && ready(s)) {
            const size_t cnt = (size_t)((volatile unsigned long long *)c->h_scnt)[s % RING];
            src.clear();
            dst.clear();
            const float *wb = c->h_wb + (size_t)(s % c->XSR) * slab;
            const unsigned long long *wd = c->h_wbdst + (size_t)(s % c->XSR) * c->T * c->n;
            for (size_t i = 0; i < cnt; i++)
                if (wd[i]) {
                    src.push_back(wb + i * c->D);
                    dst.push_back(reinterpret_cast<float *>((uintptr_t)wd[i]));
                }
            const auto t0 = std::chrono::steady_clock::now();
            c->spool.copy(src.data(), dst.data(), (long)src.size(), rowb);
            c->x_scatter_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(
                                   std::chrono::steady_clock::now() - t0).count();
            c->x_rows_s += (long long)src.size();
            s++;
            c->x_scattered.store(s, std::memory_order_release);
            std::atomic_thread_fence(std::memory_order_seq_cst);
            *(volatile unsigned long long *)c->h_scat = (unsigned long long)s;  // GPU wait-value
            idle = 0;
        } else if (++idle > 2048) {
            std::this_thread::yield();
        } else {
            _mm_pause();
        }
    }
}

// [Collect] CPU gather of batch b's missed rows into the contiguous pinned
// slot b % XSR, in batch order, once Plan(b) has mirrored its lists, the
// write-back of batch b-F-1 has landed in the host tables (RAW-4: a row
// evicted at b-F-1 or earlier may be missed again at b) and Transfer(b-XSR)
// has finished reading the slot.  Publishes gathered = b + 1 (the transfer
// stream waits on it).  No CUDA API call.
void gather_main(sp_ctx *c) {
    long long recent[16] = {};
    const size_t rowb = (size_t)c->D * sizeof(float);
    const size_t slab = (size_t)c->T * c->n * c->D;
    std::vector<const float *> src;
    std::vector<float *> dst;
    long long g = 0;
    int idle = 0;
    auto ready = [&](long long b) {
        const int r = (int)(b % RING);
        for (int t = 0; t < c->T; t++)
            if (((volatile unsigned long long *)c->hl_ready)[(size_t)r * c->T + t] != (unsigned long long)(b + 1))
                return false;
        if (c->gpu_wb) {  // the write-backs of Transfer(b-F-1) have landed
            const long long w = b - c->F - 1;
            if (w >= 0 && ((volatile unsigned long long *)c->h_staged)[w % RING] < (unsigned long long)(w + 1)) return false;
        } else if (c->x_scattered.load(std::memory_order_acquire) < b - c->F) {
            return false;
        }
        const long long prev = b - c->XSR;
        if (prev >= 0 && ((volatile unsigned long long *)c->h_staged)[prev % RING] < (unsigned long long)(prev + 1))
            return false;
        std::atomic_thread_fence(std::memory_order_acquire);
        return true;
    };
    while (!c->stop.load(std::memory_order_relaxed)) {
        if (*(volatile unsigned long long *)c->h_errflag) {
            release_engine_waits(c);
            break;
        }
        if (ready(g)) {
            const int r = (int)(g % RING);
            src.clear();
            dst.clear();
            float *in = c->h_in + (size_t)(g % c->XSR) * slab;
            size_t k0 = 0;
            // per group of 64 tables (the transfer kernel's unit), the first
            // Kg = total * q >> 16 fills in table order (hybrid split)
            for (int t0 = 0; t0 < c->T; t0 += 64) {
                const int t1 = std::min(c->T, t0 + 64);
                unsigned long long total = 0;
                for (int t = t0; t < t1; t++) total += c->hl_m[(size_t)r * c->T + t];
                const unsigned long long Kg = c->gather_q16 >= 65536 ? total : (total * c->gather_q16) >> 16;
                unsigned long long item = 0;
                for (int t = t0; t < t1 && item < Kg; t++) {
                    const uint32_t m = c->hl_m[(size_t)r * c->T + t];
                    const uint32_t *rows = c->hl_row + ((size_t)r * c->T + t) * c->n;
                    for (uint32_t k = 0; k < m && item < Kg; k++, item++) {
                        src.push_back(c->host[t] + (size_t)rows[k] * c->D);
                        dst.push_back(in + (k0 + item) * c->D);
                    }
                }
                k0 += total;
            }
            const auto t0 = std::chrono::steady_clock::now();
            (c->shared_pool ? c->spool : c->gpool).copy(src.data(), dst.data(), (long)src.size(), rowb);
            c->x_gather_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(
                                  std::chrono::steady_clock::now() - t0).count();
            c->x_rows_g += (long long)src.size();
            {   // largest of the last 16 batches (cold-start bursts age out)
                recent[g % 16] = (long long)src.size();
                long long mx = 0;
                for (long long v : recent) mx = std::max(mx, v);
                c->x_max_m.store(mx, std::memory_order_relaxed);
            }
            g++;
            c->x_gathered.store(g, std::memory_order_release);
            std::atomic_thread_fence(std::memory_order_seq_cst);
            *(volatile unsigned long long *)c->h_gathered = (unsigned long long)g;
            idle = 0;
        } else if (++idle > 2048) {
            std::this_thread::yield();
        } else {
            _mm_pause();
        }
    }
}

// Plan(b) reuses the missed-row mirror slot of Plan(b - RING): the gather
// thread must be done with it (CPU gather only).
sp_status wait_gather_slot(sp_ctx *c, long long b) {
    if (!c->cpu_gather || b - RING < 0) return SP_OK;
    return wait_engine(c, [&] { return c->x_gathered.load(std::memory_order_acquire) > b - RING; });
}

void stop_engine(sp_ctx *c) {
    c->stop = true;
    release_engine_waits(c);
    if (c->scatter_worker.joinable()) c->scatter_worker.join();
    if (c->gather_worker.joinable()) c->gather_worker.join();
    c->spool.shutdown();
    c->gpool.shutdown();
}

// stream wait on a 64-bit pinned counter (cuStreamWaitValue64 through the
// runtime's driver entry point: no link-time dependency on libcuda)
typedef CUresult (*wait_value64_fn)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
wait_value64_fn wait_value64() {
    static wait_value64_fn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<wait_value64_fn>(p);
    }
    return fn;
}

// Enqueue every Transfer(b) whose preconditions exist: Plan(b) enqueued and
// Train(b-P-1) enqueued (its event recorded).  Caller's thread only.
sp_status pump(sp_ctx *c) {
    while (c->xfer_enq < c->planned) {
        const long long b = c->xfer_enq, dep = b - c->P - 1;
        if (dep >= 0 && c->trained <= dep) break;
        const int r = (int)(b % RING);
        cudaStream_t xs = (b & 1) ? c->xfer_s2 : c->xfer_s;
        CK(cudaStreamWaitEvent(xs, c->ev_plan[r], 0));
        if (dep >= 0) CK(cudaStreamWaitEvent(xs, c->ev_train[dep % RING], 0));
        // RAW-4 + staging reuse: the CPU write-back of batch b-F-1 has landed
        const long long need = b - c->F;  // scattered >= b-F
        if (c->gpu_wb) {
            // the GPU wrote the victims of Transfer(b-F-1) into their host rows
            if (need > 0) CK(cudaStreamWaitEvent(xs, c->ev_xfer[(need - 1) % RING], 0));
        } else if (need > 0) {
            wait_value64_fn wv = wait_value64();
            if (!wv) return fail(c, SP_ERR_CUDA, "cuStreamWaitValue64 unavailable");
            CUresult cr = wv((CUstream)xs, (CUdeviceptr)c->d_scat, (cuuint64_t)need, CU_STREAM_WAIT_VALUE_GEQ);
            if (cr != CUDA_SUCCESS) return fail(c, SP_ERR_CUDA, "cuStreamWaitValue64 failed");
        }
        const bool hybrid = c->cpu_gather && c->gather_q16 < 65536;
        if (c->cpu_gather && !hybrid) {  // the CPU has gathered batch b's missed rows
            wait_value64_fn wv = wait_value64();
            if (!wv) return fail(c, SP_ERR_CUDA, "cuStreamWaitValue64 unavailable");
            CUresult cr = wv((CUstream)xs, (CUdeviceptr)c->d_gathered, (cuuint64_t)(b + 1), CU_STREAM_WAIT_VALUE_GEQ);
            if (cr != CUDA_SUCCESS) return fail(c, SP_ERR_CUDA, "cuStreamWaitValue64 failed");
        }
        XferArgs a{};
        a.g = c->g;
        a.bb = c->ring[r];
        if (c->cpu_gather) a.in_stage = c->hd_in + (size_t)(b % c->XSR) * c->T * c->n * c->D;
        a.gfrac_q16 = c->gather_q16;
        a.gwait = hybrid ? c->d_gathered : nullptr;  // hybrid: gathered rows awaited in-kernel
        if (c->cpu_gather && c->gather_dma && !hybrid) {
            // rows to DMA: 1.5x the largest of the last 16 gathered batches
            // (+256), at most the slot; rows past them are read zero-copy
            const long long Tn = (long long)c->T * c->n;
            long long rows = c->x_max_m.load(std::memory_order_relaxed);
            rows = rows ? std::min(Tn, rows + rows / 2 + 256) : Tn;
            const size_t off = (size_t)(b % c->XSR) * Tn * c->D;
            CK(cudaMemcpyAsync(c->d_in + off, c->h_in + off, (size_t)rows * c->D * sizeof(float),
                               cudaMemcpyHostToDevice, xs));
            a.in_dev = c->d_in + off;
            a.in_dev_rows = (uint32_t)rows;
        }
        a.storage = c->d_storage;
        a.host = c->d_host;
        a.wb_stage = c->hd_wb + (size_t)(b % c->XSR) * c->T * c->n * c->D;
        a.done_ctr = c->d_xdone + r;
        a.staged = c->hd_staged + r;
        a.wb_dst = c->hd_wbdst + (size_t)(b % c->XSR) * c->T * c->n;
        a.staged_cnt = c->hd_scnt + r;
        a.wb_direct = c->gpu_wb ? 1 : 0;
        a.wb_q16 = c->gpu_wb ? 65536u : c->wb_q16;
        a.span = c->span_on ? c->d_span : nullptr;
        a.b = b;
        if (c->diag & 1) a.g.T = 0;  // diagnostic: transfer launched, no rows moved
        if (c->diag & 4) a.diag_nowb = 1;  // diagnostic: victims not staged (pull only)
        a.err = c->d_err;
        if (c->stage_timing) CK(cudaEventRecord(c->sev[r][6], xs));
        CK(launch(c, SP_K_TRANSFER, b, xs, [&] {
            return c->xfer_warp ? launch_xfer_warp(a, c->xfer_ctas ? c->xfer_ctas : 2 * device_sms(), xs)
                                : launch_pullfill(a, c->pull_ctas, xs);
        }));
        if (c->stage_timing) CK(cudaEventRecord(c->sev[r][7], xs));
        c->sev_used[r][1] = c->stage_timing;
        CK(cudaEventRecord(c->ev_xfer[r], xs));
        c->xfer_enq = b + 1;
        c->x_enqueued.store(b + 1, std::memory_order_release);
    }
    return SP_OK;
}

void drop_graphs(sp_ctx *c);

// Sharded exchange (world > 1), on the compute stream.  forward: local
// pooled [T][N][D] -> caller's [T_all][N/G][D] (rank g gets samples
// g*Ns .. (g+1)*Ns-1 of every table); backward: caller's gradient
// [T_all][Ns][D] -> local [T][N][D].  Every message is one table's Ns
// contiguous rows, so no pack / unpack kernel is needed.
sp_status exchange(sp_ctx *c, bool forward, float *bufA, const float *bufB) {
    NcclApi &nc = nccl();
    const size_t Ns = (size_t)c->N / c->world, rowf = (size_t)c->D, msg = Ns * rowf;
    int r = nc.group_start();
    for (const auto &m : c->x_send) {  // (peer, local table, global table)
        if (r) break;
        if (forward) r = nc.send(c->d_pooled_local + ((size_t)m[1] * c->N + (size_t)m[0] * Ns) * rowf, msg,
                                 NCCL_FLOAT32, m[0], c->comm, c->compute);
        else r = nc.recv(c->d_grad_local + ((size_t)m[1] * c->N + (size_t)m[0] * Ns) * rowf, msg, NCCL_FLOAT32,
                         m[0], c->comm, c->compute);
    }
    for (const auto &m : c->x_recv) {  // (peer, global table)
        if (r) break;
        if (forward) r = nc.recv(bufA + (size_t)m[1] * msg, msg, NCCL_FLOAT32, m[0], c->comm, c->compute);
        else r = nc.send(bufB + (size_t)m[1] * msg, msg, NCCL_FLOAT32, m[0], c->comm, c->compute);
    }
    const int r2 = nc.group_end();
    if (r || r2) {
        c->poisoned = SP_ERR_NCCL;
        c->err = std::string("NCCL exchange: ") + nc.err(r ? r : r2);
        return SP_ERR_NCCL;
    }
    return SP_OK;
}

void destroy_all(sp_ctx *c) {
    if (!c) return;
    stop_engine(c);
    drop_graphs(c);
    cudaSetDevice(c->device);
    if (c->plan_s) cudaStreamSynchronize(c->plan_s);
    if (c->xfer_s) cudaStreamSynchronize(c->xfer_s);
    if (c->xfer_s2) cudaStreamSynchronize(c->xfer_s2);
    cudaStreamSynchronize(c->compute);
    {
        std::lock_guard<std::mutex> lk(c->prof_mu);
        harvest_profile(c, true);
        for (auto e : c->ev_pool) cudaEventDestroy(e);
    }
    for (int r = 0; r < RING; r++)
        for (cudaEvent_t e : {c->ev_plan[r], c->ev_xfer[r], c->ev_train[r], c->ev_h2d[r]})
            if (e) cudaEventDestroy(e);
    if (c->ev_user) cudaEventDestroy(c->ev_user);
    for (int r = 0; r < RING; r++)
        for (int k = 0; k < 8; k++)
            if (c->sev[r][k]) cudaEventDestroy(c->sev[r][k]);
    if (c->prof_ref) cudaEventDestroy(c->prof_ref);
    for (void *p : c->allocs) cudaFree(p);
    for (void *p : {(void *)c->h_stage, (void *)c->h_csr, (void *)c->h_err, (void *)c->h_errflag, (void *)c->h_scat, (void *)c->h_wb, (void *)c->h_staged,
                    (void *)c->h_wbdst, (void *)c->h_scnt,
                    (void *)c->hl_ready, (void *)c->hl_m, (void *)c->hl_row, (void *)c->h_in, (void *)c->h_gathered})
        if (p) cudaFreeHost(p);
    if (c->registered)
        for (int t = 0; t < c->T; t++) cudaHostUnregister(c->host[t]);
    if (c->own_plan_s) cudaStreamDestroy(c->own_plan_s);
    if (c->own_xfer_s) cudaStreamDestroy(c->own_xfer_s);
    if (c->own_xfer_s2) cudaStreamDestroy(c->own_xfer_s2);
    if (c->cap_s) cudaStreamDestroy(c->cap_s);
    if (c->cap_hi) cudaStreamDestroy(c->cap_hi);
    if (c->comm && nccl().ok) nccl().destroy(c->comm);
    (void)cudaGetLastError();
    delete c;
}

}  // namespace

extern "C" {

int32_t sp_abi_version(void) { return SP_ABI_VERSION; }

sp_status sp_nccl_unique_id(void *out) {
    if (!out) return SP_ERR_INVALID_ARG;
    if (!nccl().ok) return SP_ERR_NCCL;
    std::array<char, 128> id;
    if (nccl().unique_id(&id) != 0) return SP_ERR_NCCL;
    std::memcpy(out, id.data(), 128);
    return SP_OK;
}

sp_status sp_shard_plan(int32_t world, int32_t rank, int32_t num_tables_all, const int32_t *table_owner,
                        int32_t *send, int64_t *nsend, int32_t *recv, int64_t *nrecv) {
    if (world < 1 || rank < 0 || rank >= world || num_tables_all < 1 || !table_owner || !nsend || !nrecv)
        return SP_ERR_INVALID_ARG;
    for (int t = 0; t < num_tables_all; t++)
        if (table_owner[t] < 0 || table_owner[t] >= world) return SP_ERR_INVALID_ARG;
    std::vector<std::array<int, 3>> sv;
    std::vector<std::array<int, 2>> rv;
    shard_plan(world, rank, num_tables_all, table_owner, sv, rv);
    if (send)
        for (size_t k = 0; k < sv.size() && (int64_t)k < *nsend; k++)
            for (int j = 0; j < 3; j++) send[3 * k + j] = sv[k][j];
    if (recv)
        for (size_t k = 0; k < rv.size() && (int64_t)k < *nrecv; k++)
            for (int j = 0; j < 2; j++) recv[2 * k + j] = rv[k][j];
    *nsend = (int64_t)sv.size();
    *nrecv = (int64_t)rv.size();
    return SP_OK;
}

sp_status sp_host_alloc(size_t bytes, void **out) {
    if (!out || !bytes) return SP_ERR_INVALID_ARG;
    *out = nullptr;
    void *p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return SP_ERR_OOM;
    madvise(p, bytes, MADV_HUGEPAGE);  // best effort (THP "madvise" mode)
    // pinning faults the pages in, so they come up as 2 MB pages when possible
    cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        munmap(p, bytes);
        return e == cudaErrorMemoryAllocation ? SP_ERR_OOM : SP_ERR_CUDA;
    }
    *out = p;
    return SP_OK;
}

sp_status sp_host_alloc_near(size_t bytes, int32_t device, void **out, int32_t *numa_node_out) {
    if (!out || !bytes) return SP_ERR_INVALID_ARG;
    *out = nullptr;
    if (numa_node_out) *numa_node_out = -1;
    int node = -1;
    if (cudaDeviceGetAttribute(&node, cudaDevAttrHostNumaId, device) != cudaSuccess) {
        (void)cudaGetLastError();
        node = -1;
    }
    void *p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return SP_ERR_OOM;
    madvise(p, bytes, MADV_HUGEPAGE);
    if (node >= 0 && node < 64) {
        // MPOL_PREFERRED (1): the node's pages first, others if it is full
        const unsigned long mask = 1ul << node;
        if (syscall(SYS_mbind, p, bytes, 1, &mask, 64ul, 0u) == 0 && numa_node_out) *numa_node_out = node;
    }
    cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        munmap(p, bytes);
        return e == cudaErrorMemoryAllocation ? SP_ERR_OOM : SP_ERR_CUDA;
    }
    *out = p;
    return SP_OK;
}

sp_status sp_host_free(void *ptr, size_t bytes) {
    if (!ptr || !bytes) return SP_ERR_INVALID_ARG;
    cudaHostUnregister(ptr);
    (void)cudaGetLastError();
    munmap(ptr, bytes);
    return SP_OK;
}

sp_status sp_create(const sp_desc *d, sp_ctx **out) {
    if (!out) return SP_ERR_INVALID_ARG;
    *out = nullptr;
    if (!d || d->num_tables < 1 || d->num_tables > 65535 || !d->rows || !d->slots || !d->host_tables)
        return SP_ERR_INVALID_ARG;
    if (d->dim < 4 || d->dim > 1024 || d->dim % 4) return SP_ERR_INVALID_ARG;
    // bf16 Storage rows move by bulk copies: 2*D bytes, a multiple of 16
    if ((d->flags & SP_FLAG_BF16) && d->dim % 8) return SP_ERR_INVALID_ARG;
    if (d->batch_size < 1 || d->pooling < 1) return SP_ERR_INVALID_ARG;
    const long long n = (long long)d->batch_size * d->pooling;
    if (n > (1ll << 26)) return SP_ERR_INVALID_ARG;
    int P = d->past, F = d->future;
    if (P < 0 || F < 0) {
        if (d->window < 0) return SP_ERR_INVALID_ARG;
        P = d->window;
        F = d->window > 0 ? d->window - 1 : 0;
    }
    if (F > P + 1) return SP_ERR_INVALID_ARG;  // one-shot future probe needs F <= P + 1
    if (d->policy < SP_POLICY_LRU || d->policy > SP_POLICY_LFU || d->reserved != 0) return SP_ERR_INVALID_ARG;
    const bool sharded = d->world > 1 || (d->world == 1 && d->nccl_id);
    if (sharded) {
        if (!d->nccl_id || d->rank < 0 || d->rank >= d->world || d->num_tables_all < d->num_tables ||
            !d->table_owner || !d->table_ids || d->batch_size % d->world != 0 || d->reserved2 != 0)
            return SP_ERR_INVALID_ARG;
        int mine = 0;
        for (int t = 0; t < d->num_tables_all; t++) {
            if (d->table_owner[t] < 0 || d->table_owner[t] >= d->world) return SP_ERR_INVALID_ARG;
            mine += d->table_owner[t] == d->rank;
        }
        if (mine != d->num_tables) return SP_ERR_INVALID_ARG;
        for (int k = 0; k < d->num_tables; k++)
            if (d->table_ids[k] < 0 || d->table_ids[k] >= d->num_tables_all ||
                d->table_owner[d->table_ids[k]] != d->rank || (k && d->table_ids[k] <= d->table_ids[k - 1]))
                return SP_ERR_INVALID_ARG;
    }
    if (P + F + 2 > RING) return SP_ERR_INVALID_ARG;
    sp_ctx *c = new sp_ctx();
    c->T = d->num_tables;
    c->D = d->dim;
    c->N = d->batch_size;
    c->L = d->pooling;
    c->n = (int)n;
    c->P = P;
    c->F = F;
    c->device = d->device;
    c->flags = d->flags;
    c->compute = (cudaStream_t)d->stream;
    c->profiling = (d->flags & SP_FLAG_PROFILE) != 0;
    c->g.T = c->T;
    c->g.N = c->N;
    c->g.L = c->L;
    c->g.D = c->D;
    c->g.n = c->n;
    c->g.n1 = c->n + 1;
    c->g.nc = c->n + c->n / CH + 1;
    c->g.hs = backward_hot_segment(c->D);
    c->g.pad = (d->flags & SP_FLAG_PADDING) ? 1 : 0;
    c->g.bf16 = (d->flags & SP_FLAG_BF16) ? 1 : 0;
    c->policy = d->policy;
    c->policy_seed = d->policy_seed;
    c->log_classes = c->policy == SP_POLICY_LFU ? LOG_CLASSES_MAX : (c->policy == SP_POLICY_RANDOM ? 0 : 1);
    // hot-row segment records: rows with > CH occurrences, ceil(len/hs) each
    c->g.nh = c->n / c->g.hs + c->n / (CH + 1) + 1;
    if ((long long)c->n / c->g.hs + 1 > HOT_NSEG_MAX) {  // segment count must fit its packing
        delete c;
        return SP_ERR_INVALID_ARG;
    }
    c->rows.resize(c->T);
    c->slots.resize(c->T);
    c->host.resize(c->T);
    c->host_dev.resize(c->T);
    c->row_off.assign(c->T + 1, 0);
    c->slot_base.assign(c->T + 1, 0);
    for (int t = 0; t < c->T; t++) {
        long long R = d->rows[t], S = d->slots[t];
        if (R < 1 || R >= 0xFFFFFFFFll || S < 1 || S > R || !d->host_tables[t]) {
            delete c;
            return SP_ERR_INVALID_ARG;
        }
        c->rows[t] = R;
        c->slots[t] = S;
        c->host[t] = d->host_tables[t];
        c->row_off[t + 1] = c->row_off[t] + (unsigned long long)R;
        c->S_total += S;
    }
    if (c->S_total >= 0xFFFFFFFFll) {
        delete c;
        return SP_ERR_INVALID_ARG;
    }
    for (int t = 0; t < c->T; t++) c->slot_base[t + 1] = c->slot_base[t] + (uint32_t)c->slots[t];
    c->hit_total = c->row_off[c->T];
    c->XSR = std::max(4, c->F + 2);  // >= F+1: Transfer(b) waits for scatter(b-F-1) >= b-XSR
    c->host_threads = d->host_threads;  // 0: sized from the node's cores below
    // transfer grid: 16 one-warp CTAs (measured best on Kaggle and Terabyte;
    // 30 / 48 CTAs were 11% / 18% slower on Terabyte: more SMs add interference,
    // not host-link throughput)
    if (const char *e = getenv("SP_PULL_CTAS")) c->pull_ctas = std::max(1, atoi(e));
    if (const char *e = getenv("SP_XFER")) c->xfer_warp = std::string(e) == "warp";
    if (const char *e = getenv("SP_BWD_TMA")) c->bwd_tma = atoi(e) != 0;
    if (const char *e = getenv("SP_BWD_DYN")) c->bwd_dyn = atoi(e) != 0;
    if (const char *e = getenv("SP_BWD_2P")) c->bwd_2p = atoi(e) != 0;
    if (const char *e = getenv("SP_BWD2_SMALL")) c->bwd2_small = std::max(1, atoi(e));
    if (const char *e = getenv("SP_FWD_DYN")) c->fwd_dyn = atoi(e) != 0;
    if (const char *e = getenv("SP_XFER_CTAS")) c->xfer_ctas = std::max(1, atoi(e));
    if (const char *e = getenv("SP_WB_GPU_FRAC")) {
        const double f = atof(e);
        c->wb_q16 = f <= 0.0 ? 0u : (f >= 1.0 ? 65536u : (uint32_t)(f * 65536.0));
    }
    if (const char *e = getenv("SP_DIAG")) c->diag = atoi(e);
    if (c->g.bf16) c->xfer_warp = false;  // bf16 Storage: k_pullfill converts rows, k_xfer_warp does not

    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) {
        sp_status s = cuda_fail(c, e, "cudaSetDevice");
        destroy_all(c);
        return s;
    }
    auto bail = [&](sp_status s) {
        destroy_all(c);
        return s;
    };
#define CKC(call)                                                                  \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) {                                                   \
            (void)cudaGetLastError();                                              \
            return bail(e_ == cudaErrorMemoryAllocation ? SP_ERR_OOM : SP_ERR_CUDA); \
        }                                                                          \
    } while (0)
    // host tables: registration / mapped device pointers
    if (c->flags & SP_FLAG_REGISTER_HOST) {
        for (int t = 0; t < c->T; t++) {
            e = cudaHostRegister(c->host[t], (size_t)c->rows[t] * c->D * sizeof(float),
                                 cudaHostRegisterMapped | cudaHostRegisterPortable);
            if (e != cudaSuccess) {
                for (int k = 0; k < t; k++) cudaHostUnregister(c->host[k]);
                (void)cudaGetLastError();
                return bail(SP_ERR_INVALID_ARG);
            }
        }
        c->registered = true;
    }
    std::vector<float *> hdev(c->T);
    for (int t = 0; t < c->T; t++) {
        void *p = nullptr;
        e = cudaHostGetDevicePointer(&p, c->host[t], 0);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            return bail(SP_ERR_INVALID_ARG);  // not pinned / registered
        }
        hdev[t] = static_cast<float *>(p);
        c->host_dev[t] = hdev[t];
        // the transfer kernel moves whole rows with cp.async.bulk: 16-B aligned
        if ((reinterpret_cast<uintptr_t>(p) & 15) != 0) return bail(SP_ERR_INVALID_ARG);
    }
    {   // Plan is the serial critical chain: its CTAs get scheduled first
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        const char *pp = getenv("SP_PLAN_PRIO");  // 0: plan stream at default priority (A/B)
        const bool plan_hi = !(pp && atoi(pp) == 0);
        CKC(cudaStreamCreateWithPriority(&c->plan_s, cudaStreamNonBlocking, plan_hi ? hi : lo));
        const char *xp = getenv("SP_XFER_PRIO");  // 1: transfer CTAs also scheduled first
        CKC(cudaStreamCreateWithPriority(&c->xfer_s, cudaStreamNonBlocking, (xp && atoi(xp) == 1) ? hi : lo));
        // SP_XFER_STREAMS=1: one transfer stream (transfers strictly in sequence)
        const char *xn = getenv("SP_XFER_STREAMS");
        if (xn && atoi(xn) == 1) c->xfer_s2 = c->xfer_s;
        else CKC(cudaStreamCreateWithPriority(&c->xfer_s2, cudaStreamNonBlocking, (xp && atoi(xp) == 1) ? hi : lo));
        c->own_xfer_s2 = c->xfer_s2 != c->xfer_s ? c->xfer_s2 : nullptr;
        c->own_plan_s = c->plan_s;
        c->own_xfer_s = c->xfer_s;
        // diagnostic: SP_DIAG_SERIAL=1 runs every GPU stage on the caller's
        // stream (no stage overlap) to time kernels free of interference
        if (const char *ds = getenv("SP_DIAG_SERIAL"))
            if (atoi(ds) == 1) c->plan_s = c->xfer_s = c->xfer_s2 = c->compute;
    }
    CKC(cudaStreamCreateWithFlags(&c->cap_s, cudaStreamNonBlocking));
    {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        const char *pp = getenv("SP_PLAN_PRIO");  // the plan graphs get the plan stream's priority
        CKC(cudaStreamCreateWithPriority(&c->cap_hi, cudaStreamNonBlocking, (pp && atoi(pp) == 0) ? lo : hi));

    }
    for (int r = 0; r < RING; r++)
        for (cudaEvent_t *ev : {&c->ev_plan[r], &c->ev_xfer[r], &c->ev_train[r], &c->ev_h2d[r]})
            CKC(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&c->ev_user, cudaEventDisableTiming));
    for (int r = 0; r < RING; r++)
        for (int k = 0; k < 8; k++) CKC(cudaEventCreate(&c->sev[r][k]));
    if (const char *e = getenv("SP_CARVEOUT")) g_carveout = atoi(e);
    if (const char *e = getenv("SP_PDL")) g_pdl = atoi(e) != 0;
    if (sharded) {  // NCCL communicator of the G contexts (collective: every rank calls sp_create)
        if (!nccl().ok) return bail(SP_ERR_NCCL);
        c->world = d->world;
        c->rank = d->rank;
        c->T_all = d->num_tables_all;
        shard_plan(c->world, c->rank, c->T_all, d->table_owner, c->x_send, c->x_recv);
        std::array<char, 128> id;
        std::memcpy(id.data(), d->nccl_id, 128);
        int r = nccl().init_rank(&c->comm, c->world, id, c->rank);
        if (r != 0) {
            c->err = std::string("ncclCommInitRank: ") + nccl().err(r);
            c->comm = nullptr;
            return bail(SP_ERR_NCCL);
        }
    }
    CKC(configure_push_kernel());
    CKC(configure_xfer_kernels());
    CKC(configure_train_kernels());

    // device allocations
    const size_t Tn = (size_t)c->T * c->n;
    CKC(dalloc(c, &c->d_row_off, c->T + 1));
    CKC(dalloc(c, &c->d_rows, c->T));
    CKC(dalloc(c, &c->d_slot_base, c->T + 1));
    CKC(dalloc(c, &c->d_hitmap, c->hit_total));
    CKC(dalloc(c, &c->d_resident, (size_t)c->S_total));
    CKC(dalloc(c, &c->d_last_use, (size_t)c->S_total));
    CKC(dalloc(c, &c->d_next_need, (size_t)c->S_total));
    // Storage: S rows of D fp32, or of D bf16 (SP_FLAG_BF16: half the bytes)
    CKC(dalloc(c, &c->d_storage, (size_t)c->S_total * c->D / (c->g.bf16 ? 2 : 1)));
    CKC(dalloc(c, &c->d_fctr, (size_t)RING * TCTR_STRIDE));
    CKC(cudaMemset(c->d_fctr, 0, (size_t)RING * TCTR_STRIDE * sizeof(uint32_t)));
    // LRU log per table (LFU: one per use-count class, c = 0 holding the
    // initial vacant slots; RANDOM: none): capacity log_factor*S_t + 4n
    // (LFU classes: 2*S_t + 4n each)
    const long long lf = d->log_factor > 0 ? d->log_factor : 32;  // HBM is plentiful: compaction rare
    const int NCl = std::max(1, c->log_classes);
    std::vector<unsigned long long> lbase((size_t)c->T * NCl), lcap((size_t)c->T * NCl), lhead((size_t)c->T * NCl, 0),
        ltail((size_t)c->T * NCl, 0);
    unsigned long long ltot = 0;
    for (int t = 0; t < c->T; t++)
        for (int k = 0; k < NCl; k++) {
            const size_t l = (size_t)t * NCl + k;
            const long long f = c->log_classes == 0 ? 0 : (c->policy == SP_POLICY_LFU ? (k == 0 ? 0 : 2) : lf);
            lcap[l] = (unsigned long long)(f * c->slots[t] + (k == 0 ? c->slots[t] : 0) + 4ll * c->n);
            if (c->log_classes == 0) lcap[l] = 1;
            lbase[l] = ltot;
            ltot += lcap[l];
            ltail[l] = (k == 0 && c->log_classes > 0) ? (unsigned long long)c->slots[t] : 0ull;  // initial vacant entries
        }
    CKC(dalloc(c, &c->d_log_slot, ltot));
    CKC(dalloc(c, &c->d_log_stamp, ltot));
    CKC(dalloc(c, &c->d_log_base, lbase.size()));
    CKC(dalloc(c, &c->d_log_cap, lbase.size()));
    CKC(dalloc(c, &c->d_log_head, lbase.size()));
    CKC(dalloc(c, &c->d_log_tail, lbase.size()));
    c->pin_base.assign(c->slot_base.begin() + 1, c->slot_base.end());
    c->pinned_t.assign(c->T, false);
    CKC(dalloc(c, &c->d_pin_base, c->T));
    CKC(dalloc(c, &c->d_nfill, c->T));
    CKC(cudaMemset(c->d_nfill, 0, c->T * sizeof(uint32_t)));
    if (c->policy == SP_POLICY_RANDOM) {
        CKC(dalloc(c, &c->d_claim, (size_t)c->S_total));
        CKC(cudaMemset(c->d_claim, 0, (size_t)c->S_total * sizeof(unsigned long long)));
    }
    if (c->policy == SP_POLICY_LFU) {
        CKC(dalloc(c, &c->d_freq, (size_t)c->S_total));
        CKC(cudaMemset(c->d_freq, 0, (size_t)c->S_total));
    }
    CKC(dalloc(c, &c->d_err, 1));
    CKC(dalloc(c, &c->d_cum, 4));
    CKC(dalloc(c, &c->d_miss_u, Tn));
    CKC(dalloc(c, &c->d_victims, Tn));
    if (c->n > SMEM_SORT_MAX) CKC(dalloc(c, &c->d_sort_tmp, 4 * Tn));
    CKC(dalloc(c, &c->d_partial, (size_t)c->T * c->g.nh * c->D));
    if (backward_tiled() || c->g.bf16) {  // (bf16 Storage: the tiled backward only)
        c->bwd_tr = backward_tile_rows(c->D);
        c->bwd_ntiles = (c->n + c->bwd_tr - 1) / c->bwd_tr;
        const size_t tiles = (size_t)c->T * c->bwd_ntiles;
        CKC(dalloc(c, &c->d_tpart, tiles * 2 * c->D));
        CKC(dalloc(c, &c->d_seg_cnt, Tn));
        CKC(dalloc(c, &c->d_grp_cnt, tiles * 2));
        CKC(cudaMemset(c->d_seg_cnt, 0, Tn * sizeof(uint32_t)));
        CKC(cudaMemset(c->d_grp_cnt, 0, tiles * 2 * sizeof(uint32_t)));
        CKC(dalloc(c, &c->d_tctr, (size_t)RING * TCTR_STRIDE));
        CKC(cudaMemset(c->d_tctr, 0, (size_t)RING * TCTR_STRIDE * sizeof(uint32_t)));
    }
    CKC(dalloc(c, &c->d_pprof, 18 * (size_t)c->T + 2 + 4096));
    CKC(cudaMemset(c->d_pprof, 0, (18 * (size_t)c->T + 2 + 4096) * sizeof(unsigned long long)));
    CKC(cudaMemset(c->d_pprof + 18 * (size_t)c->T + 2, 0xFF, 1024 * sizeof(unsigned long long)));
    CKC(dalloc(c, &c->d_host, c->T));
    if (c->comm) {
        CKC(dalloc(c, &c->d_pooled_local, Tn / c->L * c->D));
        CKC(dalloc(c, &c->d_grad_local, Tn / c->L * c->D));
    }
    CKC(dalloc(c, &c->d_ctl, RING));
    CKC(dalloc(c, &c->d_xdone, RING));
    CKC(cudaMemset(c->d_xdone, 0, RING * sizeof(uint32_t)));
    c->idx_bytes = Tn * ((c->flags & SP_FLAG_INDEX_I32) ? 4 : 8);
    for (int r = 0; r < RING; r++) {
        cudaError_t st;
        c->ring[r] = carve(c, &st);
        CKC(st);
        void *p = nullptr;
        CKC(cudaMalloc(&p, c->idx_bytes));
        c->allocs.push_back(p);
        c->d_idx[r] = p;
    }
    CKC(cudaHostAlloc(&c->h_stage, c->idx_bytes * RING, cudaHostAllocDefault));
    CKC(cudaHostAlloc((void **)&c->h_err, sizeof(unsigned long long), cudaHostAllocDefault));
    *c->h_err = NO_ERR;
    CKC(cudaHostAlloc((void **)&c->h_errflag, sizeof(unsigned long long), cudaHostAllocMapped));
    *c->h_errflag = 0;
    CKC(cudaHostGetDevicePointer((void **)&c->d_errflag, c->h_errflag, 0));
    CKC(cudaHostAlloc((void **)&c->h_scat, sizeof(unsigned long long), cudaHostAllocMapped));
    *c->h_scat = 0;
    CKC(cudaHostGetDevicePointer((void **)&c->d_scat, c->h_scat, 0));
    CKC(cudaHostAlloc((void **)&c->h_wb, (size_t)c->XSR * Tn * c->D * sizeof(float), cudaHostAllocMapped));
    CKC(cudaHostGetDevicePointer((void **)&c->hd_wb, c->h_wb, 0));
    CKC(cudaHostAlloc((void **)&c->h_staged, RING * sizeof(unsigned long long), cudaHostAllocMapped));
    std::memset(c->h_staged, 0, RING * sizeof(unsigned long long));
    CKC(cudaHostGetDevicePointer((void **)&c->hd_staged, c->h_staged, 0));
    // CPU gather when a batch's rows are few (latency, not copy bandwidth,
    // dominates): +8-9% on Kaggle (T*n*D*4 = 13.6 MB); the GPU pull wins on
    // Terabyte (54.5 MB: 7.0k vs 6.0k it/s) and high-pooling (671 MB: 96 vs
    // 54 it/s), where the CPU copy threads become the bound
    // Missed rows: all gathered by the CPU when a batch's rows are few
    // (latency, not copy bandwidth, dominates: Kaggle); above 32 MB of rows
    // per batch the hybrid split, half gathered by the CPU while the transfer
    // kernel pulls the other half (Terabyte, measured: 8.0k vs 7.0k it/s for
    // the pure GPU pull, whose random host reads are bound by host-side
    // address translation and slow the Train kernels; profiles/r02_a3_sweep)
    c->cpu_gather = true;
    if ((double)c->T * c->n * c->D * sizeof(float) > 32.0 * (1 << 20)) c->gather_q16 = 32768;
    if (const char *e = getenv("SP_CPU_GATHER")) {  // 1: every missed row gathered, 0: every one pulled
        c->cpu_gather = atoi(e) != 0;
        c->gather_q16 = 65536;
    }
    // hybrid split (SP_GATHER_FRAC in (0, 1)): the CPU gathers that share of
    // each batch's missed rows while the transfer kernel pulls the rest
    if (const char *e = getenv("SP_GATHER_FRAC")) {
        const double f = atof(e);
        if (f > 0.0 && f < 1.0) {
            c->cpu_gather = true;
            c->gather_q16 = (uint32_t)(f * 65536.0);
        } else if (f >= 1.0) {
            c->cpu_gather = true;
        } else {
            c->cpu_gather = false;
        }
    }
    if (const char *e = getenv("SP_WRITEBACK")) c->gpu_wb = std::string(e) == "gpu";
    if (c->host_threads <= 0) {
        // row-copy helpers per pool from the node's cores, shared by the
        // contexts of one node (one per GPU: desc.world of them), at most 6
        const long ncpu = std::max(1L, sysconf(_SC_NPROCESSORS_ONLN));
        const long ctx = std::max(1, d->world);
        const long pools = (c->cpu_gather ? 2 : 1) * ctx;
        c->host_threads = (int)std::max(1L, std::min(6L, (ncpu - pools) / pools));
    }
    c->scatter_helpers = c->gather_helpers = c->host_threads;
    if (const char *e = getenv("SP_SCATTER_THREADS")) c->scatter_helpers = std::max(1, atoi(e) - 1);
    if (const char *e = getenv("SP_GATHER_THREADS")) c->gather_helpers = std::max(1, atoi(e) - 1);
    if (c->cpu_gather) {
        CKC(cudaHostAlloc((void **)&c->hl_ready, (size_t)RING * c->T * sizeof(unsigned long long), cudaHostAllocMapped));
        CKC(cudaHostAlloc((void **)&c->hl_m, (size_t)RING * c->T * sizeof(uint32_t), cudaHostAllocMapped));
        CKC(cudaHostAlloc((void **)&c->hl_row, (size_t)RING * Tn * sizeof(uint32_t), cudaHostAllocMapped));
        std::memset(c->hl_ready, 0, (size_t)RING * c->T * sizeof(unsigned long long));
        unsigned long long *dr;
        uint32_t *dm, *drow;
        CKC(cudaHostGetDevicePointer((void **)&dr, c->hl_ready, 0));
        CKC(cudaHostGetDevicePointer((void **)&dm, c->hl_m, 0));
        CKC(cudaHostGetDevicePointer((void **)&drow, c->hl_row, 0));
        for (int r = 0; r < RING; r++) {
            c->hl_dev[r].ready = dr + (size_t)r * c->T;
            c->hl_dev[r].m = dm + (size_t)r * c->T;
            c->hl_dev[r].row = drow + (size_t)r * Tn;
        }
        CKC(cudaHostAlloc((void **)&c->h_in, (size_t)c->XSR * Tn * c->D * sizeof(float), cudaHostAllocMapped));
        if (const char *e = getenv("SP_GATHER_DMA")) c->gather_dma = atoi(e) != 0;
        if (c->gather_dma) CKC(dalloc(c, &c->d_in, (size_t)c->XSR * Tn * c->D));
        CKC(cudaHostGetDevicePointer((void **)&c->hd_in, c->h_in, 0));
        CKC(cudaHostAlloc((void **)&c->h_gathered, sizeof(unsigned long long), cudaHostAllocMapped));
        *c->h_gathered = 0;
        CKC(cudaHostGetDevicePointer((void **)&c->d_gathered, c->h_gathered, 0));
    }
    CKC(cudaHostAlloc((void **)&c->h_wbdst, (size_t)c->XSR * Tn * sizeof(unsigned long long), cudaHostAllocMapped));
    CKC(cudaHostGetDevicePointer((void **)&c->hd_wbdst, c->h_wbdst, 0));
    CKC(cudaHostAlloc((void **)&c->h_scnt, RING * sizeof(unsigned long long), cudaHostAllocMapped));
    std::memset(c->h_scnt, 0, RING * sizeof(unsigned long long));
    CKC(cudaHostGetDevicePointer((void **)&c->hd_scnt, c->h_scnt, 0));

    // initial state
    std::vector<long long> rows64(c->rows.begin(), c->rows.end());
    CKC(cudaMemcpy(c->d_row_off, c->row_off.data(), (c->T + 1) * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    CKC(cudaMemcpy(c->d_rows, rows64.data(), c->T * sizeof(long long), cudaMemcpyHostToDevice));
    CKC(cudaMemcpy(c->d_slot_base, c->slot_base.data(), (c->T + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice));
    CKC(cudaMemcpy(c->d_host, hdev.data(), c->T * sizeof(float *), cudaMemcpyHostToDevice));
    CKC(cudaMemset(c->d_hitmap, 0xFF, c->hit_total * sizeof(uint32_t)));
    CKC(cudaMemset(c->d_resident, 0xFF, (size_t)c->S_total * sizeof(uint32_t)));
    {
        std::vector<int32_t> vac((size_t)c->S_total, VACANT);
        CKC(cudaMemcpy(c->d_last_use, vac.data(), vac.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(c->d_next_need, vac.data(), vac.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    // initial log (class 0): every slot vacant, ascending slot order
    if (c->log_classes > 0) {
        std::vector<unsigned long long> lb0(c->T);
        for (int t = 0; t < c->T; t++) lb0[t] = lbase[(size_t)t * NCl];
        unsigned long long *d_lb0 = nullptr;
        CKC(dalloc(c, &d_lb0, c->T));
        CKC(cudaMemcpy(d_lb0, lb0.data(), c->T * sizeof(unsigned long long), cudaMemcpyHostToDevice));
        CKC(launch_log_init(c->d_slot_base, d_lb0, c->T, c->S_total, c->d_log_slot, c->d_log_stamp, nullptr));
    }
    CKC(cudaMemcpy(c->d_log_base, lbase.data(), lbase.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    CKC(cudaMemcpy(c->d_log_cap, lcap.data(), lbase.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    CKC(cudaMemcpy(c->d_log_head, lhead.data(), lbase.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    CKC(cudaMemcpy(c->d_log_tail, ltail.data(), lbase.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    CKC(cudaMemcpy(c->d_pin_base, c->pin_base.data(), c->T * sizeof(uint32_t), cudaMemcpyHostToDevice));
    c->log_skip.assign(c->T, 0);
    for (int t = 0; t < c->T; t++) c->log_skip[t] = c->slots[t] >= c->rows[t] ? 1 : 0;
    CKC(dalloc(c, &c->d_log_skip, c->T));
    CKC(cudaMemcpy(c->d_log_skip, c->log_skip.data(), c->T, cudaMemcpyHostToDevice));
    CKC(cudaMemset(c->d_err, 0xFF, sizeof(unsigned long long)));
    CKC(cudaMemset(c->d_cum, 0, 4 * sizeof(unsigned long long)));
    CKC(cudaMemset(c->d_storage, 0, (size_t)c->S_total * c->D * (c->g.bf16 ? 2 : sizeof(float))));
    CKC(cudaDeviceSynchronize());
#undef CKC
    // transfer engine: helpers + worker
    if (!c->gpu_wb) {
        if (const char *e = getenv("SP_SHARED_POOL")) c->shared_pool = atoi(e) != 0 && c->cpu_gather;
        c->spool.start(c->shared_pool ? c->scatter_helpers + c->gather_helpers : c->scatter_helpers);
        c->scatter_worker = std::thread(scatter_main, c);
    }
    if (c->cpu_gather) {
        if (!c->shared_pool) c->gpool.start(c->gather_helpers);
        c->gather_worker = std::thread(gather_main, c);
    }
    *out = c;
    return SP_OK;
}

// csr != nullptr: a ragged batch {values, offsets} (host), expanded on the
// GPU into the padded [T][N][L] layout of ring slot r (sp_plan_csr)
static sp_status plan_impl(sp_ctx *c, const void *idx, bool on_device, const int64_t *const *csr = nullptr) {
    if (!c || (!idx && !csr)) return SP_ERR_INVALID_ARG;
    if (sp_status s = check_async_error(c)) return s;
    if (c->eod) return fail(c, SP_ERR_STATE, "sp_plan after sp_end_of_data (call sp_flush first)");
    const long long j = c->pushed;
    const int r = (int)(j % RING);
    if (j >= RING && c->trained < j - RING + 1)
        return fail(c, SP_ERR_STATE, "sp_plan: more than 16 batches ahead of sp_train");
    CK(cudaSetDevice(c->device));
    // Plan(b) runs beside dedup(j) once B(b+F) = B(j-1) has been deduped
    const long long b = j - c->F - 1;
    const bool do_plan = b >= 0 && b == c->planned;
    if (do_plan)
        if (sp_status s = wait_gather_slot(c, b)) return s;
    if (j >= RING) CK(cudaStreamWaitEvent(c->plan_s, c->ev_train[r], 0));  // ring slot r reused
    const void *dev_idx;
    if (csr) {
        const int64_t *vals = csr[0], *offs = csr[1];
        const long long nbags = (long long)c->T * c->N, nnz = offs[nbags];
        const size_t per = (size_t)c->T * c->n + (size_t)nbags + 1;
        if (!c->h_csr) {
            CK(cudaHostAlloc((void **)&c->h_csr, per * RING * sizeof(int64_t), cudaHostAllocDefault));
            void *p = nullptr;
            CK(cudaMalloc(&p, per * RING * sizeof(int64_t)));
            c->allocs.push_back(p);
            c->d_csr = static_cast<int64_t *>(p);
        }
        int64_t *hs = c->h_csr + (size_t)r * per;
        if (c->h2d_used[r]) CK(cudaEventSynchronize(c->ev_h2d[r]));
        std::memcpy(hs, offs, (nbags + 1) * sizeof(int64_t));
        std::memcpy(hs + nbags + 1, vals, (size_t)nnz * sizeof(int64_t));
        int64_t *ds = c->d_csr + (size_t)r * per;
        const size_t bytes = ((size_t)nbags + 1 + (size_t)nnz) * sizeof(int64_t);
        CK(cudaMemcpyAsync(ds, hs, bytes, cudaMemcpyHostToDevice, c->plan_s));
        CK(cudaEventRecord(c->ev_h2d[r], c->plan_s));
        c->h2d_used[r] = true;
        c->h2d_index_bytes += (long long)bytes;
        CK(launch_csr_pad(reinterpret_cast<const long long *>(ds + nbags + 1), reinterpret_cast<const long long *>(ds), nbags, c->L, c->d_idx[r], (c->flags & SP_FLAG_INDEX_I32) ? 1 : 0,
                          c->plan_s));
        dev_idx = c->d_idx[r];
    } else if (on_device) {
        // indices produced on the caller's stream
        CK(cudaEventRecord(c->ev_user, c->compute));
        CK(cudaStreamWaitEvent(c->plan_s, c->ev_user, 0));
        dev_idx = idx;
    } else {
        char *stage = static_cast<char *>(c->h_stage) + (size_t)r * c->idx_bytes;
        if (c->h2d_used[r]) CK(cudaEventSynchronize(c->ev_h2d[r]));
        std::memcpy(stage, idx, c->idx_bytes);
        CK(cudaMemcpyAsync(c->d_idx[r], stage, c->idx_bytes, cudaMemcpyHostToDevice, c->plan_s));
        CK(cudaEventRecord(c->ev_h2d[r], c->plan_s));
        c->h2d_used[r] = true;
        c->h2d_index_bytes += (long long)c->idx_bytes;
        dev_idx = c->d_idx[r];
    }
    PushArgs a = push_args(c);
    a.has_new = 1;
    a.j = j;
    a.idx = dev_idx;
    a.nb = c->ring[r];
    a.do_plan = do_plan ? 1 : 0;
    if (do_plan) {
        a.b = b;
        a.pb = c->ring[b % RING];
        if (c->cpu_gather) a.hl = c->hl_dev[b % RING];
        a.has_future = 1;
        a.fb = c->ring[(b + c->F) % RING];
    }
    CK(launch(c, SP_K_PLAN, do_plan ? b : j, c->plan_s, [&] { return launch_push(a, c->plan_s); }));
    if (do_plan) {
        CK(cudaEventRecord(c->ev_plan[b % RING], c->plan_s));
        c->planned = b + 1;
    }
    c->pushed = j + 1;
    return pump(c);
}

sp_status sp_plan(sp_ctx *c, const void *idx) {
    return plan_impl(c, idx, c && (c->flags & SP_FLAG_INDEX_DEVICE));
}

sp_status sp_plan_device(sp_ctx *c, const void *idx) { return plan_impl(c, idx, true); }

sp_status sp_plan_csr(sp_ctx *c, const int64_t *values, const int64_t *offsets) {
    if (!c || !offsets) return SP_ERR_INVALID_ARG;
    if (!(c->flags & SP_FLAG_PADDING)) return fail(c, SP_ERR_INVALID_ARG, "sp_plan_csr needs SP_FLAG_PADDING");
    const long long nbags = (long long)c->T * c->N;
    if (offsets[0] != 0) return fail(c, SP_ERR_INVALID_ARG, "sp_plan_csr: offsets[0] must be 0");
    for (long long k = 0; k < nbags; k++) {
        const long long len = offsets[k + 1] - offsets[k];
        if (len < 0 || len > c->L)
            return fail(c, SP_ERR_INVALID_ARG, "sp_plan_csr: bag " + std::to_string(k) + " has " +
                                                   std::to_string(len) + " lookups (pooling " + std::to_string(c->L) + ")");
    }
    if (offsets[nbags] > 0 && !values) return SP_ERR_INVALID_ARG;
    const int64_t *csr[2] = {values, offsets};
    return plan_impl(c, nullptr, false, csr);
}

sp_status sp_pin_rows(sp_ctx *c, int32_t t, const int64_t *ids, int64_t count) {
    if (!c || t < 0 || t >= c->T || count < 0 || (count > 0 && !ids)) return SP_ERR_INVALID_ARG;
    if (sp_status s = check_async_error(c)) return s;
    if (c->pushed != 0 || c->pinned_t[t]) return fail(c, SP_ERR_STATE, "sp_pin_rows: only once per table, before the first sp_plan");
    if (count > c->slots[t]) return fail(c, SP_ERR_INVALID_ARG, "sp_pin_rows: more rows than slots");
    std::vector<int64_t> sorted(ids, ids + count);
    std::sort(sorted.begin(), sorted.end());
    for (int64_t k = 0; k < count; k++)
        if (sorted[k] < 0 || sorted[k] >= c->rows[t] || (k && sorted[k] == sorted[k - 1]))
            return fail(c, SP_ERR_INVALID_ARG, "sp_pin_rows: IDs must be distinct and in range");
    CK(cudaSetDevice(c->device));
    const uint32_t base = c->slot_base[t + 1] - (uint32_t)count;
    if (count) {
        // rows -> Storage[base + k] (host gather into pinned staging, one H2D)
        float *h = nullptr;
        CK(cudaHostAlloc((void **)&h, (size_t)count * c->D * sizeof(float), cudaHostAllocDefault));
        std::vector<uint32_t> slot((size_t)count), res((size_t)count);
        for (int64_t k = 0; k < count; k++) {
            std::memcpy(h + (size_t)k * c->D, c->host[t] + (size_t)ids[k] * c->D, (size_t)c->D * sizeof(float));
            res[k] = (uint32_t)ids[k];
            slot[k] = base + (uint32_t)k;
        }
        cudaError_t e = c->g.bf16  // bf16 Storage: rows rounded on the GPU (R28)
                            ? launch_rows_to_bf16(h, reinterpret_cast<char *>(c->d_storage) + (size_t)base * c->D * 2,
                                                  count, c->D, nullptr)
                            : cudaMemcpy(c->d_storage + (size_t)base * c->D, h, (size_t)count * c->D * sizeof(float),
                                         cudaMemcpyHostToDevice);
        if (e == cudaSuccess && c->g.bf16) e = cudaDeviceSynchronize();
        cudaFreeHost(h);
        CK(e);
        CK(cudaMemcpy(c->d_resident + base, res.data(), count * sizeof(uint32_t), cudaMemcpyHostToDevice));
        for (int64_t k = 0; k < count; k++)  // Hit-Map entries (count small: one copy each is fine)
            CK(cudaMemcpy(c->d_hitmap + c->row_off[t] + (size_t)ids[k], &slot[k], sizeof(uint32_t), cudaMemcpyHostToDevice));
    }
    c->pin_base[t] = base;
    c->pinned_t[t] = true;
    CK(cudaMemcpy(c->d_pin_base + t, &base, sizeof(uint32_t), cudaMemcpyHostToDevice));
    // never evicts iff the dynamic slots can hold every unpinned row
    c->log_skip[t] = (long long)(base - c->slot_base[t]) >= c->rows[t] - count ? 1 : 0;
    CK(cudaMemcpy(c->d_log_skip + t, &c->log_skip[t], 1, cudaMemcpyHostToDevice));
    return SP_OK;
}

sp_status sp_copy_batch_stats(sp_ctx *c, int64_t b, uint32_t *host_out) {
    if (!c || !host_out) return SP_ERR_INVALID_ARG;
    if (b < 0 || b >= c->planned || c->pushed > b + RING)
        return fail(c, SP_ERR_STATE, "sp_copy_batch_stats: batch not planned or ring entry recycled");
    CK(cudaSetDevice(c->device));
    CK(cudaStreamWaitEvent(c->compute, c->ev_plan[b % RING], 0));
    CK(cudaMemcpyAsync(host_out, c->ring[b % RING].stats, (size_t)c->T * 4 * sizeof(uint32_t),
                       cudaMemcpyDeviceToHost, c->compute));
    return SP_OK;
}

sp_status sp_set_profiling(sp_ctx *c, int32_t on) {
    if (!c) return SP_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    std::lock_guard<std::mutex> lk(c->prof_mu);
    if (on) {
        // per-launch k_push spans restart with this profiling window
        const size_t so = 18 * (size_t)c->T + 2;
        CK(cudaMemsetAsync(c->d_pprof + so, 0xFF, 1024 * sizeof(unsigned long long), c->plan_s));
        CK(cudaMemsetAsync(c->d_pprof + so + 1024, 0, 3072 * sizeof(unsigned long long), c->plan_s));
        if (!c->prof_ref) CK(cudaEventCreate(&c->prof_ref));
        CK(cudaEventRecord(c->prof_ref, c->compute));
        c->timeline.clear();
        c->profiling = true;
    } else {
        c->profiling = false;
    }
    return SP_OK;
}

sp_status sp_get_timeline(sp_ctx *c, int32_t *kind, int64_t *batch, double *start_ms, double *end_ms,
                          int64_t cap, int64_t *n) {
    if (!c || !n) return SP_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    CK(cudaDeviceSynchronize());
    std::lock_guard<std::mutex> lk(c->prof_mu);
    harvest_profile(c, true);
    *n = (int64_t)c->timeline.size();
    for (int64_t i = 0; i < std::min<int64_t>(cap, *n); i++) {
        kind[i] = c->timeline[i].kind;
        batch[i] = c->timeline[i].batch;
        start_ms[i] = c->timeline[i].start_ms;
        end_ms[i] = c->timeline[i].end_ms;
    }
    return SP_OK;
}

sp_status sp_end_of_data(sp_ctx *c) {
    if (!c) return SP_ERR_INVALID_ARG;
    if (sp_status s = check_async_error(c)) return s;
    CK(cudaSetDevice(c->device));
    c->eod = true;
    while (c->planned < c->pushed)
        if (sp_status s = enqueue_plan_only(c, c->planned)) return s;
    return pump(c);
}

sp_status sp_forward(sp_ctx *c, float *pooled) {
    if (!c || !pooled) return SP_ERR_INVALID_ARG;
    if (sp_status s = check_async_error(c)) return s;
    if (c->fwd_pending) return fail(c, SP_ERR_STATE, "sp_forward twice without sp_train");
    const long long b = c->forwarded;
    if (b >= c->planned)
        return fail(c, SP_ERR_STATE, "sp_forward: batch not planned yet (push B(b+F+1) or call sp_end_of_data)");
    CK(cudaSetDevice(c->device));
    if (sp_status s = pump(c)) return s;
    if (c->xfer_enq <= b) return fail(c, SP_ERR_STATE, "sp_forward: transfer not schedulable");
    CK(cudaStreamWaitEvent(c->compute, c->ev_xfer[b % RING], 0));
    TrainArgs a = train_args(c, b);
    a.pooled = c->comm ? c->d_pooled_local : pooled;
    CK(launch(c, SP_K_FORWARD, b, c->compute, [&] { return launch_forward(a, c->compute); }));
    if (c->comm)
        if (sp_status s = exchange(c, true, pooled, nullptr)) return s;
    c->forwarded = b + 1;
    c->fwd_pending = true;
    return SP_OK;
}

sp_status sp_train(sp_ctx *c, const float *grad, float lr) {
    if (!c || !grad) return SP_ERR_INVALID_ARG;
    if (sp_status s = check_async_error(c)) return s;
    if (!c->fwd_pending) return fail(c, SP_ERR_STATE, "sp_train without a preceding sp_forward");
    CK(cudaSetDevice(c->device));
    const long long b = c->trained;
    if (c->comm)
        if (sp_status s = exchange(c, false, nullptr, grad)) return s;
    TrainArgs a = train_args(c, b);
    a.grad = c->comm ? c->d_grad_local : grad;
    a.lr = lr;
    CK(launch(c, SP_K_BACKWARD, b, c->compute, [&] {
        return launch_backward(a, c->compute);
    }));
    CK(cudaEventRecord(c->ev_train[b % RING], c->compute));
    c->trained = b + 1;
    c->trained_pub.store(b + 1, std::memory_order_release);
    c->fwd_pending = false;
    return pump(c);
}

sp_status sp_surrogate_grad(sp_ctx *c, const float *pooled, float *grad, int64_t count, float gamma,
                            float delta) {
    if (!c || !pooled || !grad || count < 0 || count % 4) return SP_ERR_INVALID_ARG;
    if (c->poisoned != SP_OK) return c->poisoned;
    CK(cudaSetDevice(c->device));
    if (count == 0) count = c->comm ? (long long)c->T_all * (c->N / c->world) * c->D : (long long)c->T * c->N * c->D;
    CK(launch(c, SP_K_SURROGATE, c->trained, c->compute,
              [&] {
                  return launch_surrogate(pooled, grad, count, gamma, delta, c->compute,
                                          c->span_on ? c->d_span : nullptr, c->trained);
              }));
    return SP_OK;
}

sp_status sp_prefill(sp_ctx *c) {
    if (!c) return SP_ERR_INVALID_ARG;
    if (sp_status s = check_async_error(c)) return s;
    if (c->pushed != 0) return fail(c, SP_ERR_STATE, "sp_prefill: only before the first sp_plan");
    for (int t = 0; t < c->T; t++)
        if (c->slots[t] != c->rows[t]) return fail(c, SP_ERR_INVALID_ARG, "sp_prefill: needs slots == rows for every table");
    CK(cudaSetDevice(c->device));
    for (int t = 0; t < c->T; t++) {
        if (c->g.bf16)  // bf16 Storage: every row rounded on the GPU as it is read (R28)
            CK(launch_rows_to_bf16(c->host_dev[t], reinterpret_cast<char *>(c->d_storage) + (size_t)c->slot_base[t] * c->D * 2,
                                   c->rows[t], c->D, c->plan_s));
        else
            CK(cudaMemcpyAsync(c->d_storage + (size_t)c->slot_base[t] * c->D, c->host[t],
                               (size_t)c->rows[t] * c->D * sizeof(float), cudaMemcpyHostToDevice, c->plan_s));
    }
    CK(launch_prefill_map(c->d_slot_base, c->d_row_off, c->T, c->S_total, c->d_resident, c->d_hitmap, c->plan_s));
    {   // RANDOM: every dynamic slot is occupied
        std::vector<uint32_t> nf(c->T);
        for (int t = 0; t < c->T; t++) nf[t] = (uint32_t)c->slots[t];
        CK(cudaMemcpyAsync(c->d_nfill, nf.data(), c->T * sizeof(uint32_t), cudaMemcpyHostToDevice, c->plan_s));
        CK(cudaStreamSynchronize(c->plan_s));
    }
    CK(cudaStreamSynchronize(c->plan_s));
    return SP_OK;
}

sp_status sp_flush(sp_ctx *c) {
    if (!c) return SP_ERR_INVALID_ARG;
    if (sp_status s = check_async_error(c)) return s;
    if (c->trained != c->pushed || c->fwd_pending)
        return fail(c, SP_ERR_STATE, "sp_flush: every pushed batch must be trained first");
    CK(cudaSetDevice(c->device));
    // the transfer engine writes back every victim of every batch
    if (sp_status s = wait_engine(c, [&] { return c->gpu_wb || c->x_scattered.load(std::memory_order_acquire) >= c->planned; }))
        return s;
    CK(cudaStreamSynchronize(c->plan_s));
    CK(cudaStreamSynchronize(c->xfer_s));
    CK(cudaStreamSynchronize(c->xfer_s2));
    CK(cudaStreamSynchronize(c->compute));
    if (sp_status s = sync_error(c)) return s;
    FlushArgs a{};
    a.g = c->g;
    a.S_total = (int)c->S_total;
    a.slot_base = c->d_slot_base;
    a.resident = c->d_resident;
    a.storage = c->d_storage;
    a.host = c->d_host;
    CK(launch(c, SP_K_FLUSH, c->trained, c->compute, [&] { return launch_flush(a, c->compute); }));
    CK(cudaStreamSynchronize(c->compute));
    c->eod = false;  // a flush is a checkpoint: the caller may continue pushing
    return SP_OK;
}

}  // extern "C"

namespace {

void drop_graphs(sp_ctx *c) {
    for (int r = 0; r < RING; r++) {
        if (c->gplan[r]) cudaGraphExecDestroy(c->gplan[r]);
        if (c->gcomp[r]) cudaGraphExecDestroy(c->gcomp[r]);
        c->gplan[r] = c->gcomp[r] = nullptr;
    }
    c->g_next_j = -1;
}

// Capture the two graphs of residue r = k % RING for step k: the push of
// B(j = k+F+P+1) with Plan(k+P), and forward / surrogate / train of batch k.
sp_status capture_step(sp_ctx *c, int r) {
    const long long ahead = c->F + c->P + 1;
    const int rj = (int)((r + ahead) % RING), rb = (int)((r + c->P) % RING),
              rf = (int)((r + c->P + c->F) % RING);
    const sp_ctx::GraphKey &k = c->gkey;
    cudaGraph_t gr = nullptr;
    // plan stream: [wait Train(j - RING): ring slot reuse] -> k_push -> [record ev_plan]
    PushArgs a = push_args(c);
    a.has_new = 1;
    a.do_plan = 1;
    a.has_future = 1;
    a.idx = k.trace;
    a.nb = c->ring[rj];
    a.pb = c->ring[rb];
    if (c->cpu_gather) a.hl = c->hl_dev[rb];
    a.fb = c->ring[rf];
    a.ctl = c->d_ctl;
    a.ctl_r = r;
    a.idx_stride = k.stride;
    CK(cudaStreamBeginCapture(c->cap_hi, cudaStreamCaptureModeThreadLocal));
    cudaStreamWaitEvent(c->cap_hi, c->ev_train[rj], cudaEventWaitExternal);
    if (c->stage_timing) cudaEventRecordWithFlags(c->sev[r][0], c->cap_hi, cudaEventRecordExternal);
    launch_push(a, c->cap_hi);
    if (c->stage_timing) cudaEventRecordWithFlags(c->sev[r][1], c->cap_hi, cudaEventRecordExternal);
    cudaEventRecordWithFlags(c->ev_plan[rb], c->cap_hi, cudaEventRecordExternal);
    CK(cudaStreamEndCapture(c->cap_hi, &gr));
    CK(cudaGraphInstantiate(&c->gplan[r], gr, 0));
    cudaGraphDestroy(gr);
    // compute stream: [wait Transfer(k)] -> forward -> surrogate -> backward -> [record ev_train]
    TrainArgs ta = train_args(c, r);
    ta.pooled = k.pooled;
    TrainArgs tb = train_args(c, r);
    tb.grad = k.grad;
    tb.lr = k.lr;
    CK(cudaStreamBeginCapture(c->cap_s, cudaStreamCaptureModeThreadLocal));
    cudaStreamWaitEvent(c->cap_s, c->ev_xfer[r], cudaEventWaitExternal);
    const bool st = c->stage_timing;
    // the event pass captures without programmatic dependent launch: an event
    // node between PDL-launched kernels would otherwise also time the early
    // launch's wait, and the events are to bracket each kernel alone
    const int pdl_saved = g_pdl;
    if (st) g_pdl = 0;
    if (st) cudaEventRecordWithFlags(c->sev[r][2], c->cap_s, cudaEventRecordExternal);
    launch_forward(ta, c->cap_s);
    if (st) cudaEventRecordWithFlags(c->sev[r][3], c->cap_s, cudaEventRecordExternal);
    launch_surrogate(k.pooled, k.grad, (long long)c->T * c->N * c->D, k.gamma, k.delta, c->cap_s,
                     c->span_on ? c->d_span : nullptr, r);
    if (st) cudaEventRecordWithFlags(c->sev[r][4], c->cap_s, cudaEventRecordExternal);
    launch_backward(tb, c->cap_s);
    if (st) cudaEventRecordWithFlags(c->sev[r][5], c->cap_s, cudaEventRecordExternal);
    g_pdl = pdl_saved;
    cudaEventRecordWithFlags(c->ev_train[r], c->cap_s, cudaEventRecordExternal);
    CK(cudaStreamEndCapture(c->cap_s, &gr));
    CK(cudaGraphInstantiate(&c->gcomp[r], gr, 0));
    cudaGraphDestroy(gr);
    c->sev_used[r][0] = st;
    return SP_OK;
}

// one steady-state step k through the graphs (2 graph launches)
sp_status graph_step(sp_ctx *c) {
    const long long k = c->trained, j = c->pushed, b = c->planned;  // j = k+F+P+1, b = k+P = j-F-1
    const int r = (int)(k % RING);
    if (!c->gplan[r])
        if (sp_status s = capture_step(c, r)) return s;
    if (c->g_next_j != j)  // (re)enter graph mode: seed the device batch-index chain
        CK(cudaMemcpyAsync(c->d_ctl + r, &j, sizeof j, cudaMemcpyHostToDevice, c->plan_s));
    if (sp_status s = wait_gather_slot(c, b)) return s;
    CK(cudaGraphLaunch(c->gplan[r], c->plan_s));
    c->pushed = j + 1;
    c->planned = b + 1;
    c->g_next_j = j + 1;
    if (sp_status s = pump(c)) return s;
    if (c->xfer_enq <= k) return fail(c, SP_ERR_STATE, "graph step: transfer not schedulable");
    CK(cudaGraphLaunch(c->gcomp[r], c->compute));
    c->forwarded = k + 1;
    c->trained = k + 1;
    c->trained_pub.store(k + 1, std::memory_order_release);
    c->graph_steps++;
    if (sp_status s = pump(c)) return s;
    {
        std::lock_guard<std::mutex> lk(c->prof_mu);
        for (int kind : {SP_K_PLAN, SP_K_FORWARD, SP_K_SURROGATE, SP_K_BACKWARD}) c->launches[kind] += 1;
    }
    return SP_OK;
}

}  // namespace

extern "C" {

sp_status sp_run_steps(sp_ctx *c, const void *indices, int64_t num_batches, int64_t stride,
                       int64_t steps, float *pooled, float *grad, float gamma, float delta,
                       float lr, uint32_t *stats_out) {
    if (!c || !indices || !pooled || !grad || num_batches < 0 || stride <= 0 || steps < 0)
        return SP_ERR_INVALID_ARG;
    if (c->fwd_pending) return fail(c, SP_ERR_STATE, "sp_run_steps between sp_forward and sp_train");
    CK(cudaSetDevice(c->device));
    {   // device memory, or pinned + mapped host memory read by k_push over the
        // host link (the batch's H2D is then part of the plan kernel)
        // (checked at the next batch to push: `indices` itself may be a base
        // offset below the caller's array, batch j living at indices + j*stride)
        const void *first = static_cast<const char *>(indices) + c->pushed * stride;
        cudaPointerAttributes pa{};
        if (steps > 0 && c->pushed < num_batches && (cudaPointerGetAttributes(&pa, first) != cudaSuccess || pa.type == cudaMemoryTypeUnregistered ||
                          (pa.type == cudaMemoryTypeHost && pa.devicePointer != first))) {
            (void)cudaGetLastError();
            return fail(c, SP_ERR_INVALID_ARG, "sp_run_steps: indices must be device memory or pinned host memory");
        }
    }
    const long long ahead = c->F + c->P + 1;
    const char *base = static_cast<const char *>(indices);
    sp_ctx::GraphKey key;
    key.trace = indices;
    key.stride = stride;
    key.pooled = pooled;
    key.grad = grad;
    key.gamma = gamma;
    key.delta = delta;
    key.lr = lr;
    if (!(key == c->gkey)) {
        drop_graphs(c);
        c->gkey = key;
    }
    const bool graphs_ok = !stats_out && !getenv("SP_NO_GRAPHS") && !c->comm;  // sharded: eager steps
    for (int64_t k = 0; k < steps; k++) {
        if (sp_status s = check_async_error(c)) return s;
        // steady state: the look-ahead is full and one push per step keeps it so
        const bool steady = graphs_ok && !c->eod && !c->profiling.load() && c->pushed == c->trained + ahead &&
                            c->planned == c->trained + c->P && c->pushed + 1 <= num_batches &&
                            c->trained >= RING;
        if (steady) {
            const auto g0 = std::chrono::steady_clock::now();
            if (sp_status s = graph_step(c)) return s;
            c->graph_step_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(
                                    std::chrono::steady_clock::now() - g0).count();
            continue;
        }
        c->g_next_j = -1;
        // keep the look-ahead full (first call: F+P+1 batches)
        while (c->pushed < std::min<long long>(num_batches, c->trained + ahead + 1) && !c->eod)
            if (sp_status s = plan_impl(c, base + c->pushed * stride, true)) return s;
        // the trace is exhausted and the next Plan needs a future that will
        // never come: truncate the window (sp_end_of_data)
        if (c->planned <= c->trained && c->pushed >= num_batches && !c->eod)
            if (sp_status s = sp_end_of_data(c)) return s;
        const long long b = c->trained;
        if (sp_status s = sp_forward(c, pooled)) return s;
        if (sp_status s = sp_surrogate_grad(c, pooled, grad, 0, gamma, delta)) return s;
        if (sp_status s = sp_train(c, grad, lr)) return s;
        if (stats_out)
            if (sp_status s = sp_copy_batch_stats(c, b, stats_out + (size_t)k * c->T * 4)) return s;
    }
    return SP_OK;
}

sp_status sp_destroy(sp_ctx *c) {
    if (!c) return SP_ERR_INVALID_ARG;
    destroy_all(c);
    return SP_OK;
}

const char *sp_error_string(const sp_ctx *c) {
    if (!c) return "null context";
    return c->err.c_str();
}

sp_status sp_last_error_batch(const sp_ctx *c, int64_t *batch, int32_t *table) {
    if (!c) return SP_ERR_INVALID_ARG;
    if (batch) *batch = c->err_batch;
    if (table) *table = c->err_table;
    return c->poisoned;
}

sp_status sp_get_stats(sp_ctx *c, sp_stats *o) {
    if (!c || !o) return SP_ERR_INVALID_ARG;
    std::memset(o, 0, sizeof *o);
    cudaSetDevice(c->device);
    o->pushed = c->pushed;
    o->planned = c->planned;
    o->transferred = c->x_enqueued.load();
    o->forwarded = c->forwarded;
    o->trained = c->trained;
    unsigned long long cum[4] = {0, 0, 0, 0};
    if (c->poisoned != SP_ERR_CUDA) {
        cudaStreamSynchronize(c->plan_s);
        cudaMemcpy(cum, c->d_cum, sizeof cum, cudaMemcpyDeviceToHost);
    }
    o->uniques = (int64_t)cum[0];
    o->hits = (int64_t)cum[1];
    o->misses = (int64_t)cum[2];
    o->evictions = (int64_t)cum[3];
    o->h2d_index_bytes = c->h2d_index_bytes;
    o->h2d_row_bytes = (int64_t)cum[2] * c->D * 4;
    o->d2h_row_bytes = (int64_t)cum[3] * c->D * 4;
    std::lock_guard<std::mutex> lk(c->prof_mu);
    o->host_gather_ms = c->x_gather_ns.load() * 1e-6;
    o->host_scatter_ms = c->x_scatter_ns.load() * 1e-6;
    o->host_rows_gathered = c->x_rows_g.load();
    o->host_rows_scattered = c->x_rows_s.load();
    o->wait_xfer_ms = c->wait_xfer_ns * 1e-6;
    o->wait_list_ms = c->wait_list_ns * 1e-6;
    o->graph_steps = c->graph_steps;
    o->graph_step_host_ms = c->graph_step_ns * 1e-6;
    o->transfer_mode = c->cpu_gather ? (c->gather_q16 < 65536 ? SP_XFER_HYBRID
                                                              : (c->gather_dma ? SP_XFER_GATHER_DMA : SP_XFER_CPU_GATHER))
                                     : SP_XFER_GPU_PULL;
    o->gather_share = c->cpu_gather ? c->gather_q16 / 65536.0 : 0.0;
    o->engine_threads = (c->gpu_wb ? 0 : 1 + c->scatter_helpers) + (c->cpu_gather ? 1 + c->gather_helpers : 0);
    o->gpu_writeback = c->gpu_wb ? 1 : 0;
    o->backward_kernels = (c->d_tpart && c->bwd_2p && !getenv("SP_BWD_WS")) ? 2 : 1;
    if (!c->prof_pending.empty()) {
        cudaStreamSynchronize(c->xfer_s);
        cudaStreamSynchronize(c->xfer_s2);
        cudaStreamSynchronize(c->compute);
        harvest_profile(c, true);
    }
    for (int k = 0; k < SP_K_COUNT; k++) {
        o->kernel_launches[k] = c->launches[k];
        o->kernel_ms[k] = c->kms[k];
        o->kernel_timed[k] = c->ktimed[k];
    }
    (void)cudaGetLastError();
    return c->poisoned;
}

sp_status sp_debug_plan(sp_ctx *c, int64_t b, int32_t t, int64_t *counts, int64_t *uniq,
                        int64_t *slot, int64_t *hit, int64_t *evicted) {
    if (!c || !counts || !uniq || !slot || !hit || !evicted || t < 0 || t >= c->T)
        return SP_ERR_INVALID_ARG;
    if (b < 0 || b >= c->planned || c->pushed > b + RING)
        return fail(c, SP_ERR_STATE, "sp_debug_plan: batch not planned or ring entry recycled");
    CK(cudaSetDevice(c->device));
    if (sp_status s = sync_error(c)) return s;
    const BatchBufs &bb = c->ring[b % RING];
    const size_t off = (size_t)t * c->n;
    uint32_t U = 0, m = 0, st[4];
    CK(cudaMemcpy(&U, bb.U + t, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&m, bb.m + t, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(st, bb.stats + 4 * t, 16, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> ids(U), su(U), ev(m);
    std::vector<uint8_t> h(U);
    if (U) {
        CK(cudaMemcpy(ids.data(), bb.uniq_id + off, U * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(su.data(), bb.slot_u + off, U * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(h.data(), bb.hit + off, U, cudaMemcpyDeviceToHost));
    }
    if (m) CK(cudaMemcpy(ev.data(), bb.evict_row + off, m * 4, cudaMemcpyDeviceToHost));
    for (int k = 0; k < 4; k++) counts[k] = st[k];
    uint32_t k = 0;
    for (uint32_t u = 0; u < U; u++) {
        uniq[u] = ids[u];
        slot[u] = (int64_t)su[u] - (int64_t)c->slot_base[t];
        hit[u] = h[u];
        evicted[u] = -1;
        if (!h[u]) {
            evicted[u] = (k < m && ev[k] != EMPTY) ? (int64_t)ev[k] : -1;
            k++;
        }
    }
    return SP_OK;
}

sp_status sp_debug_resident(sp_ctx *c, int32_t t, int64_t *ids, int64_t cap, int64_t *n) {
    if (!c || t < 0 || t >= c->T || !n) return SP_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->plan_s));
    std::vector<uint32_t> res((size_t)c->slots[t]);
    CK(cudaMemcpy(res.data(), c->d_resident + c->slot_base[t], res.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<int64_t> v;
    for (uint32_t x : res)
        if (x != EMPTY) v.push_back(x);
    std::sort(v.begin(), v.end());
    *n = (int64_t)v.size();
    for (int64_t i = 0; i < std::min<int64_t>(cap, *n); i++) ids[i] = v[i];
    return SP_OK;
}

sp_status sp_debug_slots(sp_ctx *c, int32_t t, int64_t *resident, int64_t *last_use) {
    if (!c || t < 0 || t >= c->T || !resident || !last_use) return SP_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->plan_s));
    const size_t S = (size_t)c->slots[t];
    std::vector<uint32_t> res(S);
    std::vector<int32_t> lu(S);
    CK(cudaMemcpy(res.data(), c->d_resident + c->slot_base[t], S * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(lu.data(), c->d_last_use + c->slot_base[t], S * 4, cudaMemcpyDeviceToHost));
    for (size_t s = 0; s < S; s++) {
        resident[s] = res[s] == EMPTY ? -1 : (int64_t)res[s];
        last_use[s] = lu[s] == VACANT ? INT64_MIN : (int64_t)lu[s];
    }
    return SP_OK;
}

sp_status sp_set_stage_timing(sp_ctx *c, int32_t on) {
    if (!c) return SP_ERR_INVALID_ARG;
    if ((on != 0) != c->stage_timing) {
        c->stage_timing = on != 0;
        drop_graphs(c);  // recaptured with / without the timing event nodes
        for (int r = 0; r < RING; r++) c->sev_used[r][0] = c->sev_used[r][1] = false;
    }
    return SP_OK;
}

sp_status sp_set_span_timing(sp_ctx *c, int32_t on) {
    if (!c) return SP_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    if (on && !c->d_span)
        CK(dalloc(c, &c->d_span, (size_t)SPAN_KINDS * RING * SPAN_MAXCTA * 2));
    if ((on != 0) != c->span_on) {
        CK(cudaDeviceSynchronize());
        c->span_on = on != 0;
        drop_graphs(c);  // recaptured with / without the span pointers
    }
    if (on) CK(cudaMemset(c->d_span, 0, (size_t)SPAN_KINDS * RING * SPAN_MAXCTA * 2 * sizeof(unsigned long long)));
    return SP_OK;
}

sp_status sp_span_times(sp_ctx *c, double *out_ms) {
    if (!c || !out_ms) return SP_ERR_INVALID_ARG;
    const size_t per = (size_t)SPAN_MAXCTA * 2, total = (size_t)SPAN_KINDS * RING * per;
    for (size_t i = 0; i < (size_t)SPAN_KINDS * RING * 2; i++) out_ms[i] = std::nan("");
    if (!c->d_span) return SP_OK;
    CK(cudaSetDevice(c->device));
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(total);
    CK(cudaMemcpy(h.data(), c->d_span, total * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull;
    std::vector<unsigned long long> lo((size_t)SPAN_KINDS * RING, ~0ull), hi((size_t)SPAN_KINDS * RING, 0);
    for (size_t q = 0; q < (size_t)SPAN_KINDS * RING; q++) {
        for (size_t k = 0; k < (size_t)SPAN_MAXCTA; k++) {
            const unsigned long long a = h[q * per + 2 * k], b = h[q * per + 2 * k + 1];
            if (a && b >= a) {
                lo[q] = std::min(lo[q], a);
                hi[q] = std::max(hi[q], b);
            }
        }
        if (hi[q]) t0 = std::min(t0, lo[q]);
    }
    for (size_t q = 0; q < (size_t)SPAN_KINDS * RING; q++)
        if (hi[q]) {
            out_ms[2 * q] = (double)(lo[q] - t0) * 1e-6;
            out_ms[2 * q + 1] = (double)(hi[q] - t0) * 1e-6;
        }
    return SP_OK;
}

sp_status sp_stage_times(sp_ctx *c, double *out_ms, int32_t *n_out) {
    if (!c || !out_ms || !n_out) return SP_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    CK(cudaDeviceSynchronize());
    double sum[5] = {0, 0, 0, 0, 0};
    int cnt[5] = {0, 0, 0, 0, 0};
    auto el = [&](cudaEvent_t a, cudaEvent_t b, int k) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, a, b) == cudaSuccess) {
            sum[k] += ms;
            cnt[k]++;
        }
        (void)cudaGetLastError();
    };
    for (int r = 0; r < RING; r++) {
        if (c->sev_used[r][0]) {
            el(c->sev[r][0], c->sev[r][1], 0);
            el(c->sev[r][2], c->sev[r][3], 2);
            el(c->sev[r][3], c->sev[r][4], 3);
            el(c->sev[r][4], c->sev[r][5], 4);
        }
        if (c->sev_used[r][1]) el(c->sev[r][6], c->sev[r][7], 1);
    }
    for (int k = 0; k < 5; k++) {
        out_ms[k] = cnt[k] ? sum[k] / cnt[k] : 0.0;
        n_out[k] = cnt[k];
    }
    return SP_OK;
}

sp_status sp_stage_events(sp_ctx *c, double *out_ms) {
    if (!c || !out_ms) return SP_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    CK(cudaDeviceSynchronize());
    for (int i = 0; i < RING * 8; i++) out_ms[i] = NAN;
    // reference: the plan-start event that comes first among the timed residues
    int ref = -1;
    for (int r = 0; r < RING; r++) {
        if (!c->sev_used[r][0]) continue;
        float ms = 0.f;
        if (ref < 0 || (cudaEventElapsedTime(&ms, c->sev[ref][0], c->sev[r][0]) == cudaSuccess && ms < 0.f)) ref = r;
        (void)cudaGetLastError();
    }
    if (ref < 0) return SP_OK;
    for (int r = 0; r < RING; r++)
        for (int k = 0; k < 8; k++) {
            if (!c->sev_used[r][k < 6 ? 0 : 1]) continue;
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, c->sev[ref][0], c->sev[r][k]) == cudaSuccess) out_ms[r * 8 + k] = ms;
            (void)cudaGetLastError();
        }
    return SP_OK;
}

sp_status sp_debug_plan_profile(sp_ctx *c, uint64_t *out) {
    if (!c || !out) return SP_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->plan_s));
    CK(cudaMemcpy(out, c->d_pprof, (18 * (size_t)c->T + 2 + 4096) * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    return SP_OK;
}

sp_status sp_debug_storage(sp_ctx *c, int32_t t, int64_t first, int64_t count, float *out) {
    if (!c || t < 0 || t >= c->T || !out || first < 0 || count < 0 || first + count > c->slots[t])
        return SP_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    CK(cudaDeviceSynchronize());
    if (c->g.bf16) {  // bf16 rows, widened here (exact: the top 16 bits of an fp32)
        std::vector<uint16_t> tmp((size_t)count * c->D);
        CK(cudaMemcpy(tmp.data(), reinterpret_cast<const char *>(c->d_storage) + ((size_t)c->slot_base[t] + first) * c->D * 2,
                      tmp.size() * 2, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < tmp.size(); i++) {
            const uint32_t u = (uint32_t)tmp[i] << 16;
            std::memcpy(out + i, &u, 4);
        }
        return SP_OK;
    }
    CK(cudaMemcpy(out, c->d_storage + ((size_t)c->slot_base[t] + first) * c->D,
                  (size_t)count * c->D * sizeof(float), cudaMemcpyDeviceToHost));
    return SP_OK;
}

}  // extern "C"
