// runtime.cu — host runtime behind include/scratchpipe.h.
//
// Pipeline schedule (Fig. 8 P:803-813 re-expressed with CUDA streams
// and events instead of lock-step cycles):
//   plan stream      push(j): H2D of B(j) -> k_push = dedup B(j) + future probe
//                    + Plan(j-F)                      -> record ev_plan[j-F]
//   transfer stream  Transfer(b) waits ev_plan[b] and ev_train[b-P-1]
//                    (a victim's last reader/writer is Train(<= b-P-1), the
//                    past-window rule P:840-861) -> record ev_xfer[b];
//                    transfers run in batch order, so a row written back by
//                    Transfer(b') is pulled again only by a later transfer
//                    (RAW-4)
//   compute stream   Train(b) = forward + caller's MLP + backward/SGD waits
//                    ev_xfer[b]                      -> record ev_train[b]
// Up to P transfers run ahead of Train; there is no host synchronisation in
// the steady state (only pinned staging-buffer recycling, 16 batches back).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
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
    cudaStream_t compute = nullptr, plan_s = nullptr;
    // Transfer(b) runs on xfer_s[b % nx]: transfers b..b+F touch disjoint
    // slots and rows (a row evicted at Plan(b) is not in B(b+1..b+F)), so up
    // to F+1 of them may overlap; Transfer(b) stays ordered after b-nx.
    static constexpr int MAX_XFER_STREAMS = 4;
    cudaStream_t xfer_s[MAX_XFER_STREAMS] = {};
    int nx = 1;
    int pull_ctas = 16, wb_ctas = 2;
    cudaStream_t wb_s = nullptr;  // rate-limited write-backs (HBM staging -> host)
    float *d_stage = nullptr;     // [RING][T][n][D]
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
                       *d_log_tail = nullptr;
    unsigned long long *d_err = nullptr, *d_cum = nullptr;
    uint32_t *d_miss_u = nullptr, *d_victims = nullptr;
    uint32_t *d_sort_tmp = nullptr;
    double *d_partial = nullptr;
    float **d_host = nullptr;
    void *d_idx[RING] = {};
    BatchBufs ring[RING];
    // pinned host
    void *h_stage = nullptr;
    unsigned long long *h_err = nullptr;
    size_t idx_bytes = 0;
    // events
    cudaEvent_t ev_plan[RING] = {}, ev_xfer[RING] = {}, ev_train[RING] = {}, ev_h2d[RING] = {};
    cudaEvent_t ev_wb[RING] = {};
    cudaEvent_t ev_user = nullptr;
    bool h2d_used[RING] = {};
    // schedule state
    long long pushed = 0, planned = 0, transferred = 0, forwarded = 0, trained = 0;
    bool eod = false, fwd_pending = false;
    // errors
    sp_status poisoned = SP_OK;
    std::string err = "no error";
    long long err_batch = -1;
    int err_table = -1;
    // stats
    long long h2d_index_bytes = 0;
    long long launches[SP_K_COUNT] = {};
    double kms[SP_K_COUNT] = {};
    long long ktimed[SP_K_COUNT] = {};
    std::vector<ProfEv> prof_pending;
    std::vector<cudaEvent_t> ev_pool;
    cudaEvent_t prof_ref = nullptr;
    std::vector<TimelineRec> timeline;
    long long cur_batch = -1;
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

// wraps one kernel launch: counts it, optionally brackets it with events
template <typename F>
cudaError_t launch(sp_ctx *c, int kind, cudaStream_t s, F &&fn) {
    const bool prof = (c->flags & SP_FLAG_PROFILE) != 0;
    ProfEv pe{kind, c->cur_batch, nullptr, nullptr};
    if (prof) {
        if (c->prof_pending.size() > 4096) harvest_profile(c, false);
        pe.a = pool_event(c);
        pe.b = pool_event(c);
        cudaEventRecord(pe.a, s);
    }
    cudaError_t e = fn();
    c->launches[kind] += 1;
    if (prof) {
        cudaEventRecord(pe.b, s);
        c->prof_pending.push_back(pe);
    }
    return e;
}

BatchBufs carve(sp_ctx *c, int r, cudaError_t *st) {
    (void)r;
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
    A(&b.hot_rec, (size_t)c->T * c->g.nh);
    A(&b.nhot, (size_t)c->T);
    A(&b.nchunks, (size_t)c->T);
    A(&b.slot_u, Tn);
    A(&b.slot_of_occ, Tn);
    A(&b.hit, Tn);
    A(&b.fill_slot, Tn);
    A(&b.fill_row, Tn);
    A(&b.evict_row, Tn);
    A(&b.m, (size_t)c->T);
    A(&b.stats, (size_t)c->T * 4);
    *st = e;
    return b;
}

sp_status check_async_error(sp_ctx *c) {
    if (c->poisoned != SP_OK) return c->poisoned;
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

PushArgs push_args(sp_ctx *c) {
    PushArgs a{};
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
    a.cum = c->d_cum;
    a.miss_u = c->d_miss_u;
    a.victims = c->d_victims;
    a.sort_tmp = c->d_sort_tmp;
    a.idx_i32 = (c->flags & SP_FLAG_INDEX_I32) ? 1 : 0;
    return a;
}

sp_status enqueue_plan_only(sp_ctx *c, long long b) {
    PushArgs a = push_args(c);
    c->cur_batch = b;
    a.has_new = 0;
    a.do_plan = 1;
    a.b = b;
    a.pb = c->ring[b % RING];
    a.has_future = (b + c->F < c->pushed) ? 1 : 0;  // future window truncates at the end
    a.fb = c->ring[(b + c->F) % RING];
    CK(launch(c, SP_K_PLAN, c->plan_s, [&] { return launch_push(a, c->plan_s); }));
    CK(cudaEventRecord(c->ev_plan[b % RING], c->plan_s));
    c->planned = b + 1;
    return SP_OK;
}

sp_status pump(sp_ctx *c) {
    while (c->transferred < c->planned) {
        const long long b = c->transferred, dep = b - c->P - 1;
        if (dep >= 0 && c->trained <= dep) break;  // Train(dep) not enqueued yet
        cudaStream_t xs = c->xfer_s[b % c->nx];
        CK(cudaStreamWaitEvent(xs, c->ev_plan[b % RING], 0));
        if (dep >= 0) CK(cudaStreamWaitEvent(xs, c->ev_train[dep % RING], 0));
        // RAW-4: a row written back by WriteBack(b-F-1) may be
        // pulled again by Pull(b); the write-back stream runs in batch order
        const long long rb = b - c->F - 1;
        if (rb >= 0) CK(cudaStreamWaitEvent(xs, c->ev_wb[rb % RING], 0));
        XferArgs a{};
        c->cur_batch = b;
        a.g = c->g;
        a.bb = c->ring[b % RING];
        a.storage = c->d_storage;
        a.stage = c->d_stage + (size_t)(b % RING) * c->T * c->n * c->D;
        a.host = c->d_host;
        a.err = c->d_err;
        // SP_DEBUG_NO_XFER=1: timing experiments only (results are wrong)
        static const bool no_xfer = getenv("SP_DEBUG_NO_XFER") != nullptr;
        if (!no_xfer) CK(launch(c, SP_K_TRANSFER, xs, [&] { return launch_pull(a, c->pull_ctas, xs); }));
        CK(cudaEventRecord(c->ev_xfer[b % RING], xs));
        CK(cudaStreamWaitEvent(c->wb_s, c->ev_xfer[b % RING], 0));
        if (!no_xfer) CK(launch(c, SP_K_WRITEBACK, c->wb_s, [&] { return launch_writeback(a, c->wb_ctas, c->wb_s); }));
        CK(cudaEventRecord(c->ev_wb[b % RING], c->wb_s));
        c->transferred = b + 1;
    }
    return SP_OK;
}

TrainArgs train_args(sp_ctx *c, long long b) {
    TrainArgs a{};
    a.g = c->g;
    a.bb = c->ring[b % RING];
    a.storage = c->d_storage;
    a.partial = c->d_partial;
    a.err = c->d_err;
    return a;
}

void destroy_all(sp_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->plan_s) cudaStreamSynchronize(c->plan_s);
    for (auto xs : c->xfer_s)
        if (xs) cudaStreamSynchronize(xs);
    if (c->wb_s) cudaStreamSynchronize(c->wb_s);
    cudaStreamSynchronize(c->compute);
    harvest_profile(c, true);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    for (int r = 0; r < RING; r++) {
        if (c->ev_plan[r]) cudaEventDestroy(c->ev_plan[r]);
        if (c->ev_xfer[r]) cudaEventDestroy(c->ev_xfer[r]);
        if (c->ev_train[r]) cudaEventDestroy(c->ev_train[r]);
        if (c->ev_h2d[r]) cudaEventDestroy(c->ev_h2d[r]);
        if (c->ev_wb[r]) cudaEventDestroy(c->ev_wb[r]);
    }
    if (c->ev_user) cudaEventDestroy(c->ev_user);
    if (c->prof_ref) cudaEventDestroy(c->prof_ref);
    for (void *p : c->allocs) cudaFree(p);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    if (c->h_err) cudaFreeHost(c->h_err);
    if (c->registered)
        for (int t = 0; t < c->T; t++) cudaHostUnregister(c->host[t]);
    if (c->plan_s) cudaStreamDestroy(c->plan_s);
    for (auto xs : c->xfer_s)
        if (xs) cudaStreamDestroy(xs);
    if (c->wb_s) cudaStreamDestroy(c->wb_s);
    (void)cudaGetLastError();
    delete c;
}

}  // namespace

extern "C" {

int32_t sp_abi_version(void) { return SP_ABI_VERSION; }

sp_status sp_create(const sp_desc *d, sp_ctx **out) {
    if (!out) return SP_ERR_INVALID_ARG;
    *out = nullptr;
    if (!d || d->num_tables < 1 || d->num_tables > 65535 || !d->rows || !d->slots || !d->host_tables)
        return SP_ERR_INVALID_ARG;
    if (d->dim < 4 || d->dim > 1024 || d->dim % 4) return SP_ERR_INVALID_ARG;
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
    c->g.T = c->T;
    c->g.N = c->N;
    c->g.L = c->L;
    c->g.D = c->D;
    c->g.n = c->n;
    c->g.n1 = c->n + 1;
    c->g.nc = c->n + c->n / CH + 1;
    c->g.nh = c->n / CH + 1;
    c->rows.resize(c->T);
    c->slots.resize(c->T);
    c->host.resize(c->T);
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
#define CKC(call)                                                          \
    do {                                                                   \
        cudaError_t e_ = (call);                                           \
        if (e_ != cudaSuccess) {                                           \
            (void)cudaGetLastError();                                      \
            return bail(e_ == cudaErrorMemoryAllocation ? SP_ERR_OOM : SP_ERR_CUDA); \
        }                                                                  \
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
    }
    CKC(cudaStreamCreateWithPriority(&c->plan_s, cudaStreamNonBlocking, -1));
    c->nx = std::min(c->F + 1, (int)sp_ctx::MAX_XFER_STREAMS);
    for (int k = 0; k < c->nx; k++) CKC(cudaStreamCreateWithFlags(&c->xfer_s[k], cudaStreamNonBlocking));
    CKC(cudaStreamCreateWithFlags(&c->wb_s, cudaStreamNonBlocking));
    for (int r = 0; r < RING; r++) {
        CKC(cudaEventCreateWithFlags(&c->ev_plan[r], cudaEventDisableTiming));
        CKC(cudaEventCreateWithFlags(&c->ev_xfer[r], cudaEventDisableTiming));
        CKC(cudaEventCreateWithFlags(&c->ev_train[r], cudaEventDisableTiming));
        CKC(cudaEventCreateWithFlags(&c->ev_h2d[r], cudaEventDisableTiming));
        CKC(cudaEventCreateWithFlags(&c->ev_wb[r], cudaEventDisableTiming));
    }
    CKC(cudaEventCreateWithFlags(&c->ev_user, cudaEventDisableTiming));
    c->pull_ctas = d->pull_ctas > 0 ? d->pull_ctas : 16;
    c->wb_ctas = d->writeback_ctas > 0 ? d->writeback_ctas : 2;
    CKC(configure_push_kernel());

    // device allocations
    const size_t Tn = (size_t)c->T * c->n;
    CKC(dalloc(c, &c->d_row_off, c->T + 1));
    CKC(dalloc(c, &c->d_rows, c->T));
    CKC(dalloc(c, &c->d_slot_base, c->T + 1));
    CKC(dalloc(c, &c->d_hitmap, c->hit_total));
    CKC(dalloc(c, &c->d_resident, (size_t)c->S_total));
    CKC(dalloc(c, &c->d_last_use, (size_t)c->S_total));
    CKC(dalloc(c, &c->d_next_need, (size_t)c->S_total));
    CKC(dalloc(c, &c->d_storage, (size_t)c->S_total * c->D));
    // LRU log per table: capacity log_factor*S_t + 4n
    const long long lf = d->log_factor > 0 ? d->log_factor : 8;
    std::vector<unsigned long long> lbase(c->T), lcap(c->T), lhead(c->T, 0), ltail(c->T);
    unsigned long long ltot = 0;
    for (int t = 0; t < c->T; t++) {
        lcap[t] = (unsigned long long)(lf * c->slots[t] + 4ll * c->n);
        lbase[t] = ltot;
        ltot += lcap[t];
        ltail[t] = (unsigned long long)c->slots[t];  // initial vacant entries
    }
    CKC(dalloc(c, &c->d_log_slot, ltot));
    CKC(dalloc(c, &c->d_log_stamp, ltot));
    CKC(dalloc(c, &c->d_log_base, c->T));
    CKC(dalloc(c, &c->d_log_cap, c->T));
    CKC(dalloc(c, &c->d_log_head, c->T));
    CKC(dalloc(c, &c->d_log_tail, c->T));
    CKC(dalloc(c, &c->d_err, 1));
    CKC(dalloc(c, &c->d_cum, 4));
    CKC(dalloc(c, &c->d_miss_u, Tn));
    CKC(dalloc(c, &c->d_victims, Tn));
    if (c->n > SMEM_SORT_MAX) CKC(dalloc(c, &c->d_sort_tmp, 4 * Tn));
    CKC(dalloc(c, &c->d_partial, (size_t)c->T * c->g.nc * c->D));
    CKC(dalloc(c, &c->d_host, c->T));
    CKC(dalloc(c, &c->d_stage, (size_t)RING * Tn * c->D));
    c->idx_bytes = Tn * ((c->flags & SP_FLAG_INDEX_I32) ? 4 : 8);
    for (int r = 0; r < RING; r++) {
        cudaError_t st;
        c->ring[r] = carve(c, r, &st);
        CKC(st);
        void *p = nullptr;
        CKC(cudaMalloc(&p, c->idx_bytes));
        c->allocs.push_back(p);
        c->d_idx[r] = p;
    }
    CKC(cudaHostAlloc(&c->h_stage, c->idx_bytes * RING, cudaHostAllocDefault));
    CKC(cudaHostAlloc((void **)&c->h_err, sizeof(unsigned long long), cudaHostAllocDefault));
    *c->h_err = NO_ERR;

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
        // initial LRU log: every slot vacant, ascending slot order
        std::vector<uint32_t> ls(ltot, 0);
        std::vector<int32_t> lst(ltot, VACANT);
        for (int t = 0; t < c->T; t++)
            for (long long s = 0; s < c->slots[t]; s++) ls[lbase[t] + s] = c->slot_base[t] + (uint32_t)s;
        CKC(cudaMemcpy(c->d_log_slot, ls.data(), ltot * sizeof(uint32_t), cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(c->d_log_stamp, lst.data(), ltot * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    CKC(cudaMemcpy(c->d_log_base, lbase.data(), c->T * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    CKC(cudaMemcpy(c->d_log_cap, lcap.data(), c->T * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    CKC(cudaMemcpy(c->d_log_head, lhead.data(), c->T * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    CKC(cudaMemcpy(c->d_log_tail, ltail.data(), c->T * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    CKC(cudaMemset(c->d_err, 0xFF, sizeof(unsigned long long)));
    CKC(cudaMemset(c->d_cum, 0, 4 * sizeof(unsigned long long)));
    CKC(cudaMemset(c->d_storage, 0, (size_t)c->S_total * c->D * sizeof(float)));
    CKC(cudaDeviceSynchronize());
#undef CKC
    *out = c;
    return SP_OK;
}

static sp_status plan_impl(sp_ctx *c, const void *idx, bool on_device) {
    if (!c || !idx) return SP_ERR_INVALID_ARG;
    if (sp_status s = check_async_error(c)) return s;
    if (c->eod) return fail(c, SP_ERR_STATE, "sp_plan after sp_end_of_data (call sp_flush first)");
    const long long j = c->pushed;
    const int r = (int)(j % RING);
    if (j >= RING && c->trained < j - RING + 1)
        return fail(c, SP_ERR_STATE, "sp_plan: more than 16 batches ahead of sp_train");
    CK(cudaSetDevice(c->device));
    if (j >= RING) {
        CK(cudaStreamWaitEvent(c->plan_s, c->ev_train[r], 0));
        CK(cudaStreamWaitEvent(c->plan_s, c->ev_wb[r], 0));  // WriteBack(j-RING) reads ring slot r
    }
    const void *dev_idx;
    if (on_device) {
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
    c->cur_batch = j;
    a.has_new = 1;
    a.j = j;
    a.idx = dev_idx;
    a.nb = c->ring[r];
    // Plan(b) runs beside dedup(j) once B(b+F) = B(j-1) has been deduped
    const long long b = j - c->F - 1;
    a.do_plan = (b >= 0 && b == c->planned) ? 1 : 0;
    if (a.do_plan) {
        a.b = b;
        a.pb = c->ring[b % RING];
        a.has_future = 1;
        a.fb = c->ring[(b + c->F) % RING];
    }
    CK(launch(c, SP_K_PLAN, c->plan_s, [&] { return launch_push(a, c->plan_s); }));
    if (a.do_plan) {
        CK(cudaEventRecord(c->ev_plan[b % RING], c->plan_s));
        c->planned = b + 1;
    }
    c->pushed = j + 1;
    CK(cudaMemcpyAsync(c->h_err, c->d_err, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->plan_s));
    return pump(c);
}

sp_status sp_plan(sp_ctx *c, const void *idx) {
    return plan_impl(c, idx, c && (c->flags & SP_FLAG_INDEX_DEVICE));
}

sp_status sp_plan_device(sp_ctx *c, const void *idx) { return plan_impl(c, idx, true); }

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
    if (on) {
        c->flags |= SP_FLAG_PROFILE;
        if (!c->prof_ref) CK(cudaEventCreate(&c->prof_ref));
        CK(cudaEventRecord(c->prof_ref, c->compute));
        c->timeline.clear();
    } else {
        c->flags &= ~SP_FLAG_PROFILE;
    }
    return SP_OK;
}

sp_status sp_get_timeline(sp_ctx *c, int32_t *kind, int64_t *batch, double *start_ms, double *end_ms,
                          int64_t cap, int64_t *n) {
    if (!c || !n) return SP_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    CK(cudaDeviceSynchronize());
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
    CK(cudaMemcpyAsync(c->h_err, c->d_err, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->plan_s));
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
    if (c->transferred <= b) return fail(c, SP_ERR_STATE, "sp_forward: transfer not schedulable");
    // every slot B(b) reads was filled by some Transfer(<= b): the last nx
    // transfers may still be running on their own streams
    for (int k = 0; k < c->nx && b - k >= 0; k++)
        CK(cudaStreamWaitEvent(c->compute, c->ev_xfer[(b - k) % RING], 0));
    TrainArgs a = train_args(c, b);
    c->cur_batch = b;
    a.pooled = pooled;
    CK(launch(c, SP_K_FORWARD, c->compute, [&] { return launch_forward(a, c->compute); }));
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
    TrainArgs a = train_args(c, b);
    c->cur_batch = b;
    a.grad = grad;
    a.lr = lr;
    CK(launch(c, SP_K_BACKWARD, c->compute, [&] {
        cudaError_t e = launch_backward(a, c->compute);
        return e != cudaSuccess ? e : launch_backward_hot(a, c->compute);
    }));
    CK(cudaEventRecord(c->ev_train[b % RING], c->compute));
    c->trained = b + 1;
    c->fwd_pending = false;
    return pump(c);
}

sp_status sp_surrogate_grad(sp_ctx *c, const float *pooled, float *grad, int64_t count, float gamma,
                            float delta) {
    if (!c || !pooled || !grad || count < 0 || count % 4) return SP_ERR_INVALID_ARG;
    if (c->poisoned != SP_OK) return c->poisoned;
    CK(cudaSetDevice(c->device));
    if (count == 0) count = (long long)c->T * c->N * c->D;
    CK(launch(c, SP_K_SURROGATE, c->compute,
              [&] { return launch_surrogate(pooled, grad, count, gamma, delta, c->compute); }));
    return SP_OK;
}

sp_status sp_flush(sp_ctx *c) {
    if (!c) return SP_ERR_INVALID_ARG;
    if (sp_status s = check_async_error(c)) return s;
    if (c->trained != c->pushed || c->fwd_pending)
        return fail(c, SP_ERR_STATE, "sp_flush: every pushed batch must be trained first");
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->plan_s));
    for (int k = 0; k < c->nx; k++) CK(cudaStreamSynchronize(c->xfer_s[k]));
    CK(cudaStreamSynchronize(c->wb_s));
    CK(cudaStreamSynchronize(c->compute));
    if (sp_status s = sync_error(c)) return s;
    FlushArgs a{};
    a.g = c->g;
    a.S_total = (int)c->S_total;
    a.slot_base = c->d_slot_base;
    a.resident = c->d_resident;
    a.storage = c->d_storage;
    a.host = c->d_host;
    CK(launch(c, SP_K_FLUSH, c->compute, [&] { return launch_flush(a, c->compute); }));
    CK(cudaStreamSynchronize(c->compute));
    c->eod = false;  // a flush is a checkpoint: the caller may continue pushing
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
    o->transferred = c->transferred;
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
    if (!c->prof_pending.empty()) {
        for (int k = 0; k < c->nx; k++) cudaStreamSynchronize(c->xfer_s[k]);
        cudaStreamSynchronize(c->wb_s);
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

sp_status sp_debug_storage(sp_ctx *c, int32_t t, int64_t first, int64_t count, float *out) {
    if (!c || t < 0 || t >= c->T || !out || first < 0 || count < 0 || first + count > c->slots[t])
        return SP_ERR_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, c->d_storage + ((size_t)c->slot_base[t] + first) * c->D,
                  (size_t)count * c->D * sizeof(float), cudaMemcpyDeviceToHost));
    return SP_OK;
}

}  // extern "C"
