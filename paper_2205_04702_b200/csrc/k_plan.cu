// k_plan.cu — the [Plan] stage (Alg. 1) as ONE
// kernel launch per sp_plan call.  Tables are independent (one cache manager
// per table), so every CTA works on one table and CTAs never
// synchronise with each other.  A launch at push(j) has 2T CTAs:
//
// CTAs [T, 2T) — dedup of the batch B(j) entering the window (pure function
// of the batch, no scratchpad state):
//   D1  ingest + range check of B(j)[t]
//   D2  stable LSD radix sort of (id, occurrence) pairs by id; heads,
//       unique IDs, segment offsets (Alg. 1 walks raw IDs; deduplicating
//       first is equivalent, reading R5)
//   D3  backward work lists: one chunk record per unique with <= CH
//       occurrences, one hot record per unique with more
//
// CTAs [0, T) — Plan(b), b = j - F - 1, on the scratchpad state of table t:
//   P1  future probe: resident IDs of B(b+F) (deduped by the previous
//       launch) get next_need = b+F (future window, RAW-4 rule, P:864-884;
//       one-shot probe, reading R12)
//   P2  probe B(b): hit -> last_use = b (HoldMask |= MSB, Alg. 1);
//       misses compacted in ascending ID order
//   P3  victims: walk the LRU log from its head; a slot is a candidate iff
//       last_use <= b-P-1 (past window) and next_need <= b; the
//       first |misses| candidates in (last_use, ID) order are taken (LRU,
//       P:1273, reading R8); too few -> SP_ERR_CAPACITY
//   P4  pair k-th miss with k-th victim (reading R6): Hit-Map, resident,
//       stamps; evict + fill lists for the transfer kernel
//   P5  append this batch's slots to the LRU log (compacting it if full)
//   P6  slot map per occurrence and per backward chunk for the Train stage
//       (frozen at Plan, reading R13)
#include "sp_internal.cuh"

namespace sp {

namespace {

constexpr int NW = PUSH_THREADS / 32;

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Exclusive block-wide scan of one u32 per thread; *total gets the sum.
// Contains __syncthreads: every thread of the CTA must call it.
__device__ uint32_t block_scan(uint32_t v, uint32_t *total) {
    __shared__ uint32_t s_warp[NW + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < NW ? s_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NW) s_warp[lane] = w;
    }
    __syncthreads();
    uint32_t pre = warp ? s_warp[warp - 1] : 0u;
    *total = s_warp[NW - 1];
    __syncthreads();
    return pre + x - v;
}

// latch a device error: exact (min) key in device memory, plus a zero-copy
// flag the host's transfer engine and API calls poll without a D2H copy
__device__ __forceinline__ void set_err(const PushArgs &A, long long b, int t, unsigned k) {
    atomicMin(A.err, err_key(b, t, k));
    __threadfence_system();
    *(volatile unsigned long long *)A.err_host = 1ull;
}

__device__ __forceinline__ int bit_width_u64(unsigned long long x) { return x ? 64 - __clzll(x) : 0; }

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Profiling only (A.prof != nullptr): thread 0 adds the time since the
// previous mark to this CTA's per-phase accumulator.
struct PhaseClock {
    unsigned long long *acc;
    unsigned long long last;
    __device__ PhaseClock(unsigned long long *prof, int T, int role, int t)
        : acc(prof ? prof + 2 * T + 2 + ((size_t)role * T + t) * 8 : nullptr), last(0) {
        if (acc && threadIdx.x == 0) last = gtimer();
    }
    __device__ void mark(int k) {
        if (acc && threadIdx.x == 0) {
            const unsigned long long now = gtimer();
            atomicAdd(&acc[k], now - last);
            last = now;
        }
    }
};

// Stable LSD radix sort of (key, val) pairs by key, 8-bit digits over the
// low `bits` bits.  Buffers may live in shared or global memory.  Warp w
// ranks a contiguous run of the tile in rounds of 32 (match_any), so equal
// digits keep their input order: stable.  Returns true if the result ends
// in (kb, vb).
// (histogram and per-warp digit counts shared by both instantiations)
__shared__ uint32_t s_hist[256];
__shared__ uint32_t s_wcnt[NW][256];
__shared__ uint32_t s_hist4[4][256];  // radix_sort_pairs: every pass's digit histogram, one read

template <int IPT>
__device__ bool radix_sort_pairs(uint32_t *ka, uint32_t *va, uint32_t *kb, uint32_t *vb, int n, int bits) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int TILE = PUSH_THREADS * IPT;
    bool swapped = false;
    // the digit histograms of every pass in ONE read of the keys (a stable
    // pass permutes the keys, it does not change their multiset)
    const int npass = (bits + 7) / 8;
    for (int k = threadIdx.x; k < 4 * 256; k += blockDim.x) (&s_hist4[0][0])[k] = 0;
    __syncthreads();
    for (int i0 = 0; i0 < n; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        const uint32_t key = i < n ? ka[i] : 0u;
        for (int p = 0; p < npass; p++) {
            const unsigned d = i < n ? ((key >> (8 * p)) & 255u) : 256u;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (d < 256u && (peers & lanemask_lt()) == 0) atomicAdd(&s_hist4[p][d], __popc(peers));
        }
    }
    __syncthreads();
    for (int sh = 0; sh < bits; sh += 8) {
        {
            uint32_t v = threadIdx.x < 256 ? s_hist4[sh / 8][threadIdx.x] : 0u, tot;
            const uint32_t ex = block_scan(v, &tot);
            if (threadIdx.x < 256) s_hist[threadIdx.x] = ex;
        }
        for (int t0 = 0; t0 < n; t0 += TILE) {
            for (int k = threadIdx.x; k < NW * 256; k += blockDim.x) (&s_wcnt[0][0])[k] = 0;
            __syncthreads();
            uint32_t key[IPT], val[IPT], rk[IPT];
            unsigned dg[IPT];
            const int wbase = t0 + warp * 32 * IPT;
#pragma unroll
            for (int r = 0; r < IPT; r++) {
                const int i = wbase + r * 32 + lane;
                key[r] = i < n ? ka[i] : 0u;
                val[r] = i < n ? va[i] : 0u;
                dg[r] = i < n ? ((key[r] >> sh) & 255u) : 256u;
            }
#pragma unroll
            for (int r = 0; r < IPT; r++) {
                const unsigned peers = __match_any_sync(0xffffffffu, dg[r]);
                const uint32_t base = dg[r] < 256u ? s_wcnt[warp][dg[r]] : 0u;
                rk[r] = base + __popc(peers & lanemask_lt());
                __syncwarp();
                if (dg[r] < 256u && (peers & lanemask_lt()) == 0) s_wcnt[warp][dg[r]] = base + __popc(peers);
                __syncwarp();
            }
            __syncthreads();
            for (int d = threadIdx.x; d < 256; d += blockDim.x) {
                uint32_t run = s_hist[d];
#pragma unroll
                for (int w = 0; w < NW; w++) {
                    const uint32_t c = s_wcnt[w][d];
                    s_wcnt[w][d] = run;
                    run += c;
                }
                s_hist[d] = run;
            }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < IPT; r++)
                if (dg[r] < 256u) {
                    const uint32_t pos = s_wcnt[warp][dg[r]] + rk[r];
                    kb[pos] = key[r];
                    vb[pos] = val[r];
                }
            __syncthreads();
        }
        uint32_t *tk = ka, *tv = va;
        ka = kb; va = vb; kb = tk; vb = tv;
        swapped = !swapped;
    }
    return swapped;
}

// Shared-memory LSD radix sort of (key, val) pairs by key for n <= IPT *
// PUSH_THREADS, one tile per pass.  Warp w owns the contiguous run
// [w*32*IPT, (w+1)*32*IPT) and ranks it in rounds of 32 in input order, so
// equal digits keep their order: stable.  Per pass: the digit peers of a lane
// come from 9 ballots (a warp multisplit), each warp counts its digits in its
// own row of s_wcnt, ONE block-wide exclusive scan over the (digit, warp)
// counters in digit-major order gives every (digit, warp) its output offset,
// and the elements are scattered.  No histogram pre-pass, no serial loop over
// warps.  Returns true if the result ends in (kb, vb).
template <int IPT>
__device__ bool radix_sort_smem(uint32_t *ka, uint32_t *va, uint32_t *kb, uint32_t *vb, int n, int bits) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    bool swapped = false;
    for (int sh = 0; sh < bits; sh += 8) {
        for (int k = threadIdx.x; k < NW * 256; k += blockDim.x) (&s_wcnt[0][0])[k] = 0;
        __syncthreads();
        uint32_t key[IPT], val[IPT], rk[IPT];
        unsigned dg[IPT];
        const int wbase = warp * 32 * IPT;
#pragma unroll
        for (int r = 0; r < IPT; r++) {
            const int i = wbase + r * 32 + lane;
            const bool ok = i < n;
            key[r] = ok ? ka[i] : 0u;
            val[r] = ok ? va[i] : 0u;
            dg[r] = ok ? ((key[r] >> sh) & 255u) : 256u;
            unsigned peers = 0xffffffffu;
#pragma unroll
            for (int b = 0; b < 9; b++) {
                const bool bit = (dg[r] >> b) & 1u;
                const unsigned bal = __ballot_sync(0xffffffffu, bit);
                peers &= bit ? bal : ~bal;
            }
            const uint32_t base = dg[r] < 256u ? s_wcnt[warp][dg[r]] : 0u;
            rk[r] = base + __popc(peers & lt);
            __syncwarp();
            if (dg[r] < 256u && (peers & lt) == 0) s_wcnt[warp][dg[r]] = base + __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        // exclusive scan of the counters in (digit, warp) order: thread t owns
        // the NW*256/blockDim consecutive entries e = d*NW + w of its range
        constexpr int PER = NW * 256 / PUSH_THREADS;
        uint32_t c[PER], sum = 0;
#pragma unroll
        for (int q = 0; q < PER; q++) {
            const int e = threadIdx.x * PER + q;
            c[q] = s_wcnt[e % NW][e / NW];
            sum += c[q];
        }
        uint32_t tot;
        uint32_t run = block_scan(sum, &tot);
#pragma unroll
        for (int q = 0; q < PER; q++) {
            const int e = threadIdx.x * PER + q;
            s_wcnt[e % NW][e / NW] = run;
            run += c[q];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < IPT; r++)
            if (dg[r] < 256u) {
                const uint32_t pos = s_wcnt[warp][dg[r]] + rk[r];
                kb[pos] = key[r];
                vb[pos] = val[r];
            }
        __syncthreads();
        uint32_t *tk = ka, *tv = va;
        ka = kb; va = vb; kb = tk; vb = tv;
        swapped = !swapped;
    }
    return swapped;
}

// ------------------------------------------------------------------ dedup
__device__ void dedup_table(const PushArgs &A, int t, unsigned char *smem_raw, long long j, const void *idx) {
    // (the chunk records of D3 use the sort's free ping-pong buffer as scratch)
    const Geometry &g = A.g;
    const int n = g.n, tid = threadIdx.x;
    const long long R = A.rows[t];
    const BatchBufs &nb = A.nb;
    const bool small = n <= SMEM_SORT_MAX;
    uint32_t *ka, *va, *kb, *vb;
    if (small) {
        ka = reinterpret_cast<uint32_t *>(smem_raw);
        va = ka + n; kb = va + n; vb = kb + n;
    } else {
        const size_t Tn = (size_t)g.T * n;
        ka = A.sort_tmp + (size_t)t * n;
        va = ka + Tn; kb = va + Tn; vb = kb + Tn;
    }
    PhaseClock pc(A.prof, g.T, 1, t);
    // D1: ingest + range check.  With SP_FLAG_PADDING an ID of -1 is "no
    // lookup" (ragged bags, reading R27): its key R sorts after every real ID
    // and it joins no unique.
    int bad = 0, npad = 0;
#pragma unroll 4
    for (int i = tid; i < n; i += blockDim.x) {
        long long id = A.idx_i32 ? (long long)((const int32_t *)idx)[(size_t)t * n + i]
                                 : ((const long long *)idx)[(size_t)t * n + i];
        if (A.pad && id == -1) { id = R; npad++; }
        else if (id < 0 || id >= R) { bad = 1; id = 0; }
        ka[i] = (uint32_t)id;
        va[i] = (uint32_t)i;
    }
    if (__syncthreads_or(bad)) {
        if (tid == 0) set_err(A, j, t, DERR_INDEX);
        return;
    }
    int n_real = n;
    if (A.pad) {  // real lookups of this table (pads sort last)
        uint32_t tot;
        (void)block_scan((uint32_t)npad, &tot);
        n_real = n - (int)tot;
    }
    pc.mark(0);
    // D2: sort by id (stable: occurrences stay ascending within an id).  LSD
    // radix over the table's id bits (1-3 passes of 8 bits).  (A shared-memory
    // bitonic sort of packed (id, occurrence) keys was measured slower:
    // 17.8 us for n = 2048, every table paying the full 66 barrier stages.)
    const int bits = bit_width_u64((unsigned long long)(A.pad ? R : R - 1));
    bool sw;
    if (n <= 2 * PUSH_THREADS) sw = radix_sort_smem<2>(ka, va, kb, vb, n, bits);
    else if (n <= 4 * PUSH_THREADS) sw = radix_sort_smem<4>(ka, va, kb, vb, n, bits);
    else if (small) sw = radix_sort_smem<SMEM_SORT_MAX / PUSH_THREADS>(ka, va, kb, vb, n, bits);
    else sw = radix_sort_pairs<4096 / PUSH_THREADS>(ka, va, kb, vb, n, bits);
    const uint32_t *keys = sw ? kb : ka;
    const uint32_t *vals = sw ? vb : va;
    __syncthreads();
    pc.mark(1);
    uint32_t *sorted_occ = nb.sorted_occ + (size_t)t * n;
    uint32_t *sorted_uid = nb.sorted_uid + (size_t)t * n;
    uint32_t *uniq_id = nb.uniq_id + (size_t)t * n;
    uint32_t *seg_off = nb.seg_off + (size_t)t * g.n1;
    uint32_t carry = 0;
    for (int i0 = 0; i0 < n; i0 += blockDim.x) {
        const int i = i0 + tid;
        uint32_t head = 0, id = 0;
        if (i < n_real) {
            id = keys[i];
            head = (i == 0) || (keys[i - 1] != id);
        }
        uint32_t tot;
        const uint32_t ex = block_scan(head, &tot);
        if (i < n) {
            const uint32_t uid = carry + ex + head - 1;
            sorted_occ[i] = vals[i];
            sorted_uid[i] = i < n_real ? uid : EMPTY;  // padding: no unique
            if (head) { uniq_id[uid] = id; seg_off[uid] = (uint32_t)i; }
        }
        carry += tot;
    }
    const uint32_t U = carry;
    if (tid == 0) { seg_off[U] = (uint32_t)n_real; nb.U[t] = U; }
    __syncthreads();
    pc.mark(2);
    if (!A.bwd_recs) {  // the tiled backward reads sorted_occ / sorted_uid / seg_off only
        if (A.prof) {
            pc.mark(3);
            pc.mark(4);
        }
        return;
    }
    // D3a: backward work lists.  A unique with <= CH occurrences is one chunk
    // record (its bag indices inline); a hot unique (> CH occurrences, the
    // Zipf head) is cut into segments of <= hs occurrences, one hot record
    // each, folded by one CTA of k_bwd.
    ChunkRec *rec = nb.chunk_rec + (size_t)t * g.nc;
    uint4 *hot = nb.hot_rec + (size_t)t * g.nh;
    uint32_t *hcnt = nb.hot_cnt + (size_t)t * g.nh;
    uint32_t *chunk_first = sw ? ka : kb;  // the sort's free buffer (>= n entries)
    const uint32_t hs = (uint32_t)g.hs;
    carry = 0;
    uint32_t hcarry = 0;
    for (uint32_t u0 = 0; u0 < U; u0 += blockDim.x) {
        const uint32_t u = u0 + tid;
        uint32_t lo = 0, len = 0;
        if (u < U) {
            lo = seg_off[u];
            len = seg_off[u + 1] - lo;
        }
        const bool normal = u < U && len <= (uint32_t)CH, is_hot = u < U && len > (uint32_t)CH;
        const uint32_t nseg = is_hot ? (len + hs - 1) / hs : 0u;
        uint32_t tot, htot, ex, hx;
        if (n <= 65535) {  // one scan: segment counts sum to < n/CH + blockDim < 2^16
            uint32_t t2;
            const uint32_t e2 = block_scan((normal ? 1u : 0u) | (nseg << 16), &t2);
            ex = e2 & 0xFFFFu;
            hx = e2 >> 16;
            tot = t2 & 0xFFFFu;
            htot = t2 >> 16;
        } else {
            ex = block_scan(normal ? 1u : 0u, &tot);
            hx = block_scan(nseg, &htot);
        }
        if (normal) {
            const uint32_t c = carry + ex;
            chunk_first[u] = c;
            rec[c].slot = u;
            rec[c].meta = len;
        } else if (is_hot) {
            chunk_first[u] = EMPTY;
            const uint32_t h0 = hcarry + hx;
            for (uint32_t k = 0; k < nseg; k++) {
                hot[h0 + k] = make_uint4(u, lo + k * hs, min(hs, len - k * hs) | (nseg << HOT_LEN_BITS), k);
                hcnt[h0 + k] = 0u;  // row counter at k = 0, group-of-8 counters after it (k_bwd)
            }
        }
        carry += tot;
        hcarry += htot;
    }
    if (tid == 0) {
        nb.nchunks[t] = carry;
        nb.nhot[t] = hcarry;
        if (t == 0)
            for (int k = 0; k < (g.T + 63) / 64; k++) nb.work[k] = 0u;  // k_bwd work counters
    }
    __syncthreads();
    pc.mark(3);
    // D3b: inline bag indices of the single-chunk rows, one occurrence per thread
#pragma unroll 4
    for (int i = tid; i < n_real; i += blockDim.x) {
        const uint32_t u = sorted_uid[i];
        const uint32_t c = chunk_first[u];
        if (c != EMPTY) rec[c].bag[(uint32_t)i - seg_off[u]] = vals[i] / (uint32_t)g.L;
    }
    if (A.prof) {
        __syncthreads();
        pc.mark(4);
    }
}

// ------------------------------------------------------------------- plan
// RANDOM eviction draw (reading R23): splitmix64 chain over (seed, t, b, i)
__device__ __forceinline__ unsigned long long sm64(unsigned long long x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__device__ __forceinline__ unsigned long long rand_draw(unsigned long long seed, int t, long long b,
                                                        unsigned long long i) {
    unsigned long long h = sm64(seed ^ 0x52414E44ull);  // "RAND"
    h = sm64(h ^ (unsigned long long)(long long)t);
    h = sm64(h ^ (unsigned long long)b);
    return sm64(h ^ i);
}

__device__ void plan_table(const PushArgs &A, int t, long long b, unsigned char *smem_raw) {
    const Geometry &g = A.g;
    const int n = g.n, tid = threadIdx.x;
    __shared__ uint32_t s_fail, s_got;
    __shared__ unsigned long long s_head, s_newhead, s_tail;
    __shared__ unsigned long long s_chead[LOG_CLASSES_MAX];  // per class log: head after P3
    const unsigned long long roff = A.row_off[t];
    const BatchBufs &pb = A.pb;
    const int NC = A.log_classes;  // 1 (LRU), LFU_FMAX + 1 (LFU), 0 (RANDOM: no log)
    // working lists of this Plan: in the CTA's dynamic shared memory (the same
    // 16n bytes the dedup role sorts in) when n <= SMEM_SORT_MAX, else global
    const bool small = n <= SMEM_SORT_MAX;
    uint32_t *w_uid = small ? reinterpret_cast<uint32_t *>(smem_raw) : nullptr;   // uniq_id of B(b)
    uint32_t *slot_l = small ? w_uid + n : pb.slot_u + (size_t)t * n;               // slot per unique
    uint32_t *miss_u = small ? w_uid + 2 * n : A.miss_u + (size_t)t * n;
    uint32_t *victims = small ? w_uid + 3 * n : A.victims + (size_t)t * n;
    uint32_t *slot_u = pb.slot_u + (size_t)t * n;                                    // global copy
    const uint32_t pin_base = A.pin_base[t];  // slots >= pin_base are pinned (never victims)

    PhaseClock pc(A.prof, g.T, 0, t);
    // P3's first window of the (class-0) LRU log, loaded now: its entries
    // (slot, stamp) are not touched before P3, so the loads overlap P1 + P2
    uint32_t *lslot = A.log_slot;
    int32_t *lstamp = A.log_stamp;
    const int lid0 = t * (NC > 0 ? NC : 1);
    unsigned long long head0 = 0, tail0 = 0;
    bool inr0 = false;
    uint32_t slot0 = 0;
    int32_t stamp0 = 0;
    if (NC > 0) {
        const unsigned long long cap = A.log_cap[lid0], lbase = A.log_base[lid0];
        head0 = A.log_head[lid0];
        tail0 = A.log_tail[lid0];
        inr0 = head0 + tid < tail0;
        if (inr0) {
            const size_t ix = (size_t)(lbase + (head0 + tid) % cap);
            slot0 = lslot[ix];
            stamp0 = lstamp[ix];
        }
    }
    // P1 + P2 in one pass (independent probes of the same Hit-Map):
    // P1 future probe: resident IDs of B(b+F) get next_need = b+F;
    // P2 probe of B(b): hits stamped last_use = b, misses compacted in
    // ascending ID order (Alg. 1); LFU: a hit adds one use (R24)
    const bool lfu = A.policy == POL_LFU;
    const uint32_t Ub = pb.U[t];
    const uint32_t Uf = A.has_future ? A.fb.U[t] : 0u;
    const uint32_t *fid = A.fb.uniq_id + (size_t)t * n;
    const uint32_t *uniq_id = pb.uniq_id + (size_t)t * n;
    const int32_t fstamp = (int32_t)(b + A.F);
    uint8_t *hitf = pb.hit + (size_t)t * n;
    const uint32_t Umax = Ub > Uf ? Ub : Uf;
    uint32_t carry = 0;
    if (small) {
        // probes first, PU uniques per thread per round with all their loads
        // in flight (the per-round scans below only compact the misses)
        constexpr int PU = 4;
        for (uint32_t u0 = tid; u0 < Umax; u0 += PU * blockDim.x) {
            uint32_t idf[PU], idb[PU], sf[PU], sb[PU];
#pragma unroll
            for (int q = 0; q < PU; q++) {
                const uint32_t u = u0 + q * blockDim.x;
                idf[q] = u < Uf ? fid[u] : 0u;
                idb[q] = u < Ub ? uniq_id[u] : 0u;
            }
#pragma unroll
            for (int q = 0; q < PU; q++) {
                const uint32_t u = u0 + q * blockDim.x;
                sf[q] = u < Uf ? A.hitmap[roff + idf[q]] : EMPTY;
                sb[q] = u < Ub ? A.hitmap[roff + idb[q]] : EMPTY;
            }
#pragma unroll
            for (int q = 0; q < PU; q++) {
                const uint32_t u = u0 + q * blockDim.x;
                if (sf[q] != EMPTY) A.next_need[sf[q]] = fstamp;
                if (u < Ub) {
                    w_uid[u] = idb[q];
                    if (sb[q] != EMPTY) {
                        A.last_use[sb[q]] = (int32_t)b;
                        if (lfu) A.freq[sb[q]] = (uint8_t)min((int)A.freq[sb[q]] + 1, LFU_FMAX);
                    }
                    slot_l[u] = sb[q];
                    slot_u[u] = sb[q];
                    hitf[u] = sb[q] != EMPTY;
                }
            }
        }
        __syncthreads();
        for (uint32_t u0 = 0; u0 < Ub; u0 += blockDim.x) {  // misses, ascending ID order
            const uint32_t u = u0 + tid;
            const uint32_t miss = (u < Ub && slot_l[u] == EMPTY) ? 1u : 0u;
            uint32_t tot;
            const uint32_t ex = block_scan(miss, &tot);
            if (miss) miss_u[carry + ex] = u;
            carry += tot;
        }
    } else {
        for (uint32_t u0 = 0; u0 < Umax; u0 += blockDim.x) {
            const uint32_t u = u0 + tid;
            const uint32_t idf = u < Uf ? fid[u] : 0u;
            const uint32_t idb = u < Ub ? uniq_id[u] : 0u;
            const uint32_t sf = u < Uf ? A.hitmap[roff + idf] : EMPTY;
            const uint32_t sb = u < Ub ? A.hitmap[roff + idb] : EMPTY;
            if (sf != EMPTY) A.next_need[sf] = fstamp;
            uint32_t miss = 0;
            if (u < Ub) {
                if (sb != EMPTY) {
                    A.last_use[sb] = (int32_t)b;
                    if (lfu) A.freq[sb] = (uint8_t)min((int)A.freq[sb] + 1, LFU_FMAX);
                } else {
                    miss = 1;
                }
                slot_l[u] = sb;
                hitf[u] = sb != EMPTY;
            }
            uint32_t tot;
            const uint32_t ex = block_scan(miss, &tot);  // barriers: stamps visible below
            if (miss) miss_u[carry + ex] = u;
            carry += tot;
        }
    }
    const uint32_t m = carry;
    const uint32_t nhit = Ub - m;
    __syncthreads();

    pc.mark(0);
    pc.mark(1);
    const long long limit = b - A.P - 1;
    if (tid == 0) {
        s_got = 0;
        s_fail = 0;
    }
    __syncthreads();
    if (NC > 0) {
        // P3 (LRU / LFU): walk the class logs in ascending class (LRU: one
        // log), each from its head.  A slot is a candidate iff its entry is
        // current (last_use == stamp), last_use <= b-P-1 (past window,
        // P:840-861), next_need <= b (future window) and it is not pinned; the
        // first |misses| candidates in (class, last_use, ID) order are taken
        // (LRU P:1273 reading R8; LFU reading R24).  Eligible entries before
        // the last one taken are dropped (stale, or future-held: those are hit
        // again at next_need and re-appended).  Too few -> SP_ERR_CAPACITY
        // (P:1030-1035).
        for (int c = 0; c < NC; c++) {
            const int lid = lid0 + c;
            const unsigned long long cap = A.log_cap[lid], lbase = A.log_base[lid];
            if (tid == 0) {
                s_head = c == 0 ? head0 : A.log_head[lid];
                s_tail = c == 0 ? tail0 : A.log_tail[lid];
            }
            __syncthreads();
            bool first = c == 0;
            while (true) {
                const unsigned long long head = s_head, tail = s_tail;
                const uint32_t got = s_got;
                if (got >= m) break;
                const unsigned long long pos = head + tid;
                bool inr;
                uint32_t slot = 0;
                int32_t stamp = 0;
                if (first) {  // head == head0: the prefetched window
                    inr = inr0;
                    slot = slot0;
                    stamp = stamp0;
                    first = false;
                } else {
                    inr = pos < tail;
                    if (inr) {
                        const size_t ix = (size_t)(lbase + pos % cap);
                        slot = lslot[ix];
                        stamp = lstamp[ix];
                    }
                }
                const bool elig = inr && (long long)stamp <= limit;  // stamps are non-decreasing
                const bool cand = elig && slot < pin_base && A.last_use[slot] == stamp &&
                                  (long long)A.next_need[slot] <= b;
                // one scan for both counts (<= blockDim each): eligible in the high half
                uint32_t tot2;
                const uint32_t ex2 = block_scan((elig ? 0x10000u : 0u) | (cand ? 1u : 0u), &tot2);
                const uint32_t n_elig = tot2 >> 16, n_cand = tot2 & 0xFFFFu, r = ex2 & 0xFFFFu;
                const uint32_t need = m - got;
                if (cand && r < need) {
                    victims[got + r] = slot;
                    if (r == need - 1) s_newhead = pos + 1;
                }
                __syncthreads();
                if (tid == 0) {
                    if (n_cand >= need) {
                        s_got = m;
                        s_head = s_newhead;
                    } else {
                        s_got = got + n_cand;
                        s_head = head + n_elig;
                        if (n_elig < blockDim.x) s_fail = 1;  // reached held entries or the tail
                    }
                }
                __syncthreads();
                if (s_fail) break;  // this class is exhausted
            }
            if (tid == 0) {
                s_chead[c] = s_head;
                s_fail = 0;
            }
            __syncthreads();
        }
        if (tid == 0 && s_got < m) s_fail = 1;  // every class exhausted
        __syncthreads();
    } else {
        // P3 (RANDOM, reading R23): vacant dynamic slots first, lowest first
        // (they are [nfill, pin_base): slots fill lowest first); then draws
        // s_i = H(seed, t, b, i) mod O over the O occupied dynamic slots, an
        // occupied candidate being taken the first time it is drawn.  Draw i
        // claims its slot with atomicMax of ((b+1) << 32 | ~i): the smallest i
        // of this Plan wins, claims of older Plans are smaller.
        const uint32_t sbase = A.slot_base[t];
        const uint32_t O = A.nfill[t];
        const uint32_t nvac = pin_base - sbase - O;
        const uint32_t v = min(m, nvac);
        for (uint32_t k = tid; k < v; k += blockDim.x) victims[k] = sbase + O + k;
        uint32_t got = v;
        bool counted = false;
        for (unsigned long long i0 = 0; got < m; i0 += blockDim.x) {
            const unsigned long long i = i0 + tid;
            const uint32_t s = sbase + (uint32_t)(rand_draw(A.seed, t, b, i) % (unsigned long long)O);
            const bool cand = (long long)A.last_use[s] <= limit && (long long)A.next_need[s] <= b;
            const unsigned long long key = ((unsigned long long)(b + 1) << 32) | (0xFFFFFFFFull - (i & 0xFFFFFFFFull));
            if (cand) atomicMax(&A.claim[s], key);
            __syncthreads();
            const bool acc = cand && atomicOr(&A.claim[s], 0ull) == key;  // (L2: every claim of this round landed)
            uint32_t tot;
            const uint32_t r = block_scan(acc ? 1u : 0u, &tot);
            if (acc && got + r < m) victims[got + r] = s;
            got += min(tot, m - got);
            if (got < m && !counted && i0 > 8ull * O + 4096) {
                // many draws without enough candidates: count them (capacity check)
                uint32_t c = 0;
                for (uint32_t q = tid; q < O; q += blockDim.x)
                    c += ((long long)A.last_use[sbase + q] <= limit && (long long)A.next_need[sbase + q] <= b) ? 1u : 0u;
                uint32_t ctot;
                (void)block_scan(c, &ctot);
                counted = true;
                if (ctot < m - v) {
                    if (tid == 0) s_fail = 1;
                    break;
                }
            }
        }
        __syncthreads();
        if (tid == 0 && !s_fail) A.nfill[t] = O + v;
    }
    if (s_fail) {
        if (tid == 0) set_err(A, b, t, DERR_CAPACITY);
        return;
    }

    pc.mark(2);
    // P4: assignment (k-th miss <-> k-th victim)
    uint32_t *fill_slot = pb.fill_slot + (size_t)t * n;
    uint32_t *fill_row = pb.fill_row + (size_t)t * n;
    uint32_t *evict_row = pb.evict_row + (size_t)t * n;
    uint32_t nev = 0;
    for (uint32_t k = tid; k < m; k += blockDim.x) {
        const uint32_t u = miss_u[k], s = victims[k], id = small ? w_uid[u] : uniq_id[u];
        const uint32_t old = A.resident[s];
        if (old != EMPTY) {
            A.hitmap[roff + old] = EMPTY;
            nev++;
        }
        A.hitmap[roff + id] = s;
        A.resident[s] = id;
        A.last_use[s] = (int32_t)b;
        A.next_need[s] = NEVER;
        if (lfu) A.freq[s] = 1;
        slot_l[u] = s;
        if (small) slot_u[u] = s;
        fill_slot[k] = s;
        fill_row[k] = id;
        evict_row[k] = old;
        if (A.hl.row) A.hl.row[(size_t)t * n + k] = id;  // pinned mirror (zero-copy)
    }
    uint32_t ev_total;
    (void)block_scan(nev, &ev_total);  // barriers: P4 writes visible below
    if (tid == 0) {
        pb.m[t] = m;  // fills of table t for k_pullfill
        if (A.hl.row) {
            // the CTA's mirror writes precede this fence through the barrier
            // above (causality order): one system-scope fence publishes them
            A.hl.m[t] = m;
            __threadfence_system();
            *(volatile unsigned long long *)&A.hl.ready[t] = (unsigned long long)(b + 1);
        }
    }

    pc.mark(3);
    // P5: log append, per class (LRU: every unique of B(b) to the one log;
    // LFU: each to the log of its use count), after an in-place compaction
    // of a log that would overflow; stamps b, ascending ID within a batch
    for (int c = 0; c < NC; c++) {
        const int lid = lid0 + c;
        const unsigned long long cap = A.log_cap[lid], lbase = A.log_base[lid];
        const unsigned long long head = s_chead[c];
        unsigned long long tail = c == 0 ? tail0 : A.log_tail[lid];
        // entries going to this class (LFU: freq == c; class 0 only holds the
        // initial vacant slots, appended to by LRU alone).  A table with at
        // least as many dynamic slots as rows never evicts: its misses always
        // find the next initial vacant entry, so nothing is appended (and its
        // log never needs compaction).
        const bool no_append = A.log_skip != nullptr && A.log_skip[t] != 0;
        uint32_t cnt = no_append ? 0u : Ub;
        if (lfu && !no_append) {
            if (c == 0) cnt = 0;
            else {
                uint32_t k = 0;
                for (uint32_t u = tid; u < Ub; u += blockDim.x) k += A.freq[slot_l[u]] == c ? 1u : 0u;
                (void)block_scan(k, &cnt);
            }
        }
        if (tail - head + cnt > cap) {
            unsigned long long w = head;
            for (unsigned long long c0 = head; c0 < tail; c0 += blockDim.x) {
                const unsigned long long pos = c0 + tid;
                const bool inr = pos < tail;
                uint32_t slot = 0;
                int32_t stamp = 0;
                if (inr) {
                    const size_t ix = (size_t)(lbase + pos % cap);
                    slot = lslot[ix];
                    stamp = lstamp[ix];
                }
                const bool keep = inr && A.last_use[slot] == stamp;
                uint32_t tot;
                const uint32_t r = block_scan(keep ? 1u : 0u, &tot);  // all reads precede writes
                if (keep) {
                    const size_t ix = (size_t)(lbase + (w + r) % cap);
                    lslot[ix] = slot;
                    lstamp[ix] = stamp;
                }
                w += tot;
                __syncthreads();
            }
            tail = w;
        }
        if (no_append) {
        } else if (!lfu) {
            for (uint32_t u = tid; u < Ub; u += blockDim.x) {
                const size_t ix = (size_t)(lbase + (tail + u) % cap);
                lslot[ix] = slot_l[u];
                lstamp[ix] = (int32_t)b;
            }
        } else if (cnt) {
            uint32_t run = 0;
            for (uint32_t u0 = 0; u0 < Ub; u0 += blockDim.x) {
                const uint32_t u = u0 + tid;
                const uint32_t sl = u < Ub ? slot_l[u] : 0u;
                const bool mine = u < Ub && A.freq[sl] == c;
                uint32_t tot;
                const uint32_t r = block_scan(mine ? 1u : 0u, &tot);
                if (mine) {
                    const size_t ix = (size_t)(lbase + (tail + run + r) % cap);
                    lslot[ix] = sl;
                    lstamp[ix] = (int32_t)b;
                }
                run += tot;
            }
        }
        if (tid == 0) {
            A.log_head[lid] = head;
            A.log_tail[lid] = tail + cnt;
        }
        __syncthreads();
    }
    if (tid == 0) {
        uint32_t *st = pb.stats + 4 * t;
        st[0] = Ub; st[1] = nhit; st[2] = m; st[3] = ev_total;
        atomicAdd(&A.cum[0], (unsigned long long)Ub);
        atomicAdd(&A.cum[1], (unsigned long long)nhit);
        atomicAdd(&A.cum[2], (unsigned long long)m);
        atomicAdd(&A.cum[3], (unsigned long long)ev_total);
    }
    pc.mark(4);
    // P6: slot maps for Train (slot_u complete: the block_scan above synced)
    const uint32_t *sorted_occ = pb.sorted_occ + (size_t)t * n;
    const uint32_t *sorted_uid = pb.sorted_uid + (size_t)t * n;
    uint32_t *slot_of_occ = pb.slot_of_occ + (size_t)t * n;
    uint32_t *sorted_slot = pb.sorted_slot + (size_t)t * n;  // same map in sorted order (backward)
    // (4 elements per thread per round: their independent loads are in flight
    // together instead of one dependent pair per loop trip)
    for (int i0 = tid; i0 < n; i0 += 4 * (int)blockDim.x) {
        uint32_t o[4], u[4], sl[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int i = i0 + q * (int)blockDim.x;
            if (i < n) { o[q] = sorted_occ[i]; u[q] = sorted_uid[i]; }
        }
#pragma unroll
        for (int q = 0; q < 4; q++)
            if (i0 + q * (int)blockDim.x < n) sl[q] = u[q] == EMPTY ? EMPTY : slot_l[u[q]];  // EMPTY: padding
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int i = i0 + q * (int)blockDim.x;
            if (i < n) {
                slot_of_occ[o[q]] = sl[q];
                sorted_slot[i] = sl[q];
            }
        }
    }
    if (A.bwd_recs) {  // (the tiled backward reads slot_u)
        ChunkRec *rec = pb.chunk_rec + (size_t)t * g.nc;
        uint4 *hot = pb.hot_rec + (size_t)t * g.nh;
        const uint32_t nch = pb.nchunks[t], nhot = pb.nhot[t];
        for (uint32_t c = tid; c < nch; c += blockDim.x) rec[c].slot = slot_l[rec[c].slot];
        for (uint32_t h = tid; h < nhot; h += blockDim.x) hot[h].x = slot_l[hot[h].x];
    }
    if (A.prof) {
        __syncthreads();
        pc.mark(5);
    }
}

}  // namespace

__global__ void __launch_bounds__(PUSH_THREADS, SP_PUSH_MIN_BLOCKS) k_push(PushArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (*A.err != NO_ERR) return;  // poisoned: nothing more is planned
    const int T = A.g.T;
    long long j = A.j, b = A.b;
    const void *idx = A.idx;
    if (A.ctl) {  // CUDA-graph replay: absolute batch indices from the device chain
        j = A.ctl[A.ctl_r];
        b = j - A.F - 1;
        idx = static_cast<const char *>(A.idx) + j * A.idx_stride;
        if (blockIdx.x == 0 && threadIdx.x == 0) A.ctl[(A.ctl_r + 1) % RING] = j + 1;
    }
    unsigned long long t_start = 0;
    if (A.prof && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    unsigned long long *spn = A.do_plan ? span_base(A.span, SPK_PLAN, b) : nullptr;
    span_mark(spn, 0);
    const bool role_plan = (int)blockIdx.x < T;
    if (role_plan) {
        if (A.do_plan) plan_table(A, blockIdx.x, b, smem_raw);
    } else if (A.has_new) {
        dedup_table(A, blockIdx.x - T, smem_raw, j, idx);
    }
    if (spn) {
        __syncthreads();
        span_mark(spn, 1);
    }
    if (A.prof && (role_plan ? A.do_plan : A.has_new)) {  // per-CTA wall time, by role and table
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t_end;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            atomicAdd(&A.prof[blockIdx.x], t_end - t_start);
            atomicAdd(&A.prof[2 * T + (role_plan ? 0 : 1)], 1ull);
            // per launch (j mod 1024): kernel span from the first CTA start to
            // the last CTA end, and the slowest CTA of each role
            unsigned long long *sp = A.prof + 18 * T + 2;
            const int q = (int)(j & 1023);
            atomicMin(&sp[q], t_start);
            atomicMax(&sp[1024 + q], t_end);
            atomicMax(&sp[2048 + (role_plan ? 0 : 1024) + q], t_end - t_start);
        }
    }
}

size_t push_smem_bytes(int n) { return n <= SMEM_SORT_MAX ? (size_t)n * 4 * sizeof(uint32_t) : 0; }

int g_carveout = -1;
int g_pdl = 1;

cudaError_t configure_push_kernel() {
    apply_carveout(k_push);
    return cudaFuncSetAttribute(k_push, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(SMEM_SORT_MAX * 4 * sizeof(uint32_t)));
}

cudaError_t launch_push(const PushArgs &a, cudaStream_t s) {
    k_push<<<2 * a.g.T, PUSH_THREADS, push_smem_bytes(a.g.n), s>>>(a);
    return cudaGetLastError();
}

}  // namespace sp
